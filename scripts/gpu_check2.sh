#!/bin/bash
# after a kernel change: GPU suite, smoke, bench c3 and the default line, c3 scaling, group-mode probe
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-chk}
: > gpurun_out/st_$TAG.txt
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 400 python bench.py --config c3 --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_c3.log 2>&1; echo "bench_c3=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 400 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_default.log 2>&1; echo "bench=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 600 python scripts/scaling_probe.py --config c3 > gpurun_out/scaling_${TAG}_c3.jsonl 2>&1; echo "scal=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 600 python scripts/attn_probe.py --heads 8,16 --flags 0,0x20,0x60 --decode --steps 100 > gpurun_out/group_mode_${TAG}.jsonl 2>&1; echo "group=$?" >> gpurun_out/st_$TAG.txt
cat gpurun_out/st_$TAG.txt
