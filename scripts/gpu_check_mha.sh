#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-mw}
: > gpurun_out/st_$TAG.txt
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 600 python scripts/stress_steps.py --replays 10 --steps 20 > gpurun_out/stress_$TAG.txt 2>&1; echo "stress=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 400 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_default.log 2>&1; echo "bench=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 900 python scripts/scaling_probe.py --config c2 > gpurun_out/scaling_${TAG}_c2.jsonl 2>&1; echo "scal=$?" >> gpurun_out/st_$TAG.txt
timeout -s KILL 900 python scripts/scaling_probe.py --config c4 --shares > gpurun_out/c4_shares_$TAG.jsonl 2>&1; echo "c4=$?" >> gpurun_out/st_$TAG.txt
cat gpurun_out/st_$TAG.txt
