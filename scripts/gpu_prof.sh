#!/bin/bash
# usage: bash scripts/gpu_prof.sh <tag> [config]
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}; CFG=${2:-c2}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" > gpurun_out/status_$TAG.txt
timeout -s KILL 300 python bench.py --config $CFG --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_$CFG.log 2>&1; echo "bench=$?" >> gpurun_out/status_$TAG.txt
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${TAG}_$CFG.csv python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu_list=$?" >> gpurun_out/status_$TAG.txt
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 3 -c 1 -o gpurun_out/prof_${TAG}_$CFG python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_${TAG}_$CFG.log 2>&1; echo "ncu_full=$?" >> gpurun_out/status_$TAG.txt
cat gpurun_out/status_$TAG.txt
