#!/bin/bash
# Evidence run for profiles/: bench lines, ncu launch lists and one full ncu capture per config.
# usage: bash scripts/gpu_profile.sh <tag> "<configs>"
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}; CFGS=${2:-"c2 c3"}
mkdir -p gpurun_out
: > gpurun_out/status_$TAG.txt
for C in $CFGS; do
  timeout -s KILL 400 python bench.py --config $C --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_$C.log 2>&1; echo "bench_$C=$?" >> gpurun_out/status_$TAG.txt
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'attn_decode|kv_append|combine_kernel|head_copy' -c 40 --csv --log-file gpurun_out/launches_${TAG}_$C.csv python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu_list_$C=$?" >> gpurun_out/status_$TAG.txt
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 3 -c 1 -o gpurun_out/prof_${TAG}_$C python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_${TAG}_$C.log 2>&1; echo "ncu_full_$C=$?" >> gpurun_out/status_$TAG.txt
done
cat gpurun_out/status_$TAG.txt
