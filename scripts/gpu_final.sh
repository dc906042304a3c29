#!/bin/bash
# Round-end evidence run: GPU tests, bench lines for every config (with cpu_baseline),
# ncu launch lists + one --set full capture of the attention kernel for c2 and c3.
# usage: bash scripts/gpu_final.sh <tag>
cd "$GRAFT_REPO_ROOT"
TAG=${1:-final}
mkdir -p gpurun_out
: > gpurun_out/status_$TAG.txt
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG.txt
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG.txt
for C in c1 c2 c3 c4 c5; do
  timeout -s KILL 400 python bench.py --config $C --steps 200 --warmup 10 > gpurun_out/bench_${TAG}_$C.log 2>&1; echo "bench_$C=$?" >> gpurun_out/status_$TAG.txt
done
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo "bench_ref=$?" >> gpurun_out/status_$TAG.txt
for C in c2 c3; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'attn|kv_append|combine_kernel|head_copy' -c 40 --csv --log-file gpurun_out/launches_${TAG}_$C.csv python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu_list_$C=$?" >> gpurun_out/status_$TAG.txt
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -o gpurun_out/prof_${TAG}_$C python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_${TAG}_$C.log 2>&1; echo "ncu_full_$C=$?" >> gpurun_out/status_$TAG.txt
done
cat gpurun_out/status_$TAG.txt
