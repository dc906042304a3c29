#!/bin/bash
# usage: bash scripts/gpu_iter.sh <tag> [ncu-config|none] [bench configs...]
cd "$GRAFT_REPO_ROOT"
TAG=${1:-it}; NCU=${2:-c2}; shift 2; CFGS=${@:-c2 c3}
mkdir -p gpurun_out
: > gpurun_out/status_$TAG.txt
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG.txt
tail -3 gpurun_out/pytest_gpu_$TAG.log
for C in $CFGS; do
  timeout -s KILL 300 python bench.py --config $C --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${TAG}_$C.log 2>&1; echo "bench_$C=$?" >> gpurun_out/status_$TAG.txt
  python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}_$C.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$C', round(d['value']), 'tok/s', round(d['ms_per_step'],4), 'ms', round(r['achieved']), 'GB/s', round(r['frac'],3), d['clocks'])" 2>&1 | tail -1
done
if [ "$NCU" != "none" ]; then
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 3 -c 1 -o gpurun_out/prof_${TAG}_$NCU python bench.py --config $NCU --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_${TAG}_$NCU.log 2>&1; echo "ncu_full=$?" >> gpurun_out/status_$TAG.txt
fi
cat gpurun_out/status_$TAG.txt
