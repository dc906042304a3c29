#!/bin/bash
# Build kernel variants on the box and bench each: bash scripts/gpu_sweep.sh <tag> "<variant specs>" [configs]
# variant spec: SIMT_NW:TC_NW:STAGES[:PRODUCER_LANES]
cd "$GRAFT_REPO_ROOT"
TAG=${1:-sw}; SPECS=${2:-"8:8:24"}; CFGS=${3:-"c2 c3"}
mkdir -p gpurun_out
OUT=gpurun_out/sweep_$TAG.txt; : > $OUT
for C in $CFGS; do
timeout -s KILL 300 python bench.py --config $C --steps 100 --warmup 5 --no-cpu-baseline --attn-flags 256 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('  STREAM-ONLY $C', round(d['roofline']['achieved']), 'GB/s')" >> $OUT 2>&1
done
for spec in $SPECS; do
  IFS=: read SNW TNW ST PL <<< "$spec"; PL=${PL:-4}
  LIB=/tmp/libhetis_${SNW}_${TNW}_${ST}_${PL}.so
  HETIS_LIB=$LIB HETIS_NVCC_FLAGS="-DHETIS_SIMT_NW=$SNW -DHETIS_TC_NW=$TNW -DHETIS_MAX_STAGES=$ST -DHETIS_PRODUCER_LANES=$PL" timeout -s KILL 600 python -m paper_2509_08309_b200.build > /tmp/build_$spec.log 2>&1 || { echo "build $spec failed" >> $OUT; tail -5 /tmp/build_$spec.log >> $OUT; continue; }
  for C in $CFGS; do
    HETIS_LIB=$LIB timeout -s KILL 300 python bench.py --config $C --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('  $spec $C', round(d['value']), 'tok/s', round(r['avg_launch_ms'],4), 'ms', round(r['achieved']), 'GB/s', round(r['frac'],3))" >> $OUT 2>&1
  done
done
cat $OUT
