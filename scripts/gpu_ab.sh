#!/bin/bash
# A/B two builds: bash scripts/gpu_ab.sh "<nvcc flags A>" "<nvcc flags B>" "<configs>"
cd "$GRAFT_REPO_ROOT"
for tag in A B; do
  if [ $tag = A ]; then F="$1"; else F="$2"; fi
  LIB=/tmp/libhetis_$tag.so
  HETIS_LIB=$LIB HETIS_NVCC_FLAGS="$F" timeout -s KILL 600 python -m paper_2509_08309_b200.build > /dev/null 2>&1 || echo "build $tag failed"
  for C in $3; do
    HETIS_LIB=$LIB timeout -s KILL 300 python bench.py --config $C --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$tag [$F] $C', round(d['ms_per_step']*1000,1), 'us/step', round(r['avg_launch_ms']*1000,1), 'us', round(r['achieved']), 'GB/s', round(r['frac'],3))"
  done
done
