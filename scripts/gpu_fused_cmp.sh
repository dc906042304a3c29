#!/bin/bash
cd "$GRAFT_REPO_ROOT"; TAG=${1:-fc}; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for C in ${2:-c2 c3 c5}; do for F in 0 1; do
timeout -s KILL 300 python bench.py --config $C --steps 200 --warmup 10 --no-cpu-baseline --fused $F 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$C fused=$F', round(d['value']), 'tok/s step', round(d['ms_per_step']*1000,1), 'us kernel', round(r['avg_launch_ms']*1000,1), 'us', round(r['achieved']), 'GB/s', round(r['frac'],3))" 2>&1 | tail -1
done; done
