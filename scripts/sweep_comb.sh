#!/bin/bash
# combine chunk size A/B (comb-only and full-step graphs) on c3 / c5 / c2
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for L in tracelib/libhetis_u4.so tracelib/libhetis_u8.so tracelib/libhetis_u16.so; do
  for C in c3 c5; do
    HETIS_LIB=$PWD/$L timeout -s KILL 150 python scripts/step_breakdown.py --config $C --ns 1,8 --steps 100 2>&1 | grep '^{' | python -c "
import json,sys
print('$(basename $L .so) $C'.ljust(20), ' '.join(f\"n{d['n']}: fapp={d['fapp_us']:.1f} comb={d['comb_us']:.1f}\" for d in map(json.loads, sys.stdin)))"
  done
done
done
