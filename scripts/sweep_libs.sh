#!/bin/bash
# Interleaved A/B/... of step_breakdown over several library builds on one box:
#   bash scripts/sweep_libs.sh "<lib1> <lib2> ..." <config> <ns> [reps]
cd "$GRAFT_REPO_ROOT"
for rep in $(seq 1 ${4:-2}); do
  for L in $1; do
    HETIS_LIB=$PWD/$L timeout -s KILL 150 python scripts/step_breakdown.py --config $2 --ns $3 --steps 100 2>&1 | grep '^{' | python -c "
import json,sys
print('$(basename $L .so)'.ljust(22), ' '.join(f\"n{d['n']}={d['full_us']:.1f}/{d['attn_us']:.1f}/{d.get('fapp_us', 0):.1f}/{d.get('pipe_us', 0):.1f}\" for d in map(json.loads, sys.stdin)))"
  done
done
