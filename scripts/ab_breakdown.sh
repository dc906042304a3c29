#!/bin/bash
# A/B of scripts/step_breakdown.py between two library builds on the same box:
#   bash scripts/ab_breakdown.sh <libA> <libB> "<configs>" [ns]
cd "$GRAFT_REPO_ROOT"
NS=${4:-1,8}
for rep in 1 2; do
  for tag in A B; do
    if [ $tag = A ]; then LIB="$1"; else LIB="$2"; fi
    for C in $3; do
      HETIS_LIB=$LIB timeout -s KILL 300 python scripts/step_breakdown.py --config $C --ns $NS 2>&1 | grep '^{' | \
        python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$tag', d['config'], d['n'], *[f\"{k[:-3]}={d[k]:.1f}\" for k in ('full_us','no_app_us','attn_us','comb_us')])"
    done
  done
done
