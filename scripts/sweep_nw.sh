cd $GRAFT_REPO_ROOT
bash scripts/sweep_libs.sh "tracelib/libhetis_nw8_sw3.so tracelib/libhetis_nw6_sw4.so tracelib/libhetis_nw4_sw6.so" c3 1,2,4,8 2
for L in tracelib/libhetis_nw8_sw3.so tracelib/libhetis_nw6_sw4.so tracelib/libhetis_nw4_sw6.so; do
  HETIS_LIB=$PWD/$L timeout -s KILL 300 python scripts/step_breakdown.py --config c2 --ns 1,8 --steps 100 --flags 8 2>&1 | grep '^{' | python -c "
import json,sys
print('mha_tc $(basename $L .so)'.ljust(30), ' '.join(f\"n{d['n']}={d['full_us']:.1f}/{d['fapp_us']:.1f}\" for d in map(json.loads, sys.stdin)))"
done
