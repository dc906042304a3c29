cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for L in tracelib/libhetis_s100.so tracelib/libhetis_s95.so paper_2509_08309_b200/libhetis.so tracelib/libhetis_s70.so; do
  for rep in 1 2; do
  HETIS_LIB=$PWD/$L timeout -s KILL 300 python scripts/step_breakdown.py --config c3 --ns 1,2,4,8 2>&1 | grep '^{' | python -c "
import json,sys
print('$L', ' '.join(f\"n{d['n']}={d['full_us']:.1f}/{d['attn_us']:.1f}\" for d in map(json.loads, sys.stdin)))"
  done
  HETIS_LIB=$PWD/$L timeout -s KILL 600 python scripts/migrate_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L migrate', [(r['max_ctas'], round(r['decode_slowdown'],3), round(r['migration_gbs_read_plus_write'])) for r in d['rows']])"
done
