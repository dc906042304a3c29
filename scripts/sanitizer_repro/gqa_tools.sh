cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash scripts/sanitizer_repro/run.sh
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in synccheck racecheck; do
  timeout -s KILL 900 $CS --tool $tool --print-limit 5 --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "edge_lengths_ragged and 16-2-128-bf16" -p no:cacheprovider > gpurun_out/san_gqa_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_gqa_$tool.log | tail -3 | tr '\n' ' ')"
done
