cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2509_08309_b200.build > gpurun_out/build_f.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='units or merge_fused or staged or edge_lengths_ragged or bf16_output or fused_append or narrow_and_wide'
for tool in memcheck initcheck; do
  timeout -s KILL 1500 $CS --tool $tool --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize2_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize2_$tool.log | tail -2 | tr '\n' ' ')"
done
timeout -s KILL 1500 $CS --tool memcheck --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_peer.py -m gpu -q -k "32-32 and None-None" -p no:cacheprovider > gpurun_out/sanitize2_peer.log 2>&1
echo "peer memcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize2_peer.log | tail -3 | tr '\n' ' ')"
