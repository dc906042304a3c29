#!/bin/bash
# memcheck + initcheck over the round-2 kernel paths (group mode, consumer refill, peer pull + group merge)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='group_mode or merge_fused or units_random or tensor_core_vs_cuda_core or edge_lengths or pipelined or fused_append'
for tool in memcheck initcheck; do
  timeout -s KILL 1500 $CS --tool $tool --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_r2i_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_r2i_$tool.log | tail -2 | tr '\n' ' ')"
done
timeout -s KILL 1500 $CS --tool memcheck --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_peer.py -q -k "not c1" -p no:cacheprovider > gpurun_out/sanitize_r2i_peer_memcheck.log 2>&1
echo "peer memcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_r2i_peer_memcheck.log | tail -2 | tr '\n' ' ')"
