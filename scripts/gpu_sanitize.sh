#!/bin/bash
# compute-sanitizer evidence on small problems (memcheck, racecheck, synccheck, initcheck)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL=${SEL:-'c1_two_virtual or edge_lengths_ragged or kv_append_memcmp or bf16_output or per_request or fused_append or pipelined or narrow_and_wide or device_claim'}
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 1200 $CS --tool $tool --error-exitcode 9 --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
