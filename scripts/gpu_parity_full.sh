#!/bin/bash
# Whole-O full-size parity (T10) against the fp64 oracle; the per-case max-abs records land in
# gpurun_out/parity_<tag>.jsonl.  usage: bash scripts/gpu_parity_full.sh <tag>
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r2}
mkdir -p gpurun_out
(free -g; nproc; lscpu | grep 'Model name') > gpurun_out/host_$TAG.txt 2>&1
rm -f gpurun_out/parity_$TAG.jsonl
HETIS_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout -s KILL 1500 python -m pytest -q -x -s \
  tests/test_gpu_parity.py -k "full_size or tensor_core_vs_cuda_core" tests/test_gpu_seqsplit.py \
  > gpurun_out/pytest_parity_$TAG.log 2>&1
echo "pytest=$?"
tail -3 gpurun_out/pytest_parity_$TAG.log
