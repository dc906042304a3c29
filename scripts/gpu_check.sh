#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?" > gpurun_out/status.txt
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout -s KILL 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
