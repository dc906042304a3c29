#!/bin/bash
# bf16 MHA: per-warp CUDA-core kernel (default) vs the shared-ring kernel (libx/libhetis_mw0.so) vs MHA_TC
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t_parity_mw.log 2>&1; echo "parity=$?" > gpurun_out/st_mw.txt
for r in 1 2; do for L in paper_2509_08309_b200/libhetis.so libx/libhetis_mw0.so; do
HETIS_LIB=$PWD/$L timeout -s KILL 400 python scripts/attn_probe.py --config c2 --heads 40,10,5 --flags 0,0x8,0x100 --decode --steps 50 2>&1 | grep '^{'
done; done > gpurun_out/ab_mha.jsonl; echo "ab=$?" >> gpurun_out/st_mw.txt
cat gpurun_out/st_mw.txt
