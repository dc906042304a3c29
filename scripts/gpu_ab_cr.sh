#!/bin/bash
# consumer-refill A/B + the parity tests that cover small launches
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t_parity.log 2>&1; echo "parity=$?" > gpurun_out/st.txt
bash scripts/exp_libs_probe.sh "paper_2509_08309_b200/libhetis.so libx/libhetis_cr0.so" 8,16,64 ab_cr.jsonl 2 "0,0x20" ; echo "ab=$?" >> gpurun_out/st.txt
timeout -s KILL 600 python scripts/stress_steps.py --replays 10 --steps 20 > gpurun_out/stress_cr.txt 2>&1; echo "stress=$?" >> gpurun_out/st.txt
cat gpurun_out/st.txt
