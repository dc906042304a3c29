#!/bin/bash
# consumer-refill A/B (HETIS_CONSUMER_REFILL 1 = small launches, 2 = every launch) + parity / stress on the variant
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
HETIS_LIB=$PWD/libx/libhetis_cr2.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t_parity_cr2.log 2>&1; echo "parity_cr2=$?" > gpurun_out/st.txt
HETIS_LIB=$PWD/libx/libhetis_cr2.so timeout -s KILL 600 python scripts/stress_steps.py --replays 10 --steps 20 > gpurun_out/stress_cr2.txt 2>&1; echo "stress_cr2=$?" >> gpurun_out/st.txt
bash scripts/exp_libs_probe.sh "paper_2509_08309_b200/libhetis.so libx/libhetis_cr2.so" 8,16,32,64 ab_cr2.jsonl 2 "0" ; echo "ab=$?" >> gpurun_out/st.txt
cat gpurun_out/st.txt
