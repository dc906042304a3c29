#!/bin/bash
# confidence soak of the final kernels: long graph-replayed stress, the parity suite three times, the peer tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/st_soak.txt
timeout -s KILL 1200 python scripts/stress_steps.py --replays 50 --steps 40 > gpurun_out/stress_soak.txt 2>&1; echo "stress=$?" >> gpurun_out/st_soak.txt
for i in 1 2 3; do timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/soak_parity_$i.log 2>&1; echo "parity$i=$?" >> gpurun_out/st_soak.txt; done
timeout -s KILL 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_bench.py -q -x > gpurun_out/soak_peer.log 2>&1; echo "peer_bench=$?" >> gpurun_out/st_soak.txt
cat gpurun_out/st_soak.txt
