#!/bin/bash
# gpu_check2.sh + graph-replayed stress + the claim A/B (default device-wide vs HETIS_ATTN_STATIC_DEAL)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-chk}
bash scripts/gpu_check2.sh $TAG > /dev/null 2>&1
timeout -s KILL 600 python scripts/stress_steps.py --replays 10 --steps 20 > gpurun_out/stress_$TAG.txt 2>&1; echo "stress=$?" >> gpurun_out/st_$TAG.txt
for r in 1 2; do timeout -s KILL 300 python scripts/attn_probe.py --heads 8,16,32,64 --flags 0,0x80 --decode --steps 100; done > gpurun_out/claim_ab_$TAG.jsonl 2>&1; echo "ab=$?" >> gpurun_out/st_$TAG.txt
cat gpurun_out/st_$TAG.txt
