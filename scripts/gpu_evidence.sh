#!/bin/bash
# Full evidence run for one tag: tests, smoke, bench lines + ncu (scripts/gpu_final.sh), then the
# probes of the next rows (scaling, head-vs-sequence split, migration).  usage: bash scripts/gpu_evidence.sh <tag>
cd "$GRAFT_REPO_ROOT"
TAG=${1:-final}
bash scripts/gpu_final.sh $TAG
timeout -s KILL 600 python scripts/scaling_probe.py --config c3 > gpurun_out/scaling_${TAG}_c3.jsonl 2>&1
timeout -s KILL 600 python scripts/scaling_probe.py --config c2 > gpurun_out/scaling_${TAG}_c2.jsonl 2>&1
timeout -s KILL 600 python scripts/seq_vs_head_probe.py --config c5 > gpurun_out/seq_vs_head_${TAG}_c5.jsonl 2>&1
timeout -s KILL 600 python scripts/seq_vs_head_probe.py --config c3 > gpurun_out/seq_vs_head_${TAG}_c3.jsonl 2>&1
timeout -s KILL 600 python scripts/migrate_probe.py > gpurun_out/migrate_${TAG}.jsonl 2>&1
timeout -s KILL 600 python scripts/stress_steps.py --replays 20 --steps 40 > gpurun_out/stress_${TAG}.txt 2>&1
timeout -s KILL 300 python scripts/step_breakdown.py --config c3 --ns 1,8 > gpurun_out/breakdown_${TAG}_c3.jsonl 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/clocks_${TAG}.txt 2>&1
echo evidence_done
