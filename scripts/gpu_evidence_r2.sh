#!/bin/bash
# Round-2 evidence run: scripts/gpu_final.sh (tests, smoke, bench c1-c5 + reference, ncu for c2/c3), then
# the probes of every row: per-rank scaling (c2, c3), the uneven c4 shares, head vs sequence split,
# migration, the graph-replayed stress, the step breakdown, the Eq. 3 / Eq. 4 fits, the N > 1 path at
# N = 1 (--force-dist, peer and NCCL exchanges) and the mbarrier sanitizer repro.
# usage: bash scripts/gpu_evidence_r2.sh <tag>
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r2f}
mkdir -p gpurun_out
bash scripts/gpu_final.sh $TAG
timeout -s KILL 600 python scripts/scaling_probe.py --config c3 > gpurun_out/scaling_${TAG}_c3.jsonl 2>&1
timeout -s KILL 600 python scripts/attn_probe.py --heads 8,16 --flags 0,0x20,0x60 --decode --steps 100 > gpurun_out/group_mode_${TAG}.jsonl 2>&1
timeout -s KILL 900 python scripts/scaling_probe.py --config c2 > gpurun_out/scaling_${TAG}_c2.jsonl 2>&1
timeout -s KILL 900 python scripts/scaling_probe.py --config c4 --shares > gpurun_out/c4_shares_${TAG}.jsonl 2>&1
timeout -s KILL 600 python scripts/seq_vs_head_probe.py --config c5 > gpurun_out/seq_vs_head_${TAG}_c5.jsonl 2>&1
timeout -s KILL 600 python scripts/seq_vs_head_probe.py --config c3 > gpurun_out/seq_vs_head_${TAG}_c3.jsonl 2>&1
timeout -s KILL 600 python scripts/migrate_probe.py > gpurun_out/migrate_${TAG}.jsonl 2>&1
timeout -s KILL 600 python scripts/stress_steps.py --replays 20 --steps 40 > gpurun_out/stress_${TAG}.txt 2>&1
timeout -s KILL 300 python scripts/step_breakdown.py --config c3 --ns 1,8 > gpurun_out/breakdown_${TAG}_c3.jsonl 2>&1
timeout -s KILL 900 python scripts/cost_model_fit.py --shape 13b > gpurun_out/cost_model_${TAG}_13b.json 2>&1
timeout -s KILL 900 python scripts/cost_model_fit.py --shape 70b --batch 64 > gpurun_out/cost_model_${TAG}_70b.json 2>&1
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29541 scripts/transfer_model_fit.py --exchange peer --share-gpu --grid 4 --steps 20 \
  > gpurun_out/transfer_fit_${TAG}_share.json 2> gpurun_out/transfer_fit_${TAG}_share.err
for X in "peer" "peer --pull 0" "nccl"; do
  N=$(echo $X | tr -d ' -')
  timeout -s KILL 400 python bench.py --config c3 --sub-config none --force-dist --exchange $X --steps 100 \
    --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_forcedist_$N.log 2>&1
done
bash scripts/sanitizer_repro/run.sh > /dev/null 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/clocks_${TAG}.txt 2>&1
echo evidence_done
