#!/bin/bash
# Interleaved A/B of scripts/attn_probe.py over several library builds on one box:
#   bash scripts/exp_libs_probe.sh "<lib1> <lib2> ..." <heads> <out> [reps] [flags]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in $(seq 1 ${4:-2}); do for L in $1; do
HETIS_LIB=$PWD/$L timeout -s KILL 300 python scripts/attn_probe.py --heads $2 --flags ${5:-0} --decode --steps 100 2>&1 | grep '^{'
done; done > gpurun_out/$3
