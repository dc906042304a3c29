#!/bin/bash
# Build the mbarrier hand-off repro and run every variant plain and under synccheck / racecheck.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
OUT=gpurun_out/mbar_repro.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o /tmp/mbar_handoff scripts/sanitizer_repro/mbar_handoff.cu || exit 1
: > $OUT
for v in 0 2 8 16 32 64 128 256 80 176; do
  echo "== variant $v" >> $OUT
  timeout -s KILL 60 /tmp/mbar_handoff $v >> $OUT 2>&1
  for tool in synccheck racecheck; do
    timeout -s KILL 300 $CS --tool $tool --print-limit 3 /tmp/mbar_handoff $v > /tmp/cs.log 2>&1
    echo "-- $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|variant' /tmp/cs.log | tr '\n' ' ')" >> $OUT
    grep -m3 -A3 -E 'Barrier error|hazard' /tmp/cs.log >> $OUT
  done
done
cat $OUT
