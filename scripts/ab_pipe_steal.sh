#!/bin/bash
# A/B of the pipelined step with and without stealing (two library builds):
#   bash scripts/ab_pipe_steal.sh  (expects libs_ab/base.so and libs_ab/steal.so)
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined" 2>&1 | tail -3
timeout 300 python scripts/stress_steps.py --replays 5 --steps 20 2>&1 | tail -9
bash scripts/sweep_libs.sh "libs_ab/base.so libs_ab/steal.so" c3 "1,2,8" 3
bash scripts/sweep_libs.sh "libs_ab/base.so libs_ab/steal.so" c2 "1,8" 2
