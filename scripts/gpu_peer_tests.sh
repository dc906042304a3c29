cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/t_peer.log 2>&1; echo "peer=$?" > gpurun_out/st.txt
timeout -s KILL 900 python -m pytest tests/test_gpu_bench.py -q -x -k "multirank" > gpurun_out/t_bench.log 2>&1; echo "bench=$?" >> gpurun_out/st.txt
cat gpurun_out/st.txt
