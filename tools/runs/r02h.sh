cd $GRAFT_REPO_ROOT
timeout 300 python tools/latency.py gpurun_out/latency_r02h.json cfg1_1d_1024 cfg2_2d_256 > gpurun_out/r02h_lat.log 2>&1
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "term_split or 1d or last_launches or host or radix or config1" > gpurun_out/r02h_t.log 2>&1; echo "exit $?" >> gpurun_out/r02h_t.log
tail -3 gpurun_out/r02h_t.log; cat gpurun_out/r02h_lat.log
