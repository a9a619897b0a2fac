cd $GRAFT_REPO_ROOT
timeout 300 python tools/latency.py gpurun_out/latency_r02g.json cfg1_1d_1024 cfg2_2d_256 > gpurun_out/r02g_lat.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_t.log 2>&1; echo "exit $?" >> gpurun_out/r02g_t.log
timeout 300 python tools/quick_time.py gpurun_out/quick_time_r02g.json > gpurun_out/r02g_qt.log 2>&1
tail -3 gpurun_out/r02g_t.log; cat gpurun_out/r02g_lat.log; cat gpurun_out/r02g_qt.log
