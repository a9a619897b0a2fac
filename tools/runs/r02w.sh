cd $GRAFT_REPO_ROOT
timeout 300 python tools/quick_time.py gpurun_out/quick_time_r02w.json > gpurun_out/r02w_qt.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r02w_t.log 2>&1; echo "exit $?" >> gpurun_out/r02w_t.log
tail -3 gpurun_out/r02w_t.log; cat gpurun_out/r02w_qt.log
