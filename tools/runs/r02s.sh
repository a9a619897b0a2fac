cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -k full_size > gpurun_out/r02s_t.log 2>&1; echo "exit $?" >> gpurun_out/r02s_t.log
JT_ACCURACY_OUT=gpurun_out/accuracy_r02s.json timeout 900 python -m pytest tests/test_accuracy_report.py -q > gpurun_out/r02s_acc.log 2>&1; echo "exit $?" >> gpurun_out/r02s_acc.log
tail -3 gpurun_out/r02s_t.log; tail -2 gpurun_out/r02s_acc.log
