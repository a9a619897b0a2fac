cd $GRAFT_REPO_ROOT
timeout 300 python tools/latency.py gpurun_out/latency_r02f.json cfg1_1d_1024 cfg2_2d_256 > gpurun_out/r02f_lat.log 2>&1
python tools/latency.py /tmp/x.json cfg2_2d_256 > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f_lat.csv python tools/latency.py /tmp/y.json cfg2_2d_256 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_next.py tests/test_gpu_dist.py -q -x > gpurun_out/r02f_t.log 2>&1; echo "exit $?" >> gpurun_out/r02f_t.log
tail -3 gpurun_out/r02f_t.log; cat gpurun_out/r02f_lat.log
