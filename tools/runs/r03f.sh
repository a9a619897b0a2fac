cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03f
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -k "checks" > gpurun_out/gputest_checks_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_checks_$T.txt
tail -12 gpurun_out/gputest_checks_$T.txt
timeout 600 python tools/latency.py > gpurun_out/latency_$T.json 2> gpurun_out/latency_$T.err; tail -c 600 gpurun_out/latency_$T.json
