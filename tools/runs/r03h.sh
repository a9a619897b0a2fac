cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03h
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -8 gpurun_out/gputest_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
tail -2 gpurun_out/smoke_$T.txt
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
head -c 600 gpurun_out/bench_$T.json
JT_CAPACITY_OUT=gpurun_out/capacity_$T.json timeout 900 python -m pytest tests/test_gpu_capacity.py -q > gpurun_out/capacity_$T.txt 2>&1; tail -3 gpurun_out/capacity_$T.txt; cat gpurun_out/capacity_$T.json
