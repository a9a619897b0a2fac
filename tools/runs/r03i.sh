cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03i
timeout 900 python -m pytest tests/test_gpu_pair.py -q > gpurun_out/gputest_pair_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_pair_$T.txt
tail -6 gpurun_out/gputest_pair_$T.txt
timeout 600 python -m pytest tests/test_gpu.py -q -x > gpurun_out/gputest_main_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_main_$T.txt
tail -3 gpurun_out/gputest_main_$T.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
head -c 400 gpurun_out/bench_$T.json
