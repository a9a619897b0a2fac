cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02za.txt 2>&1; tail -3 gpurun_out/gputest_r02za.txt
timeout 300 python tools/quick_time.py gpurun_out/quick_time_r02za.json > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/bench_r02za.json 2> gpurun_out/bench_r02za.err
tail -c 600 gpurun_out/bench_r02za.json
