cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zz2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -15 gpurun_out/gputest_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
tail -2 gpurun_out/smoke_$T.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
tail -c 2500 gpurun_out/bench_$T.json
