cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zu
L=paper_1901_07275_b200/libjt.so
# auto k0 (20 at N = 4096, 24 at 2048 when the rank holds) vs the previous default 27
timeout 600 python tools/ab_time.py $L $L@27 --configs cfg3_2d_4096,grid:2048x2048 --reps 20 --rounds 2 > gpurun_out/ab_$T.txt 2>&1
cat gpurun_out/ab_$T.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -3 gpurun_out/gputest_$T.txt
timeout 300 python bench.py --config cfg3_2d_4096 --no-cpu-baseline > gpurun_out/bench_${T}_cfg3_2d_4096.json 2> gpurun_out/bench_${T}_cfg3.err
tail -c 600 gpurun_out/bench_${T}_cfg3_2d_4096.json
