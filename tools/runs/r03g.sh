cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03g
timeout 900 python -m pytest tests/test_gpu_pair.py -x -q -k "2048 or 2000 or full_compare" > gpurun_out/gputest_pair_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_pair_$T.txt
tail -8 gpurun_out/gputest_pair_$T.txt
timeout 1200 python tools/pair_check.py > gpurun_out/pair_$T.txt 2>&1
grep -o '"grid[^}]*}\|JT_PAIR=[01] [0-9]*' gpurun_out/pair_$T.txt
