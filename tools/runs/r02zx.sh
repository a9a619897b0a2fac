cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zx
L=paper_1901_07275_b200/libjt.so
# inverse (N <= 512): paired (W V)^T y warp reduction (default) vs two separate reductions (P0)
timeout 900 python tools/ab_time.py $L build/var/libjt_P0.so --configs cfg5_3d_512,cfg4_3d_256,cfg2_2d_256,grid:128x128x128 --reps 20 --rounds 3 > gpurun_out/ab_$T.txt 2>&1
cat gpurun_out/ab_$T.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -3 gpurun_out/gputest_$T.txt
