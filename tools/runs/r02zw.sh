cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zw
L=paper_1901_07275_b200/libjt.so
V=build/var
# N = 4096 inverse: TMEM twiddles (B), + factor loads not first (C), + 4 twiddles per TMEM wait (D), loads-first off (E)
timeout 900 python tools/ab_time.py $L $V/libjt_B.so $V/libjt_C.so $V/libjt_D.so $V/libjt_E.so --configs cfg3_2d_4096,grid:2048x2048 --reps 20 --rounds 2 > gpurun_out/ab_$T.txt 2>&1
cat gpurun_out/ab_$T.txt
