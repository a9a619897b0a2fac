cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zt
L=paper_1901_07275_b200/libjt.so
# dense block width k0 vs rank at N >= 1024 (W V read through L1 at batch start: k0 x MAXR x NBINS x 8 B per line)
timeout 1200 python tools/ab_time.py $L@32 $L@27 $L@24 $L@20 $L@16 $L@12 $L@8 \
  --configs cfg3_2d_4096,grid:2048x2048,grid:1024x1024,cfg1_1d_1024 --reps 20 --rounds 2 > gpurun_out/ab_$T.txt 2>&1
cat gpurun_out/ab_$T.txt
