cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1901_07275_b200
JT_LIB=$L/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zh.txt 2>&1
timeout 900 python tools/ab_time.py $L/libjt_prev.so $L/libjt.so --configs cfg1_1d_1024,cfg2_2d_256,grid:128x128,grid:512x512,grid:4096 --rounds 2 --reps 200 > gpurun_out/ab_r02zh.txt 2>&1
cat gpurun_out/ab_r02zh.txt
grep -A9 "k0_i1 n256\|k0_i1 n1024" gpurun_out/phases_r02zh.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02zh.txt 2>&1; tail -3 gpurun_out/gputest_r02zh.txt
