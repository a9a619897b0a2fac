cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 900 python tools/ab_time.py $L/libjt.so $L/libjt_twinv.so --configs cfg5_3d_512,grid:128x128x128,grid:1024x1024,cfg4_3d_256 --rounds 2 --reps 20 > gpurun_out/ab_r02zn.txt 2>&1
cat gpurun_out/ab_r02zn.txt
