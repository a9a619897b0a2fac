cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_wg512.so --configs cfg5_3d_512,grid:512x512x64 --rounds 2 > gpurun_out/r02q_ab.txt 2>&1
cat gpurun_out/r02q_ab.txt
