cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_twpre.so --configs cfg5_3d_512,cfg4_3d_256,grid:1024x1024x16,cfg3_2d_4096 --rounds 2 > gpurun_out/r02v_ab.txt 2>&1
cat gpurun_out/r02v_ab.txt
