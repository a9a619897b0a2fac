cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_lg2.so --configs cfg3_2d_4096,grid:4096x512 --rounds 2 > gpurun_out/r02l_ab.txt 2>&1
cat gpurun_out/r02l_ab.txt
