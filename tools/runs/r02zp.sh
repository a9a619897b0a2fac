cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "512 or term_split or graph or repeat or determin" > gpurun_out/gputest_r02zp_quick.txt 2>&1; tail -3 gpurun_out/gputest_r02zp_quick.txt
timeout 900 python tools/ab_time.py $L/libjt_novtm.so $L/libjt.so --configs cfg5_3d_512,grid:512x512,grid:512x64x32 --rounds 2 --reps 20 > gpurun_out/ab_r02zp.txt 2>&1
cat gpurun_out/ab_r02zp.txt
