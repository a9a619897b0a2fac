cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_early.so --configs cfg5_3d_512,cfg4_3d_256,cfg3_2d_4096,grid:1024x1024x16,nu_3d_256 --rounds 3 > gpurun_out/r02i_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_next.py -q -x > gpurun_out/r02i_t.log 2>&1; echo "exit $?" >> gpurun_out/r02i_t.log
tail -3 gpurun_out/r02i_t.log; cat gpurun_out/r02i_ab.txt
