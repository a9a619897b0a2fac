cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_nosub.so $L/libjt_vu4.so $L/libjt_vu1.so $L/libjt.so@32 --configs cfg3_2d_4096,grid:2048x2048,grid:1024x1024x16,cfg5_3d_512 --rounds 2 > gpurun_out/r02e_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_next.py -q -x > gpurun_out/r02e_t.log 2>&1; echo "exit $?" >> gpurun_out/r02e_t.log
tail -3 gpurun_out/r02e_t.log; cat gpurun_out/r02e_ab.txt
