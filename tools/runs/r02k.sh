cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 600 python tools/ab_time.py $L/libjt.so $L/libjt_m3r168.so $L/libjt_nosub.so --configs nu_3d_256,cfg4_3d_256 --rounds 2 > gpurun_out/r02k_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu.py -q -x > gpurun_out/r02k_t.log 2>&1; echo "exit $?" >> gpurun_out/r02k_t.log
tail -3 gpurun_out/r02k_t.log; cat gpurun_out/r02k_ab.txt
