cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 300 python tools/ab_time.py $L/libjt.so $L/libjt_nosub.so --configs cfg3_2d_4096,grid:4096x512 --rounds 3 > gpurun_out/r02c_ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "4096 or cfg3 or 3000 or repeat or term_split or radix" > gpurun_out/r02c_t.log 2>&1; echo "exit $?" >> gpurun_out/r02c_t.log
tail -3 gpurun_out/r02c_t.log; cat gpurun_out/r02c_ab.txt
