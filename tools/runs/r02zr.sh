cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 900 python tools/ab_time.py $L/libjt.so $L/libjt_jt_regs16m3_168.so $L/libjt_jt_regs16m4_144.so --configs nu_3d_256 --rounds 2 --reps 20 > gpurun_out/ab_r02zr.txt 2>&1
cat gpurun_out/ab_r02zr.txt
