cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1901_07275_b200
JT_LIB=$L/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zi.txt 2>&1
grep -A12 "k0_i1 n256\|k0_i1 n1024" gpurun_out/phases_r02zi.txt
tools/cluster_probe 256 111744; tools/cluster_probe 512 185472; tools/cluster_probe 256 205312
timeout 900 python tools/ab_time.py $L/libjt.so $L/libjt_noz.so $L/libjt_nowg.so --configs cfg1_1d_1024,cfg2_2d_256,cfg5_3d_512,cfg4_3d_256,cfg3_2d_4096 --rounds 2 --reps 20 > gpurun_out/ab_r02zi.txt 2>&1
cat gpurun_out/ab_r02zi.txt
