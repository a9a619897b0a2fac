cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
JT_LIB=paper_1901_07275_b200/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zb.txt 2>&1
cat gpurun_out/phases_r02zb.txt
