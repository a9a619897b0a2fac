cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
for lib in libjt.so libjt_nosub.so libjt.so libjt_nosub.so; do JT_LIB=$L/$lib timeout 300 python tools/e2e_ab.py cfg5_3d_512 8; JT_LIB=$L/$lib timeout 300 python tools/e2e_ab.py cfg4_3d_256 8; done > gpurun_out/r02z.txt 2>&1
cat gpurun_out/r02z.txt
