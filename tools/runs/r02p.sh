cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
for lib in libjt_hs1.so libjt_nosub.so libjt_hs1.so libjt_nosub.so; do JT_LIB=$L/$lib timeout 300 python tools/e2e_ab.py cfg5_3d_512 8; done > gpurun_out/r02p.txt 2>&1
for lib in libjt_hs1.so libjt_nosub.so; do JT_LIB=$L/$lib timeout 300 python tools/e2e_ab.py cfg3_2d_4096 8; JT_LIB=$L/$lib timeout 300 python tools/e2e_ab.py cfg4_3d_256 8; done >> gpurun_out/r02p.txt 2>&1
cat gpurun_out/r02p.txt
