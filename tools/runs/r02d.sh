cd $GRAFT_REPO_ROOT
python tools/prof_run.py cfg3_2d_4096 > gpurun_out/r02d_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -c 4 -o gpurun_out/prof_cfg3_r02d python tools/prof_run.py cfg3_2d_4096 > gpurun_out/ncu_r02d.log 2>&1
cp paper_1901_07275_b200/libjt.so gpurun_out/libjt_r02d.so
tail -2 gpurun_out/ncu_r02d.log
