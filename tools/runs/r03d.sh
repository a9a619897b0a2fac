cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03d
timeout 1200 python tools/pair_check.py > gpurun_out/pair_$T.txt 2>&1
cat gpurun_out/pair_$T.txt
