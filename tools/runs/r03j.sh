cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03j
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -6 gpurun_out/gputest_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
tail -1 gpurun_out/smoke_$T.txt
