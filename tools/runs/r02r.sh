cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r02r_t.log 2>&1; echo "exit $?" >> gpurun_out/r02r_t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02r_smoke.log
tail -3 gpurun_out/r02r_t.log; tail -2 gpurun_out/r02r_smoke.log
