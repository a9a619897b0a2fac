cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02n_t.log 2>&1; echo "exit $?" >> gpurun_out/r02n_t.log
tail -3 gpurun_out/r02n_t.log
