cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r02u_t.log 2>&1; echo "exit $?" >> gpurun_out/r02u_t.log
timeout 300 python bench.py --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_r02u_slab.json 2> gpurun_out/bench_r02u_slab.err
tail -4 gpurun_out/r02u_t.log; tail -c 600 gpurun_out/bench_r02u_slab.json
