cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/r02t_t.log 2>&1; echo "exit $?" >> gpurun_out/r02t_t.log
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "nccl or chunk_major or split" >> gpurun_out/r02t_t.log 2>&1; echo "exit $?" >> gpurun_out/r02t_t.log
timeout 300 python bench.py --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_r02t_slab.json 2> gpurun_out/bench_r02t_slab.err
tail -5 gpurun_out/r02t_t.log; tail -c 700 gpurun_out/bench_r02t_slab.json
