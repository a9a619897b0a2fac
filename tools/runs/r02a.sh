cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/r02a_dist.log 2>&1; echo "dist exit $?" >> gpurun_out/r02a_dist.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_dist.py > gpurun_out/r02a_gpu.log 2>&1; echo "gpu exit $?" >> gpurun_out/r02a_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 300 python bench.py --slab --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_slab.json 2> gpurun_out/r02a_slab.err
tail -3 gpurun_out/r02a_dist.log gpurun_out/r02a_gpu.log
