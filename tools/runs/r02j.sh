cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err
timeout 300 python bench.py --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_r02j_slab.json 2> gpurun_out/bench_r02j_slab.err
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --slab --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02j_torchrun.json 2> gpurun_out/bench_r02j_torchrun.err
timeout 300 python bench.py --config cfg3_2d_4096 --no-cpu-baseline > gpurun_out/bench_r02j_cfg3.json 2> gpurun_out/bench_r02j_cfg3.err
timeout 300 python bench.py --config cfg4_3d_256 --no-cpu-baseline > gpurun_out/bench_r02j_cfg4.json 2> gpurun_out/bench_r02j_cfg4.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_r02j.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02j.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r02j.log 2>&1
python tools/prof_run.py cfg5_3d_512 > gpurun_out/r02j_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -s 1 -c 3 -o gpurun_out/prof_cfg5_r02j python tools/prof_run.py cfg5_3d_512 > gpurun_out/ncu_r02j.log 2>&1
cp paper_1901_07275_b200/libjt.so gpurun_out/libjt_r02j.so
tail -c 600 gpurun_out/bench_r02j.json; tail -c 800 gpurun_out/bench_r02j_torchrun.json; grep -c "NCCL INFO" gpurun_out/bench_r02j_torchrun.err
