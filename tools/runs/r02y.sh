cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_r02y.json 2> gpurun_out/bench_r02y.err
timeout 300 python bench.py --config cfg3_2d_4096 --no-cpu-baseline > gpurun_out/bench_r02y_cfg3.json 2> gpurun_out/bench_r02y_cfg3.err
timeout 300 python bench.py --config cfg4_3d_256 --no-cpu-baseline > gpurun_out/bench_r02y_cfg4.json 2> gpurun_out/bench_r02y_cfg4.err
timeout 300 python bench.py --config nu_3d_256 --no-cpu-baseline > gpurun_out/bench_r02y_nu.json 2> gpurun_out/bench_r02y_nu.err
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_r02y_torchrun.json 2> gpurun_out/bench_r02y_torchrun.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_r02y_ref.json 2> gpurun_out/bench_r02y_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_r02y.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02y.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r02y.log 2>&1
python tools/prof_run.py cfg5_3d_512 > gpurun_out/r02y_plain2.log 2>&1 && python tools/prof_run.py cfg3_2d_4096 >> gpurun_out/r02y_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -s 1 -c 2 -o gpurun_out/prof_cfg5_r02y python tools/prof_run.py cfg5_3d_512 > gpurun_out/ncu_r02y.log 2>&1

for f in bench_r02y bench_r02y_cfg3 bench_r02y_cfg4 bench_r02y_nu bench_r02y_torchrun bench_r02y_ref; do echo $f; tail -c 300 gpurun_out/$f.json; echo; done
