cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02zv
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
for c in cfg4_3d_256 nu_3d_256 cfg1_1d_1024 cfg2_2d_256; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_${T}_torchrun.json 2> gpurun_out/bench_${T}_torchrun.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$T.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
python tools/prof_run.py cfg3_2d_4096 > gpurun_out/${T}_plain3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -c 4 -o gpurun_out/prof_cfg3_$T python tools/prof_run.py cfg3_2d_4096 > gpurun_out/ncu_cfg3_$T.log 2>&1
for f in bench_$T bench_${T}_cfg4_3d_256 bench_${T}_nu_3d_256 bench_${T}_cfg1_1d_1024 bench_${T}_cfg2_2d_256 bench_${T}_torchrun bench_${T}_ref; do echo $f; tail -c 300 gpurun_out/$f.json; echo; done
cat gpurun_out/smoke_$T.txt | tail -2
ls -la gpurun_out | tail -5
