cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r03e
timeout 900 python -m pytest tests/test_gpu_pair.py -x -q > gpurun_out/gputest_pair_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_pair_$T.txt
tail -5 gpurun_out/gputest_pair_$T.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_$T.txt 2>&1; echo "exit $?" >> gpurun_out/gputest_$T.txt
tail -8 gpurun_out/gputest_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1
tail -2 gpurun_out/smoke_$T.txt
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
for c in cfg3_2d_4096 cfg4_3d_256 nu_3d_256 cfg1_1d_1024 cfg2_2d_256; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --slab --steps 10 --no-cpu-baseline > gpurun_out/bench_${T}_torchrun.json 2> gpurun_out/bench_${T}_torchrun.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$T.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
python tools/prof_run.py cfg5_3d_512 > gpurun_out/${T}_plain5.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -s 1 -c 2 -o gpurun_out/prof_cfg5_$T python tools/prof_run.py cfg5_3d_512 > gpurun_out/ncu_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:inv_axis_kernel -s 1 -c 1 -o gpurun_out/prof_cfg5inv_$T python tools/prof_run.py cfg5_3d_512 > gpurun_out/ncu_inv_$T.log 2>&1
python tools/prof_run.py cfg3_2d_4096 > gpurun_out/${T}_plain3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:axis_kernel -c 4 -o gpurun_out/prof_cfg3_$T python tools/prof_run.py cfg3_2d_4096 > gpurun_out/ncu_cfg3_$T.log 2>&1
for f in bench_$T bench_${T}_cfg3_2d_4096 bench_${T}_cfg4_3d_256 bench_${T}_cfg2_2d_256 bench_${T}_torchrun; do echo $f; head -c 2300 gpurun_out/$f.json | tail -c 1700; echo; done
ls -la gpurun_out | tail -8
