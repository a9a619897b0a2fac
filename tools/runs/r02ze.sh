cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1901_07275_b200
timeout 900 python tools/ab_time.py $L/libjt_head.so $L/libjt.so $L/libjt_nopdl.so --configs cfg1_1d_1024,cfg2_2d_256,cfg4_3d_256,cfg5_3d_512,cfg3_2d_4096,nu_3d_256 --rounds 2 > gpurun_out/ab_r02ze.txt 2>&1
cat gpurun_out/ab_r02ze.txt
timeout 300 python tools/latency.py gpurun_out/latency_r02ze.json > gpurun_out/latency_r02ze.log 2>&1
python - <<'P'
import json
d=json.load(open('gpurun_out/latency_r02ze.json'))
for k,v in d.items(): print(k, v['stream_us_per_call'], v['graph_us_per_call'], v['kernels_per_call'])
P
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02ze.txt 2>&1; tail -3 gpurun_out/gputest_r02ze.txt
