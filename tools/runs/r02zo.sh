cd $GRAFT_REPO_ROOT
L=paper_1901_07275_b200
timeout 900 python tools/ab_time.py $L/libjt_twinv.so $L/libjt.so --configs cfg1_1d_1024,cfg2_2d_256,grid:128x128,grid:512x512,grid:64x64x64,grid:32x32x32,grid:4096,grid:3x1024,grid:7x256x5,cfg5_3d_512 --rounds 2 --reps 100 > gpurun_out/ab_r02zo.txt 2>&1
cat gpurun_out/ab_r02zo.txt
timeout 300 python tools/latency.py gpurun_out/latency_r02zo.json > /dev/null 2>&1
python - <<'P'
import json
d=json.load(open('gpurun_out/latency_r02zo.json'))
for k,v in d.items(): print(k, v['stream_us_per_call'], v['graph_us_per_call'], v['kernels_per_call'], v['graph_result_equal'])
P
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02zo.txt 2>&1; tail -3 gpurun_out/gputest_r02zo.txt
