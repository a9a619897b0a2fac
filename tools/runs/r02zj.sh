cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1901_07275_b200
JT_LIB=$L/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zj.txt 2>&1
grep -A12 "k0_i1 n256\|k0_i1 n1024" gpurun_out/phases_r02zj.txt
timeout 900 python tools/ab_time.py $L/libjt_pull.so $L/libjt.so --configs cfg1_1d_1024,cfg2_2d_256,grid:128x128,grid:512x512,grid:4096,grid:3x1024 --rounds 2 --reps 200 > gpurun_out/ab_r02zj.txt 2>&1
cat gpurun_out/ab_r02zj.txt
timeout 300 python tools/latency.py gpurun_out/latency_r02zj.json > /dev/null 2>&1
python - <<'P'
import json
d=json.load(open('gpurun_out/latency_r02zj.json'))
for k,v in d.items(): print(k, v['stream_us_per_call'], v['graph_us_per_call'], v['kernels_per_call'])
P
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02zj.txt 2>&1; tail -3 gpurun_out/gputest_r02zj.txt
