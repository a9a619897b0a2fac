cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
JT_LIB=paper_1901_07275_b200/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zf.txt 2>&1
cat gpurun_out/phases_r02zf.txt
timeout 300 python tools/latency.py gpurun_out/latency_r02zf.json > gpurun_out/latency_r02zf.log 2>&1
python - <<'P'
import json
d=json.load(open('gpurun_out/latency_r02zf.json'))
for k,v in d.items(): print(k, v['stream_us_per_call'], v['graph_us_per_call'], v['kernels_per_call'])
P
