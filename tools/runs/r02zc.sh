cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
JT_LIB=paper_1901_07275_b200/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zc.txt 2>&1
timeout 300 python tools/latency.py gpurun_out/latency_r02zc.json > gpurun_out/latency_r02zc.log 2>&1
timeout 300 python tools/quick_time.py gpurun_out/quick_time_r02zc.json > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02zc.txt 2>&1; tail -3 gpurun_out/gputest_r02zc.txt
cat gpurun_out/phases_r02zc.txt; cat gpurun_out/latency_r02zc.json
python - <<'P'
import json
d=json.load(open('gpurun_out/quick_time_r02zc.json'))
for k,v in d.items(): print(k, v['ms'])
P
