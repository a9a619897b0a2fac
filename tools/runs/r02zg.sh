cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1901_07275_b200
JT_LIB=$L/libjt_phases.so timeout 300 python tools/phases.py cfg1_1d_1024 cfg2_2d_256 > gpurun_out/phases_r02zg.txt 2>&1
timeout 900 python tools/ab_time.py $L/libjt_head.so $L/libjt.so $L/libjt_wg4.so --configs cfg1_1d_1024,cfg2_2d_256,grid:128x128,grid:512x512,grid:64x64x64 --rounds 2 --reps 200 > gpurun_out/ab_r02zg.txt 2>&1
cat gpurun_out/ab_r02zg.txt
for lib in libjt.so libjt_wg4.so; do JT_LIB=$L/$lib timeout 300 python tools/latency.py gpurun_out/latency_r02zg_$lib.json > /dev/null 2>&1; done
python - <<'P'
import json
for lib in ['libjt.so','libjt_wg4.so']:
    d=json.load(open(f'gpurun_out/latency_r02zg_{lib}.json'))
    for k,v in d.items(): print(lib, k, v['stream_us_per_call'], v['graph_us_per_call'], v['kernels_per_call'])
P
cat gpurun_out/phases_r02zg.txt
