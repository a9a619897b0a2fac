cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02zq.txt 2>&1; tail -3 gpurun_out/gputest_r02zq.txt
timeout 300 python tools/quick_time.py gpurun_out/quick_time_r02zq.json > /dev/null 2>&1
python - <<'P'
import json
d=json.load(open('gpurun_out/quick_time_r02zq.json'))
for k,v in d.items(): print(k, v['ms'])
P
