cd $GRAFT_REPO_ROOT
TL_MARCH=1 timeout 400 python scripts/tile_timeline.py 2>&1 | grep -A14 "march (fluid"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bexp.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bexp.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], d['clocks']['sm_mhz'])
PY
