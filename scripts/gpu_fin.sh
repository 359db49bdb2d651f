cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_tc.py tests/test_gpu_relu_masks.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
TL_MARCH=1 timeout 400 python scripts/tile_timeline.py 2>&1 | grep -A75 "march (fluid" | grep -v "MMA: K" | tail -12
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bexp.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bexp.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], d['clocks']['sm_mhz'])
PY
