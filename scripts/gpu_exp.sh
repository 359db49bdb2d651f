cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fluid.py tests/test_gpu_tc.py tests/test_gpu_relu_masks.py tests/test_gpu_skip_tc.py -x -q 2>&1 | tail -3
for d in 0 0; do DIST_TC_DEBUG=$d timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1; done
TL_MARCH=1 timeout 400 python scripts/tile_timeline.py > gpurun_out/tl_march2.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bexp.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bexp.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], d['clocks']['sm_mhz'])
PY
