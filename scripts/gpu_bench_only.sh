cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bo
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bo/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bo/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], d['clocks'])
PY
timeout 900 python -m pytest tests/test_gpu_heads.py tests/test_gpu_relu_masks.py tests/test_gpu_tc.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
