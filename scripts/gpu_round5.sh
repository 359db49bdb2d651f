cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_skip_tc.py tests/test_gpu_edge_cases.py tests/test_gpu_multishape_skip.py -q -m gpu --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_skip.log 2>&1; echo "pytest-skip rc=$?"
grep -E "passed|failed|FAILED|ERROR|^E  " gpurun_out/pytest_skip.log | head -30
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'e2e', d['e2e']['value'], d['gpu_launches'], d['clocks'])
PY
