cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/stage
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stage/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/stage/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], d['clocks'])
PY
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/stage/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|^E  " gpurun_out/stage/pytest.log | head -12
