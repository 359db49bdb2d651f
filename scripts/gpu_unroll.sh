cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/unroll
for d in 0 2; do DIST_TC_DEBUG=$d timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/unroll/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/unroll/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], d['clocks'])
PY
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/unroll/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|^E  " gpurun_out/unroll/pytest.log | head -12
