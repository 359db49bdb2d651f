# one gpurun call: GPU tests, timeline, a short bench (args: extra pytest selection)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_SEL:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -25
if [ -n "$TIMELINE" ]; then timeout 600 python scripts/tile_timeline.py > gpurun_out/timeline.log 2>&1; echo "timeline rc=$?"; grep -E "tile|colsum" gpurun_out/timeline.log | head -20; fi
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); r=d.get('roofline',{})
    print('bench', d['value'], d['ms_per_step'], 'trace', r.get('trace_ms_per_step'), 'obj', r.get('objective_ms_per_step'), 'e2e', d.get('e2e',{}).get('value'))
PY
