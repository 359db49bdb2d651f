cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 scripts/tc_rate_bench > gpurun_out/tc_rate.jsonl 2>&1; echo "tc_rate rc=$?"; cat gpurun_out/tc_rate.jsonl
python scripts/fbias_probe.py > gpurun_out/fbias_cal.json 2>gpurun_out/fbias_cal.err; echo "probe rc=$?"; head -c 1500 gpurun_out/fbias_cal.json; echo
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider -rA -k "graph or configs or refuses or nan or batched" > gpurun_out/pytest_sel.log 2>&1; echo "pytest-sel rc=$?"
grep -E "passed|failed|FAILED|ERROR|ms per iterate" gpurun_out/pytest_sel.log | tail -25
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'e2e', d['e2e']['value'], d['gpu_launches'], d['clocks'])
PY
