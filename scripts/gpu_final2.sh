cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final2/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final2/bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --skip 4 --no-cpu-baseline > gpurun_out/final2/bench_skip4.log 2>&1; echo "bench skip rc=$?"
python - <<'PY'
import json
for f in ['gpurun_out/final2/bench.log','gpurun_out/final2/bench_ref.log','gpurun_out/final2/bench_skip4.log']:
    l=[x for x in open(f) if x.startswith('{')]
    d=json.loads(l[-1])
    r=d.get('roofline',{})
    print(f, d['value'], d.get('ms_per_step'), r.get('trace_ms_per_step'), r.get('objective_ms_per_step'), r.get('frac'), d.get('e2e',{}).get('value'), d.get('clocks',{}).get('sm_mhz'), (d.get('cpu_baseline') or {}).get('value'))
PY
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final2/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final2/pytest.log
