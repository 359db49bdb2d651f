cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/fbias_probe.py > gpurun_out/fbias_cal.json 2>gpurun_out/fbias_cal.err; echo "probe rc=$?"; cat gpurun_out/fbias_cal.json; tail -3 gpurun_out/fbias_cal.err
timeout 900 python scripts/fullsize_parity.py --out gpurun_out/r02_fullsize_parity.jsonl > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"
python - <<'PY'
import json, collections
for l in open('gpurun_out/r02_fullsize_parity.jsonl'):
    s = json.loads(l)
    if 'out_of_band_rays' in s:
        c = collections.Counter((r['status_ref'], r['status'], (r['steps'] > r['steps_ref']) - (r['steps'] < r['steps_ref'])) for r in s['out_of_band_rays'])
        print(s['config'][:8], s.get('view', ''), s['precision'], 'oob', s['mismatch_out_of_band'], 'hit', s['hitmask_diff_out_of_band'], 'depth', '%.2e' % s['depth_rel_max'], 'n', s.get('normal_max', ''), dict(c))
    else:
        print(s)
PY
timeout 2000 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.log
