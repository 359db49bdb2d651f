cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gain
python scripts/fbias_probe.py > gpurun_out/gain/fbias.json 2>gpurun_out/gain/fbias.err; echo "probe rc=$?"; cat gpurun_out/gain/fbias.json
for g in 1.0 1.000002 1.000004 1.000006 1.000008 1.000012; do
  DIST_TC_HEAD_GAIN=$g timeout 300 python scripts/fullsize_parity.py --precisions fp16x3 --c3-precisions fp16x3 --out gpurun_out/gain/g$g.jsonl > /dev/null 2>&1
  python - "$g" <<'PY'
import json, sys, collections
g = sys.argv[1]
L = [json.loads(l) for l in open(f'gpurun_out/gain/g{g}.jsonl')]
tot = collections.Counter(); oob = 0
for s in L:
    if 'out_of_band_rays' in s:
        oob += s['mismatch_out_of_band']
        for r in s['out_of_band_rays']:
            tot[(r['status_ref'], r['status'], (r['steps'] > r['steps_ref']) - (r['steps'] < r['steps_ref']))] += 1
print('gain', g, 'oob', oob, dict(tot), 'normal_max', [s.get('normal_max') for s in L if 'normal_max' in s], 'depth', max(s.get('depth_rel_max', 0) for s in L))
PY
done
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_heads.py -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu2.log | tail -12
