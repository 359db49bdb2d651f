cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in "" "--skip 4"; do
timeout 600 python bench.py --steps 10 --warmup 3 $a > gpurun_out/bench$(echo $a | tr -d ' -').log 2>&1; echo "bench '$a' rc=$?"
python - "$a" <<'PY'
import json, sys
l=[x for x in open('gpurun_out/bench'+sys.argv[1].replace(' ','').replace('-','')+'.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', sys.argv[1], d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], 'e2e', d['e2e']['value'], d['gpu_launches'], d['clocks'], d.get('cpu_baseline',{}).get('value'), d.get('cpu_baseline',{}).get('kind'))
PY
done
