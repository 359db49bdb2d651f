cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu.log | tail -25
timeout 900 python scripts/fullsize_parity.py --out gpurun_out/r02_fullsize_parity.jsonl > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --force-tiles --no-cpu-baseline > gpurun_out/bench_tiles.log 2>&1; echo "bench tiles rc=$?"
DIST_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2rank_gloo.log 2>&1; echo "bench 2-rank (one GPU, gloo, correctness only) rc=$?"
python - <<'PY'
import json
for f in ['bench.log','bench_tiles.log','bench_2rank_gloo.log']:
    l=[x for x in open('gpurun_out/'+f) if x.startswith('{')]
    if l:
        d=json.loads(l[-1]); r=d.get('roofline',{})
        print(f, d['value'], d['ms_per_step'], 'trace', r.get('trace_ms_per_step'), 'obj', r.get('objective_ms_per_step'), 'e2e', d.get('e2e',{}).get('value'), 'consistent', d.get('replicas_bit_identical'), d.get('scaling'))
PY
