cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tworank
DIST_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/tworank/bench.log 2>&1; echo "2-rank bench rc=$?"
grep "^{" gpurun_out/tworank/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['scaling'], d['config']['parallelism'][:60], d['replicas_bit_identical'], d['n_gpus'])"
