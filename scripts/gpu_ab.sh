# A/B two builds of libdist_b200.so on ONE box (box-to-box clocks differ by
# up to 10%): put them at ab_old/libA.so and ab_old/libB.so (git-ignored
# scratch), then
#   gpurun -- 'bash scripts/gpu_ab.sh'
# Each variant runs bench.py twice, interleaved; DIST_LIB_PATH selects the build.
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in A B; do
  DIST_LIB_PATH=$PWD/ab_old/lib$v.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python - $v <<'PY'
import json,sys
l=[x for x in open('gpurun_out/ab_%s.log' % sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print(sys.argv[1], 'bench', round(d['value']), round(d['ms_per_step'],2), 'trace', round(r['trace_ms_per_step'],2), 'obj', round(r['objective_ms_per_step'],2), d['clocks']['sm_mhz'])
PY
done; done
