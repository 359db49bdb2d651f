set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/sanitize_cases.py tiny64 fp64 > gpurun_out/san/plain.log 2>&1; echo plain rc=$?
for tool in memcheck racecheck synccheck initcheck; do
  for c in "tiny64 fp64" "geo32s1 fp64" "geo64 fp16x3" "geo64 bf16x3"; do
    set -- $c
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py $1 $2 > gpurun_out/san/${tool}_$1_$2.log 2>&1
    echo "$tool $1 $2 rc=$?"
    tail -3 gpurun_out/san/${tool}_$1_$2.log
  done
done
