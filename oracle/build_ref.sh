#!/bin/sh
# Stage the UNMODIFIED reference package for the CPU baseline (bench.py
# --impl reference and the cpu_baseline leg): a verbatim copy of
# /root/reference/pkg/src/sdftrace into oracle/_ref/ (git-ignored, so it stays
# out of history; not gpurun-ignored, so it travels to the GPU box, where
# /root/reference does not exist).  TEST/BASELINE INFRASTRUCTURE ONLY.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg/src/sdftrace}
if [ ! -d "$SRC" ]; then
  echo "reference not present ($SRC): keeping the existing oracle/_ref" >&2
  exit 0
fi
rm -rf "$HERE/_ref/sdftrace"
mkdir -p "$HERE/_ref"
cp -r "$SRC" "$HERE/_ref/sdftrace"
find "$HERE/_ref" -name __pycache__ -prune -exec rm -rf {} +
echo "staged $(ls "$HERE/_ref/sdftrace" | wc -l) files of the reference in oracle/_ref/sdftrace"
