#!/usr/bin/env bash
# ncu --set full (with source) of the two LDL^T sweep kernels on the bench workload.
#   bash tools/profile_sweeps.sh [tag] [workload]
set -u
TAG=${1:-r1}
WL=${2:-cfg2}
OUT=gpurun_out/ncu_${TAG}_${WL}
mkdir -p "$OUT"
CMD="python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu-baseline"
for k in lower_sweep upper_sweep; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${k}" -s 3 -c 1 \
      -o "$OUT/full_${k}" -f $CMD > "$OUT/full_${k}.log" 2>&1
  echo "$k rc=$?"
done
