#!/usr/bin/env bash
# ncu evidence for the device refactorisation (run under gpurun, 1 GPU).
#   bash tools/profile_refactor.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/ncu_refactor_${TAG}
mkdir -p "$OUT"
for WL in cfg2 cfg3; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
      --log-file "$OUT/launches_${WL}.csv" python tools/refactor_bench.py --workload $WL --reps 1 > "$OUT/launches_${WL}.log" 2>&1
  echo "launch list $WL rc=$?"
done
CMD="python tools/refactor_bench.py --workload cfg3 --reps 1"
for spec in "update_kernel:400" "diag_kernel:100" "tupdate_kernel:100" "extend_kernel:10"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${k}" -s "$s" -c 1 \
      -o "$OUT/full_${k}" -f $CMD > "$OUT/full_${k}.log" 2>&1
  echo "$k rc=$?"
done
ls "$OUT"
