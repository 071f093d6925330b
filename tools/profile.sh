#!/usr/bin/env bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU).
#   bash tools/profile.sh [tag] [workload] [kernels...]
# 1) launch list (gpu__time_duration per launch) of a short bench run
# 2) one --set full capture per hot kernel (-lineinfo build => source page)
set -u
TAG=${1:-r1}
WL=${2:-cfg2}
shift 2 || true
KERNELS=${*:-"pcg_persistent<(int)2>:8 pcg_persistent<(int)1>:8 lower_sweep:3 upper_sweep:3 elem_kernel:10 gather_kernel:10 spmv_kernel:3"}
OUT=gpurun_out/ncu_${TAG}_${WL}
mkdir -p "$OUT"
CMD="python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$OUT/launches.csv" $CMD > "$OUT/launches.log" 2>&1
echo "launch list rc=$?"
for spec in $KERNELS; do
  k=${spec%%:*}; s=${spec##*:}
  name=$(echo "$k" | tr -c 'a-zA-Z0-9_\n' '_')
  kre=$(echo "$k" | sed 's/[()<>]/./g')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${kre}" -s "$s" -c 1 -o "$OUT/full_${name}" -f $CMD > "$OUT/full_${name}.log" 2>&1
  echo "$k rc=$?"
done
ls "$OUT"
