#!/usr/bin/env bash
# Round-2 ncu evidence (run under gpurun, 1 GPU): launch list of the bench
# command and one --set full capture per hot kernel via tools/ncu_driver.py.
#   bash tools/profile_r2.sh [tag] [workload]
set -u
TAG=${1:-r2}
WL=${2:-cfg3}
OUT=gpurun_out/ncu_${TAG}_${WL}
mkdir -p "$OUT"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --workload "$WL" --steps 3 --warmup 3 --no-cpu-baseline \
    > "$OUT/launches.log" 2>&1
echo "launch list rc=$?"
for spec in elem_kernel:1 gather_kernel:1 spmv_kernel:1 lower_sweep:1 upper_sweep:1 "pcg_persistent<(int)1:1" "pcg_persistent<(int)2:1"; do
  k=${spec%%:*}; s=${spec##*:}
  name=$(echo "$k" | tr -c 'a-zA-Z0-9_\n' '_')
  kre=$(echo "$k" | sed 's/[()<>]/./g')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${kre}" -s "$s" -c 1 -o "$OUT/full_${name}" -f python tools/ncu_driver.py --workload "$WL" \
      > "$OUT/full_${name}.log" 2>&1
  echo "$k rc=$?"
done
ls "$OUT"
