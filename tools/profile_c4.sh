#!/bin/bash
# C4 launch list + one ncu --set full capture per hot kernel (run through gpurun from the repo root).
# Each ncu step runs only after the same command exited 0 without ncu.  Development aid.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CFG=${CFG:-C4}
KERNELS=${KERNELS:-"rhals_sweeps_kernel tc_xht_resid_kernel tc_xw_kernel tc_xtw_kernel"}
timeout 900 python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_short_$CFG.json 2>&1 || { echo "short bench failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$CFG.csv \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$CFG.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/run_fit.py --config $CFG --fits 1 > $OUT/fit_$CFG.json 2>&1 || { echo "fit failed"; exit 1; }
for K in $KERNELS; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 \
    -o $OUT/${K}_${CFG} python tools/run_fit.py --config $CFG --fits 1 > $OUT/ncu_${K}_$CFG.log 2>&1
  echo "ncu $K rc=$?"
done
