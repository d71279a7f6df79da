#!/bin/bash
# Round profile on the GPU box (run through gpurun from the repo root):
#   1. bench.py (no profiler)                         -> gpurun_out/prof/bench.json
#   2. ncu launch list of the same bench command      -> gpurun_out/prof/launches.csv
#   3. ncu --set full of one launch of each hot kernel (sweeps, metrics, xw/xtw) -> *.ncu-rep
# Each ncu step runs only after its command exited 0 without ncu.  Development aid.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CFG=${CFG:-C4}
timeout 900 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err || { echo "bench failed"; tail $OUT/bench.err; exit 1; }
timeout 900 python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_short.json 2>&1 || { echo "short bench failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/run_fit.py --config $CFG --fits 1 > $OUT/fit.json 2>&1 || { echo "fit failed"; exit 1; }
for K in rhals_sweeps_kernel tc_xht_resid_w_kernel tc_xw_kernel tc_xtw_kernel; do
  timeout 900 ncu --set full --clock-control none -k regex:$K -s 1 -c 1 \
    -o $OUT/${K}_${CFG} python tools/run_fit.py --config $CFG --fits 1 > $OUT/ncu_${K}.log 2>&1
  echo "ncu $K rc=$?"
done
# other configs (bench lines) and the accuracy / streaming probes
for C2 in C2 C3 C1 C5; do
  timeout 600 python bench.py --config $C2 --steps 3 --no-cpu-baseline > $OUT/bench_$C2.json 2> $OUT/bench_$C2.err
  echo "bench $C2 rc=$?"
done
[ -x tools/sketch_acc ] && ./tools/sketch_acc 32256 2410 36 10 > $OUT/sketch_acc_c2.txt 2>&1
timeout 600 python tools/bench_streaming.py > $OUT/streaming_c2.json 2>&1
echo "streaming rc=$?"
