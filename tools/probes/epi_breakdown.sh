#!/bin/bash
# Forward / input-gradient epilogue breakdown on the training step: launch
# list of one bench_train step with the debug-hook build and PNN_IGEMM_DEBUG
# bits (1 no conversion, 8 no TMEM loads, 16 no output stores, 2 no MMA, 4 no TMA).
# Results are wrong by design under the flags; only the times matter.
mkdir -p gpurun_out
for d in ${DEBUGS:-0 1 16 17 25 2 4}; do
  PNN_B200_LIB=build_exp/dbg/libpnn_b200.so PNN_IGEMM_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/epi_$d.csv -k regex:igemm_kernel \
    python tools/bench_train.py --configs 3b --steps 1 --warmup 0 > /dev/null 2>&1
  echo "== debug $d"
  python tools/ncu_summary.py sequence gpurun_out/epi_$d.csv | awk '$1 > 8'
done
