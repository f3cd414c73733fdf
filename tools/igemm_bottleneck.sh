#!/bin/bash
# Profiling experiment: device time of the implicit conv kernels with parts of
# the pipeline disabled (PNN_IGEMM_DEBUG bits: 1 no quire->posit conversion,
# 2 no MMA, 4 no TMA operand loads).  Results are wrong by design under the
# flag; only the launch times (ncu launch list) are of interest.
#   bash tools/igemm_bottleneck.sh <fmt> <layer>      e.g.  12,1 conv2
fmt=${1:-12,1}; layer=${2:-conv2}
mkdir -p gpurun_out
for d in ${DEBUGS:-0 1 2 4 3 7}; do
  PNN_IGEMM_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/dbg_${layer}_$d.csv python tools/profile_conv.py --fmt $fmt --layers $layer \
    --iters 1 --algos 0 > /dev/null 2>&1
done
