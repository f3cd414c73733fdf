#!/bin/bash
# Launch list (per-kernel device time, ncu gpu__time_duration, cold/serialised)
# of training steps: first the same command without ncu (must exit 0), then
# under ncu.  Usage (GPU box): tools/train_launches.sh <config> <tag>
set -e
cfg=${1:-3b}; tag=${2:-train}
mkdir -p gpurun_out
python tools/bench_train.py --configs $cfg --steps 5 --warmup 3 --graph > gpurun_out/${tag}_bench.json
python tools/bench_train.py --configs $cfg --steps 2 --warmup 1 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python tools/bench_train.py --configs $cfg --steps 2 --warmup 1 > gpurun_out/${tag}_ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_summary.json
