#!/bin/bash
# ncu --set full (with SASS source) of ONE launch of a kernel matching $1
# (skip $2 matching launches first) in a bench_train step of config $3;
# exports raw / details / source CSVs into gpurun_out/<tag>_*.
set -e
regex=$1; skip=${2:-0}; cfg=${3:-3b}; tag=${4:-one}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:${regex}" -s ${skip} -c 1 -o /tmp/${tag} -f \
    python tools/bench_train.py --configs $cfg --steps 1 --warmup 0 > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
rm -f /tmp/${tag}.ncu-rep
