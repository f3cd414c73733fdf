#!/bin/bash
# ncu --set full of the igemm / act_digits kernels of ONE training step
# (config given as $1), exported to CSV on the box (the .ncu-rep itself is too
# large to bring back).  Run only after tools/train_launches.sh (the same
# command without ncu) exited 0.
set -e
cfg=${1:-3b}; tag=${2:-full}; regex=${3:-"igemm_kernel|act_digits"}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:${regex}" -o /tmp/${tag} -f \
    python tools/bench_train.py --configs $cfg --steps 1 --warmup 0 > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv
for k in "igemm_kernel<4" "igemm_kernel<6, 32, 1, 1, 4, unsigned short, 1" "act_digits_kernel<6"; do
  n=$(echo "$k" | tr -c 'a-zA-Z0-9' '_')
  ncu -i /tmp/${tag}.ncu-rep --page source --csv -k "regex:^${k}" -c 1 > gpurun_out/${tag}_src_${n}.csv 2>&1 || true
done
rm -f /tmp/${tag}.ncu-rep
ls -la gpurun_out/${tag}*
