#!/bin/bash
# ncu --set full (with SASS source) of the config-1 pack kernels: one launch of
# the A (row-major) and B (column-major) pack per format; details / source CSVs
# into gpurun_out/<tag>_pack_<fmt>_<k>_*.  bash tools/ncu_pack.sh r02
tag=${1:-pack}
mkdir -p gpurun_out
python tools/profile_gemm.py > /dev/null || exit 1
for fmt in 16,1 8,0; do
  n=${fmt/,/}
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k regex:pack_ -s 2 -c 2 -o /tmp/${tag}_p$n -f python tools/profile_gemm.py $fmt > gpurun_out/${tag}_p${n}_ncu.log 2>&1
  ncu -i /tmp/${tag}_p$n.ncu-rep --page details --csv > gpurun_out/${tag}_pack_p${n}_details.csv
  ncu -i /tmp/${tag}_p$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_pack_p${n}_sass.csv
  ncu -i /tmp/${tag}_p$n.ncu-rep --page raw --csv > gpurun_out/${tag}_pack_p${n}_raw.csv
done
echo done
