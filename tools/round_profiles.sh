#!/bin/bash
# Round-end measurement set (GPU box): bench line + reference arm, the bench's
# ncu launch list, one `ncu --set full` capture of each config-1 GEMM, the
# training-step launch list and all BASELINE training configs.  Every ncu pass
# runs only after the same command exited 0 without ncu.
#   bash tools/round_profiles.sh r02
set -e
tag=${1:-r02}
mkdir -p gpurun_out
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${tag}.txt
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}_reference.json
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-train > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-train > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_${tag}_bench.csv > gpurun_out/launches_${tag}_bench.json
python tools/profile_gemm.py > /dev/null
for fmt in 16,1 8,0; do
  n=${fmt/,/}
  skip=0; [ $fmt = 16,1 ] && skip=1  # (16,1): the first launch is the 4-digit variant, which exits
  ncu --set full --import-source on --clock-control none -k regex:quire_gemm_tc_kernel -s $skip -c 1 \
      -o /tmp/prof_${tag}_p$n -f python tools/profile_gemm.py $fmt > /dev/null 2>&1
done
python tools/ncu_summary.py report /tmp/prof_${tag}_p161.ncu-rep /tmp/prof_${tag}_p80.ncu-rep > gpurun_out/ncu_full_${tag}.json
python tools/bench_train.py --configs 0,2,3,4a,4b,4c,4d,3b --steps 10 --warmup 3 --graph > gpurun_out/train_${tag}_graph.jsonl
bash tools/train_launches.sh 3b train_${tag} > /dev/null 2>&1
python tools/ncu_summary.py sequence gpurun_out/train_${tag}_launches.csv > gpurun_out/train_${tag}_sequence.txt
echo done
