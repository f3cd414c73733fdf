#!/bin/bash
# How much of the config-1 MMA kernels is the TMEM drain / the rounding?
# Needs build_exp/libpnn_b200_dbg.so (quire_gemm.cu built with -DPNN_GEMM_DEBUG_HOOKS).
# PNN_GEMM_DEBUG: 1 = no TMEM loads, 2 = no rounding / stores, 3 = both.
for d in 0 1 2 3; do
  echo -n "debug=$d "
  PNN_B200_LIB=$PWD/build_exp/libpnn_b200_dbg.so PNN_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train \
    | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:round(v['mma_ms'],4) for k,v in b['per_format'].items()})"
done
