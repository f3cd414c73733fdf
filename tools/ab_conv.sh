#!/bin/bash
# A/B of the conv passes: the in-tree library vs an alternative build ($1).
alt=$1; shift
for fmt in 8,1 12,1; do
  echo "== base $fmt"; python tools/profile_conv.py --batch 1024 --fmt $fmt --algos 0 --iters 20 "$@"
  echo "== alt $fmt";  PNN_B200_LIB=$alt python tools/profile_conv.py --batch 1024 --fmt $fmt --algos 0 --iters 20 "$@"
done
