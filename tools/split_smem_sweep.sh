#!/bin/bash
# split decode per-step time across the GEMV ring budget and the static
# half's staging piece (co-residency of the two halves on an SM)
for cfg in "112000 96" "112000 48" "112000 32" "150000 48" "80000 96"; do
  set -- $cfg
  SVT_SPLIT_GEMV_SMEM=$1 SVT_SPLIT_PIECE=$2 timeout 300 python tools/time_split.py > gpurun_out/split_b$1_p$2.json 2>/dev/null
done
