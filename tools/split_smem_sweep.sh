#!/bin/bash
# split decode per-step time across the GEMV ring budget and the static
# half's staging piece (co-residency of the two halves on an SM). Measured at
# cfg2 (us per step): 112 KB/96 29.9, 112 KB/48 26.8, 112 KB/32 27.2,
# 150 KB/48 26.8, 80 KB/96 31.8; full ring/96 32.5. 4-warp static CTAs
# (8 requests each) were slower: 27.7-35.8.
for cfg in "112000 96" "112000 48" "112000 32" "150000 48" "80000 96"; do
  set -- $cfg
  SVT_SPLIT_GEMV_SMEM=$1 SVT_SPLIT_PIECE=$2 timeout 300 python tools/time_split.py \
      > gpurun_out/split_b$1_p$2.json 2>/dev/null
done
