#!/bin/bash
# ncu --set full over one split decode step's kernels (cfg2): DRAM traffic
# and throughput of static_rows_kernel, the dynamic GEMV, its finalize and
# the combine. Run under gpurun; reads gpurun_out/split_full.ncu-rep after.
ncu --set full --clock-control none --import-source on \
    -k regex:"static_rows|gemv_ring|argmax_finalize|split_combine" -c 4 \
    -o gpurun_out/split_full python tools/split_only.py
