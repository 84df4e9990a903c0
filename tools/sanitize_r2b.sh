#!/bin/bash
# compute-sanitizer over the round-2 kernels: the resident-hidden rows kernel
# (rows_hs_kernel: TMA ring, in-grid finalizer, record clearing) and the
# certified static half of the split decode (static_gemm_kernel with tcgen05,
# static_select_kernel, split_combine_cert_kernel).
# Usage: tools/sanitize_r2b.sh [outdir]   (run on the GPU box)
OUT=${1:-gpurun_out/sanitize_r2b}
mkdir -p "$OUT"
T1="tests/test_gpu_rows_hs.py"
K1="shapes or special_values or alternating"
T2="tests/test_gpu_parity.py"
K2="split_decode_matches"
for tool in memcheck synccheck racecheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis --kernel-name-exclude kns=gemv_ring_kernel"
  echo "== $tool" > "$OUT/$tool.log"
  for pair in "$T1|$K1" "$T2|$K2"; do
    t=${pair%%|*}; k=${pair#*|}
    timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --error-exitcode 99 \
       --target-processes all python -m pytest $t -q -x -k "$k" -p no:cacheprovider \
       >> "$OUT/$tool.log" 2>&1
    echo "exit=$? ($t -k $k)" >> "$OUT/$tool.log"
  done
  grep -E "ERROR SUMMARY|exit=|passed|failed" "$OUT/$tool.log" | tail -6
done
