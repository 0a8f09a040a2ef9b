#!/bin/bash
# Runs scripts/gemm_lab.cu on the GPU box, one variant per process (a hung
# variant is killed by its own 20 s timeout and the sweep continues).
set -u
out=${1:-gpurun_out/lab/lab.txt}
mkdir -p "$(dirname "$out")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/gemm_lab.cu -o /tmp/gemm_lab -lcuda || exit 1
echo "BN S CN ST skip ctas smemKB | graph_us iso_us exact" > "$out"
/tmp/gemm_lab list | while read -r bn s cn red skip; do
  timeout 20 /tmp/gemm_lab "$bn" "$s" "$cn" "$red" "$skip" >> "$out" 2>&1 || echo "$bn $s $cn $red $skip rc=$?" >> "$out"
done
