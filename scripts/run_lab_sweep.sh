#!/bin/bash
# gemm_lab sweep: one process per variant ("BN S CN ST skip"), 20 s cap each.
out=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/gemm_lab.cu -o /tmp/gemm_lab -lcuda || exit 1
mkdir -p "$(dirname "$out")"
echo "BN S CN ST skip ctas smemKB | graph_us(median) iso_us exact" > "$out"
for v in "$@"; do timeout 20 /tmp/gemm_lab $v >> "$out" 2>&1 || echo "$v rc=$?" >> "$out"; done
