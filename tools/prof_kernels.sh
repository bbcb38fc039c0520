#!/bin/bash
# ncu --set full captures of individual CSR-stream kernels on the c2 hierarchy.
# usage (on the GPU box): bash tools/prof_kernels.sh "L1.A:0:0" "L0.R:0:0" "L0.A:3:3"
#   each spec = matrix:kind:epi-template-value
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r mat kind epi <<< "$spec"
  tag="${mat/./_}_${kind}"
  timeout 300 ncu --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "regex:Epi\\)${epi}[,>]" -c 2 \
    -o "gpurun_out/prof_${tag}" python tools/kernel_bench.py --only "${mat}:${kind}" --reps 2 \
    > "gpurun_out/ncu_${tag}.log" 2>&1
done
