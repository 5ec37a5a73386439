#!/bin/bash
# ncu --set full of the first launch of kernels matching $1 (one bench step)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} \
  -o gpurun_out/prof_${3:-one} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_${3:-one}.log 2>&1
echo "ncu rc=$?"
