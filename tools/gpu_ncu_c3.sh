#!/bin/bash
# ncu --set full of the c3 (GQA) step kernels: qk5, select, pv6
mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none -k regex:"qk5_kernel|select_kernel|pv6_kernel|append_token|combine" -c 5 \
  -o /tmp/prof_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-validate > gpurun_out/prof_c3.log 2>&1
echo "ncu c3 rc=$?"
ncu -i /tmp/prof_c3.ncu-rep --page raw --csv > gpurun_out/prof_c3_raw.csv 2>&1
