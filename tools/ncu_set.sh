#!/bin/bash
# ncu --set full --import-source of kernels matching $1 in one bench step of config $2; CSV exports
# (raw metrics + SASS source counters) into gpurun_out/ (the .ncu-rep stays on the box).
mkdir -p gpurun_out
tag=$3
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"$1" -c ${4:-1} \
  -o /tmp/prof_$tag python bench.py --config $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-validate ${BENCH_ARGS} > gpurun_out/prof_$tag.log 2>&1
echo "ncu $tag rc=$?"
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_sass.csv 2>&1
