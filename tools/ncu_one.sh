#!/bin/bash
# ncu (speed-of-light, memory, warp state, source counters) of kernels matching $1 in one bench step;
# exports raw metrics + SASS source counters as CSV (the .ncu-rep embeds the whole module and is too big to ship back)
mkdir -p gpurun_out
tag=${3:-one}
timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SourceCounters \
  --section LaunchStats --section Occupancy --clock-control none -k regex:"$1" -c ${2:-1} \
  -o /tmp/prof_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/prof_$tag.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_sass.csv 2>&1
ls -la gpurun_out/
