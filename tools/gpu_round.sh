#!/bin/bash
# One GPU call: smoke, gpu parity tests, bench (default = the driver's command, with CPU baseline),
# reference arm, launch list, ncu of the hot kernels (CSV exports; the .ncu-rep stays on the box).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 150 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-200
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"qk_kernel|select_kernel|pv3_kernel|append_token|combine" -c 5 \
  -o /tmp/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_bench.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv 2>&1
ls -la gpurun_out
