#!/bin/bash
# Round-2 full GPU pass: smoke, -m gpu tests, the driver's default bench (c2, with CPU baseline + e2e),
# reference arm, per-config lines (c3, c4, c2 paper-like, c5 sweep), launch list, ncu of the top kernels.
# Usage: bash tools/gpu_r2.sh [skip-tests]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
if [ "$1" != "skip-tests" ]; then
  timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
  tail -2 gpurun_out/smoke.log
  timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -4 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-300
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -1 gpurun_out/bench_ref.log | cut -c1-300
for a in "--config c3" "--config c4" "--config c2 --scale 0.5" "--config c3 --scale 0.5" "--config c1"; do
  f=gpurun_out/b_$(echo $a|tr -d ' -.').log
  timeout 400 python bench.py $a --steps 20 --warmup 5 --no-cpu-baseline > $f 2>&1
  python - "$f" "$a" <<'PY'
import json,sys
f=sys.argv[1]
try:
  d=json.loads(open(f).read().strip().splitlines()[-1])
  print(sys.argv[2], round(d['ms_per_step']*1000,1),'us frac', round(d.get('step_roofline_frac',0),3), 'speedup', round(d.get('speedup_vs_fp16_control',0),3), 'bytes',round(d.get('bytes_read_fraction',0),3), 'parity', d.get('parity',{}).get('mismatches'), {k:round(v*1000,1) for k,v in d.get('kernel_ms',{}).items()}, 'ctl', {k:round(v*1000,1) for k,v in d.get('kernel_ms_control',{}).items()})
except Exception as e: print(sys.argv[2], 'fail', e); print(open(f).read()[-2000:])
PY
done
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5.log 2>&1; echo "c5 rc=$?"
tail -1 gpurun_out/b_c5.log | cut -c1-400
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-validate > gpurun_out/launches_bench.log 2>&1
echo "launches rc=$?"
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"qk_kernel|select_kernel|pv6_kernel|append_token|combine" -c 5 \
  -o /tmp/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-validate > gpurun_out/prof_bench.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv 2>&1
ls -la gpurun_out | head -40
