#!/bin/bash
# A/B/C of the pv kernels: default (pv5) vs AKV_PV_KERNEL=pv4 vs pv3
for c in ${CFGS:-c2 c3}; do
  for mode in default pv4 pv3; do
    if [ $mode = default ]; then unset AKV_PV_KERNEL; else export AKV_PV_KERNEL=$mode; fi
    timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ab3_${c}_$mode.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab3_${c}_$mode.log').read().strip().splitlines()[-1])
print('$c $mode', round(d['ms_per_step']*1000,1),'us frac', round(d['step_roofline_frac'],3), 'speedup', round(d['speedup_vs_fp16_control'],3), 'parity', d['parity']['mismatches'], {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'ctl', {k:round(v*1000,1) for k,v in d['kernel_ms_control'].items()})" || tail -3 gpurun_out/ab3_${c}_$mode.log
  done
done
unset AKV_PV_KERNEL
