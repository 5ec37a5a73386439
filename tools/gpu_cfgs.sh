#!/bin/bash
# quick per-config kernel times (no CPU baseline, no e2e)
for c in ${CFGS:-c2 c3}; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step']*1000,1),'us frac', round(d['step_roofline_frac'],3), 'speedup', round(d['speedup_vs_fp16_control'],3), {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'ctl', {k:round(v*1000,1) for k,v in d['kernel_ms_control'].items()})" || tail -3 gpurun_out/bench_$c.log
done
