#!/bin/bash
# A/B over environment settings: AB_SETS="VAR=a,VAR2=b;VAR=c" CFGS="c2 c3" bash tools/ab_env.sh
mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${AB_SETS}"
for c in ${CFGS:-c2}; do
  for set in "${SETS[@]}"; do
    envs=$(echo "$set" | tr ',' ' ')
    tag=$(echo "${c}_$set" | tr -c 'A-Za-z0-9_' '_')
    env $envs timeout 400 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e --no-validate ${BENCH_ARGS} > gpurun_out/ab_$tag.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1])
print('$c [$set]', round(d['ms_per_step']*1000,1),'us frac', round(d['step_roofline_frac'],3), 'x', round(d['speedup_vs_fp16_control'],3), {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'ctl', {k:round(v*1000,1) for k,v in d['kernel_ms_control'].items()})" || tail -3 gpurun_out/ab_$tag.log
  done
done
