bash tools/gpu_check.sh
for a in "--config c3" "--config c4" "--config c2 --scale 0.5"; do
  timeout 400 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$(echo $a|tr -d ' -.').log 2>&1
  python - "$a" <<'PY'
import json,sys,glob
f='gpurun_out/b_'+sys.argv[1].replace(' ','').replace('-','').replace('.','')+'.log'
try:
  d=json.loads(open(f).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1),'us frac', round(d['step_roofline_frac'],3), 'speedup', round(d['speedup_vs_fp16_control'],3), 'bytes',round(d['bytes_read_fraction'],3), d.get('avg_bits'), 'parity', d['parity'], {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'ctl', {k:round(v*1000,1) for k,v in d['kernel_ms_control'].items()})
except Exception as e: print(sys.argv[1], 'fail', e); print(open(f).read()[-2000:])
PY
done
