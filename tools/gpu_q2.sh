#!/bin/bash
# quick GPU iteration: -m gpu tests (unless NOTEST) + kernel breakdown for each bench arg set in RUNS (';'-separated)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_gpu.log | tail -5
fi
IFS=';' read -ra R <<< "${RUNS:---config c2;--config c3;--config c2 --scale 0.5;--config c3 --scale 0.5}"
for a in "${R[@]}"; do
  f=gpurun_out/q_$(echo $a|tr -d ' -.').log
  timeout 400 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${EXTRA} > $f 2>&1
  python - "$f" "$a" <<'PY'
import json,sys
f=sys.argv[1]
try:
  d=json.loads(open(f).read().strip().splitlines()[-1])
  print(sys.argv[2], '|', round(d['ms_per_step']*1000,1),'us frac', round(d.get('step_roofline_frac',0),3), 'x', round(d.get('speedup_vs_fp16_control',0),3), 'B',round(d.get('bytes_read_fraction',0),3), 'par', d.get('parity',{}).get('mismatches'), d.get('parity',{}).get('knife_edges'), {k:round(v*1000,1) for k,v in d.get('kernel_ms',{}).items()}, 'ctl', {k:round(v*1000,1) for k,v in d.get('kernel_ms_control',{}).items()})
except Exception as e: print(sys.argv[2], 'fail', e); print(open(f).read()[-1500:])
PY
done
