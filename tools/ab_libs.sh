#!/bin/bash
# A/B of libakv builds in one GPU call: for each build/ab/<name>.so (LIBS, space-separated names),
# install it as the package library and run the bench arg sets in RUNS (';'-separated), REPS times.
mkdir -p gpurun_out
LIB=paper_2409_16546_b200/libakv.so
cp $LIB /tmp/libakv_orig.so
IFS=';' read -ra R <<< "${RUNS:---config c2}"
for rep in $(seq ${REPS:-1}); do
for name in $LIBS; do
  cp build/ab/$name.so $LIB
  for a in "${R[@]}"; do
    f=gpurun_out/ab_${name}_$(echo $a|tr -d ' -.').log
    timeout 400 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-validate ${EXTRA} > $f 2>&1
    python - "$f" "$name $a" <<'PY'
import json,sys
f=sys.argv[1]
try:
  d=json.loads(open(f).read().strip().splitlines()[-1])
  print(sys.argv[2], '|', round(d['ms_per_step']*1000,1),'us x', round(d.get('speedup_vs_fp16_control',0),3), {k:round(v*1000,1) for k,v in d.get('kernel_ms',{}).items()}, 'ctl', {k:round(v*1000,1) for k,v in d.get('kernel_ms_control',{}).items()})
except Exception as e: print(sys.argv[2], 'fail', e); print(open(f).read()[-1500:])
PY
  done
done
done
cp /tmp/libakv_orig.so $LIB
