for v in 0; do
  if [ $v = 0 ]; then unset AKV_LIB_PROBE; else export AKV_LIB_PROBE=build/probe/libakv_$v.so; fi
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/probe$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/probe$v.log').read().strip().splitlines()[-1])
print('probe $v', 'aligned', {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'control', {k:round(v*1000,1) for k,v in d['kernel_ms_control'].items()}, 'bytes', round(d['bytes_read_fraction'],3))" || tail -5 gpurun_out/probe$v.log
done
