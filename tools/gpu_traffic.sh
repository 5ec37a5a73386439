#!/bin/bash
# DRAM read + write of the dominant kernel per config (ncu, one launch each) for roofline.traffic
mkdir -p gpurun_out
run() {  # regex config tag extra-args
  timeout 600 ncu -f --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"$1" -c 1 --csv \
    python bench.py --config $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-validate $4 > gpurun_out/traffic_$3.csv 2>gpurun_out/traffic_$3.err
  echo "$3 rc=$?"
}
run "qk5_kernel" c3 c3_qk ""
run "qk_kernel" c4 c4_qk ""
run "pv6_kernel" c2 c2s05_pv "--scale 0.5"
run "pv6_kernel" c3 c3s05_pv "--scale 0.5"
run "qk_kernel" c2 c2_qk ""
