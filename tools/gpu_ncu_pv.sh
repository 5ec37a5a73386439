#!/bin/bash
mkdir -p gpurun_out
BENCH_ARGS="--scale 0.5" bash tools/ncu_set.sh "pv6_kernel" c2 pv6b_c2s05 1
BENCH_ARGS="--scale 0.5" bash tools/ncu_set.sh "pv6_kernel" c3 pv6b_c3s05 1
