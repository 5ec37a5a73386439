#!/bin/bash
# ncu --set full of pv6 in the paper-like regime (c2, c3) and of qk5 / select at c3
mkdir -p gpurun_out
BENCH_ARGS="--scale 0.5" bash tools/ncu_set.sh "pv6_kernel" c2 pv6_c2s05 1
BENCH_ARGS="--scale 0.5" bash tools/ncu_set.sh "pv6_kernel" c3 pv6_c3s05 1
bash tools/ncu_set.sh "qk5_kernel" c3 qk5_c3 1
BENCH_ARGS="--scale 0.5" bash tools/ncu_set.sh "select_kernel" c3 sel_c3s05 1
ls -la gpurun_out
