#!/bin/bash
# quick GPU iteration: smoke + gpu tests + per-config kernel times
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q --timeout 150 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CFGS=${CFGS:-c2} bash tools/gpu_cfgs.sh
