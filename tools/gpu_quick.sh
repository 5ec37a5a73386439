#!/bin/bash
# quick GPU iteration: smoke + gpu tests + probe decomposition (bench kernel times) + QK ring accounting
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q --timeout 150 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
bash tools/probe_run.sh
# timeout 300 python tools/probe3.py
