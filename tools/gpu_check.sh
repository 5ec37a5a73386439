#!/bin/bash
# One GPU call: build check, smoke, the -m gpu suite, the default bench line (and optional extra bench args).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q --timeout 400 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -15
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-3000; tail -3 gpurun_out/bench.err
fi
