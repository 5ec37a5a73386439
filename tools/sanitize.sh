#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the smoke step and small GQA /
# forced-tier steps (race detection).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool smoke rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_cases.log 2>&1
  echo "$tool cases rc=$?"; tail -5 gpurun_out/sanitize_${tool}_cases.log
  AKV_QK_KERNEL=qk9 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_qk9.log 2>&1
  echo "$tool cases (qk9) rc=$?"; tail -2 gpurun_out/sanitize_${tool}_qk9.log
done
