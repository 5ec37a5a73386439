mkdir -p gpurun_out
# launch list of one bench run (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
echo "launches rc=$?"
# full sections of qk / select / pv (first launch of each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qk_kernel|select_kernel|pv_kernel" -c 3 \
  -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_bench.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out
