#!/bin/bash
# Measurement-aid variants of libakv (kernel-time decomposition, not shipped):
#   probe1: consumers skip compute  -> load-pipeline-bound time
#   probe2: producers skip plane loads -> consumer-bound time
set -e
cd "$(dirname "$0")/.."
mkdir -p build/probe
for v in 1 2 3; do
  objs=""
  for f in akv_append akv_qk akv_select akv_pv akv_api akv_analysis; do
    nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DAKV_PROBE=$v \
      -Iinclude -Ipaper_2409_16546_b200/csrc -c paper_2409_16546_b200/csrc/$f.cu -o build/probe/${f}_$v.o &
    objs="$objs build/probe/${f}_$v.o"
  done
  wait
  nvcc -gencode=arch=compute_100a,code=sm_100a -shared -o build/probe/libakv_probe$v.so $objs
done
ls -la build/probe/*.so
