#!/bin/bash
# Build libevr.so variants with -D overrides into build_variants/ (tuning
# sweeps; select one with EVR_LIBRARY=build_variants/<name>.so).
# usage: tools/build_variants.sh "name:-DA=1 -DB=2" ...
cd "$(dirname "$0")/../paper_1607_06283_b200/csrc" || exit 1
mkdir -p ../../build_variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
    -fmad=false -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $defs -shared \
    -o ../../build_variants/$name.so evr_capi.cu evr_simulate.cu evr_events.cpp -lcudart 2>&1 | grep -iE "error" &
done
wait
