#!/bin/bash
# float32 instruction-count switches (evr_math.cuh / evr_tile.cuh), built by tools/build_variants.sh
for v in ${VARS:-main m ms msi i}; do
  if [ $v = main ]; then L=paper_1607_06283_b200/libevr.so; else L=build_variants/$v.so; fi
  for rep in 1 2; do for c in C3 C4 C5 C2; do
    EVR_LIBRARY=$L timeout 300 python bench.py --config $c --precision f32 --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c f32', d['ms_per_step'], d['roofline']['frac'])"
  done; done
done
EVR_LIBRARY=build_variants/${TESTVAR:-msi}.so timeout 600 python -m pytest tests -m gpu -x -q -k "float32 or f32 or tile" > gpurun_out/pytest_f32var.log 2>&1; tail -3 gpurun_out/pytest_f32var.log
