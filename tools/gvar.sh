#!/bin/bash
# tile CTA shape sweep: warps per CTA (G) x CTAs per SM, built by tools/build_variants.sh
for v in ${VARS:-main g16 g12}; do
  if [ $v = main ]; then L=paper_1607_06283_b200/libevr.so; else L=build_variants/$v.so; fi
  for c in C3 C4 C5; do for p in f32 f64; do
    EVR_LIBRARY=$L timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c $p', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'][:90])"
  done; done
done
