#!/bin/bash
# float64 tile occupancy variants (rows per thread x CTAs per SM) on the headline shapes
for v in main r3m3 r2m3 r2m4 r4m2g6; do
  if [ $v = main ]; then L=$PWD/paper_1607_06283_b200/libevr.so; else L=$PWD/build_variants/$v.so; fi
  for c in C3 C4; do for k in 2 3 4; do
    EVR_LIBRARY=$L EVR_TILE_K=$k timeout 120 python bench.py --config $c --precision f64 --no-cpu-baseline --no-f32-leg --steps 60 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c K=$k', d['ms_per_step'], d['roofline']['kernel_us'])"
  done; done
done
