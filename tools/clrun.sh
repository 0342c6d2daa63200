#!/bin/bash
# A/B of the clustered primal-dual tiles (EVR_TILE_CLUSTER) on the float64 headline shapes.
for cl in none 2x2 4x2 2x4; do
  if [ $cl = none ]; then unset EVR_TILE_CLUSTER; else export EVR_TILE_CLUSTER=$cl; fi
  timeout 300 python -m pytest tests/test_gpu_long_chains.py -x -q -k "c3_float64" 2>&1 | tail -1
  for c in C3 C4 C5; do for k in 3 4; do
    EVR_TILE_K=$k timeout 120 python bench.py --config $c --precision f64 --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cl $c f64 K=$k', d['ms_per_step'], d['roofline']['frac'])"
  done; done
done
