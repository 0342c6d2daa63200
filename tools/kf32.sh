#!/bin/bash
# float32 tiles: iterations per launch (EVR_TILE_K) after the instruction cuts
for c in C3 C4 C5; do for k in ${KS:-4 5 6}; do
  EVR_TILE_K=$k timeout 300 python bench.py --config $c --precision f32 --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c f32 K=$k', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'][40:100])"
done; done
