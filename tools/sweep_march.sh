#!/bin/bash
for lib in paper_1607_06283_b200/libevr.so build_variants/*.so; do
  for c in C3 C4 C5; do for p in f32 f64; do
    EVR_LIBRARY=$lib timeout 120 python bench.py --config $c --steps 20 --warmup 3 --engine streaming --precision $p --no-cpu-baseline > gpurun_out/sw.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$(basename $lib) $c $p', d['ms_per_step'])" 2>&1 | tail -1
  done; done
done
