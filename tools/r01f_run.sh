#!/bin/bash
# round-1f check: full gpu suite + C3/C4/C5 bench lines in both precisions
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/bench_r01f
for c in C3 C4 C5; do for p in f32 f64; do
  timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/bench_r01f/bench_${c}_$p.json 2>gpurun_out/bench_r01f/bench_${c}_$p.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r01f/bench_${c}_$p.json').read().strip().splitlines()[-1]); print('$c $p', d['ms_per_step'], d['value'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
done; done
