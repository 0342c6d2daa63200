#!/bin/bash
# quick perf matrix: engine x precision x config (diagnostic)
for c in ${CONFIGS:-C2 C1}; do for e in ${ENGINES:-streaming resident}; do for p in ${PRECS:-f64 f32}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --engine $e --precision $p --no-cpu-baseline > gpurun_out/bench_${c}_${e}_$p.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${c}_${e}_$p.log').read().strip().splitlines()[-1]); print('$c $e $p', d['config']['engine'], 'ms/pkt', d['ms_per_step'], 'ev/s', d['value'], 'e2e', d['e2e']['value'])" 2>&1 | tail -1
done; done; done
