#!/bin/bash
# A/B a runtime knob: tools/ab_env.sh "ENV=a" "ENV=b" -- configs...
# (CONFIGS, PRECS, ENGINE, STEPS from the environment)
for setting in "$@"; do
  for c in ${CONFIGS:-C3 C4 C5}; do for p in ${PRECS:-f32 f64}; do
    env $setting timeout 120 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --engine ${ENGINE:-streaming} --precision $p --no-cpu-baseline > gpurun_out/ab.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$setting $c $p', d['ms_per_step'], d['config'].get('engine'))" 2>&1 | tail -1
  done; done
done
