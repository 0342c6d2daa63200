#!/bin/bash
# resident engine check: gpu tests of the resident path + C1/C2 bench lines
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in C2 C1; do for p in f64 f32; do
  timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 200 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $p', d['ms_per_step'], d['value'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
done; done
python tools/probe_timeline.py C2 0 > gpurun_out/timeline_C2_f64.txt 2>&1; tail -12 gpurun_out/timeline_C2_f64.txt
