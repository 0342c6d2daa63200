#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   plain runs first, then the ncu launch lists, then one --set full capture
#   of each top kernel.  Outputs under gpurun_out/prof/.
set -u
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_C2_f64.json 2> $O/bench_C2_f64.err
python bench.py --config C3 --precision f32 --no-cpu-baseline > $O/bench_C3_f32.json 2>&1
python bench.py --config C1 --no-cpu-baseline > $O/bench_C1_f64.json 2>&1
python bench.py --config C4 --precision f32 --no-cpu-baseline > $O/bench_C4_f32.json 2>&1
python bench.py --config C5 --precision f32 --no-cpu-baseline > $O/bench_C5_f32.json 2>&1
python tools/probe_timeline.py C2 0 > $O/timeline_C2_f64.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_f64.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 600 --log-file $O/launches_C3_f32.csv \
    python bench.py --config C3 --precision f32 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_resident -s 10 -c 1 \
    -o $O/full_k_resident_col_C2_f64 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pd_march -s 40 -c 1 \
    -o $O/full_k_pd_march_C3_f32 python bench.py --config C3 --precision f32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tv_march -s 40 -c 1 \
    -o $O/full_k_tv_march_C3_f32 python bench.py --config C3 --precision f32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la $O
