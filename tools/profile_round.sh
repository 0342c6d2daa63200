#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   plain runs first, then the ncu launch lists, then one --set full capture
#   of each top kernel.  Outputs under gpurun_out/prof/.
set -u
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_C2_f64.json 2> $O/bench_C2_f64.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_C2_f64.json 2>&1
python bench.py --precision f32 --no-cpu-baseline > $O/bench_C2_f32.json 2>&1
for c in C1 C3 C4 C5; do for p in f64 f32; do
  python bench.py --config $c --precision $p --no-cpu-baseline > $O/bench_${c}_$p.json 2>&1
done; done
python tools/probe_timeline.py C2 0 > $O/timeline_C2_f64.txt 2>&1
for b in 1 2 4; do python tools/probe_group.py C5 $b f32; done > $O/group_C5_f32.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_f64.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 400 --log-file $O/launches_C3_f32.csv \
    python bench.py --config C3 --precision f32 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 400 --log-file $O/launches_C3_f64.csv \
    python bench.py --config C3 --precision f64 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_resident -s 10 -c 1 \
    -o $O/full_k_resident_col_C2_f64 python bench.py --steps 3 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pd_tile -s 30 -c 1 \
    -o $O/full_k_pd_tile_C3_f32 python bench.py --config C3 --precision f32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pd_tile -s 30 -c 1 \
    -o $O/full_k_pd_tile_C3_f64 python bench.py --config C3 --precision f64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tv_tile -s 15 -c 1 \
    -o $O/full_k_tv_tile_C3_f32 python bench.py --config C3 --precision f32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# keep the text exports (the .ncu-rep files exceed what gpurun brings back)
for r in $O/*.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  python tools/stall_mix.py $r > ${r%.ncu-rep}_stalls.txt 2>/dev/null
  python tools/sass_mix.py $r 30 > ${r%.ncu-rep}_sass_mix.txt 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
