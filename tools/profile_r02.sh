#!/bin/bash
# Round 2 profile capture (run on the GPU box from the repo root): plain
# bench lines first, then the ncu launch list and one --set full capture of
# each dominant kernel.  Outputs under gpurun_out/prof/ (text exports only).
set -u
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_C3_f64.json 2> $O/bench_C3_f64.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_C3_f64.json 2>&1
python bench.py --config C1 > $O/bench_C1_f64.json 2> $O/bench_C1_f64.err
python bench.py --config C1 --impl reference --steps 40 --warmup 3 > $O/bench_ref_C1_f64.json 2>&1
python bench.py --config C2 --no-cpu-baseline > $O/bench_C2_f64.json 2>&1
python bench.py --config C4 > $O/bench_C4_f64.json 2> $O/bench_C4_f64.err
for c in C1 C2 C3 C4 C5; do
  python bench.py --config $c --precision f32 --no-cpu-baseline > $O/bench_${c}_f32.json 2>&1
done
python bench.py --config C5 --no-cpu-baseline > $O/bench_C5_f64.json 2>&1
for v in rof l1 tgv; do
  python bench.py --config C2 --variant $v --steps 50 --warmup 5 > $O/bench_C2_$v.json 2>&1
done
python bench.py --config C5 --bands 2 --steps 20 --warmup 3 > $O/bench_C5_bands2_1gpu.json 2>&1
for fz in 0 3; do EVR_FUSE=$fz python bench.py --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_C3_f64_fuse$fz.json 2>&1; done
for cl in 2x2 4x2; do EVR_TILE_CLUSTER=$cl python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_C3_f64_cluster$cl.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 300 --log-file $O/launches_C3_f64.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_f64.csv \
    python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pd_tile -s 40 -c 1 \
    -o $O/full_k_pd_tile_C3_f64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tv_tile -s 20 -c 1 \
    -o $O/full_k_tv_tile_C3_f64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_resident -s 5 -c 1 \
    -o $O/full_k_resident_col_C2_f64 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_resident -s 5 -c 1 \
    -o $O/full_k_resident_col_C1_f64 python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_metric_pack|k_unpack_rel" -s 2 -c 2 \
    -o $O/full_k_fused_C3_f64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pd_tile -s 40 -c 1 \
    -o $O/full_k_pd_tile_C3_f32 python bench.py --precision f32 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for r in $O/*.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  python tools/stall_mix.py $r > ${r%.ncu-rep}_stalls.txt 2>/dev/null
  python tools/sass_mix.py $r 30 > ${r%.ncu-rep}_sass_mix.txt 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
