#!/bin/bash
# A/B of the TMA region loads of the float64 primal-dual tile (EVR_TILE_TMA).
for v in 0 1; do
  for c in C3 C4; do
    EVR_TILE_TMA=$v timeout 120 python bench.py --config $c --precision f64 --no-cpu-baseline --no-f32-leg --steps 100 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tma=$v $c f64', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_us'])"
  done
done
EVR_TILE_TMA=1 timeout 300 ncu --metrics sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__shared_mem_per_block_dynamic,launch__shared_mem_config_size,gpu__time_duration.sum,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct -k regex:k_pd_tile -s 40 -c 1 --clock-control none python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-f32-leg 2>&1 | grep -E "k_pd_tile|warps_active|occupancy|shared_mem|duration|stalled" | head -12
