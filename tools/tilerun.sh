timeout 600 python -m pytest tests -m gpu -x -q -k "tile or stream_packets or full_size or fused_streaming or float32" > gpurun_out/pytest_tile.log 2>&1; tail -5 gpurun_out/pytest_tile.log
for c in C3 C4 C5; do for k in 1 2 3 4; do
EVR_TILE_K=$k timeout 300 python bench.py --config $c --precision f32 --no-cpu-baseline --steps 30 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c f32 K=$k', d['ms_per_step'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
done; done
for c in C3 C4; do for k in 1 2 3; do
EVR_TILE_K=$k timeout 300 python bench.py --config $c --precision f64 --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c f64 K=$k', d['ms_per_step'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
done; done
