timeout 600 python -m pytest tests -m gpu -x -q -k "float32 or tile or stream_packets" 2>&1 | tail -2
for c in C3 C4 C5; do for k in 3 4; do
EVR_TILE_K=$k timeout 300 python bench.py --config $c --precision f32 --no-cpu-baseline --steps 50 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c f32 K=$k', d['ms_per_step'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
done; done
timeout 300 python bench.py --config C2 --precision f32 --no-cpu-baseline --steps 100 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 f32', d['ms_per_step'], 'e2e', d['e2e']['value'], d['roofline']['frac'])"
