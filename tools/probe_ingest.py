"""Probe: time evr_ingest alone vs packet size (diagnostic, GPU)."""
import sys, time, ctypes, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib

H, W = 260, 346
st = evr.init_state(evr.SensorGeometry(W, H), evr.SolverConfig())
ctx = st.context()
rng = np.random.default_rng(0)
for n in [1, 10, 100, 500, 1000, 2000, 5000]:
    ev = evr.make_event_array(rng.integers(0, W, n), rng.integers(0, H, n), rng.choice([-1, 1], n),
                              np.arange(n, dtype=np.int64))
    for _ in range(3):
        ctx.call("evr_ingest", _lib.ptr(ev), n)
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.call("evr_ingest", _lib.ptr(ev), n)
    dt = (time.perf_counter() - t0) / 20
    print(f"ingest n={n:5d}: {dt*1e6:9.1f} us/call", flush=True)
