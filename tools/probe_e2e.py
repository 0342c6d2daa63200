"""Probe: where the end-to-end per-packet time goes (diagnostic, GPU)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
H, W, epp, pd, tv, rate = bench.CONFIGS[cfgname]
sc = evr.SolverConfig(max_iterations=pd)
mc = evr.ManifoldConfig(denoise_iterations=tv)
th = evr.Thresholds()
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec)
ctx = st.context()
pk = list(bench.gen_packets(H, W, epp, 60, rate, 1))
for p in pk[:10]:
    evr.process_packet_arrays(st, p, mc, sc, th)
T = {"api_total": 0.0, "process": 0.0, "get_frame": 0.0, "py_prep": 0.0}
frame = np.empty((H, W))
pinned = np.empty((H, W))
for p in pk[10:]:
    t0 = time.perf_counter()
    evr.process_packet_arrays(st, p, mc, sc, th)
    T["api_total"] += time.perf_counter() - t0
for p in pk[10:]:
    t0 = time.perf_counter()
    c = evr.pipeline._prepare(st, mc, sc, th)
    w = evr.pipeline._window(st, int(p["t"][-1]), mc)
    info = _lib.SolveInfo()
    t1 = time.perf_counter()
    c.call("evr_process_packet", _lib.ptr(p), len(p), float(w), ctypes.byref(info))
    t2 = time.perf_counter()
    c.call("evr_get_frame", _lib.ptr(frame))
    t3 = time.perf_counter()
    T["py_prep"] += t1 - t0
    T["process"] += t2 - t1
    T["get_frame"] += t3 - t2
n = len(pk) - 10
print(cfgname, {k: round(v / n * 1e6, 1) for k, v in T.items()}, "us/packet", ctx.engine_detail())
