"""Probe: end-to-end per-packet time split (diagnostic, GPU)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib

H, W, epp, pd, tv, rate = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
sc, mc, th = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(denoise_iterations=tv), evr.Thresholds()
st = evr.init_state(evr.SensorGeometry(W, H), sc)
ctx = st.context()
pk = [np.ascontiguousarray(p) for p in bench.gen_packets(H, W, epp, 80, rate, 1)]
for p in pk[:10]:
    evr.process_packet_arrays(st, p, mc, sc, th)
frame = _lib.pinned_empty((H, W))
info = _lib.SolveInfo()
T = {}


def add(k, v):
    T[k] = T.get(k, 0.0) + v


n = 0
for p in pk[10:]:
    t0 = time.perf_counter()
    c = evr.pipeline._prepare(st, mc, sc, th)
    w = evr.pipeline._window(st, int(p["t"][-1]), mc)
    t1 = time.perf_counter()
    c.call("evr_process_packet_async", _lib.ptr(p), len(p), float(w))
    t2 = time.perf_counter()
    c.call("evr_get_frame_async", _lib.ptr(frame))
    t3 = time.perf_counter()
    c.call("evr_synchronize", ctypes.byref(info))
    t4 = time.perf_counter()
    add("py_prepare", t1 - t0)
    add("enqueue_packet", t2 - t1)
    add("enqueue_frame", t3 - t2)
    add("sync", t4 - t3)
    n += 1
# kernel-only reference: device packets back to back, one sync each
t0 = time.perf_counter()
for p in pk[10:]:
    c.call("evr_process_packet_async", _lib.ptr(p), len(p), 1000.0)
    c.call("evr_synchronize", None)
T["packet+sync, no frame"] = time.perf_counter() - t0
t0 = time.perf_counter()
for p in pk[10:]:
    evr.process_packet_arrays(st, p, mc, sc, th)
T["api_total"] = time.perf_counter() - t0
print({k: round(v / n * 1e6, 1) for k, v in T.items()}, "us/packet")
