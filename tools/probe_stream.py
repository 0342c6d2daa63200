"""Probe: pipelined stream (stream_packets) vs device time (diagnostic, GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1607_06283_b200 as evr

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 1
H, W, epp, pd, tv, rate = bench.CONFIGS[cfg]
sc, mc, th = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(denoise_iterations=tv), evr.Thresholds()
pk = bench.gen_packets(H, W, epp, 120, rate, 1)
pinned = [torch.from_numpy(p.view(np.uint8)).pin_memory().numpy().view(evr.EVENT_DTYPE) for p in pk]
for depth in (1, 2, 3, 4):
    for want in (True, False):
        st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec)
        for _ in evr.stream_packets(st, pinned[:10], mc, sc, th):
            pass
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in evr.stream_packets(st, pinned[10:], mc, sc, th, depth=depth, want_frames=want):
            pass
        dt = (time.perf_counter() - t0) / 110
        print(f"{cfg} prec={prec} depth={depth} frames={want}: {dt*1e3:.3f} ms/packet")
# host cost of one async submit
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec)
ctx = evr.pipeline._prepare(st, mc, sc, th)
from paper_1607_06283_b200 import _lib
import ctypes
ts = []
for p in pinned[:40]:
    t0 = time.perf_counter()
    ctx.call("evr_process_packet_async", _lib.ptr(p), len(p), 1000.0)
    ts.append(time.perf_counter() - t0)
    ctx.call("evr_synchronize", None)
print("submit host us", np.median(ts[5:]) * 1e6)
# device-only back-to-back (no frame, no sync)
torch.cuda.synchronize()
t0 = time.perf_counter()
for p in pinned[40:100]:
    ctx.call("evr_process_packet_async", _lib.ptr(p), len(p), 1000.0)
ctx.call("evr_synchronize", None)
print("back-to-back ms/packet", (time.perf_counter() - t0) / 60 * 1e3)
