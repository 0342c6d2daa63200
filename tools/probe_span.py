"""Probe: where the resident kernel's time goes outside its phases (GPU).

Uses the timeline marks (thread 0 of each CTA, globaltimer ns) with PD capped
at 49 iterations so the last mark (kernel end, after the epilogue and the
rel_change fold) fits the 256 slots.  Reports the CTA start skew, the solve
end, the kernel end, and the host-measured packet time for comparison.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
H, W, epp, pd, tv, rate = bench.CONFIGS[cfgname]
pd = min(pd, 49)
sc = evr.SolverConfig(max_iterations=pd)
mc = evr.ManifoldConfig(denoise_iterations=tv)
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=2)
ctx = st.context()
evr.pipeline._prepare(st, mc, sc, evr.Thresholds())
pk = bench.gen_packets(H, W, epp, 12, rate, 1)
for p in pk[:6]:
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
torch.cuda.synchronize()
t = time.perf_counter()
for p in pk[6:11]:
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
torch.cuda.synchronize()
host_us = (time.perf_counter() - t) / 5 * 1e6
ctx.call("evr_debug_timeline", 1, None, 0)
evr.process_packet_arrays(st, pk[11], mc, sc, evr.Thresholds(), want_frame=False)
buf = np.zeros(256 * 160, dtype=np.uint64)
ctx.call("evr_debug_timeline", -1, _lib.ptr(buf), buf.size)
tr = buf.reshape(-1, 256).astype(np.int64)
rows = [r for r in range(tr.shape[0]) if tr[r, 0] > 0]
a = tr[rows]
k_solve_end = 2 + tv + 2 + 4 * pd
k_end = k_solve_end + 1
t0 = a[:, 0].min()
st_ = (a[:, 0] - t0) / 1e3
print(f"{cfgname} f{'64' if prec == 0 else '32'} pd={pd} tv={tv} CTAs={len(rows)}")
print(f"CTA start skew: max {st_.max():.2f} us, median {np.median(st_):.2f}")
print(f"ingest done (max over CTAs): {(a[:, 1].max() - t0) / 1e3:.2f} us")
print(f"solve end (max): {(a[:, k_solve_end].max() - t0) / 1e3:.2f} us")
print(f"kernel end (max): {(a[:, k_end].max() - t0) / 1e3:.2f} us, "
      f"epilogue {((a[:, k_end] - a[:, k_solve_end]).max()) / 1e3:.2f} us")
print(f"host time per synchronous packet (untraced, no frame): {host_us:.1f} us")
