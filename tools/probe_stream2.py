"""Probe: per-packet yield intervals of stream_packets (diagnostic, GPU)."""
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
pk = bench.gen_packets(H, W, epp, 80, rate, 1)
pinned = [torch.from_numpy(p.view(np.uint8)).pin_memory().numpy().view(evr.EVENT_DTYPE) for p in pk]
for rep in range(3):
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec)
    for _ in evr.stream_packets(st, pinned[:5], mc, sc, th):
        pass
    torch.cuda.synchronize()
    ts = [time.perf_counter()]
    for _ in evr.stream_packets(st, pinned[5:], mc, sc, th):
        ts.append(time.perf_counter())
    d = np.diff(ts) * 1e3
    print(cfg, "rep", rep, "mean %.3f med %.3f max %.3f min %.3f" % (d.mean(), np.median(d), d.max(), d.min()),
          "slow:", [round(x, 2) for x in d if x > 2 * np.median(d)][:10])
