"""Probe: a few packets through a 1-band group (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
H, W, epp, pd, tv, rate = bench.CONFIGS[cfg]
sc, mc = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(denoise_iterations=tv)
pk = [np.ascontiguousarray(p) for p in bench.gen_packets(H, W, epp, 4, rate, 3)]
grp = evr.BandedStream(evr.SensorGeometry(W, H), sc, mc, bands=int(sys.argv[2]) if len(sys.argv) > 2 else 1, precision=1)
for p in pk:
    grp.process_packet(p, want_frame=False)
