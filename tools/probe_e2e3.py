"""Probe: cProfile of process_packet_arrays (diagnostic, GPU)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr

H, W, epp, pd, tv, rate = bench.CONFIGS["C2"]
sc, mc, th = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(denoise_iterations=tv), evr.Thresholds()
st = evr.init_state(evr.SensorGeometry(W, H), sc)
pk = [np.ascontiguousarray(p) for p in bench.gen_packets(H, W, epp, 80, rate, 1)]
for p in pk[:10]:
    evr.process_packet_arrays(st, p, mc, sc, th)
pr = cProfile.Profile()
pr.enable()
for p in pk[10:]:
    evr.process_packet_arrays(st, p, mc, sc, th)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
