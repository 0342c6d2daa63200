"""Probe: banded group (evr_group) time per packet on one GPU, fused vs split
(diagnostic, GPU).  usage: probe_group.py CONFIG BANDS [f32]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
bands = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = 1 if len(sys.argv) > 3 and sys.argv[3] == "f32" else 0
H, W, epp, pd, tv, rate = bench.CONFIGS[cfg]
sc, mc = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(denoise_iterations=tv)
pk = [np.ascontiguousarray(p) for p in bench.gen_packets(H, W, epp, 14, rate, 3)]
for split in ("0", "1"):
    os.environ["EVR_GROUP_SPLIT"] = split
    grp = evr.BandedStream(evr.SensorGeometry(W, H), sc, mc, bands=bands, precision=prec)
    for p in pk[:4]:
        grp.process_packet(p, want_frame=False)
    t0 = time.perf_counter()
    for p in pk[4:]:
        grp.process_packet(p, want_frame=False)  # synchronous: returns after the solve
    dt = (time.perf_counter() - t0) / (len(pk) - 4)
    print(f"{cfg} {'f32' if prec else 'f64'} bands={bands} {'split' if split == '1' else 'fused'}: "
          f"{dt * 1e3:.3f} ms/packet (host clock, no frame download)")
# the whole-sensor context, same host clock (synchronous packet, no frame)
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec)
for p in pk[:4]:
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
t0 = time.perf_counter()
for p in pk[4:]:
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
dt = (time.perf_counter() - t0) / (len(pk) - 4)
print(f"{cfg} {'f32' if prec else 'f64'} single context: {dt * 1e3:.3f} ms/packet (host clock, no frame download)")
