"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
the resident column kernel (C2 shape, float64 and float32, with and without
the device early stop), the fused streaming list (tiles + march), a banded
group of 3 bands and the ROF tile solve.
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1607_06283_b200 as evr  # noqa: E402


def packets(H, W, n, epp, seed):
    rng = np.random.default_rng(seed)
    m = n * epp
    ev = evr.make_event_array(rng.integers(0, W, m), rng.integers(0, H, m),
                              rng.choice([-1, 1], m), np.arange(m, dtype=np.int64))
    return [ev[s:s + epp] for s in range(0, m, epp)]


mc, th = evr.ManifoldConfig(denoise_iterations=6), evr.Thresholds()
for prec in (0, 1):
    for tol in (0.0, 1e-3):
        sc = evr.SolverConfig(max_iterations=6, convergence_tol=tol)
        st = evr.init_state(evr.SensorGeometry(346, 260), sc, precision=prec)
        for p in packets(260, 346, 2, 500, 1):
            evr.process_packet_arrays(st, p, mc, sc, th)
        print("resident", prec, tol, st.context().engine_detail())
sc = evr.SolverConfig(max_iterations=7)
st = evr.init_state(evr.SensorGeometry(200, 150), sc, engine=1)
for p in packets(150, 200, 2, 500, 2):
    evr.process_packet_arrays(st, p, mc, sc, th)
print("streaming", st.context().engine_detail())
from paper_1607_06283_b200.group import BandedStream  # noqa: E402

bs = BandedStream(evr.SensorGeometry(120, 90), sc, mc, th, bands=3)
for p in packets(90, 120, 2, 400, 3):
    bs.process_packet(p)
print("bands ok")
yy, xx = np.mgrid[0:40, 0:50]
m = evr.compute_metric(3.0 * np.sin(xx / 6.0) * np.cos(yy / 9.0) ** 2)
evr.rof_manifold_solve(np.full((40, 50), 1.5), m, 8.0, 7)
print("sanitize workload done")
