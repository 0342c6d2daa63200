"""One-off: float32 vs float64 chained drift on log u over a long DVS128
S-stream (diagnostic, GPU).  python tools/drift_long.py [packets]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import paper_1607_06283_b200 as evr
from test_gpu_long_chains import s_packets, u_packets

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for name, pk in (("C1 S-stream", s_packets(128, 128, n, 500, frames=16)),
                 ("C1 U-stream", u_packets(128, 128, n, 500, seed=0, t_step=10))):
    sc, mc, th = evr.SolverConfig(max_iterations=50), evr.ManifoldConfig(), evr.Thresholds()
    s64 = evr.init_state(evr.SensorGeometry(128, 128), sc, precision=0)
    s32 = evr.init_state(evr.SensorGeometry(128, 128), sc, precision=1)
    worst, marks = 0.0, []
    for k, (a, b) in enumerate(zip(evr.stream_packets(s64, pk, mc, sc, th),
                                   evr.stream_packets(s32, pk, mc, sc, th))):
        d = float(np.abs(np.log(a[0]) - np.log(b[0])).max())
        worst = max(worst, d)
        if (k + 1) % (n // 10) == 0:
            marks.append(f"{k + 1}:{d:.2e}")
    print(f"{name}: {n} chained packets, worst max|dlog u| {worst:.3e}; {' '.join(marks)}")
