import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_06283_b200 as evr


def uniform_packets(H, W, n_packets, epp, seed, t_step):
    rng = np.random.default_rng(seed)
    n = n_packets * epp
    ev = evr.make_event_array(rng.integers(0, W, n), rng.integers(0, H, n),
                              rng.choice([-1, 1], n), np.arange(n, dtype=np.int64) * t_step)
    return [ev[s:s + epp] for s in range(0, n, epp)]


H, W = 300, 1000
for tv, pd in ((10, 20), (1, 1), (0, 1), (1, 0)):
    sc = evr.SolverConfig(max_iterations=max(pd,1))
    mc = evr.ManifoldConfig(denoise_iterations=max(tv,1), enabled=tv > 0)
    out = {}
    for eng in (1, 4):
        st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=1, engine=eng)
        seen = []
        for pk in uniform_packets(H, W, 3, 1000, seed=21, t_step=1):
            _, frame, _ = evr.process_packet(st, pk, mc, sc, evr.Thresholds())
            seen.append((frame.copy(), st.p.copy()))
        out[eng] = seen
    for k, (a, b) in enumerate(zip(out[1], out[4])):
        d = np.argwhere(a[0] != b[0])
        print(tv, pd, k, "u", np.abs(a[0]-b[0]).max(), len(d), d[:5].tolist(), "p", np.abs(a[1]-b[1]).max())
