import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1607_06283_b200 as e
rng = np.random.default_rng(0)
for shape in [(16, 16), (32, 32)]:
    t = rng.normal(0, 1, shape); u = rng.normal(0, 1, shape); p = rng.normal(0, 1, shape + (3,))
    for rep in range(3):
        t0 = time.perf_counter(); m = e.compute_metric(t); t1 = time.perf_counter()
        e.surface_gradient(u, m); t2 = time.perf_counter(); e.surface_gradient_adjoint(p, m); t3 = time.perf_counter()
        print(shape, rep, "metric %.3f ms grad %.3f ms adj %.3f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3))
