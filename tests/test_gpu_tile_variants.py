"""The opt-in forms of the primal-dual tile must give the oracle's bits
exactly -- chained packets at the headline shape and at 640x480, K = 3 and 4:
clustered tiles (k_pd_tile<..., CX, CY>, EVR_TILE_CLUSTER; the region of a
thread-block cluster, neighbour values crossing between its CTAs through
DSMEM each half-step) for every cluster shape, and TMA tiles (EVR_TILE_TMA;
the region loaded as two 2-D tensor boxes, off-sensor pixels zero-filled).
The switches are read once per process, so each case runs in a subprocess."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys
    import numpy as np
    import paper_1607_06283_b200 as evr
    from oracle import oracle as O

    H, W, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    rng = np.random.default_rng(7)
    m = n * 1000
    ev = evr.make_event_array(rng.integers(0, W, m), rng.integers(0, H, m),
                              rng.choice([-1, 1], m), 50_000 + np.arange(m, dtype=np.int64))
    sc, mc, th = evr.SolverConfig(max_iterations=100), evr.ManifoldConfig(), evr.Thresholds()
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0, engine=1)
    ref = O.OracleStream(H, W, O.make_config(max_iterations=100))
    for k in range(n):
        p = ev[k * 1000:(k + 1) * 1000]
        _, frame, res = evr.process_packet_arrays(st, p, mc, sc, th)
        ref.process(np.ascontiguousarray(p))
        assert np.array_equal(frame, ref.u), f"u differs at packet {k}"
    assert np.array_equal(st.p, ref.p)
    print("ok")
""")


@pytest.mark.parametrize("variant", ["cluster2x2", "cluster4x2", "cluster2x4", "tma"])
@pytest.mark.parametrize("K", [3, 4])
@pytest.mark.parametrize("H,W,n", [(720, 1280, 2), (480, 640, 3)])
def test_tile_variants_bit_exact(variant, K, H, W, n):
    env = dict(os.environ, EVR_TILE_K=str(K))
    if variant == "tma":
        env["EVR_TILE_TMA"] = "1"
    else:
        env["EVR_TILE_CLUSTER"] = variant[len("cluster"):]
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(H), str(W), str(n)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "ok" in r.stdout
