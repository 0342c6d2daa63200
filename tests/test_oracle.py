"""Pin the C oracle against the reference's own outputs (CPU only).

The fixtures in tests/golden/ were produced by running the unmodified
reference (tests/golden/make_golden.py).  Every hot-path stage must be
bit-identical (np.array_equal); only the norm/energy reductions, whose
summation order differs from numpy's BLAS/pairwise sums, are compared with
a tolerance.  Known-answer vectors come from SURVEY.md 8(c) and the
reference tests cited beside each check.
"""

import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def packets(d):
    ev = O.events_array(d["ev_x"], d["ev_y"], d["ev_pol"], d["ev_t"])
    epp = int(d["epp"])
    return [ev[s:s + epp] for s in range(0, len(ev), epp)]


STREAMS = {
    "stream_u_32x24.npz": dict(),
    "stream_s_dvs128.npz": dict(),
    "stream_flat_9x2.npz": dict(manifold_enabled=False, max_iterations=20),
    "stream_window_2x7.npz": dict(t_window=50.0, t_scale=2.0, denoise_weight=0.5,
                                  denoise_iterations=7, lam=1.3, max_iterations=9,
                                  pos=0.2, neg=0.1),
}


def start_stream(d, cfg, t_window):
    """Oracle stream at the fixture's starting state (init_* when the
    fixture skipped warm-up packets)."""
    s = O.OracleStream(int(d["height"]), int(d["width"]), cfg, t_window=t_window)
    if "init_u" in d:
        s.u, s.f = d["init_u"].copy(), d["init_f"].copy()
        s.raw, s.p = d["init_raw"].copy(), d["init_p"].copy()
        s.packet_starts.extend(int(v) for v in d["init_starts"])
        s.frame_index = int(d["init_frame_index"])
    return s


def oracle_cfg(opts):
    kw = {k: v for k, v in opts.items() if k != "t_window"}
    return O.make_config(**kw), opts.get("t_window")


@pytest.mark.parametrize("name", sorted(STREAMS))
def test_chained_stream_bit_exact(name):
    """pipeline.py:142-171 chained over packets: f, raw after ingest and the
    solved u, p are bit-identical to the reference at every packet."""
    d = load(name)
    cfg, t_window = oracle_cfg(STREAMS[name])
    s = start_stream(d, cfg, t_window)
    for k, pk in enumerate(packets(d)):
        # teacher-forced ingest check (apply_event on the previous state)
        f_chk, raw_chk = s.f.copy(), s.raw.copy()
        O.ingest(f_chk, raw_chk, pk, cfg)
        assert np.array_equal(f_chk, d["f_ing"][k])
        assert np.array_equal(raw_chk, d["raw_ing"][k])
        it, rel = s.process(pk)
        assert it == d["iterations"][k]
        assert np.array_equal(s.u, d["u"][k]), f"packet {k}"
        if "p" in d:
            assert np.array_equal(s.p, d["p"][k])
        assert np.array_equal(s.f, s.u)
        assert rel == pytest.approx(d["rel_change"][k], rel=1e-10, abs=1e-300)
    if "p_last" in d:
        assert np.array_equal(s.p, d["p_last"])


def test_stage_by_stage_u_stream():
    """normalize -> denoise -> metric -> solve, teacher-forced per packet."""
    d = load("stream_u_32x24.npz")
    cfg = O.make_config()
    for k in range(len(d["u"])):
        now = int(packets(d)[k]["t"][-1])
        t = O.normalize(d["raw_ing"][k], now, 3.0, float(d["window"][k]))
        assert np.array_equal(t, d["t_norm"][k])
        td = O.denoise(t, 1.0, 50, 3.0)
        assert np.array_equal(td, d["t_den"][k])
        tx, ty, G, sg = O.metric(td)
        for a, key in ((tx, "tx"), (ty, "ty"), (G, "G"), (sg, "sqrtG")):
            assert np.array_equal(a, d[key][k])
        u0 = d["u"][k - 1] if k else np.full(tx.shape, 1.5)
        p0 = d["p"][k - 1] if k else np.zeros(tx.shape + (3,))
        u, p, it, _ = O.pd_solve(d["f_ing"][k], tx, ty, G, sg, cfg, u0, p0)
        assert np.array_equal(u, d["u"][k]) and np.array_equal(p, d["p"][k])


def test_dvs128_surface_is_steep():
    """The S stream exercises non-trivial metrics (max G ~ 4)."""
    d = load("stream_s_dvs128.npz")
    assert d["G_last"].max() > 2.0


def test_operator_cases():
    o = load("ops.npz")
    assert np.array_equal(O.normalize(o["norm_raw"], 1000, 3.0, 1000.0), o["norm_t"])
    assert np.array_equal(O.denoise(o["den_in"], 0.3, 50, 3.0), o["den_out"])
    tx, ty, G, sg = O.metric(o["met_in"])
    assert np.array_equal(tx, o["met_tx"]) and np.array_equal(ty, o["met_ty"])
    assert np.array_equal(G, o["met_G"]) and np.array_equal(sg, o["met_sqrtG"])
    assert np.array_equal(np.stack(O.coeffs(tx, ty, G)), o["met_coeffs"])
    assert np.array_equal(O.div(o["div_qx"], o["div_qy"]), o["div_out"])
    assert np.array_equal(O.surface_gradient(o["sg_u"], tx, ty, G), o["sg_out"])
    assert np.array_equal(O.surface_gradient_adjoint(o["sg_p"], tx, ty, G), o["sga_out"])
    step = O.DEFAULT_STEP
    assert np.array_equal(O.prox_data(o["pd_ubar"], o["pd_f"], sg, 0.3, 3.0, 1.0, 2.0),
                          o["prox_data_out"])
    assert np.array_equal(O.prox_dual(o["prox_dual_in"], sg), o["prox_dual_out"])
    e = O.energy(o["sg_u"], o["pd_f"], tx, ty, G, sg, 0.7)
    assert e == pytest.approx(o["energy_val"][0], rel=1e-12)
    assert step == 1.0 / math.sqrt(8.0 + 4.0 * math.sqrt(2.0))


def test_warm_started_solve_and_trace():
    o = load("ops.npz")
    cfg = O.make_config(lam=0.9, max_iterations=60)
    u, p, it, rel, et, rt = O.pd_solve(o["solve_f"], o["solve_tx"], o["solve_ty"],
                                       o["solve_G"], o["solve_sqrtG"], cfg,
                                       o["solve_u0"], o["solve_p0"], trace=True)
    assert np.array_equal(u, o["solve_u"]) and np.array_equal(p, o["solve_p"])
    assert it == o["solve_iters"][0]
    tr = o["solve_trace"]
    assert np.array_equal(tr[:, 0], np.arange(1, it + 1))
    np.testing.assert_allclose(et, tr[:, 1], rtol=1e-12)
    np.testing.assert_allclose(rt, tr[:, 2], rtol=1e-9)


def test_early_stop_iteration_count():
    o = load("ops.npz")
    cfg = O.make_config(lam=0.7, max_iterations=500, convergence_tol=1e-5)
    z = np.zeros((10, 10))
    u, p, it, rel = O.pd_solve(o["tol_f"], z, z, np.ones_like(z), np.ones_like(z), cfg)
    assert it == o["tol_iters"][0]
    assert np.array_equal(u, o["tol_u"]) and np.array_equal(p, o["tol_p"])
    assert rel == pytest.approx(o["tol_rel"][0], rel=1e-9)


def test_rof_variants():
    o = load("ops.npz")
    z = np.zeros((20, 20))
    one = np.ones_like(z)
    assert np.array_equal(O.rof_solve(o["rof_f"], z, z, one, one, 8.0, 250), o["rof_flat"])
    tx, ty, G, sg = O.metric(o["rof_h"])
    assert np.array_equal(O.rof_solve(o["rof_f"], tx, ty, G, sg, 4.0, 120), o["rof_steep"])


def test_known_answers():
    """SURVEY.md 8(c) known-answer vectors."""
    cfg = O.make_config()
    f = np.full((4, 4), 1.5)
    raw = np.zeros((4, 4), dtype=np.int64)
    O.ingest(f, raw, O.events_array([3, 1], [2, 0], [1, -1], [7, 9]), cfg)
    assert f[2, 3] == 1.5 * math.exp(0.15)  # test_pipeline.py:52-56
    assert f[0, 1] == 1.5 * math.exp(-0.15)  # test_pipeline.py:59-62
    assert raw[2, 3] == 7 and raw[0, 1] == 9
    # clamp at the box (test_pipeline.py:65-70)
    f[1, 1] = 2.0
    O.ingest(f, raw, O.events_array([1], [1], [1], [11]), cfg)
    assert f[1, 1] == 2.0
    # normalize raw=1000/500/0 at now=1000, win=1000 (test_surface.py:50-57)
    t = O.normalize(np.array([[1000, 500, 0]]), 1000, 3.0, 1000.0)
    assert np.array_equal(t, [[3.0, 1.5, 0.0]])
    # ramp a=2 -> G = 5 away from the last column (test_surface.py:129-134)
    tx, ty, G, sg = O.metric(2.0 * np.mgrid[0:5, 0:6][1].astype(float))
    assert np.all(G[:, :-1] == 5.0)
    # prox instance of test_solve.py:77-83 against the closed form
    out = O.prox_data(np.array([1.3]), np.array([1.6]), np.array([1.0]), 0.2, 1.0, 1.0, 2.0)
    beta = 0.2
    s = 1.3 - beta
    assert out[0] == min(max((s + math.sqrt(s * s + 4 * beta * 1.6)) * 0.5, 1.0), 2.0)


def test_duplicate_events_are_order_sensitive():
    """Multiply-then-clamp does not commute: the ingest must
    apply duplicates sequentially in stream order."""
    cfg = O.make_config()
    f = np.full((2, 2), 1.95)
    raw = np.zeros((2, 2), dtype=np.int64)
    seq = O.events_array([0, 0, 0], [0, 0, 0], [1, -1, 1], [1, 2, 3])
    O.ingest(f, raw, seq, cfg)
    c_pos, c_neg = math.exp(0.15), math.exp(-0.15)
    want = min(max(min(max(min(max(1.95 * c_pos, 1.0), 2.0) * c_neg, 1.0), 2.0) * c_pos, 1.0), 2.0)
    assert f[0, 0] == want
    assert raw[0, 0] == 3


# --- variants the reference does not ship (parity unpinned) -----------------
# TGV and the L1 data term restate published algorithms; these property
# tests pin the restatement's behaviour instead of reference vectors.


def _flat(H, W):
    z = np.zeros((H, W))
    return z, z, np.ones((H, W)), np.ones((H, W))


def test_tgv_keeps_affine_ramps_that_tv_flattens():
    """TGV's w absorbs a constant gradient (E w = 0), so an affine ramp is a
    minimiser of TGV-ROF; TV-ROF shrinks its contrast at the borders."""
    H, W = 40, 50
    yy, xx = np.mgrid[0:H, 0:W]
    f = 1.2 + 0.01 * xx + 0.005 * yy
    m = _flat(H, W)
    u, w = O.tgv_solve(f, *m, lam=8.0, data="rof", iterations=500)
    ut = O.rof_solve(f, *m, 8.0, 500)
    assert np.abs(u - f).max() < 0.2 * np.abs(ut - f).max()
    inner = (slice(2, -2), slice(2, -2))
    assert abs(w[..., 0][inner].mean() - 0.01) < 2e-3 and abs(w[..., 1][inner].mean() - 0.005) < 2e-3


def test_tgv_and_l1_fixed_points_and_denoising():
    H, W = 24, 30
    m = _flat(H, W)
    c = np.full((H, W), 1.4)
    for data in ("kl", "rof", "l1"):  # a constant image is a fixed point
        u, w = O.tgv_solve(c, *m, lam=2.0, data=data, iterations=60)
        assert np.array_equal(u, c) and not w.any()
    assert np.array_equal(O.l1_solve(c, *m, 2.0, 60), c)
    rng = np.random.default_rng(0)
    xx = np.mgrid[0:H, 0:W][1]
    clean = np.where(xx < W // 2, 1.3, 1.7)
    noisy = np.clip(clean + rng.normal(0, 0.05, (H, W)), 1.0, 2.0)
    for data, lam in (("kl", 8.0), ("rof", 8.0), ("l1", 1.0)):
        u, _ = O.tgv_solve(noisy, *m, lam=lam, data=data, iterations=300)
        assert np.abs(u - clean).mean() < 0.6 * np.abs(noisy - clean).mean()
    # L1 removes an isolated outlier completely (TV-L1's defining property)
    spike = c.copy()
    spike[10, 10] = 1.9
    assert abs(O.l1_solve(spike, *m, 1.0, 400)[10, 10] - 1.4) < 1e-3
