"""Parity of the CUDA path with the reference (golden fixtures) and with the
C oracle (seeded inputs at full sensor sizes).  float64: bit-exact
(np.array_equal) for f, raw, t, metric, u, p at every packet; float32:
log-intensity within 1e-4 max-abs (the north_star tolerance).
"""

import math
import os

import numpy as np
import pytest

import paper_1607_06283_b200 as evr
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOG_TOL = 1e-4  # north_star: max-abs on log intensity (float32 engine)


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def packets_of(d):
    ev = evr.make_event_array(d["ev_x"], d["ev_y"], d["ev_pol"], d["ev_t"])
    epp = int(d["epp"])
    return [ev[s:s + epp] for s in range(0, len(ev), epp)]


STREAMS = {
    "stream_u_32x24.npz": (evr.ManifoldConfig(), evr.SolverConfig(), evr.Thresholds()),
    "stream_s_dvs128.npz": (evr.ManifoldConfig(), evr.SolverConfig(), evr.Thresholds()),
    "stream_flat_9x2.npz": (evr.ManifoldConfig(enabled=False),
                            evr.SolverConfig(max_iterations=20), evr.Thresholds()),
    "stream_window_2x7.npz": (evr.ManifoldConfig(t_window=50.0, t_scale=2.0,
                                                 denoise_weight=0.5, denoise_iterations=7),
                              evr.SolverConfig(lam=1.3, max_iterations=9),
                              evr.Thresholds(0.2, 0.1)),
}

ENGINES = ["streaming", "resident"]


def device_state(d, cfg, precision=0, engine=None):
    H, W = int(d["height"]), int(d["width"])
    st = evr.init_state(evr.SensorGeometry(width=W, height=H), cfg, precision=precision,
                        engine=engine)
    if "init_u" in d:
        st.u, st.f = d["init_u"].copy(), d["init_f"].copy()
        st.raw_timestamps, st.p = d["init_raw"].copy(), d["init_p"].copy()
        st.packet_starts.extend(int(v) for v in d["init_starts"])
        st.frame_index = int(d["init_frame_index"])
    return st


def engine_id(name):
    return {"streaming": 1, "resident": 2}[name]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", sorted(STREAMS))
def test_golden_stream_bit_exact(name, engine):
    """Chained packets through the device state machine equal the
    reference's own per-packet outputs bit for bit."""
    d = load(name)
    mc, sc, th = STREAMS[name]
    st = device_state(d, sc, engine=engine_id(engine))
    seen = []
    for k, pk in enumerate(packets_of(d)):
        _, frame, res = evr.process_packet(
            st, pk, mc, sc, th, debug_sink=(lambda i, s, m: seen.append((s, m))) if k == 0 else None)
        assert res.iterations == int(d["iterations"][k])
        assert np.array_equal(frame, d["u"][k]), f"u packet {k}"
        if "p" in d:
            assert np.array_equal(st.p, d["p"][k]), f"p packet {k}"
        assert np.array_equal(st.raw_timestamps, d["raw_ing"][k])
        assert np.array_equal(st.f, frame)
        assert res.rel_change == pytest.approx(float(d["rel_change"][k]), rel=1e-9)
    if "p_last" in d:
        assert np.array_equal(st.p, d["p_last"])
    # the debug view of packet 0 is the reference's surface and metric
    s, m = seen[0]
    if "t_den" in d and mc.enabled:
        assert np.array_equal(s.t, d["t_den"][0])
        assert np.array_equal(m.G, d["G"][0]) and np.array_equal(m.tx, d["tx"][0])


@pytest.mark.parametrize("name", ["stream_u_32x24.npz", "stream_s_dvs128.npz"])
def test_teacher_forced_ingest_bit_exact(name):
    """apply_event over a packet (duplicates included) == reference f, raw."""
    d = load(name)
    sc = evr.SolverConfig()
    st = device_state(d, sc)
    pk = packets_of(d)
    prev_u = d["init_u"] if "init_u" in d else np.full(d["u"][0].shape, 1.5)
    prev_raw = d["init_raw"] if "init_raw" in d else np.zeros(d["u"][0].shape, np.int64)
    for k in range(len(pk)):
        st.f = (prev_u if k == 0 else d["u"][k - 1]).copy()
        st.raw_timestamps = (prev_raw if k == 0 else d["raw_ing"][k - 1]).copy()
        ctx = evr.pipeline._prepare(st, evr.ManifoldConfig(), sc, evr.Thresholds())
        from paper_1607_06283_b200 import _lib
        ctx.call("evr_ingest", _lib.ptr(pk[k]), len(pk[k]))
        st._after_device_write(in_place=("f", "raw_timestamps"))
        assert np.array_equal(st.f, d["f_ing"][k])
        assert np.array_equal(st.raw_timestamps, d["raw_ing"][k])


def test_operator_api_bit_exact():
    o = load("ops.npz")
    t = evr.normalize_timestamps(o["norm_raw"], 1000, 3.0, 1000.0)
    assert np.array_equal(t.t, o["norm_t"])
    td = evr.denoise_timestamps(evr.TimeSurface(o["den_in"], 3.0), 0.3, 50)
    assert np.array_equal(td.t, o["den_out"])
    m = evr.compute_metric(o["met_in"])
    for a, k in ((m.tx, "met_tx"), (m.ty, "met_ty"), (m.G, "met_G"), (m.sqrtG, "met_sqrtG")):
        assert np.array_equal(a, o[k])
    assert np.array_equal(np.stack(m.coeffs), o["met_coeffs"])
    assert np.array_equal(evr.div_xy(o["div_qx"], o["div_qy"]), o["div_out"])
    assert np.array_equal(evr.surface_gradient(o["sg_u"], m), o["sg_out"])
    assert np.array_equal(evr.surface_gradient_adjoint(o["sg_p"], m), o["sga_out"])
    cfg = evr.SolverConfig(lam=3.0)
    assert np.array_equal(evr.prox_data(o["pd_ubar"], o["pd_f"], m, 0.3, cfg), o["prox_data_out"])
    assert np.array_equal(evr.prox_dual(o["prox_dual_in"], m), o["prox_dual_out"])
    assert evr.energy(o["sg_u"], o["pd_f"], m, 0.7) == pytest.approx(o["energy_val"][0], rel=1e-12)


def test_operator_solve_warm_start_and_trace():
    o = load("ops.npz")
    m = evr.MetricField(tx=o["solve_tx"], ty=o["solve_ty"], G=o["solve_G"], sqrtG=o["solve_sqrtG"])
    trace = []
    res = evr.primal_dual_solve(o["solve_f"], m, evr.SolverConfig(lam=0.9, max_iterations=60),
                                u_init=o["solve_u0"], p_init=o["solve_p0"], trace=trace)
    assert np.array_equal(res.u, o["solve_u"]) and np.array_equal(res.p, o["solve_p"])
    tr = np.array(trace)
    assert np.array_equal(tr[:, 0], o["solve_trace"][:, 0])
    np.testing.assert_allclose(tr[:, 1], o["solve_trace"][:, 1], rtol=1e-12)
    np.testing.assert_allclose(tr[:, 2], o["solve_trace"][:, 2], rtol=1e-9)


def test_operator_early_stop():
    o = load("ops.npz")
    cfg = evr.SolverConfig(lam=0.7, max_iterations=500, convergence_tol=1e-5)
    res = evr.primal_dual_solve(o["tol_f"], evr.flat_metric((10, 10)), cfg)
    assert res.iterations == int(o["tol_iters"][0])
    assert np.array_equal(res.u, o["tol_u"]) and np.array_equal(res.p, o["tol_p"])


def test_operator_rof():
    o = load("ops.npz")
    out = evr.rof_manifold_solve(o["rof_f"], evr.flat_metric((20, 20)), 8.0, 250)
    assert np.array_equal(out, o["rof_flat"])
    out = evr.rof_manifold_solve(o["rof_f"], evr.compute_metric(o["rof_h"]), 4.0, 120)
    assert np.array_equal(out, o["rof_steep"])


def uniform_packets(H, W, n_packets, epp, seed, t_step):
    rng = np.random.default_rng(seed)
    n = n_packets * epp
    ev = evr.make_event_array(rng.integers(0, W, n), rng.integers(0, H, n),
                              rng.choice([-1, 1], n), np.arange(n, dtype=np.int64) * t_step)
    return [ev[s:s + epp] for s in range(0, n, epp)]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("H,W,epp,iters", [(260, 346, 500, 50), (128, 128, 500, 50),
                                           (33, 70, 1500, 17), (500, 200, 700, 20),
                                           (140, 600, 500, 12), (296, 512, 500, 20),
                                           (148, 512, 500, 20)])
def test_full_size_chained_vs_oracle(H, W, epp, iters, engine):
    """DAVIS346 / DVS128 generator-U streams, plus a packet
    larger than one ingest chunk: bit-exact with the C oracle, chained.  The
    resident engine runs its column kernel (bands <= 2 rows, W <= 512) on
    the first three shapes and the last two (its largest shapes: 148 CTAs of
    512 threads, bands of 2 and 1 rows) and its plane-frame kernel on the
    other two."""
    sc = evr.SolverConfig(max_iterations=iters)
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0, engine=engine_id(engine))
    ref = O.OracleStream(H, W, O.make_config(max_iterations=iters))
    for pk in uniform_packets(H, W, 3, epp, seed=H + W, t_step=1):
        _, frame, res = evr.process_packet(st, pk, evr.ManifoldConfig(), sc, evr.Thresholds())
        it, rel = ref.process(np.ascontiguousarray(pk))
        assert res.iterations == it
        assert np.array_equal(frame, ref.u)
        assert res.rel_change == pytest.approx(rel, rel=1e-9)
    assert np.array_equal(st.p, ref.p)
    assert np.array_equal(st.raw_timestamps, ref.raw)


@pytest.mark.parametrize("H,W,tv,pd", [(45, 97, 13, 9), (17, 33, 1, 1), (9, 40, 2, 3)])
def test_fused_streaming_odd_iterations_vs_oracle(H, W, tv, pd):
    """The fused one-launch-per-iteration streaming kernels ping-pong their
    fields; odd TV-L1 / primal-dual counts end on the second set, ragged
    tiles at the right / bottom edges: bit-exact with the oracle, chained,
    including the dual carried to the next packet."""
    sc = evr.SolverConfig(max_iterations=pd)
    mc = evr.ManifoldConfig(denoise_iterations=tv)
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0, engine=1)
    ref = O.OracleStream(H, W, O.make_config(max_iterations=pd, denoise_iterations=tv))
    for pk in uniform_packets(H, W, 4, 300, seed=H * tv + pd, t_step=2):
        _, frame, res = evr.process_packet(st, pk, mc, sc, evr.Thresholds())
        it, rel = ref.process(np.ascontiguousarray(pk))
        assert res.iterations == it
        assert np.array_equal(frame, ref.u)
        assert np.array_equal(st.p, ref.p)


def test_float32_engine_within_log_tolerance():
    """float32 surface+solver: max |log u - log u_ref| <= 1e-4, teacher-forced
    per packet and chained over the DVS128 S-stream fixture."""
    d = load("stream_s_dvs128.npz")
    sc = evr.SolverConfig()
    st = device_state(d, sc, precision=1)
    worst = 0.0
    for k, pk in enumerate(packets_of(d)):
        _, frame, res = evr.process_packet(st, pk, evr.ManifoldConfig(), sc, evr.Thresholds())
        worst = max(worst, float(np.abs(np.log(frame) - np.log(d["u"][k])).max()))
    assert worst <= LOG_TOL, worst
    # ingest stays float64: f after ingest equals the reference given the same f
    st.f = d["u"][0].copy()
    st.raw_timestamps = d["raw_ing"][0].copy()
    evr.apply_event(st, evr.Event(x=3, y=4, polarity=1, timestamp=10**9), evr.Thresholds(), sc)
    assert st.f[4, 3] == min(max(d["u"][0][4, 3] * math.exp(0.15), 1.0), 2.0)


def test_float32_chained_u_stream_tolerance():
    H, W = 260, 346
    sc = evr.SolverConfig()
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=1)
    ref = O.OracleStream(H, W, O.make_config())
    worst = 0.0
    for pk in uniform_packets(H, W, 6, 500, seed=11, t_step=1):
        _, frame, _ = evr.process_packet(st, pk, evr.ManifoldConfig(), sc, evr.Thresholds())
        ref.process(np.ascontiguousarray(pk))
        worst = max(worst, float(np.abs(np.log(frame) - np.log(ref.u)).max()))
    assert worst <= LOG_TOL, worst


@pytest.mark.parametrize("engine", [0, 1])
def test_float32_streaming_tolerance_vs_oracle(engine):
    """float32 fused streaming list (packed state, FFMA, MUFU) at a sensor
    AUTO sends to it: within the north_star log tolerance, chained."""
    H, W = 300, 400
    sc = evr.SolverConfig()
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=1, engine=engine)
    ref = O.OracleStream(H, W, O.make_config())
    worst = 0.0
    for pk in uniform_packets(H, W, 4, 1000, seed=17, t_step=1):
        _, frame, _ = evr.process_packet(st, pk, evr.ManifoldConfig(), sc, evr.Thresholds())
        ref.process(np.ascontiguousarray(pk))
        worst = max(worst, float(np.abs(np.log(frame) - np.log(ref.u)).max()))
    assert st.engine() == "streaming"
    assert worst <= LOG_TOL, worst


def test_duplicates_and_clamp_order():
    """Multiply-then-clamp per event in stream order."""
    geom = evr.SensorGeometry(4, 3)
    sc = evr.SolverConfig()
    st = evr.init_state(geom, sc)
    st.f = np.full((3, 4), 1.95)
    seq = [evr.Event(0, 0, 1, 1), evr.Event(1, 2, -1, 2), evr.Event(0, 0, -1, 3),
           evr.Event(0, 0, 1, 4), evr.Event(1, 2, -1, 5)] * 300  # 1500 events, 2 chunks
    ev = evr.events_to_array(seq)
    ev["t"] = np.arange(len(ev))
    ctx = evr.pipeline._prepare(st, evr.ManifoldConfig(), sc, evr.Thresholds())
    from paper_1607_06283_b200 import _lib
    ctx.call("evr_ingest", _lib.ptr(ev), len(ev))
    st._after_device_write(in_place=("f", "raw_timestamps"))
    f = np.full((3, 4), 1.95)
    raw = np.zeros((3, 4), np.int64)
    O.ingest(f, raw, ev, O.make_config())
    assert np.array_equal(st.f, f) and np.array_equal(st.raw_timestamps, raw)


def test_out_of_range_event_raises():
    st = evr.init_state(evr.SensorGeometry(8, 8), evr.SolverConfig())
    with pytest.raises(IndexError):
        evr.process_packet(st, [evr.Event(8, 0, 1, 1)], evr.ManifoldConfig(),
                           evr.SolverConfig(), evr.Thresholds())


def test_repeat_runs_bitwise_deterministic():
    H, W = 96, 80
    outs = []
    for _ in range(2):
        st = evr.init_state(evr.SensorGeometry(W, H), evr.SolverConfig())
        for pk in uniform_packets(H, W, 2, 700, seed=5, t_step=3):
            _, frame, _ = evr.process_packet(st, pk, evr.ManifoldConfig(), evr.SolverConfig(),
                                             evr.Thresholds())
        outs.append((frame.copy(), st.p.copy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_engines_agree_bitwise():
    H, W = 150, 211
    res = {}
    for eng in ENGINES:
        st = evr.init_state(evr.SensorGeometry(W, H), evr.SolverConfig(), engine=engine_id(eng))
        for pk in uniform_packets(H, W, 3, 500, seed=9, t_step=2):
            _, frame, _ = evr.process_packet(st, pk, evr.ManifoldConfig(), evr.SolverConfig(),
                                             evr.Thresholds())
        res[eng] = (frame.copy(), st.p.copy(), st.engine())
    for eng in ENGINES[1:]:
        assert np.array_equal(res["streaming"][0], res[eng][0]), eng
        assert np.array_equal(res["streaming"][1], res[eng][1]), eng


@pytest.mark.parametrize("precision", [0, 1])
def test_resident_plane_frames_match_streaming_bitwise(precision):
    """Sensors wider than the column kernel's 512 threads run the resident
    engine's shared-memory plane-frame kernel: bit-identical to the streaming
    engine in both precisions."""
    H, W = 120, 600
    sc = evr.SolverConfig(max_iterations=20)
    mc = evr.ManifoldConfig(denoise_iterations=10)
    out = {}
    for eng in ("streaming", "resident"):
        st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=precision,
                            engine=engine_id(eng))
        for pk in uniform_packets(H, W, 3, 1000, seed=21, t_step=1):
            _, frame, _ = evr.process_packet(st, pk, mc, sc, evr.Thresholds())
        out[eng] = (frame.copy(), st.p.copy(), st.context().engine_detail())
    assert "smem frames" in out["resident"][2]
    assert np.array_equal(out["resident"][0], out["streaming"][0])
    assert np.array_equal(out["resident"][1], out["streaming"][1])


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("H,W,tv,pd", [(150, 97, 13, 9), (61, 29, 4, 5), (7, 300, 3, 2),
                                        (260, 346, 50, 50), (720, 1280, 9, 10),
                                        (2048, 1100, 5, 6)])
def test_tile_kernels_bitwise_equal_to_march(H, W, tv, pd, precision):
    """Temporally blocked tiles (K = 2, 3, 4 iterations per launch) give the
    bits of one march launch per iteration, chained over packets, in float64
    and float32, with tile edges crossing the sensor edges."""
    from paper_1607_06283_b200 import _lib

    rng = np.random.default_rng(H * W + tv)
    sc = evr.SolverConfig(max_iterations=pd)
    mc = evr.ManifoldConfig(denoise_iterations=tv)
    n = 400
    ev = evr.make_event_array(rng.integers(0, W, 3 * n), rng.integers(0, H, 3 * n),
                              rng.choice([-1, 1], 3 * n), np.arange(3 * n, dtype=np.int64) * 7)
    out = {}
    for k in (1, 2, 3, 4):
        st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=precision, engine=1)
        st.context().call("evr_set_tile_k", k)
        frames = []
        for s in range(0, 3 * n, n):
            _, fr, res = evr.process_packet_arrays(st, ev[s:s + n], mc, sc, evr.Thresholds())
            frames.append((fr.copy(), res.rel_change))
        out[k] = (frames, st.p.copy(), st.context().engine_detail())
    for k in (2, 3, 4):
        assert f"K={k}" in out[k][2]
        for (a, ra), (b, rb) in zip(out[1][0], out[k][0]):
            assert np.array_equal(a, b) and ra == rb
        assert np.array_equal(out[1][1], out[k][1])
    if precision == 0 and H * W <= 100_000:  # and the oracle
        ref = O.OracleStream(H, W, O.make_config(max_iterations=pd, denoise_iterations=tv))
        for s in range(0, 3 * n, n):
            ref.process(np.ascontiguousarray(ev[s:s + n]))
        assert np.array_equal(out[2][0][-1][0], ref.u)


@pytest.mark.parametrize("data", ["kl", "rof", "l1"])
def test_tgv_and_l1_solvers_bit_exact_vs_oracle(data):
    """TGV (three data terms) and the L1 data term on a steep manifold: the
    CUDA operator kernels reproduce the C restatement bit for bit."""
    rng = np.random.default_rng(7)
    H, W = 37, 53
    yy, xx = np.mgrid[0:H, 0:W]
    t = 3.0 * np.sin(xx / 6.0) * np.cos(yy / 9.0) ** 2
    m = evr.compute_metric(t)
    f = np.clip(1.5 + 0.3 * np.sin(xx / 5.0) + rng.normal(0, 0.05, (H, W)), 1.0, 2.0)
    u, w = evr.tgv_manifold_solve(f, m, 6.0, alpha0=1.7, alpha1=0.9, iterations=40, data=data,
                                  return_w=True)
    ru, rw = O.tgv_solve(f, m.tx, m.ty, m.G, m.sqrtG, 6.0, alpha0=1.7, alpha1=0.9, data=data,
                         iterations=40)
    assert np.array_equal(u, ru) and np.array_equal(w, rw)
    if data == "l1":
        assert np.array_equal(evr.l1_manifold_solve(f, m, 3.0, 50),
                              O.l1_solve(f, m.tx, m.ty, m.G, m.sqrtG, 3.0, 50))
    with pytest.raises(ValueError, match="positive"):
        evr.tgv_manifold_solve(f, m, 1.0, alpha0=0.0)
    with pytest.raises(ValueError, match="data term"):
        evr.tgv_manifold_solve(f, m, 1.0, data="huber")


@pytest.mark.parametrize("cfg", ["C4", "C3", "C5"])
def test_baseline_sizes_streaming_vs_oracle(cfg):
    """BASELINE configs at their full sizes on the streaming engine (tile
    kernels, 4 iterations per launch): 640x480 (2 chained packets), 1280x720
    at 100 primal-dual iterations and 2048x2048 (1 packet each), generator U
    at 1 Mev/s, 1000-event packets: float64 bit-exact with the C oracle, and
    the float32 engine within the north-star 1e-4 on log u."""
    H, W, pd, n = {"C4": (480, 640, 50, 2), "C3": (720, 1280, 100, 1),
                   "C5": (2048, 2048, 50, 1)}[cfg]
    sc = evr.SolverConfig(max_iterations=pd)
    mc = evr.ManifoldConfig()
    pks = uniform_packets(H, W, n, 1000, seed=H + W + pd, t_step=1)
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0, engine=1)
    s32 = evr.init_state(evr.SensorGeometry(W, H), sc, precision=1, engine=1)
    ref = O.OracleStream(H, W, O.make_config(max_iterations=pd))
    for pk in pks:
        _, frame, res = evr.process_packet(st, pk, mc, sc, evr.Thresholds())
        _, f32, _ = evr.process_packet(s32, pk, mc, sc, evr.Thresholds())
        it, rel = ref.process(np.ascontiguousarray(pk))
        assert res.iterations == it == pd
        assert np.array_equal(frame, ref.u)
        assert res.rel_change == pytest.approx(rel, rel=1e-9)
        assert np.abs(np.log(f32) - np.log(ref.u)).max() <= LOG_TOL
    assert np.array_equal(st.p, ref.p) and np.array_equal(st.f, ref.f)
    assert "k_pd_tile" in st.context().engine_detail()


@pytest.mark.parametrize("iters", [1, 2, 3, 4, 5, 7, 13])
@pytest.mark.parametrize("H,W", [(37, 53), (260, 346)])
def test_rof_and_l1_tiles_bit_exact_vs_oracle(H, W, iters):
    """rof_manifold_solve (solve.py:264-293) and the L1 data term run on the
    temporally blocked tiles (K iterations per launch, remainders merged
    into the last tile): bit-identical to the C oracle for every iteration
    count, on a steep manifold, at DAVIS346 size too."""
    rng = np.random.default_rng(iters)
    yy, xx = np.mgrid[0:H, 0:W]
    t = 3.0 * np.sin(xx / 6.0) * np.cos(yy / 9.0) ** 2
    m = evr.compute_metric(t)
    f = np.clip(1.5 + 0.3 * np.sin(xx / 5.0) + rng.normal(0, 0.05, (H, W)), 1.0, 2.0)
    got = evr.rof_manifold_solve(f, m, 8.0, iters)
    assert np.array_equal(got, O.rof_solve(f, m.tx, m.ty, m.G, m.sqrtG, 8.0, iters))
    got = evr.l1_manifold_solve(f, m, 3.0, iters)
    assert np.array_equal(got, O.l1_solve(f, m.tx, m.ty, m.G, m.sqrtG, 3.0, iters))


@pytest.mark.parametrize("tol", [0.0, 1e-3])
def test_resident_exchange_repeatable_under_load(tol):
    """Race evidence without a sanitizer (closed on this pool): the resident
    kernel's relaxed tagged-word halo exchange and (tol > 0) its per-iteration
    rel_change fold, replayed 40 times from the same state at the DAVIS346
    shape, with a concurrent streaming context loading the GPU from another
    stream -- every replay bit-identical to the oracle."""
    H, W = 260, 346
    sc = evr.SolverConfig(max_iterations=30, convergence_tol=tol)
    mc, th = evr.ManifoldConfig(denoise_iterations=20), evr.Thresholds()
    pk = uniform_packets(H, W, 2, 500, seed=11, t_step=2)
    ref = O.OracleStream(H, W, O.make_config(max_iterations=30, denoise_iterations=20,
                                             convergence_tol=tol))
    ref.process(np.ascontiguousarray(pk[0]))
    u0, f0, raw0, p0 = ref.u.copy(), ref.f.copy(), ref.raw.copy(), ref.p.copy()
    it_ref, _ = ref.process(np.ascontiguousarray(pk[1]))
    noise = evr.init_state(evr.SensorGeometry(1280, 720), evr.SolverConfig(), engine=1)
    noise_pk = uniform_packets(720, 1280, 1, 1000, seed=3, t_step=1)[0]
    st = evr.init_state(evr.SensorGeometry(W, H), sc)
    for rep in range(40):
        st.u, st.f, st.raw_timestamps, st.p = u0.copy(), f0.copy(), raw0.copy(), p0.copy()
        st.packet_starts.clear()
        st.packet_starts.append(int(pk[0]["t"][0]))
        noise.context().call("evr_process_packet_async", evr._lib.ptr(noise_pk), len(noise_pk),
                             1000.0)
        _, frame, res = evr.process_packet_arrays(st, pk[1], mc, sc, th)
        assert st.engine() == "resident"
        assert res.iterations == it_ref
        assert np.array_equal(frame, ref.u) and np.array_equal(st.p, ref.p), rep
    noise.context().call("evr_synchronize", None)
