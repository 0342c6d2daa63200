"""The reference's own behavioural tests, restated against the drop-in API
(reference: pkg/tests/test_pipeline.py, test_solve.py, test_surface.py).
Each test names the reference test it mirrors."""

import io
import math
import sys

import numpy as np
import pytest

import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import (Event, ManifoldConfig, PacketPolicy, SensorGeometry,
                                   SolverConfig, Thresholds)

pytestmark = pytest.mark.gpu

GEOM = SensorGeometry(width=16, height=16)


def make_events(n, geom=GEOM, seed=0, t_step=10):
    rng = np.random.default_rng(seed)
    return [Event(x=int(rng.integers(0, geom.width)), y=int(rng.integers(0, geom.height)),
                  polarity=int(rng.choice([-1, 1])), timestamp=k * t_step) for k in range(n)]


# --- test_pipeline.py ---------------------------------------------------------


def test_init_state_midpoint():  # test_pipeline.py:40-46
    state = evr.init_state(GEOM, SolverConfig(u_min=1.0, u_max=2.0))
    np.testing.assert_array_equal(state.u, 1.5)
    np.testing.assert_array_equal(state.f, state.u)
    np.testing.assert_array_equal(state.p, 0.0)
    np.testing.assert_array_equal(state.raw_timestamps, 0)
    assert state.frame_index == 0


def test_apply_event_quanta_clamp_locality():  # test_pipeline.py:52-79
    cfg = SolverConfig()
    state = evr.init_state(GEOM, cfg)
    evr.apply_event(state, Event(x=3, y=5, polarity=1, timestamp=7), Thresholds(), cfg)
    assert state.f[5, 3] == 1.5 * math.exp(0.15)
    assert state.raw_timestamps[5, 3] == 7
    evr.apply_event(state, Event(x=1, y=1, polarity=-1, timestamp=3), Thresholds(), cfg)
    assert state.f[1, 1] == 1.5 * math.exp(-0.15)
    state.f[2, 2] = cfg.u_max  # caller edit of the host view is honoured
    evr.apply_event(state, Event(x=2, y=2, polarity=1, timestamp=1), Thresholds(), cfg)
    assert state.f[2, 2] == cfg.u_max
    before = state.f.copy()
    evr.apply_event(state, Event(x=4, y=6, polarity=1, timestamp=1), Thresholds(), cfg)
    np.testing.assert_array_equal(np.argwhere(state.f != before), [[6, 4]])


def test_empty_packet_is_identity():  # test_pipeline.py:85-94
    state = evr.init_state(GEOM, SolverConfig())
    u_before = state.u.copy()
    state, frame, result = evr.process_packet(state, [], ManifoldConfig(), SolverConfig(),
                                              Thresholds())
    np.testing.assert_array_equal(frame, u_before)
    assert result is None and state.frame_index == 0


def test_packet_reanchors_measurement_to_solution():  # test_pipeline.py:97-106
    state = evr.init_state(GEOM, SolverConfig())
    state, frame, result = evr.process_packet(state, make_events(40), ManifoldConfig(),
                                              SolverConfig(), Thresholds())
    np.testing.assert_array_equal(state.f, state.u)
    np.testing.assert_array_equal(frame, state.u)
    assert frame is state.u
    assert state.frame_index == 1 and result.iterations == SolverConfig().max_iterations


def test_packet_monotone_raw_timestamps():  # test_pipeline.py:109-118
    state = evr.init_state(GEOM, SolverConfig())
    events = make_events(60, seed=1)
    snaps = []
    for chunk in (events[:20], events[20:40], events[40:]):
        snaps.append(state.raw_timestamps.copy())
        evr.process_packet(state, chunk, ManifoldConfig(), SolverConfig(), Thresholds())
    snaps.append(state.raw_timestamps.copy())
    for a, b in zip(snaps, snaps[1:]):
        assert np.all(b >= a)


def test_frame_counts_skip_and_short_final():  # test_pipeline.py:124-159
    frames = []
    _, stats = evr.run_stream(make_events(1500), GEOM, PacketPolicy(500), ManifoldConfig(),
                              SolverConfig(), Thresholds(), sink=lambda i, fr: frames.append(i))
    assert frames == [0, 1, 2] and stats.packets == 3 and stats.events_consumed == 1500
    frames = []
    evr.run_stream(make_events(1500), GEOM, PacketPolicy(500, frames_to_skip=2),
                   ManifoldConfig(), SolverConfig(), Thresholds(),
                   sink=lambda i, fr: frames.append(i))
    assert len(frames) == 1
    frames = []
    _, stats = evr.run_stream(make_events(650), GEOM, PacketPolicy(500), ManifoldConfig(),
                              SolverConfig(), Thresholds(), sink=lambda i, fr: frames.append(fr))
    assert stats.packets == 2 and len(frames) == 2


def test_split_run_bit_identical():  # test_pipeline.py:162-183
    geom = SensorGeometry(width=24, height=24)
    events = make_events(2000, geom=geom, seed=3, t_step=2)
    args = (geom, PacketPolicy(500), ManifoldConfig(), SolverConfig(), Thresholds())
    whole, first, second = [], [], []
    evr.run_stream(events, *args, sink=lambda i, fr: whole.append(fr.copy()))
    state, _ = evr.run_stream(events[:500], *args, sink=lambda i, fr: first.append(fr.copy()))
    evr.run_stream(events[500:], *args, sink=lambda i, fr: second.append(fr.copy()), state=state)
    assert len(whole) == len(first + second)
    for a, b in zip(whole, first + second):
        np.testing.assert_array_equal(a, b)


def test_fidelity_dominant_limit_reproduces_integration():  # test_pipeline.py:186-204
    geom = SensorGeometry(width=12, height=12)
    events = make_events(900, geom=geom, seed=5)
    cfg = SolverConfig(lam=1e6)
    frames = []
    evr.run_stream(events, geom, PacketPolicy(300), ManifoldConfig(enabled=False), cfg,
                   Thresholds(), sink=lambda i, fr: frames.append(fr.copy()))
    f = np.full((12, 12), 1.5)
    for ev in events:
        c = math.exp(0.15) if ev.polarity > 0 else math.exp(-0.15)
        f[ev.y, ev.x] = min(max(f[ev.y, ev.x] * c, cfg.u_min), cfg.u_max)
    assert np.abs(frames[-1] - f).max() <= 1e-3


def test_stats_line_and_energy_trace(capsys):  # test_pipeline.py:207-214, test_cli.py:80-89
    trace = io.StringIO()
    evr.run_stream(make_events(600), GEOM, PacketPolicy(200), ManifoldConfig(), SolverConfig(),
                   Thresholds(), stats_every=2, log=sys.stderr, trace=trace)
    err = capsys.readouterr().err
    assert "packet 2:" in err and "iterations" in err
    rows = trace.getvalue().strip().splitlines()
    assert rows[0] == "packet,iteration,energy,rel_change" and len(rows) == 1 + 3 * 50


# --- test_solve.py ------------------------------------------------------------


def test_config_validation():  # test_solve.py:32-46
    with pytest.raises(ValueError, match="step sizes"):
        SolverConfig(tau=1.0, sigma=1.0)
    with pytest.raises(ValueError):
        SolverConfig(u_min=0.0, u_max=1.0)


def test_prox_data_cases():  # test_solve.py:52-72
    m = evr.flat_metric((1, 3))
    out = evr.prox_data(np.array([[0.2, 1.4, 3.0]]), np.array([[1.5, 1.5, 1.5]]), m, 0.3,
                        SolverConfig(lam=0.0))
    np.testing.assert_allclose(out, [[1.0, 1.4, 2.0]])
    f = np.array([[1.2, 1.5], [1.8, 1.01]])
    np.testing.assert_allclose(evr.prox_data(f.copy(), f, evr.flat_metric((2, 2)), 0.7,
                                             SolverConfig(lam=2.0)), f, atol=1e-14)
    with pytest.raises(ValueError, match="positive"):
        evr.prox_data(np.ones((1, 1)), np.zeros((1, 1)), evr.flat_metric((1, 1)), 0.1,
                      SolverConfig())


def test_solve_fixed_point_box_and_errors():  # test_solve.py:190-247
    res = evr.primal_dual_solve(np.full((8, 8), 1.3), evr.flat_metric((8, 8)),
                                SolverConfig(lam=0.7))
    np.testing.assert_allclose(res.u, 1.3, atol=1e-12)
    with pytest.raises(ValueError, match="box"):
        evr.primal_dual_solve(np.full((4, 4), 5.0), evr.flat_metric((4, 4)), SolverConfig())
    with pytest.raises(ValueError):
        evr.primal_dual_solve(np.full((4, 4), 1.5), evr.flat_metric((5, 5)), SolverConfig())


def test_solve_single_iteration_matches_op_composition():  # test_solve.py:261-273
    rng = np.random.default_rng(32)
    cfg = SolverConfig(lam=0.9, max_iterations=1)
    f = np.clip(1.5 + 0.4 * rng.normal(0, 1, (11, 7)), 1, 2)
    m = evr.compute_metric(rng.normal(0, 1.3, (11, 7)))
    u0 = np.clip(1.5 + 0.4 * rng.normal(0, 1, (11, 7)), 1, 2)
    p0 = rng.normal(0, 0.5, (11, 7, 3))
    res = evr.primal_dual_solve(f, m, cfg, u_init=u0, p_init=p0)
    u1 = evr.prox_data(u0 - cfg.tau * evr.surface_gradient_adjoint(p0, m), f, m, cfg.tau, cfg)
    p1 = evr.prox_dual(p0 + cfg.sigma * evr.surface_gradient(2 * u1 - u0, m), m)
    np.testing.assert_allclose(res.u, u1, atol=1e-14)
    np.testing.assert_allclose(res.p, p1, atol=1e-14)


# --- test_surface.py ----------------------------------------------------------


def test_adjointness():  # test_surface.py:217-236
    rng = np.random.default_rng(7)
    for shape in [(9, 13), (2, 2), (31, 17)]:
        m = evr.compute_metric(rng.normal(0, 2, shape))
        u = rng.normal(0, 1, shape)
        p = rng.normal(0, 1, shape + (3,))
        lhs = np.sum(evr.surface_gradient(u, m) * p)
        rhs = np.sum(u * evr.surface_gradient_adjoint(p, m))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def test_denoise_validation_and_range():  # test_surface.py:78-115
    with pytest.raises(ValueError):
        evr.denoise_timestamps(evr.TimeSurface(np.zeros((4, 4)), 3.0), 0.0)
    t = np.random.default_rng(1).uniform(0, 3, (10, 12))
    out = evr.denoise_timestamps(evr.TimeSurface(t, 3.0), 0.5, 30)
    assert out.t.min() >= 0 and out.t.max() <= 3.0


def test_install_reroutes_reference_stream():
    """install() patches an evrecon.pipeline module's seam."""
    import types

    fake = types.ModuleType("evrecon.pipeline")
    fake.init_state = fake.process_packet = fake.primal_dual_solve = fake.run_stream = None
    cli = types.ModuleType("evrecon.cli")
    cli.run_stream = None
    evr.install(fake, cli)
    try:
        assert fake.process_packet is evr.process_packet
        assert fake.init_state is evr.init_state
        assert fake.run_stream is evr.run_stream and cli.run_stream is evr.run_stream
    finally:
        evr.uninstall()
    assert fake.process_packet is None and cli.run_stream is None


def test_engine_detail_names_the_kernel():
    st = evr.init_state(SensorGeometry(width=346, height=260), SolverConfig())
    evr.process_packet(st, make_events(50, SensorGeometry(width=346, height=260)),
                       ManifoldConfig(), SolverConfig(), Thresholds())
    d = st.context().engine_detail()
    assert d.startswith("k_resident_col<f64,NT=352,RB=2>") and "x130 CTAs" in d
    st = evr.init_state(SensorGeometry(width=640, height=480), SolverConfig(), precision=1)
    evr.process_packet(st, make_events(50, SensorGeometry(width=640, height=480)),
                       ManifoldConfig(), SolverConfig(), Thresholds())
    assert st.context().engine_detail().startswith("streaming k_tv_tile/k_pd_tile<f32,K=4>")


def test_frames_are_fresh_pinned_arrays():
    """Each packet's frame is a new array (the reference's result.u), served
    from the pinned pool; an old frame keeps its values after later packets
    and after being dropped and reallocated."""
    from paper_1607_06283_b200 import _lib

    st = evr.init_state(GEOM, SolverConfig())
    ev = make_events(90)
    _, f1, _ = evr.process_packet(st, ev[:30], ManifoldConfig(), SolverConfig(), Thresholds())
    keep = f1.copy()
    _, f2, _ = evr.process_packet(st, ev[30:60], ManifoldConfig(), SolverConfig(), Thresholds())
    assert f1 is not f2 and np.array_equal(f1, keep) and not np.array_equal(f1, f2)
    assert f2.flags.c_contiguous and f2.dtype == np.float64
    # a read-only snapshot: an in-place edit would not reach the device state
    assert not f2.flags.writeable
    with pytest.raises(ValueError):
        f2[0, 0] = 1.5
    del f1
    _, f3, _ = evr.process_packet(st, ev[60:], ManifoldConfig(), SolverConfig(), Thresholds())
    assert np.array_equal(f3, st.u) and not np.array_equal(f2, f3)
    a = _lib.pinned_empty((3, 5), np.int64)
    a[:] = 7
    assert a.sum() == 105


def test_get_frame_async_matches_get_frame():
    from paper_1607_06283_b200 import _lib

    st = evr.init_state(GEOM, SolverConfig(), precision=1)
    evr.process_packet(st, make_events(40), ManifoldConfig(), SolverConfig(), Thresholds())
    ctx = st.context()
    a = np.empty(GEOM.height * GEOM.width)
    b = _lib.pinned_empty((GEOM.height, GEOM.width))
    ctx.call("evr_get_frame", _lib.ptr(a))
    ctx.call("evr_get_frame_async", _lib.ptr(b))
    ctx.call("evr_synchronize", None)
    assert np.array_equal(a.reshape(b.shape), b)


@pytest.mark.parametrize("precision,engine,depth", [(0, 0, 2), (0, 1, 3), (1, 0, 4), (1, 1, 1)])
def test_stream_packets_matches_process_packet(precision, engine, depth):
    """The pipelined stream (packet k+1 in flight while frame k is read back)
    yields exactly the frames and results of one process_packet per packet
    and leaves the same state behind."""
    geom = SensorGeometry(width=37, height=23)
    ev = evr.events_to_array(make_events(700, geom, seed=3))
    pk = [ev[s:s + 100] for s in range(0, len(ev), 100)]
    mc, sc, th = ManifoldConfig(), SolverConfig(max_iterations=20), Thresholds()
    a = evr.init_state(geom, sc, precision=precision, engine=engine)
    ref = [evr.process_packet_arrays(a, p, mc, sc, th) for p in pk]
    b = evr.init_state(geom, sc, precision=precision, engine=engine)
    got = list(evr.stream_packets(b, pk, mc, sc, th, depth=depth))
    assert len(got) == len(ref)
    for (_, fr, rr), (fg, rg) in zip(ref, got):
        assert np.array_equal(fr, fg)
        assert rr.iterations == rg.iterations and rr.rel_change == rg.rel_change
    assert np.array_equal(a.u, b.u) and np.array_equal(a.p, b.p)
    assert np.array_equal(a.f, b.f) and np.array_equal(a.raw_timestamps, b.raw_timestamps)
    assert a.frame_index == b.frame_index == len(pk)
    assert list(a.packet_starts) == list(b.packet_starts)
    assert np.array_equal(got[-1][1].p, a.p)  # last result still holds the state's dual


def test_stream_packets_decimation_and_errors():
    geom = SensorGeometry(width=16, height=16)
    ev = evr.events_to_array(make_events(600))
    pk = [ev[s:s + 100] for s in range(0, 600, 100)]
    mc, sc, th = ManifoldConfig(), SolverConfig(max_iterations=10), Thresholds()
    st = evr.init_state(geom, sc)
    got = list(evr.stream_packets(st, pk, mc, sc, th, want_frames=lambda i: i % 3 == 0))
    assert [f is not None for f, _ in got] == [True, False, False, True, False, False]
    with pytest.raises(ValueError):
        list(evr.stream_packets(st, pk, mc, sc, th, depth=5))
    with pytest.raises(ValueError, match="ticket"):
        st.context().call("evr_frame_wait", 12345, None)
    # an event outside the sensor is reported by its packet's wait
    bad = evr.make_event_array([3, 99], [2, 2], [1, 1], [10_000, 10_010])
    with pytest.raises((ValueError, IndexError)):
        list(evr.stream_packets(st, [bad], mc, sc, th))
    # an empty packet yields the current frame after the ones before it
    st2 = evr.init_state(geom, sc)
    out = list(evr.stream_packets(st2, [pk[0], pk[0][:0]], mc, sc, th))
    assert out[1][1] is None and np.array_equal(out[0][0], out[1][0])


def _acceptance8_stream(seed_scene="moving_sine", n=60):
    """The convergence-budget workload of acceptance criterion 8
    (test_acceptance.py:273-308): 64x64 simulator stream, 500-event packets."""
    from paper_1607_06283_b200.simulate import generate_events_array, render_scene

    geom = SensorGeometry(width=64, height=64)
    ev = generate_events_array(render_scene(seed_scene, geom, n), 0.15, 0.15)
    return geom, [ev[s:s + 500] for s in range(0, len(ev), 500)]


@pytest.mark.parametrize("precision", [0, 1])
def test_device_early_stop_matches_host_loop(precision):
    """convergence_tol > 0 on the resident engine: rel_change folded on the
    device every iteration and the stop taken there (one launch per packet,
    no host round trip per iteration) -- the same iteration counts, frames
    and duals as the host-driven loop of the streaming engine, and (float64)
    the same as the C oracle."""
    from oracle import oracle as O

    geom, pk = _acceptance8_stream()
    mc, th = ManifoldConfig(), Thresholds()
    sc = SolverConfig(lam=2.0, max_iterations=50, convergence_tol=1e-3)
    dev = evr.init_state(geom, sc, precision=precision)
    host = evr.init_state(geom, sc, precision=precision, engine=1)
    ref = O.OracleStream(64, 64, O.make_config(lam=2.0, max_iterations=50, convergence_tol=1e-3))
    its = []
    for k, p in enumerate(pk[:30]):
        n0 = dev.context().launch_count()
        _, fd, rd = evr.process_packet_arrays(dev, p, mc, sc, th)
        launches = dev.context().launch_count() - n0
        _, fh, rh = evr.process_packet_arrays(host, p, mc, sc, th)
        assert dev.engine() == "resident" and launches == 1
        assert rd.iterations == rh.iterations, k
        assert np.array_equal(fd, fh), k
        assert rd.rel_change == pytest.approx(rh.rel_change, rel=1e-9)
        if precision == 0:
            it, _ = ref.process(np.ascontiguousarray(p))
            assert rd.iterations == it and np.array_equal(fd, ref.u), k
        its.append(rd.iterations)
    assert np.array_equal(dev.p, host.p)
    assert min(its) < 50  # the stop is taken


def test_stream_packets_early_stop_pipelined():
    """The pipelined stream keeps packets in flight with convergence_tol > 0
    when the engine stops on the device (no per-packet fallback)."""
    geom, pk = _acceptance8_stream("two_bars", 80)
    mc, th = ManifoldConfig(), Thresholds()
    sc = SolverConfig(lam=2.0, max_iterations=50, convergence_tol=1e-3)
    a = evr.init_state(geom, sc)
    ref = [evr.process_packet_arrays(a, p, mc, sc, th) for p in pk[:12]]
    b = evr.init_state(geom, sc)
    got = list(evr.stream_packets(b, pk[:12], mc, sc, th))
    for (_, fr, rr), (fg, rg) in zip(ref, got):
        assert np.array_equal(fr, fg) and rr.iterations == rg.iterations
        assert rg.packet_ms is not None and rg.packet_ms > 0


def test_stream_source_error_delivers_computed_frames():
    """A packet source that fails (e.g. StreamOrderError from read_stream)
    still gets every frame computed before the failure, in order, and then
    the exception -- as the reference's run_stream, which hands frame k to
    the sink before it reads packet k+1."""
    geom = SensorGeometry(width=20, height=14)
    ev = evr.events_to_array(make_events(400, geom, seed=4))
    pk = [ev[s:s + 100] for s in range(0, 400, 100)]
    mc, sc, th = ManifoldConfig(), SolverConfig(max_iterations=10), Thresholds()
    ref_state = evr.init_state(geom, sc)
    ref = [evr.process_packet_arrays(ref_state, p, mc, sc, th)[1].copy() for p in pk[:3]]

    def source():
        yield from pk[:3]
        raise evr.StreamOrderError(0, "timestamp went backwards")

    st = evr.init_state(geom, sc)
    got = []
    with pytest.raises(evr.StreamOrderError):
        for frame, _ in evr.stream_packets(st, source(), mc, sc, th, depth=3):
            got.append(frame.copy())
    assert len(got) == 3 and all(np.array_equal(a, b) for a, b in zip(got, ref))
    # run_stream: the sink saw the three frames, then the error propagated
    seen = []
    with pytest.raises(evr.StreamOrderError):
        evr.run_stream(_bad_events(pk), geom, PacketPolicy(events_per_packet=100), mc, sc, th,
                       sink=lambda i, f: seen.append(i))
    assert seen == [0, 1, 2]


def _bad_events(pk):
    for p in pk[:3]:
        for e in p:
            yield Event(int(e["x"]), int(e["y"]), int(e["polarity"]), int(e["t"]))
    raise evr.StreamOrderError(0, "timestamp went backwards")


def test_run_stream_solve_ms_is_per_packet_device_time():
    """run_stream's solve_ms is each packet's own processing time (event
    upload .. frame download on the device), not the pipeline's inter-arrival
    time (pipeline.py:239-249)."""
    geom = SensorGeometry(width=40, height=30)
    ev = evr.events_to_array(make_events(600, geom, seed=8))
    _, stats = evr.run_stream(ev, geom, PacketPolicy(events_per_packet=100), ManifoldConfig(),
                              SolverConfig(), Thresholds(), sink=lambda i, f: None)
    assert stats.packets == 6 and len(stats.solve_ms) == 6
    assert all(0 < ms < 1000 for ms in stats.solve_ms)


@pytest.mark.parametrize("H,W,precision", [(400, 300, 0), (360, 640, 0), (360, 640, 1)])
def test_streaming_engine_device_early_stop(H, W, precision):
    """convergence_tol > 0 on the fused streaming list (sensors the resident
    engine does not take): one march launch + rel_change per iteration behind
    a device stop flag, no host round trip per iteration -- iteration counts
    and (float64) frames identical to the C oracle, a constant launch count
    per packet whatever the stop iteration."""
    from oracle import oracle as O

    rng = np.random.default_rng(H)
    sc = SolverConfig(lam=2.0, max_iterations=40, convergence_tol=2e-3)
    mc, th = ManifoldConfig(), Thresholds()
    st = evr.init_state(SensorGeometry(W, H), sc, precision=precision)
    ref = O.OracleStream(H, W, O.make_config(lam=2.0, max_iterations=40, convergence_tol=2e-3))
    n = 6 * 800
    ev = evr.make_event_array(rng.integers(0, W, n), rng.integers(0, H, n),
                              rng.choice([-1, 1], n), np.arange(n, dtype=np.int64) * 2)
    its, per_packet = [], set()
    for k in range(6):
        p = ev[k * 800:(k + 1) * 800]
        n0 = st.context().launch_count()
        _, frame, res = evr.process_packet_arrays(st, p, mc, sc, th)
        per_packet.add(st.context().launch_count() - n0)
        it, rel = ref.process(np.ascontiguousarray(p))
        assert st.engine() == "streaming"
        assert res.iterations == it, k
        if precision == 0:
            assert np.array_equal(frame, ref.u), k
            assert res.rel_change == pytest.approx(rel, rel=1e-9)
        its.append(res.iterations)
    assert len(per_packet) == 1
    assert min(its) < 40


def test_time_iteration_kernel_hook_leaves_state_alone():
    """evr_time_iteration_kernel (bench.py's live roofline timing) runs the
    streaming list's tiles on the packed scratch sets only: the next packet
    gives the same frame as without the timing call."""
    import ctypes

    from paper_1607_06283_b200 import _lib

    geom = SensorGeometry(width=300, height=400)
    ev = evr.events_to_array(make_events(2000, geom, seed=12))
    pk = [ev[:1000], ev[1000:]]
    mc, sc, th = ManifoldConfig(), SolverConfig(max_iterations=12), Thresholds()
    a = evr.init_state(geom, sc, engine=1)
    b = evr.init_state(geom, sc, engine=1)
    evr.process_packet_arrays(a, pk[0], mc, sc, th)
    evr.process_packet_arrays(b, pk[0], mc, sc, th)
    us, k = ctypes.c_float(0), ctypes.c_int(0)
    for which in (0, 1):
        b.context().call("evr_time_iteration_kernel", which, 5, ctypes.byref(us), ctypes.byref(k))
        assert us.value > 0 and k.value >= 2
    _, fa, _ = evr.process_packet_arrays(a, pk[1], mc, sc, th)
    _, fb, _ = evr.process_packet_arrays(b, pk[1], mc, sc, th)
    assert np.array_equal(fa, fb) and np.array_equal(a.p, b.p)
    with pytest.raises(Exception):  # the resident engine has no iteration kernels
        st = evr.init_state(GEOM, SolverConfig())
        evr.process_packet(st, make_events(30), ManifoldConfig(), SolverConfig(), Thresholds())
        st.context().call("evr_time_iteration_kernel", 0, 5, ctypes.byref(us), None)
