"""Long chained streams at the BASELINE sizes (VERDICT round 1, items 1 and
weak 1-2): float64 bit-exact over >= 5 chained 1280x720 packets for both
synthetic generators -- U (uniform events, nearly flat surfaces) and S (the
simulator's moving scene, steep metrics) -- and the
float32 engine's chained drift on log intensity against the float64 engine
over 300 DVS128 S-stream packets and 50 1280x720 packets, each held to the
north-star 1e-4 (SURVEY.md B.4 measured 6.7e-5 after 300 packets at 128^2).

The worst drift of every run is appended to gpurun_out/drift.log (when that
directory exists) so the numbers travel back with the GPU run.
"""

import os

import numpy as np
import pytest

import paper_1607_06283_b200 as evr
from oracle import oracle as O
from paper_1607_06283_b200.simulate import generate_events_array, render_scene

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG_TOL = 1e-4


def _log(msg):
    d = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "drift.log"), "a") as fh:
            fh.write(msg + "\n")
    print(msg)


def u_packets(H, W, n, epp, seed, t_step=1):
    rng = np.random.default_rng(seed)
    m = n * epp
    ev = evr.make_event_array(rng.integers(0, W, m), rng.integers(0, H, m),
                              rng.choice([-1, 1], m), np.arange(m, dtype=np.int64) * t_step)
    return [ev[s:s + epp] for s in range(0, m, epp)]


def s_packets(H, W, n, epp, scene="moving_sine", frames=16, skip=0):
    """Generator S: the simulator's scene (cli.py:256-264 doubles the frame
    count until the stream is long enough), events in its (t, y, x, p)
    order; `skip` packets dropped from the front."""
    geom = evr.SensorGeometry(width=W, height=H)
    need = (n + skip) * epp
    while True:
        ev = generate_events_array(render_scene(scene, geom, frames), 0.15, 0.15)
        if len(ev) >= need or frames >= 4096:
            break
        frames *= 2
    assert len(ev) >= need, (len(ev), need)
    ev = ev[skip * epp:need]
    return [ev[s:s + epp] for s in range(0, len(ev), epp)]


@pytest.mark.parametrize("gen", ["U", "S", "steep"])
def test_c3_float64_chained_bit_exact(gen):
    """1280x720, 1000-event packets, 100 primal-dual + 50 TV-L1 iterations,
    six packets chained through the streaming engine's tiles: u, p, f and
    the timestamp map identical to the C oracle after every packet.  U:
    uniform events (nearly flat surfaces); S: the simulator's moving scene
    (at this size 1000 events cover under one row of a frame, so its
    surfaces stay flat too); steep: U events on a state whose timestamp map
    carries a sawtooth of ages, so every packet's metric is steep (max G
    above 1.5) and the fast float64 division / square-root paths and the
    projections run away from sqrt(G) = 1 at full size."""
    H, W, pd = 720, 1280, 100
    t0 = 100_000
    if gen == "S":
        pk = s_packets(H, W, 6, 1000, frames=8, skip=3)
    else:
        pk = u_packets(H, W, 6, 1000, seed=2 if gen == "U" else 5)
        for p in pk:
            p["t"] += t0
    sc, mc, th = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(), evr.Thresholds()
    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0)
    ref = O.OracleStream(H, W, O.make_config(max_iterations=pd))
    if gen == "steep":
        yy, xx = np.mgrid[0:H, 0:W]
        # ages rising over 16 columns and dropping back: a ramp of slope
        # ~0.2 per pixel on the surface, then an edge of ~3 that TV-L1 keeps
        raw = (t0 - (xx % 16) * 400 - (yy % 9) * 100).astype(np.int64)
        st.raw_timestamps = raw.copy()
        ref.raw[...] = raw
        st.packet_starts.append(t0 - 6400)
        ref.packet_starts.append(t0 - 6400)
    gmax = 1.0
    for k, p in enumerate(pk):
        _, frame, res = evr.process_packet_arrays(st, p, mc, sc, th)
        it, rel = ref.process(np.ascontiguousarray(p))
        assert res.iterations == it == pd
        assert np.array_equal(frame, ref.u), f"u differs at packet {k}"
        assert res.rel_change == pytest.approx(rel, rel=1e-9)
        if k == len(pk) - 1:  # the metric of the last packet's surface (device planes)
            from paper_1607_06283_b200 import _lib

            G = np.empty((H, W))
            st.context().call("evr_get_metric", None, None, _lib.ptr(G), None)
            gmax = float(G.max())
    assert np.array_equal(st.p, ref.p) and np.array_equal(st.f, ref.f)
    assert np.array_equal(st.raw_timestamps, ref.raw)
    _log(f"C3 f64 {gen}-stream: {len(pk)} chained packets bit-exact, max G of the last "
         f"surface {gmax:.3f}")
    if gen == "steep":
        assert gmax > 1.5  # the steep-metric paths are exercised


def test_c2_float64_s_stream_both_engines_bit_exact():
    """DAVIS346 S-stream (steep metrics at full size), 8 chained packets on
    the resident and the streaming engine: both identical to the oracle."""
    H, W = 260, 346
    pk = s_packets(H, W, 8, 500, frames=16, skip=2)
    sc, mc, th = evr.SolverConfig(), evr.ManifoldConfig(), evr.Thresholds()
    ref = O.OracleStream(H, W, O.make_config())
    states = {e: evr.init_state(evr.SensorGeometry(W, H), sc, precision=0, engine=e)
              for e in (1, 2)}
    for k, p in enumerate(pk):
        ref.process(np.ascontiguousarray(p))
        for e, st in states.items():
            _, frame, _ = evr.process_packet_arrays(st, p, mc, sc, th)
            assert np.array_equal(frame, ref.u), f"engine {e}, packet {k}"
    for st in states.values():
        assert np.array_equal(st.p, ref.p)


def _drift(H, W, pk, pd, tag):
    sc, mc, th = evr.SolverConfig(max_iterations=pd), evr.ManifoldConfig(), evr.Thresholds()
    s64 = evr.init_state(evr.SensorGeometry(W, H), sc, precision=0)
    s32 = evr.init_state(evr.SensorGeometry(W, H), sc, precision=1)
    worst, at = 0.0, 0
    marks = []
    for k, (a, b) in enumerate(zip(evr.stream_packets(s64, pk, mc, sc, th),
                                   evr.stream_packets(s32, pk, mc, sc, th))):
        d = float(np.abs(np.log(a[0]) - np.log(b[0])).max())
        if d > worst:
            worst, at = d, k
        if (k + 1) % max(1, len(pk) // 6) == 0:
            marks.append(f"{k + 1}:{d:.2e}")
    _log(f"{tag}: float32 vs float64, {len(pk)} chained packets, worst max|dlog u| {worst:.3e} "
         f"(packet {at}); after packet n: {' '.join(marks)}")
    return worst


def test_c1_float32_drift_300_packets_s_stream():
    """DVS128 S-stream, 300 chained 500-event packets: the float32 engine
    stays within 1e-4 on log u of the bit-exact float64 engine."""
    pk = s_packets(128, 128, 300, 500, frames=16)
    assert _drift(128, 128, pk, 50, "C1 S-stream") <= LOG_TOL


def test_c1_float32_drift_300_packets_u_stream():
    pk = u_packets(128, 128, 300, 500, seed=0, t_step=10)
    assert _drift(128, 128, pk, 50, "C1 U-stream") <= LOG_TOL


def test_c3_float32_drift_50_packets():
    """1280x720, 50 chained 1000-event packets at 1 Mev/s (100 primal-dual
    iterations): float32 within 1e-4 on log u of float64 throughout."""
    pk = u_packets(720, 1280, 50, 1000, seed=2)
    assert _drift(720, 1280, pk, 100, "C3 U-stream") <= LOG_TOL


def test_c3_float32_drift_s_stream():
    pk = s_packets(720, 1280, 30, 1000, frames=8, skip=3)
    assert _drift(720, 1280, pk, 100, "C3 S-stream") <= LOG_TOL
