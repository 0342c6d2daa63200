"""Event simulator: scene rendering and the oracle against
the reference's own outputs (tests/golden/simulate.npz, made by
tests/golden/make_sim_golden.py); the GPU generator against both."""

import ast
import os

import numpy as np
import pytest

import paper_1607_06283_b200 as evr
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "simulate.npz")


def golden():
    d = dict(np.load(GOLD))
    specs = ast.literal_eval(str(d["specs"]))
    return d, specs


def test_render_scene_bit_identical_to_reference():
    d, specs = golden()
    geom = evr.SensorGeometry(width=40, height=24)
    for i, (kind, n, dt, params) in enumerate(specs):
        v = evr.render_scene(kind, geom, n, dt=dt, **dict(params))
        assert np.array_equal(v.frames, d[f"c{i}_frames"]), kind
        assert np.array_equal(v.frame_timestamps, d[f"c{i}_ts"])


def test_oracle_generate_matches_reference_events():
    d, specs = golden()
    for i in range(len(specs)):
        out = O.sim_generate(np.log(d[f"c{i}_frames"]), d[f"c{i}_ts"], 0.15, float(d[f"c{i}_dn"]))
        assert np.array_equal(out, d[f"c{i}_ev"]), i
    out = O.sim_generate(np.log(d["r_frames"]), d["r_ts"], 0.2, 0.13)
    assert np.array_equal(out, d["r_ev"])


def test_video_and_scene_validation():  # simulate.py:30-48, :150-199
    with pytest.raises(ValueError, match="n>=2"):
        evr.GroundTruthVideo(np.ones((1, 2, 2)), [0])
    with pytest.raises(ValueError, match="differ"):
        evr.GroundTruthVideo(np.ones((2, 2, 2)), [0, 1, 2])
    with pytest.raises(ValueError, match="strictly increasing"):
        evr.GroundTruthVideo(np.ones((2, 2, 2)), [1, 1])
    with pytest.raises(ValueError, match="positive"):
        evr.GroundTruthVideo(np.zeros((2, 2, 2)), [0, 1])
    geom = evr.SensorGeometry(width=8, height=8)
    with pytest.raises(ValueError, match="at least 2 frames"):
        evr.render_scene("moving_sine", geom, 1)
    with pytest.raises(ValueError, match="unknown scene kind"):
        evr.render_scene("spiral", geom, 4)
    with pytest.raises(ValueError, match="unknown parameters"):
        evr.render_scene("two_bars", geom, 4, colour=3)


def test_psnr_aligned():  # simulate.py:209-225
    a = np.random.default_rng(0).uniform(1, 2, (6, 7))
    assert evr.psnr_aligned(a, a) == float("inf")
    assert evr.psnr_aligned(a, a + 0.25) > 200  # offset removed up to rounding
    assert 20 < evr.psnr_aligned(a, a + np.sin(a) * 0.01) < 80
    with pytest.raises(ValueError, match="shape mismatch"):
        evr.psnr_aligned(a, a[:3])


def _rows(arr):
    return np.stack([arr["t"], arr["x"], arr["y"], arr["polarity"]], axis=1).astype(np.int64)


@pytest.mark.gpu
def test_gpu_generator_bit_identical_to_reference():
    d, specs = golden()
    sim = evr.EventSimulator()
    for i in range(len(specs)):
        v = evr.GroundTruthVideo(d[f"c{i}_frames"], d[f"c{i}_ts"])
        arr = evr.generate_events_array(v, 0.15, float(d[f"c{i}_dn"]), simulator=sim)
        assert np.array_equal(_rows(arr), d[f"c{i}_ev"]), i
    v = evr.GroundTruthVideo(d["r_frames"], d["r_ts"])
    assert np.array_equal(_rows(evr.generate_events_array(v, 0.2, 0.13, simulator=sim)), d["r_ev"])
    evs = evr.generate_events(v, 0.2, 0.13)
    assert [(e.timestamp, e.x, e.y, e.polarity) for e in evs[:5]] == [tuple(r) for r in d["r_ev"][:5]]


@pytest.mark.gpu
def test_gpu_generator_megapixel_scale_vs_oracle():
    geom = evr.SensorGeometry(width=640, height=480)
    v = evr.render_scene("moving_square", geom, 24, dt=800, velocity=(1.7, -0.9))
    sim = evr.EventSimulator()
    n = sim.generate(v, 0.15, 0.12)
    ref = O.sim_generate(np.log(v.frames), v.frame_timestamps, 0.15, 0.12)
    assert n == len(ref) and n > 10000
    assert np.array_equal(_rows(sim.events()), ref)


@pytest.mark.gpu
def test_gpu_generated_stream_feeds_the_pipeline_from_device():
    """Events generated on the device drive process_packet_device with no
    host round trip; frames equal the host-fed path bit for bit."""
    import ctypes

    from paper_1607_06283_b200 import _lib

    geom = evr.SensorGeometry(width=64, height=48)
    v = evr.render_scene("moving_sine", geom, 16)
    sim = evr.EventSimulator()
    n = sim.generate(v, 0.15, 0.15)
    host = sim.events()
    dptr, dn = sim.device_events()
    assert dn == n and n >= 1000
    sc, mc, th = evr.SolverConfig(max_iterations=20), evr.ManifoldConfig(), evr.Thresholds()
    a = evr.init_state(geom, sc)
    b = evr.init_state(geom, sc)
    epp = 250
    for s in range(0, 4 * epp, epp):
        _, fa, _ = evr.process_packet_arrays(a, host[s:s + epp], mc, sc, th)
        ctx = evr.pipeline._prepare(b, mc, sc, th)
        b.packet_starts.append(int(host["t"][s]))
        w = evr.pipeline._window(b, int(host["t"][s + epp - 1]), mc)
        ctx.call("evr_process_packet_device", ctypes.c_void_p(dptr + 16 * s), epp, float(w))
        ctx.call("evr_synchronize", None)
        b.frame_index += 1
        b._after_device_write(replaced=("u", "f", "p"), in_place=("raw_timestamps",))
        assert np.array_equal(fa, b.u)
