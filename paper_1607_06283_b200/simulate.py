"""Synthetic ground truth and the GPU event simulator.

Mirror of the reference's ``evrecon.simulate`` (simulate.py:24-225):

* ``GroundTruthVideo`` -- a positive (n, h, w) frame stack with strictly
  increasing integer timestamps (simulate.py:24-48, same validation).
* ``render_scene`` -- the deterministic test scenes (simulate.py:136-199),
  rendered on the host with numpy in the reference's operation order, so the
  frames are bit-identical to the reference's.
* ``generate_events`` / ``generate_events_array`` -- the comparator-model
  event stream (simulate.py:51-103).  The host takes ``np.log`` of the frames
  (the reference's own step, simulate.py:60); crossing counts, crossing
  times and the (t, y, x, polarity) ordering run on the GPU
  (``csrc/evr_simulate.cu``) -- bit-identical to the reference's stream.
* ``psnr_aligned`` (simulate.py:209-225).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .events import EVENT_DTYPE, array_to_events

__all__ = ["GroundTruthVideo", "EventSimulator", "generate_events", "generate_events_array",
           "render_scene", "psnr_aligned"]


@dataclass
class GroundTruthVideo:
    """(n >= 2, h, w) positive intensities with strictly increasing integer
    timestamps (simulate.py:24-48)."""

    frames: np.ndarray
    frame_timestamps: np.ndarray

    def __post_init__(self):
        self.frames = np.asarray(self.frames, dtype=np.float64)
        self.frame_timestamps = np.asarray(self.frame_timestamps, dtype=np.int64)
        if self.frames.ndim != 3 or self.frames.shape[0] < 2:
            raise ValueError(f"need a (n>=2, h, w) frame stack, got shape {self.frames.shape}")
        if self.frames.shape[0] != self.frame_timestamps.shape[0]:
            raise ValueError("frame count and timestamp count differ")
        if np.any(np.diff(self.frame_timestamps) <= 0):
            raise ValueError("frame timestamps must be strictly increasing")
        if np.any(self.frames <= 0):
            raise ValueError("frame intensities must be positive")

    @property
    def shape(self):
        return self.frames.shape[1:]


class EventSimulator:
    """Device-side event generator (one ``evr_sim`` handle on one GPU).

    ``generate`` returns the event count; ``events()`` downloads them as an
    EVENT_DTYPE array, ``device_events()`` gives the device pointer for
    ``evr_process_packet_device`` (no host round trip)."""

    def __init__(self, device=None):
        if _lib.device_count() < 1:
            raise RuntimeError("the event simulator runs on the GPU only (no CUDA device)")
        import os

        dev = int(os.environ.get("EVR_DEVICE", "0")) if device is None else int(device)
        h = ctypes.c_void_p()
        rc = _lib.lib().evr_sim_create(ctypes.byref(h), dev)
        if rc != 0:
            raise RuntimeError(f"evr_sim_create failed ({rc})")
        self._h = h
        self.n_events = 0

    def close(self):
        if self._h:
            _lib.lib().evr_sim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != 0:
            msg = _lib.lib().evr_sim_last_error(self._h).decode()
            if rc == -1:
                raise ValueError(msg)
            raise RuntimeError(f"{what}: {msg} ({rc})")

    def generate(self, video, dp, dn):
        if dp <= 0 or dn <= 0:  # simulate.py:57-58
            raise ValueError(f"thresholds must be positive, got dp={dp}, dn={dn}")
        log_frames = np.ascontiguousarray(np.log(video.frames))  # simulate.py:60
        ts = np.ascontiguousarray(video.frame_timestamps, dtype=np.int64)
        n, h, w = log_frames.shape
        count = ctypes.c_int64(0)
        self._check(_lib.lib().evr_sim_generate(self._h, _lib.ptr(log_frames), _lib.ptr(ts), n,
                                                h, w, float(dp), float(dn),
                                                ctypes.byref(count)), "evr_sim_generate")
        self.n_events = int(count.value)
        return self.n_events

    def events(self):
        out = np.empty(self.n_events, dtype=EVENT_DTYPE)
        self._check(_lib.lib().evr_sim_events(self._h, _lib.ptr(out), self.n_events),
                    "evr_sim_events")
        return out

    def device_events(self):
        p, n = ctypes.c_void_p(), ctypes.c_int64(0)
        self._check(_lib.lib().evr_sim_device_events(self._h, ctypes.byref(p), ctypes.byref(n)),
                    "evr_sim_device_events")
        return p.value, int(n.value)


def generate_events_array(video, dp, dn, simulator=None):
    """generate_events (simulate.py:51-103) as an EVENT_DTYPE array."""
    sim = simulator if simulator is not None else EventSimulator()
    sim.generate(video, dp, dn)
    return sim.events()


def generate_events(video, dp, dn):
    """generate_events (simulate.py:51-103): list[Event] sorted by timestamp,
    ties by (y, x, polarity)."""
    arr = generate_events_array(video, dp, dn)
    return array_to_events(arr) if len(arr) else []


# --- scenes (host, numpy; simulate.py:106-206) ---------------------------------


def _grid(h, w):
    yy, xx = np.mgrid[0:h, 0:w]
    return yy.astype(np.float64), xx.astype(np.float64)


def _soft_box(coord, half_width, edge=1.5):
    """1 inside |coord| < half_width, 0 outside, linear ramp of width edge
    (simulate.py:130-133)."""
    return np.clip((half_width - np.abs(coord)) / edge + 0.5, 0.0, 1.0)


def _shifted(template, dx, dy, wrap):
    """Bilinear sample of template at (y - dy, x - dx), wrapped or clamped
    (simulate.py:106-127)."""
    h, w = template.shape
    iy, ix = np.mgrid[0:h, 0:w]
    sy, sx = iy - dy, ix - dx
    y0, x0 = np.floor(sy).astype(np.int64), np.floor(sx).astype(np.int64)
    wy, wx = sy - y0, sx - x0
    if wrap:
        def at(yi, xi):
            return template[np.mod(yi, h), np.mod(xi, w)]
    else:
        def at(yi, xi):
            return template[np.clip(yi, 0, h - 1), np.clip(xi, 0, w - 1)]
    upper = at(y0, x0) * (1 - wx) + at(y0, x0 + 1) * wx
    lower = at(y0 + 1, x0) * (1 - wx) + at(y0 + 1, x0 + 1) * wx
    return upper * (1 - wy) + lower * wy


def _scene_moving_square(h, w, n_frames, p):
    size = p.pop("size", min(h, w) * 0.4)
    vx, vy = p.pop("velocity", (0.5, 0.25))
    background = p.pop("background", 1.5)
    amplitude = p.pop("amplitude", 0.4)
    period = p.pop("texture_period", 8.0)
    yy, xx = _grid(h, w)
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    box = _soft_box(xx - cx, size / 2.0) * _soft_box(yy - cy, size / 2.0)
    texture = 0.5 + 0.5 * np.cos(2 * np.pi * (xx - cx) / period) * np.cos(
        2 * np.pi * (yy - cy) / period)
    template = background + box * amplitude * texture
    for k in range(n_frames):
        s = k - (n_frames - 1) / 2.0  # symmetric path keeps the square inside
        yield _shifted(template, vx * s, vy * s, wrap=False)


def _scene_moving_sine(h, w, n_frames, p):
    period = p.pop("period", 16.0)
    amplitude = p.pop("amplitude", 0.45)
    vx, vy = p.pop("velocity", (0.5, 0.0))
    yy, xx = _grid(h, w)
    for k in range(n_frames):
        ax = 2 * np.pi * (xx - vx * k) / period
        ay = 2 * np.pi * (yy - vy * k) / period
        yield 1.5 + amplitude * np.sin(ax) * np.cos(ay)


def _scene_two_bars(h, w, n_frames, p):
    bar = p.pop("bar_width", 6.0)
    amplitude = p.pop("amplitude", 0.35)
    speed = p.pop("speed", 0.5)
    background = p.pop("background", 1.2)
    cols = np.arange(w, dtype=np.float64)

    def ring_distance(c):
        d = np.abs(cols - c)
        return np.minimum(d, w - d)

    for k in range(n_frames):
        c1 = np.mod(w * 0.25 + speed * k, w)
        c2 = np.mod(w * 0.75 - speed * k, w)
        row = background + amplitude * (_soft_box(ring_distance(c1), bar / 2.0)
                                        + _soft_box(ring_distance(c2), bar / 2.0))
        yield np.tile(row, (h, 1))


_SCENES = {"moving_square": _scene_moving_square, "moving_sine": _scene_moving_sine,
           "two_bars": _scene_two_bars}


def render_scene(kind, geometry, n_frames, dt=1000, **params):
    """Deterministic synthetic scenes with sub-pixel motion, intensities in
    [1, 2], frame k at timestamp k * dt (simulate.py:136-199)."""
    if n_frames < 2:
        raise ValueError(f"need at least 2 frames, got {n_frames}")
    if kind not in _SCENES:
        raise ValueError(f"unknown scene kind {kind!r}")
    h, w = geometry.height, geometry.width
    frames = np.empty((n_frames, h, w), dtype=np.float64)
    gen = _SCENES[kind](h, w, n_frames, params)
    first = next(gen)  # pops the scene's own parameters
    if params:
        raise ValueError(f"unknown parameters for {kind!r}: {sorted(params)}")
    frames[0] = first
    for k, fr in enumerate(gen, start=1):
        frames[k] = fr
    return GroundTruthVideo(frames=frames,
                            frame_timestamps=np.arange(n_frames, dtype=np.int64) * int(dt))


def psnr_aligned(a, b, peak=1.0):
    """PSNR in dB after removing the mean difference; identical images give
    inf (simulate.py:209-225)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    d = a - b
    d -= d.mean()
    mse = float(np.mean(d * d))
    if mse == 0.0:
        return float("inf")
    return float(10.0 * np.log10(peak * peak / mse))
