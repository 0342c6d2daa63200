"""Row-band split of one sensor over several GPUs (SURVEY.md 8(e), configs[4]).

``BandedStream`` is the stream state machine of pipeline.py:142-171 for a
megapixel sensor whose rows are divided into contiguous bands, one evr
context per band (one per GPU, or several on one GPU), driven by the C
group API (evr_group_*): every packet runs the streaming step list on all
bands in lock step with one halo row exchanged per half-step over
device-to-device / NVLink peer copies.  Results are bit-identical to the
single-context path for any band count.
"""

from __future__ import annotations

import ctypes
from collections import deque

import numpy as np

from . import _lib
from .events import events_to_array
from .pipeline import (ADAPTIVE_WINDOW_PACKETS, ManifoldConfig, Thresholds, default_precision,
                       device_config)
from .solve import SolveResult, SolverConfig


def band_rows(height, n_bands):
    """Row ranges [y0, y1) of the bands (same split as evr_group_create)."""
    return [(height * b // n_bands, height * (b + 1) // n_bands) for b in range(n_bands)]


class BandedStream:
    def __init__(self, geometry, solver_cfg=None, manifold_cfg=None, thresholds=None, bands=2,
                 devices=None, precision=None):
        self.geometry = geometry
        self.solver_cfg = solver_cfg or SolverConfig()
        self.manifold_cfg = manifold_cfg or ManifoldConfig()
        self.thresholds = thresholds or Thresholds()
        self.precision = default_precision() if precision is None else precision
        L = _lib.lib()
        if _lib.device_count() < 1:
            raise RuntimeError("no CUDA device visible: the evr hot path runs on the GPU only")
        if devices is None:
            devices = [0] * bands
        if len(devices) != bands:
            raise ValueError(f"need one device per band, got {len(devices)} for {bands}")
        devs = (ctypes.c_int * bands)(*devices)
        h = ctypes.c_void_p()
        rc = L.evr_group_create(ctypes.byref(h), bands, devs, geometry.height, geometry.width,
                                self.precision)
        if rc != _lib.EVR_OK:
            raise _lib.EvrError(rc, f"evr_group_create({bands} bands) failed")
        self._h = h
        self.bands = bands
        self.devices = list(devices)
        c = device_config(self.manifold_cfg, self.solver_cfg, self.thresholds,
                          engine=_lib.ENGINE_STREAMING)
        self._call("evr_group_set_config", ctypes.byref(c))
        self._call("evr_group_init_state")
        self.frame_index = 0
        self.packet_starts = deque(maxlen=ADAPTIVE_WINDOW_PACKETS)

    def _call(self, name, *args):
        rc = getattr(_lib.lib(), name)(self._h, *args)
        if rc != _lib.EVR_OK:
            msg = _lib.lib().evr_group_last_error(self._h).decode()
            if rc == _lib.EVR_ERR_INVALID:
                raise ValueError(msg)
            if rc == _lib.EVR_ERR_RANGE:
                raise IndexError(msg)
            raise _lib.EvrError(rc, f"{name}: {msg}")

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().evr_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _get(self, which):
        H, W = self.geometry.height, self.geometry.width
        out = np.empty((H, W, 3) if which == 3 else (H, W),
                       dtype=np.int64 if which == 2 else np.float64)
        ptrs = [None] * 4
        ptrs[which] = _lib.ptr(out)
        self._call("evr_group_get_state", *ptrs)
        return out

    u = property(lambda s: s._get(0))
    f = property(lambda s: s._get(1))
    raw_timestamps = property(lambda s: s._get(2))
    p = property(lambda s: s._get(3))

    def set_state(self, u=None, f=None, raw_timestamps=None, p=None):
        def c(a, dt):
            return None if a is None else np.ascontiguousarray(a, dtype=dt)
        arrs = [c(u, np.float64), c(f, np.float64), c(raw_timestamps, np.int64), c(p, np.float64)]
        self._call("evr_group_set_state", *[_lib.ptr(a) for a in arrs])

    def process_packet(self, events, want_frame=True):
        """pipeline.py:142-171 over the bands -> (frame or None, SolveResult)."""
        ev = events_to_array(events)
        if len(ev) == 0:
            return self.u, None
        self.packet_starts.append(int(ev["t"][0]))
        now = int(ev["t"][-1])
        mc = self.manifold_cfg
        if mc.t_window is not None:
            window = float(mc.t_window)
        else:
            window = max(float(now - self.packet_starts[0]), 1.0)
        info = _lib.SolveInfo()
        self._call("evr_group_process_packet", _lib.ptr(ev), len(ev), window, ctypes.byref(info))
        self.frame_index += 1
        frame = self.u if want_frame else None
        return frame, SolveResult(u=frame, p=None, iterations=int(info.iterations),
                                  rel_change=float(info.rel_change))

    def launch_count(self):
        return int(_lib.lib().evr_group_launch_count(self._h))
