"""Time surface, metric and the manifold operators (reference: surface.py).

Same names, arguments, return types and ValueError messages as the
reference module; every array computation runs in the CUDA library
(evr_op_* entry points of include/evr.h) on a float64 operator context
cached per shape, bit-identical to the numpy reference.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# surface.py:30 -- step-size contract tau*sigma <= 1/(8 + 4 sqrt 2)
OPERATOR_NORM_BOUND_SQ = 8.0 + 4.0 * np.sqrt(2.0)

_OP_CTX: "OrderedDict[tuple, _lib.Context]" = OrderedDict()
_OP_CTX_MAX = 8


def op_context(shape):
    """float64 operator context for a 2-D shape (LRU cache)."""
    key = (int(shape[0]), int(shape[1]))
    ctx = _OP_CTX.get(key)
    if ctx is None:
        ctx = _lib.Context(key[0], key[1], _lib.PREC_F64)
        _OP_CTX[key] = ctx
        while len(_OP_CTX) > _OP_CTX_MAX:
            _OP_CTX.popitem(last=False)[1].close()
    else:
        _OP_CTX.move_to_end(key)
    return ctx


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _as2d(shape):
    """Operator contexts are 2-D; fold any shape into (rows, last)."""
    if len(shape) == 2:
        return shape
    if len(shape) == 0:
        return (1, 1)
    return (int(np.prod(shape[:-1])), int(shape[-1]))


@dataclass
class TimeSurface:
    """Normalised event-age field in [0, t_scale] (surface.py:33-49)."""

    t: np.ndarray
    t_scale: float

    def __post_init__(self):
        self.t = np.asarray(self.t, dtype=np.float64)
        if not np.all(np.isfinite(self.t)):
            raise ValueError("time surface contains non-finite values")
        if self.t.min() < 0 or self.t.max() > self.t_scale + 1e-9:
            raise ValueError(
                f"time surface values must lie in [0, {self.t_scale}], got "
                f"[{self.t.min()}, {self.t.max()}]"
            )


@dataclass
class MetricField:
    """Per-pixel surface geometry (surface.py:52-90); ``coeffs`` are the
    entries (a11, a12, a22, a31, a32) of the 3x2 metric matrix, computed on
    the device and cached."""

    tx: np.ndarray
    ty: np.ndarray
    G: np.ndarray
    sqrtG: np.ndarray
    _coeffs: tuple = field(default=None, init=False, repr=False)

    @property
    def shape(self):
        return self.G.shape

    @property
    def is_flat(self):
        return not (self.tx.any() or self.ty.any())

    @property
    def coeffs(self):
        if self._coeffs is None:
            tx, ty, G = _f64(self.tx), _f64(self.ty), _f64(self.G)
            out = np.empty((5,) + tx.shape)
            op_context(_as2d(tx.shape)).call("evr_op_coeffs", _lib.ptr(tx), _lib.ptr(ty),
                                              _lib.ptr(G), _lib.ptr(out))
            self._coeffs = tuple(out[m] for m in range(5))
        return self._coeffs


def _grad(u):
    u = _f64(u)
    gx, gy = np.empty_like(u), np.empty_like(u)
    op_context(u.shape).call("evr_op_grad", _lib.ptr(u), _lib.ptr(gx), _lib.ptr(gy))
    return gx, gy


def grad_x(u):
    """Forward difference along x, zero on the last column (surface.py:93-97)."""
    return _grad(u)[0]


def grad_y(u):
    """Forward difference along y, zero on the last row (surface.py:100-104)."""
    return _grad(u)[1]


def div_xy(qx, qy):
    """Backward-difference divergence, -adjoint of the gradient
    (surface.py:107-121)."""
    qx, qy = _f64(qx), _f64(qy)
    out = np.empty_like(qx)
    op_context(qx.shape).call("evr_op_div", _lib.ptr(qx), _lib.ptr(qy), _lib.ptr(out))
    return out


def update_timestamp_map(raw_map, event):
    """Record the event's timestamp in a caller-owned host map
    (surface.py:124-127).  The stream path does this on the device inside
    the ingest kernel; this helper only edits the numpy array it is given."""
    raw_map[event.y, event.x] = event.timestamp
    return raw_map


def normalize_timestamps(raw_map, now, t_scale, t_window):
    """Raw last-event timestamps -> surface heights (surface.py:130-143)."""
    if t_window <= 0:
        raise ValueError(f"t_window must be positive, got {t_window}")
    if t_scale < 0:
        raise ValueError(f"t_scale must be non-negative, got {t_scale}")
    raw = _f64(raw_map)
    t = np.empty_like(raw)
    op_context(_as2d(raw.shape)).call("evr_op_normalize", _lib.ptr(raw), ctypes.c_double(now),
                                      ctypes.c_double(t_scale), ctypes.c_double(t_window),
                                      _lib.ptr(t))
    return TimeSurface(t=t, t_scale=t_scale)


def denoise_timestamps(surface, weight, iterations=50):
    """TV-L1 denoising of the time surface (surface.py:146-196)."""
    if weight <= 0:
        raise ValueError(f"denoise weight must be positive, got {weight}")
    if iterations < 1:
        raise ValueError(f"iterations must be >= 1, got {iterations}")
    t = _f64(surface.t)
    out = np.empty_like(t)
    op_context(t.shape).call("evr_op_denoise", _lib.ptr(t), ctypes.c_double(weight),
                             int(iterations), ctypes.c_double(surface.t_scale), _lib.ptr(out))
    return TimeSurface(t=out, t_scale=surface.t_scale)


def compute_metric(surface):
    """Metric field of a time surface or bare 2-D height array
    (surface.py:199-205)."""
    t = surface.t if isinstance(surface, TimeSurface) else surface
    t = _f64(t)
    tx, ty, G, sg = (np.empty_like(t) for _ in range(4))
    op_context(t.shape).call("evr_op_metric", _lib.ptr(t), _lib.ptr(tx), _lib.ptr(ty),
                             _lib.ptr(G), _lib.ptr(sg))
    return MetricField(tx=tx, ty=ty, G=G, sqrtG=sg)


def flat_metric(shape):
    """Identity metric (surface.py:208-211)."""
    z = np.zeros(shape, dtype=np.float64)
    return MetricField(tx=z, ty=z.copy(), G=np.ones(shape), sqrtG=np.ones(shape))


def surface_gradient(u, m):
    """Surface gradient in embedding coordinates, (H, W, 3)
    (surface.py:214-236)."""
    if u.shape != m.shape:
        raise ValueError(f"image shape {u.shape} != metric shape {m.shape}")
    u = _f64(u)
    out = np.empty(u.shape + (3,))
    op_context(u.shape).call("evr_op_surface_gradient", _lib.ptr(u), _lib.ptr(_f64(m.tx)),
                             _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)), _lib.ptr(out))
    return out


def surface_gradient_adjoint(p, m):
    """Exact adjoint of surface_gradient (surface.py:239-252)."""
    if p.shape[:2] != m.shape or p.shape[2:] != (3,):
        raise ValueError(f"dual shape {p.shape} incompatible with metric {m.shape}")
    p = _f64(p)
    out = np.empty(p.shape[:2])
    op_context(out.shape).call("evr_op_surface_gradient_adjoint", _lib.ptr(p),
                               _lib.ptr(_f64(m.tx)), _lib.ptr(_f64(m.ty)),
                               _lib.ptr(_f64(m.G)), _lib.ptr(out))
    return out


def operator_norm_bound():
    """Squared-norm bound used for the step-size product (surface.py:255-257)."""
    return OPERATOR_NORM_BOUND_SQ
