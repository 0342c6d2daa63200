"""ctypes front-end of the CPU test oracle (oracle/evr_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker for the CUDA path and the CPU
baseline leg of bench.py.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs import this module; the
product package (paper_1607_06283_b200) never does.

Each wrapper names the reference function it restates (file:line under
/root/reference/pkg/src/evrecon).  The packet driver below mirrors the
host-side bookkeeping of pipeline.py:142-171 (packet_starts deque, window,
frame_index) around the C restatement.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from collections import deque

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

EVENT_DTYPE = np.dtype(
    [("t", "<i8"), ("x", "<i4"), ("y", "<i2"), ("polarity", "<i2")], align=False
)
assert EVENT_DTYPE.itemsize == 16

# pipeline.py:32
ADAPTIVE_WINDOW_PACKETS = 10
# surface.py:30 / solve.py:38
DEFAULT_STEP = 1.0 / np.sqrt(8.0 + 4.0 * np.sqrt(2.0))


class _Config(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double),
        ("u_min", ctypes.c_double),
        ("u_max", ctypes.c_double),
        ("tau", ctypes.c_double),
        ("sigma", ctypes.c_double),
        ("convergence_tol", ctypes.c_double),
        ("max_iterations", ctypes.c_int32),
        ("manifold_enabled", ctypes.c_int32),
        ("t_scale", ctypes.c_double),
        ("denoise_weight", ctypes.c_double),
        ("denoise_iterations", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("c_pos", ctypes.c_double),
        ("c_neg", ctypes.c_double),
    ]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.evo_ingest.argtypes = [P, P, i32, i32, P, i64, d, d, d, d]
        L.evo_normalize.argtypes = [P, i64, d, d, d, P]
        L.evo_grad.argtypes = [P, i32, i32, P, P]
        L.evo_div.argtypes = [P, P, i32, i32, P]
        L.evo_denoise.argtypes = [P, i32, i32, d, i32, d, P]
        L.evo_metric.argtypes = [P, i32, i32, P, P, P, P]
        L.evo_coeffs.argtypes = [P, P, P, i64, P, P, P, P, P]
        L.evo_surface_gradient.argtypes = [P, P, P, P, i32, i32, P]
        L.evo_surface_gradient_adjoint.argtypes = [P, P, P, P, i32, i32, P]
        L.evo_prox_data.argtypes = [P, P, P, i64, d, d, d, d, P]
        L.evo_prox_dual.argtypes = [P, P, i64, P]
        L.evo_energy.argtypes = [P, P, P, P, P, P, i32, i32, d]
        L.evo_energy.restype = d
        L.evo_pd_solve.argtypes = [P, P, P, P, P, i32, i32, P, P, P, P, P, P]
        L.evo_pd_solve.restype = i32
        L.evo_rof_solve.argtypes = [P, P, P, P, P, i32, i32, d, i32, P]
        L.evo_l1_solve.argtypes = [P, P, P, P, P, i32, i32, d, i32, P]
        L.evo_tgv_solve.argtypes = [P, P, P, P, P, i32, i32, d, d, d, i32, d, d, i32, P, P]
        L.evo_process_packet.argtypes = [P, P, P, P, i32, i32, P, i64, d, P, P, P, P]
        L.evo_process_packet.restype = i32
        L.evo_num_threads.restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads():
    return lib().evo_num_threads()


def make_config(lam=180.0 / 255.0, u_min=1.0, u_max=2.0, tau=DEFAULT_STEP,
                sigma=DEFAULT_STEP, convergence_tol=0.0, max_iterations=50,
                manifold_enabled=True, t_scale=3.0, denoise_weight=1.0,
                denoise_iterations=50, pos=0.15, neg=0.15):
    """Defaults of SolverConfig (solve.py:52-58), ManifoldConfig
    (pipeline.py:80-84) and Thresholds (pipeline.py:55-68)."""
    return _Config(lam, u_min, u_max, tau, sigma, convergence_tol,
                   int(max_iterations), int(bool(manifold_enabled)), t_scale,
                   denoise_weight, int(denoise_iterations), 0,
                   math.exp(pos), math.exp(-neg))


def events_array(xs, ys, pols, ts):
    ev = np.empty(len(xs), dtype=EVENT_DTYPE)
    ev["x"], ev["y"], ev["polarity"], ev["t"] = xs, ys, pols, ts
    return ev


# --- operators -------------------------------------------------------------


def ingest(f, raw, events, cfg):
    """pipeline.py:114-121 over a packet (in place)."""
    H, W = f.shape
    lib().evo_ingest(_p(f), _p(raw), H, W, _p(events), len(events),
                     cfg.c_pos, cfg.c_neg, cfg.u_min, cfg.u_max)


def normalize(raw, now, t_scale, window):
    """surface.py:130-143."""
    r = _f64(raw)
    t = np.empty_like(r)
    lib().evo_normalize(_p(r), r.size, float(now), t_scale, window, _p(t))
    return t


def grad(u):
    u = _f64(u)
    gx, gy = np.empty_like(u), np.empty_like(u)
    lib().evo_grad(_p(u), u.shape[0], u.shape[1], _p(gx), _p(gy))
    return gx, gy


def div(qx, qy):
    qx, qy = _f64(qx), _f64(qy)
    out = np.empty_like(qx)
    lib().evo_div(_p(qx), _p(qy), qx.shape[0], qx.shape[1], _p(out))
    return out


def denoise(t, weight=1.0, iterations=50, t_scale=3.0):
    """surface.py:146-196."""
    t = _f64(t)
    out = np.empty_like(t)
    lib().evo_denoise(_p(t), t.shape[0], t.shape[1], weight, iterations, t_scale, _p(out))
    return out


def metric(t):
    """surface.py:199-205 -> (tx, ty, G, sqrtG)."""
    t = _f64(t)
    outs = [np.empty_like(t) for _ in range(4)]
    lib().evo_metric(_p(t), t.shape[0], t.shape[1], *map(_p, outs))
    return tuple(outs)


def coeffs(tx, ty, G):
    tx, ty, G = _f64(tx), _f64(ty), _f64(G)
    outs = [np.empty_like(tx) for _ in range(5)]
    lib().evo_coeffs(_p(tx), _p(ty), _p(G), tx.size, *map(_p, outs))
    return tuple(outs)


def surface_gradient(u, tx, ty, G):
    u = _f64(u)
    out = np.empty(u.shape + (3,))
    lib().evo_surface_gradient(_p(u), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)),
                               u.shape[0], u.shape[1], _p(out))
    return out


def surface_gradient_adjoint(p, tx, ty, G):
    p = _f64(p)
    out = np.empty(p.shape[:2])
    lib().evo_surface_gradient_adjoint(_p(p), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)),
                                       p.shape[0], p.shape[1], _p(out))
    return out


def prox_data(u_bar, f, sqrtG, tau, lam, u_min, u_max):
    u_bar, f, sqrtG = _f64(u_bar), _f64(f), _f64(sqrtG)
    out = np.empty_like(u_bar)
    lib().evo_prox_data(_p(u_bar), _p(f), _p(sqrtG), u_bar.size, tau, lam, u_min, u_max, _p(out))
    return out


def prox_dual(p, sqrtG):
    p, sqrtG = _f64(p), _f64(sqrtG)
    out = np.empty_like(p)
    lib().evo_prox_dual(_p(p), _p(sqrtG), sqrtG.size, _p(out))
    return out


def energy(u, f, tx, ty, G, sqrtG, lam):
    u = _f64(u)
    return lib().evo_energy(_p(u), _p(_f64(f)), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)),
                            _p(_f64(sqrtG)), u.shape[0], u.shape[1], lam)


def pd_solve(f, tx, ty, G, sqrtG, cfg, u_init=None, p_init=None, trace=False):
    """solve.py:207-261 -> (u, p, iterations, rel_change[, energies, rels])."""
    f = _f64(f)
    u = _f64(f if u_init is None else u_init).copy()
    p = np.zeros(f.shape + (3,)) if p_init is None else _f64(p_init).copy()
    rel = ctypes.c_double(0.0)
    et = np.zeros(cfg.max_iterations) if trace else None
    rt = np.zeros(cfg.max_iterations) if trace else None
    it = lib().evo_pd_solve(_p(f), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)), _p(_f64(sqrtG)),
                            f.shape[0], f.shape[1], ctypes.byref(cfg), _p(u), _p(p),
                            ctypes.byref(rel), _p(et), _p(rt))
    if trace:
        return u, p, it, rel.value, et[:it], rt[:it]
    return u, p, it, rel.value


def rof_solve(f, tx, ty, G, sqrtG, lam, iterations=200):
    """solve.py:264-293."""
    f = _f64(f)
    out = np.empty_like(f)
    lib().evo_rof_solve(_p(f), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)), _p(_f64(sqrtG)),
                        f.shape[0], f.shape[1], lam, iterations, _p(out))
    return out


def l1_solve(f, tx, ty, G, sqrtG, lam, iterations=200):
    """Manifold TV + L1 data term (not in the reference: parity unpinned)."""
    f = _f64(f)
    out = np.empty_like(f)
    lib().evo_l1_solve(_p(f), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)), _p(_f64(sqrtG)),
                       f.shape[0], f.shape[1], lam, iterations, _p(out))
    return out


DATA_TERMS = {"kl": 0, "rof": 1, "l1": 2}


def tgv_solve(f, tx, ty, G, sqrtG, lam, alpha0=2.0, alpha1=1.0, data="kl", u_min=1.0,
              u_max=2.0, iterations=200):
    """Second-order manifold TGV (not in the reference: parity unpinned).
    Returns (u, w) with w of shape (H, W, 2)."""
    f = _f64(f)
    out = np.empty_like(f)
    w = np.empty(f.shape + (2,))
    lib().evo_tgv_solve(_p(f), _p(_f64(tx)), _p(_f64(ty)), _p(_f64(G)), _p(_f64(sqrtG)),
                        f.shape[0], f.shape[1], lam, alpha0, alpha1, DATA_TERMS[data], u_min,
                        u_max, iterations, _p(out), _p(w))
    return out, w


# --- packet driver -----------------------------------------------------------


class OracleStream:
    """State machine of pipeline.py:87-171 around the C restatement.

    Holds u, f, raw, p (reference layouts) plus the packet_starts deque;
    ``process(events)`` runs one packet and returns (iterations, rel_change).
    """

    def __init__(self, height, width, cfg, t_window=None):
        self.cfg = cfg
        self.t_window = t_window
        mid = 0.5 * (cfg.u_min + cfg.u_max)  # pipeline.py:105
        self.u = np.full((height, width), mid)
        self.f = np.full((height, width), mid)
        self.raw = np.zeros((height, width), dtype=np.int64)
        self.p = np.zeros((height, width, 3))
        self.frame_index = 0
        self.packet_starts = deque(maxlen=ADAPTIVE_WINDOW_PACKETS)
        self.last_t = None
        self.last_G = None

    def window_for(self, now):
        # pipeline.py:128-132
        if self.t_window is not None:
            return float(self.t_window)
        oldest = self.packet_starts[0] if self.packet_starts else now
        return max(float(now - oldest), 1.0)

    def process(self, events, keep_surface=False):
        if len(events) == 0:  # pipeline.py:151-153
            return None, None
        self.packet_starts.append(int(events["t"][0]))  # pipeline.py:155
        now = int(events["t"][-1])
        window = self.window_for(now)
        H, W = self.u.shape
        rel = ctypes.c_double(0.0)
        t_out = np.empty((H, W)) if keep_surface else None
        G_out = np.empty((H, W)) if keep_surface else None
        ev = np.ascontiguousarray(events)
        it = lib().evo_process_packet(_p(self.u), _p(self.f), _p(self.raw), _p(self.p),
                                      H, W, _p(ev), len(ev), window, ctypes.byref(self.cfg),
                                      ctypes.byref(rel), _p(t_out), _p(G_out))
        self.last_t, self.last_G = t_out, G_out
        self.frame_index += 1
        return it, rel.value


def sim_generate(log_frames, frame_ts, dp, dn):
    """generate_events (simulate.py:51-103) restated per pixel in numpy on a
    (n, H, W) LOG-intensity stack; returns an (E, 4) int64 array of
    [t, x, y, polarity] rows in the reference's (t, y, x, polarity) order."""
    n, h, w = log_frames.shape
    ref = log_frames[0].copy()
    yy, xx = np.mgrid[0:h, 0:w]
    rows = []
    for k in range(n - 1):
        l0, l1 = log_frames[k], log_frames[k + 1]
        t0, t1 = int(frame_ts[k]), int(frame_ts[k + 1])
        up = np.maximum(np.floor((l1 - ref) / dp + 1e-9).astype(np.int64), 0)
        down = np.maximum(np.floor((ref - l1) / dn + 1e-9).astype(np.int64), 0)
        for counts, sign, step in ((up, 1, dp), (down, -1, dn)):
            for j in range(1, int(counts.max(initial=0)) + 1):
                m = counts >= j
                level = ref + j * step if sign > 0 else ref - j * step
                frac = (level[m] - l0[m]) / (l1[m] - l0[m])
                t = np.rint(t0 + frac * (t1 - t0)).astype(np.int64)
                rows.append(np.stack([t, xx[m], yy[m], np.full(t.shape, sign)], axis=1))
        ref += up * dp - down * dn
    if not rows:
        return np.zeros((0, 4), np.int64)
    ev = np.concatenate(rows).astype(np.int64)
    order = np.lexsort((ev[:, 3], ev[:, 1], ev[:, 2], ev[:, 0]))
    return ev[order]
