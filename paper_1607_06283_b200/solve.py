"""Primal-dual reconstruction solver (reference: solve.py).

Energy (solve.py:3-7):  sum sqrt(G |S u|^2) + lam sum (u - f log u) sqrtG
on the box [u_min, u_max], minimised with Chambolle-Pock steps whose
proximal maps are closed form.  Names, signatures, defaults, results and
error messages follow the reference; the iterations run in the CUDA
library (evr_op_pd_solve / evr_op_rof_solve), float64, bit-identical.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .surface import _as2d, _f64, op_context, operator_norm_bound

# solve.py:38
_DEFAULT_STEP = 1.0 / np.sqrt(operator_norm_bound())


@dataclass
class SolverConfig:
    """Solve parameters, validated at construction (solve.py:41-78)."""

    lam: float = 180.0 / 255.0
    u_min: float = 1.0
    u_max: float = 2.0
    max_iterations: int = 50
    tau: float = _DEFAULT_STEP
    sigma: float = _DEFAULT_STEP
    convergence_tol: float = 0.0

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError(f"lam must be non-negative, got {self.lam}")
        if not (0 < self.u_min < self.u_max):
            raise ValueError(f"need 0 < u_min < u_max, got [{self.u_min}, {self.u_max}]")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")
        limit = 1.0 / operator_norm_bound()
        if self.tau * self.sigma > limit * (1.0 + 1e-9):
            raise ValueError(
                f"step sizes violate tau*sigma <= 1/{operator_norm_bound():.6f}: "
                f"tau={self.tau}, sigma={self.sigma}"
            )

    @property
    def bounds(self):
        return (self.u_min, self.u_max)


class SolveResult(NamedTuple):
    u: np.ndarray
    p: np.ndarray
    iterations: int
    rel_change: float


def solver_config_struct(cfg: SolverConfig, base=None) -> _lib.Config:
    c = _lib.Config() if base is None else base
    c.lam, c.u_min, c.u_max = cfg.lam, cfg.u_min, cfg.u_max
    c.tau, c.sigma, c.convergence_tol = cfg.tau, cfg.sigma, cfg.convergence_tol
    c.max_iterations = int(cfg.max_iterations)
    return c


def prox_data(u_bar, f, m, tau, cfg):
    """Closed-form KL prox on the intensity box (solve.py:88-100)."""
    f = _f64(f)
    if np.any(f <= 0):
        raise ValueError("measurement f must be positive (log undefined)")
    u_bar = _f64(u_bar)
    sg = _f64(np.broadcast_to(m.sqrtG, u_bar.shape))
    out = np.empty_like(u_bar)
    op_context(_as2d(u_bar.shape)).call(
        "evr_op_prox_data", _lib.ptr(u_bar), _lib.ptr(_f64(np.broadcast_to(f, u_bar.shape))),
        _lib.ptr(sg), ctypes.c_double(tau), ctypes.c_double(cfg.lam),
        ctypes.c_double(cfg.u_min), ctypes.c_double(cfg.u_max), _lib.ptr(out))
    return out


def prox_dual(p_bar, m):
    """Radial projection onto the ball of radius sqrtG (solve.py:103-108)."""
    p = _f64(p_bar)
    out = np.empty_like(p)
    sg = _f64(np.broadcast_to(m.sqrtG, p.shape[:-1]))
    op_context(_as2d(p.shape[:-1])).call("evr_op_prox_dual", _lib.ptr(p), _lib.ptr(sg),
                                         _lib.ptr(out))
    return out


def energy(u, f, m, lam):
    """G-weighted TV plus weighted KL fidelity (solve.py:111-118)."""
    if np.any(u <= 0):
        raise ValueError("u must be positive (log undefined)")
    u = _f64(u)
    out = ctypes.c_double(0.0)
    op_context(u.shape).call("evr_op_energy", _lib.ptr(u), _lib.ptr(_f64(f)),
                             _lib.ptr(_f64(m.tx)), _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)),
                             _lib.ptr(_f64(m.sqrtG)), ctypes.c_double(lam), ctypes.byref(out))
    return float(out.value)


def primal_dual_solve(f, m, cfg, u_init=None, p_init=None, trace=None):
    """Chambolle-Pock iteration (solve.py:207-261) -> SolveResult.

    Warm starts default to u = f, p = 0; early stop when convergence_tol > 0;
    ``trace`` (a list) receives (iteration, energy, rel_change) rows.
    """
    if f.shape != m.shape:
        raise ValueError(f"measurement shape {f.shape} != metric shape {m.shape}")
    if np.any(f < cfg.u_min) or np.any(f > cfg.u_max):
        raise ValueError("measurement f outside the intensity box")
    f = _f64(f)
    u0 = None if u_init is None else _f64(u_init)
    p0 = None if p_init is None else _f64(p_init)
    u = np.empty_like(f)
    p = np.empty(f.shape + (3,))
    info = _lib.SolveInfo()
    et = rt = None
    if trace is not None:
        et = np.zeros(cfg.max_iterations)
        rt = np.zeros(cfg.max_iterations)
    c = solver_config_struct(cfg)
    op_context(f.shape).call(
        "evr_op_pd_solve", ctypes.byref(c), _lib.ptr(f), _lib.ptr(_f64(m.tx)),
        _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)), _lib.ptr(_f64(m.sqrtG)), _lib.ptr(u0),
        _lib.ptr(p0), _lib.ptr(u), _lib.ptr(p), ctypes.byref(info), _lib.ptr(et), _lib.ptr(rt))
    if trace is not None:
        for k in range(info.iterations):
            trace.append((k + 1, float(et[k]), float(rt[k])))
    return SolveResult(u=u, p=p, iterations=int(info.iterations),
                       rel_change=float(info.rel_change))


def rof_manifold_solve(f, m, lam, iterations=200):
    """Quadratic-fidelity (ROF) variant on the same surface (solve.py:264-293)."""
    if lam <= 0:
        raise ValueError(f"lam must be positive, got {lam}")
    if f.shape != m.shape:
        raise ValueError(f"image shape {f.shape} != metric shape {m.shape}")
    f = _f64(f)
    out = np.empty_like(f)
    op_context(f.shape).call("evr_op_rof_solve", _lib.ptr(f), _lib.ptr(_f64(m.tx)),
                             _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)), _lib.ptr(_f64(m.sqrtG)),
                             ctypes.c_double(lam), int(iterations), _lib.ptr(out))
    return out


# --- variants the reference does not ship -----------------------------------
# BASELINE configs[1] names "TV and TGV regularisers, KL vs ROF/L1 data
# terms"; the reference has the KL (primal_dual_solve) and ROF
# (rof_manifold_solve) data terms with manifold TV only.  These two follow
# the published algorithms on the reference's manifold operators; their
# parity is against the CPU restatement (oracle/evr_oracle.c), not the
# reference.

DATA_TERMS = {"kl": 0, "rof": 1, "l1": 2}


def l1_manifold_solve(f, m, lam, iterations=200):
    """Manifold TV with the L1 data term lam * sum |u - f| sqrtG:
    rof_manifold_solve's loop with the soft-shrink prox (no box, cold start)."""
    if lam <= 0:
        raise ValueError(f"lam must be positive, got {lam}")
    if f.shape != m.shape:
        raise ValueError(f"image shape {f.shape} != metric shape {m.shape}")
    f = _f64(f)
    out = np.empty_like(f)
    op_context(f.shape).call("evr_op_l1_solve", _lib.ptr(f), _lib.ptr(_f64(m.tx)),
                             _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)), _lib.ptr(_f64(m.sqrtG)),
                             ctypes.c_double(lam), int(iterations), _lib.ptr(out))
    return out


def tgv_manifold_solve(f, m, lam, alpha0=2.0, alpha1=1.0, iterations=200, data="kl",
                       cfg: SolverConfig | None = None, return_w=False):
    """Second-order manifold TGV:

        min_{u,w}  alpha1 |A (grad u - w)|_g + alpha0 |E w| + D(u, f)

    with the reference's metric matrix A (surface_gradient) and
    g-tensor norm, the symmetrised gradient E w, and D the KL (box from
    ``cfg``, default SolverConfig()), ROF or L1 data term.  Chambolle-Pock,
    tau = sigma = 1/sqrt(17 + 4 sqrt 2), cold start u = f.  Returns u, or
    (u, w) with w of shape (H, W, 2) when ``return_w``."""
    if lam <= 0:
        raise ValueError(f"lam must be positive, got {lam}")
    if alpha0 <= 0 or alpha1 <= 0:
        raise ValueError(f"TGV weights must be positive, got alpha0={alpha0} alpha1={alpha1}")
    if data not in DATA_TERMS:
        raise ValueError(f"data term must be one of {sorted(DATA_TERMS)}, got {data!r}")
    if f.shape != m.shape:
        raise ValueError(f"image shape {f.shape} != metric shape {m.shape}")
    cfg = cfg or SolverConfig()
    f = _f64(f)
    if data == "kl" and (np.any(f < cfg.u_min) or np.any(f > cfg.u_max)):
        raise ValueError(f"f must lie in the box [{cfg.u_min}, {cfg.u_max}]")
    out = np.empty_like(f)
    w = np.empty(f.shape + (2,)) if return_w else None
    op_context(f.shape).call("evr_op_tgv_solve", _lib.ptr(f), _lib.ptr(_f64(m.tx)),
                             _lib.ptr(_f64(m.ty)), _lib.ptr(_f64(m.G)), _lib.ptr(_f64(m.sqrtG)),
                             ctypes.c_double(lam), ctypes.c_double(alpha0),
                             ctypes.c_double(alpha1), DATA_TERMS[data],
                             ctypes.c_double(cfg.u_min), ctypes.c_double(cfg.u_max),
                             int(iterations), _lib.ptr(out), _lib.ptr(w))
    return (out, w) if return_w else out

