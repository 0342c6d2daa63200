"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (needs /root/reference; never runs on the GPU box):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
and records, for seeded synthetic inputs, the reference's own outputs of
every hot-path stage (pipeline.py:142-171 decomposed into apply_event,
normalize_timestamps, denoise_timestamps, compute_metric,
primal_dual_solve) plus operator-level cases (solve.py / surface.py).
The fixtures pin the C oracle (tests/test_oracle.py) and, through the
oracle or directly, the CUDA path (tests/test_gpu_*.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.path.insert(0, REF)
    import evrecon  # noqa: F401  (the reference package)
    from evrecon import pipeline, solve, surface, simulate

    return evrecon, pipeline, solve, surface, simulate


def _events_to_arrays(events):
    return (
        np.array([e.x for e in events], dtype=np.int32),
        np.array([e.y for e in events], dtype=np.int32),
        np.array([e.polarity for e in events], dtype=np.int32),
        np.array([e.timestamp for e in events], dtype=np.int64),
    )


def uniform_events(ev_mod, n, width, height, seed, t_step, t0=0):
    """Generator U of SURVEY.md 8(d) (mirrors test_pipeline.py:24-34)."""
    rng = np.random.default_rng(seed)
    xs = rng.integers(0, width, n)
    ys = rng.integers(0, height, n)
    ps = rng.choice([-1, 1], n)
    return [
        ev_mod.Event(x=int(xs[k]), y=int(ys[k]), polarity=int(ps[k]),
                     timestamp=int(t0 + k * t_step))
        for k in range(n)
    ]


def record_stream(ev, pl, so, su, geom, events, epp, manifold_cfg, solver_cfg,
                  thresholds, full=True, skip=0):
    """Teacher-forced stage dump of a chained stream, stage by stage, and a
    cross-check that the stage composition equals process_packet.  The
    first ``skip`` packets only warm the state up; the state they leave is
    stored as init_* so a checker can start from it."""
    state = pl.init_state(geom, solver_cfg)
    twin = pl.init_state(geom, solver_cfg)
    for start in range(0, skip * epp, epp):
        for st in (state, twin):
            pl.process_packet(st, events[start:start + epp], manifold_cfg, solver_cfg,
                              thresholds)
    init = dict(init_u=state.u.copy(), init_f=state.f.copy(),
                init_raw=state.raw_timestamps.copy(), init_p=state.p.copy(),
                init_starts=np.array(list(state.packet_starts), dtype=np.int64),
                init_frame_index=state.frame_index)
    events = events[skip * epp:]
    rec = {k: [] for k in ("f_ing", "raw_ing", "window", "t_norm", "t_den", "tx",
                           "ty", "G", "sqrtG", "u", "p", "iterations", "rel_change")}
    for start in range(0, len(events), epp):
        packet = events[start:start + epp]
        # reference process_packet on the twin state (ground truth)
        _, frame, result = pl.process_packet(twin, packet, manifold_cfg, solver_cfg,
                                             thresholds)
        # the same packet, stage by stage (pipeline.py:151-171)
        state.packet_starts.append(packet[0].timestamp)
        for e in packet:
            pl.apply_event(state, e, thresholds, solver_cfg)
        now = packet[-1].timestamp
        if manifold_cfg.enabled:
            if manifold_cfg.t_window is not None:
                window = manifold_cfg.t_window
            else:
                window = max(float(now - state.packet_starts[0]), 1.0)
            tn = su.normalize_timestamps(state.raw_timestamps, now, manifold_cfg.t_scale, window)
            td = su.denoise_timestamps(tn, manifold_cfg.denoise_weight,
                                       manifold_cfg.denoise_iterations)
            m = su.compute_metric(td)
            t_norm, t_den = tn.t, td.t
        else:
            window = 0.0
            m = su.flat_metric(state.f.shape)
            t_norm = t_den = np.zeros(state.f.shape)
        rec["f_ing"].append(state.f.copy())
        rec["raw_ing"].append(state.raw_timestamps.copy())
        res = so.primal_dual_solve(state.f, m, solver_cfg, u_init=state.u, p_init=state.p)
        state.u, state.p, state.f = res.u, res.p, res.u.copy()
        state.frame_index += 1
        assert np.array_equal(res.u, frame) and np.array_equal(res.p, twin.p)
        assert res.iterations == result.iterations
        rec["window"].append(window)
        rec["t_norm"].append(t_norm)
        rec["t_den"].append(t_den)
        rec["tx"].append(m.tx)
        rec["ty"].append(m.ty)
        rec["G"].append(m.G)
        rec["sqrtG"].append(m.sqrtG)
        rec["u"].append(res.u.copy())
        rec["p"].append(res.p.copy())
        rec["iterations"].append(res.iterations)
        rec["rel_change"].append(res.rel_change)
    out = {k: np.asarray(v) for k, v in rec.items()}
    if not full:
        keep = ("f_ing", "raw_ing", "window", "u", "iterations", "rel_change")
        out = {k: out[k] for k in keep}
        out["p_last"] = rec["p"][-1]
        out["t_den_last"] = rec["t_den"][-1]
        out["G_last"] = rec["G"][-1]
    x, y, pol, t = _events_to_arrays(events)
    out.update(ev_x=x, ev_y=y, ev_pol=pol, ev_t=t, epp=epp,
               height=geom.height, width=geom.width)
    if skip:
        out.update(init)
    return out


def main():
    evrecon, pl, so, su, sim = _import_reference()
    ev = sys.modules["evrecon.events"]
    th = pl.Thresholds()
    scfg = so.SolverConfig()

    # 1. small chained U stream with many intra-packet duplicates
    geom = ev.SensorGeometry(width=32, height=24)
    events = uniform_events(ev, 1200, 32, 24, seed=7, t_step=10)
    d = record_stream(ev, pl, so, su, geom, events, 200, pl.ManifoldConfig(), scfg, th)
    np.savez_compressed(os.path.join(OUT, "stream_u_32x24.npz"), **d)

    # 2. the reference bench stream S (cli.py:256-264) on DVS128, 3 packets
    geom = ev.SensorGeometry(width=128, height=128)
    n_frames, evs = 16, []
    while len(evs) < 9000:
        video = sim.render_scene("moving_sine", geom, n_frames)
        evs = sim.generate_events(video, 0.15, 0.15)
        n_frames *= 2
    evs = evs[:9000]
    # packets 15-17 carry the steepest surfaces of the first 20 (max G ~ 2.4-4.2)
    d = record_stream(ev, pl, so, su, geom, evs, 500, pl.ManifoldConfig(), scfg, th,
                      full=False, skip=15)
    np.savez_compressed(os.path.join(OUT, "stream_s_dvs128.npz"), **d)

    # 3. manifold disabled (flat metric) and a fixed window, odd shapes
    geom = ev.SensorGeometry(width=9, height=2)
    events = uniform_events(ev, 90, 9, 2, seed=3, t_step=7)
    d = record_stream(ev, pl, so, su, geom, events, 30, pl.ManifoldConfig(enabled=False),
                      so.SolverConfig(max_iterations=20), th)
    np.savez_compressed(os.path.join(OUT, "stream_flat_9x2.npz"), **d)
    geom = ev.SensorGeometry(width=2, height=7)
    events = uniform_events(ev, 60, 2, 7, seed=4, t_step=3)
    d = record_stream(ev, pl, so, su, geom, events, 20,
                      pl.ManifoldConfig(t_window=50.0, t_scale=2.0, denoise_weight=0.5,
                                        denoise_iterations=7),
                      so.SolverConfig(lam=1.3, max_iterations=9), pl.Thresholds(0.2, 0.1))
    np.savez_compressed(os.path.join(OUT, "stream_window_2x7.npz"), **d)

    # 4. operator-level cases
    rng = np.random.default_rng(2024)
    ops = {}
    raw = np.array([[1000, 500], [0, 1200]], dtype=np.int64)
    ops["norm_raw"] = raw
    ops["norm_t"] = su.normalize_timestamps(raw, 1000, 3.0, 1000.0).t
    t_rand = rng.uniform(0, 3, (17, 13))
    ops["den_in"] = t_rand
    ops["den_out"] = su.denoise_timestamps(su.TimeSurface(t_rand, 3.0), 0.3, 50).t
    h = rng.normal(0, 1.3, (11, 7))
    m = su.compute_metric(h)
    ops["met_in"] = h
    ops["met_tx"], ops["met_ty"], ops["met_G"], ops["met_sqrtG"] = m.tx, m.ty, m.G, m.sqrtG
    ops["met_coeffs"] = np.stack(m.coeffs)
    ops["div_qx"], ops["div_qy"] = rng.normal(0, 1, (2, 5, 6))
    ops["div_out"] = su.div_xy(ops["div_qx"], ops["div_qy"])
    u = rng.uniform(1, 2, (11, 7))
    p = rng.normal(0, 0.7, (11, 7, 3))
    ops["sg_u"], ops["sg_p"] = u, p
    ops["sg_out"] = su.surface_gradient(u, m)
    ops["sga_out"] = su.surface_gradient_adjoint(p, m)
    ub = rng.uniform(-1, 4, (11, 7))
    ff = rng.uniform(1, 2, (11, 7))
    pcfg = so.SolverConfig(lam=3.0)
    ops["pd_ubar"], ops["pd_f"] = ub, ff
    ops["prox_data_out"] = so.prox_data(ub, ff, m, 0.3, pcfg)
    pbig = rng.normal(0, 2, (11, 7, 3))
    ops["prox_dual_in"] = pbig
    ops["prox_dual_out"] = so.prox_dual(pbig, m)
    ops["energy_val"] = np.array([so.energy(u, ff, m, 0.7)])
    # warm-started solve on a steep random metric, with trace rows
    cfg = so.SolverConfig(lam=0.9, max_iterations=60)
    f = np.clip(1.5 + 0.4 * rng.normal(0, 1, (12, 10)), 1.0, 2.0)
    hm = su.compute_metric(rng.normal(0, 1.5, (12, 10)))
    u0 = np.clip(1.5 + 0.4 * rng.normal(0, 1, (12, 10)), 1.0, 2.0)
    p0 = rng.normal(0, 0.5, (12, 10, 3))
    trace = []
    res = so.primal_dual_solve(f, hm, cfg, u_init=u0, p_init=p0, trace=trace)
    ops.update(solve_f=f, solve_h=rng.normal(0, 0, (1,)), solve_u0=u0, solve_p0=p0,
               solve_tx=hm.tx, solve_ty=hm.ty, solve_G=hm.G, solve_sqrtG=hm.sqrtG,
               solve_u=res.u, solve_p=res.p, solve_iters=np.array([res.iterations]),
               solve_rel=np.array([res.rel_change]),
               solve_trace=np.array(trace))
    # early stop on tolerance (test_solve.py:222-229 shape)
    cfg = so.SolverConfig(lam=0.7, max_iterations=500, convergence_tol=1e-5)
    f = np.clip(1.5 + 0.4 * rng.normal(0, 1, (10, 10)), 1.0, 2.0)
    res = so.primal_dual_solve(f, su.flat_metric((10, 10)), cfg)
    ops.update(tol_f=f, tol_u=res.u, tol_p=res.p, tol_iters=np.array([res.iterations]),
               tol_rel=np.array([res.rel_change]))
    # ROF (flat and steep metric)
    f = rng.normal(0.5, 0.25, (20, 20))
    ops["rof_f"] = f
    ops["rof_flat"] = so.rof_manifold_solve(f, su.flat_metric((20, 20)), 8.0, 250)
    hr = rng.normal(0, 2, (20, 20))
    mr = su.compute_metric(hr)
    ops["rof_h"] = hr
    ops["rof_steep"] = so.rof_manifold_solve(f, mr, 4.0, 120)
    np.savez_compressed(os.path.join(OUT, "ops.npz"), **ops)

    # 5. text event front-end (events.py:65-130) and gray mapping (pgm.py:14-22)
    import json

    cases = {
        "clean": ("# hdr\n0 1 2 1\n5 3 4 0\n\n5 0 0 -1\n", 8, 6, 0),
        "crlf_and_signs": ("1 +2 3 1\r\n2 1_0 0 0\r\n3\t4   5 -1\n", 16, 8, 0),
        "slack_ok": ("10 1 1 1\n8 1 1 1\n12 0 0 0\n", 4, 4, 3),
        "slack_fail": ("10 1 1 1\n8 1 1 1\n6 0 0 0\n", 4, 4, 3),
        "order": ("5 1 1 1\n4 1 1 1\n", 4, 4, 0),
        "bounds": ("1 1 1 1\n2 9 0 1\n", 8, 8, 0),
        "fields": ("1 1 1\n", 4, 4, 0),
        "token": ("1 1 x 1\n", 4, 4, 0),
        "neg_t": ("-1 1 1 1\n", 4, 4, 0),
        "neg_xy": ("1 -1 1 1\n", 4, 4, 0),
        "polarity": ("1 1 1 2\n", 4, 4, 0),
        "comment_only": ("# a\n   # b\n\n", 4, 4, 0),
    }
    out_cases = {}
    for name, (text, w, h, slack) in cases.items():
        geom = ev.SensorGeometry(width=w, height=h)
        rec = {"text": text, "width": w, "height": h, "slack": slack}
        try:
            evs = ev.events_from_text(text, geom, slack=slack)
            rec["events"] = [[e.timestamp, e.x, e.y, e.polarity] for e in evs]
        except Exception as exc:  # the reference's own error
            rec["error"] = type(exc).__name__
            rec["message"] = str(exc)
            rec["line_no"] = getattr(exc, "line_no", None)
            rec["index"] = getattr(exc, "index", None)
        out_cases[name] = rec
    with open(os.path.join(OUT, "events_cases.json"), "w") as fh:
        json.dump(out_cases, fh, indent=1)
    pgm = sys.modules["evrecon.pgm"]
    img = np.concatenate([1.0 + (np.arange(256) + 0.5) / 255.0, 1.0 + np.arange(256) / 255.0,
                          rng.uniform(0.5, 2.5, 512)]).reshape(32, 32)
    np.savez_compressed(os.path.join(OUT, "gray.npz"), image=img,
                        gray=pgm.to_gray(img, (1.0, 2.0)))
    for name in sorted(os.listdir(OUT)):
        if name.endswith(".npz"):
            print(name, os.path.getsize(os.path.join(OUT, name)))


if __name__ == "__main__":
    main()
