"""Golden fixtures of the reference's event simulator (simulate.py), made by
running the REFERENCE itself in the build container:

    python tests/golden/make_sim_golden.py

Records rendered frames of every scene kind and the events generate_events
produces from them (plus an irregular-timestamp random video with dp != dn),
which pin render_scene (CPU test) and the GPU simulator (GPU test).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from evrecon import events as ev
    from evrecon import simulate as sim

    cases = {}
    geom = ev.SensorGeometry(width=40, height=24)
    specs = [("moving_square", 9, 1000, {}), ("moving_sine", 12, 1000, {}),
             ("two_bars", 10, 700, {"speed": 1.3}),
             ("moving_sine", 7, 250, {"period": 9.0, "velocity": (0.7, 0.4)}),
             ("moving_square", 6, 500, {"size": 11.0, "velocity": (1.1, -0.6)})]
    for i, (kind, n, dt, params) in enumerate(specs):
        video = sim.render_scene(kind, geom, n, dt=dt, **dict(params))
        evs = sim.generate_events(video, 0.15, 0.15 if i % 2 == 0 else 0.11)
        cases[f"c{i}_frames"] = video.frames
        cases[f"c{i}_ts"] = video.frame_timestamps
        cases[f"c{i}_dn"] = np.array(0.15 if i % 2 == 0 else 0.11)
        cases[f"c{i}_ev"] = np.array([[e.timestamp, e.x, e.y, e.polarity] for e in evs],
                                     dtype=np.int64).reshape(-1, 4)
    # irregular timestamps, random positive frames, dp != dn
    rng = np.random.default_rng(11)
    frames = np.exp(rng.normal(0.4, 0.35, (8, 13, 17)))
    ts = np.cumsum(rng.integers(1, 900, 8)).astype(np.int64)
    video = sim.GroundTruthVideo(frames=frames, frame_timestamps=ts)
    evs = sim.generate_events(video, 0.2, 0.13)
    cases["r_frames"], cases["r_ts"] = frames, ts
    cases["r_ev"] = np.array([[e.timestamp, e.x, e.y, e.polarity] for e in evs],
                             dtype=np.int64).reshape(-1, 4)
    cases["specs"] = np.array(repr(specs))
    np.savez_compressed(os.path.join(OUT, "simulate.npz"), **cases)
    print({k: v.shape for k, v in cases.items() if k.endswith("_ev")})


if __name__ == "__main__":
    main()
