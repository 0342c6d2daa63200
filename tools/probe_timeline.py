"""Probe: per-phase timeline of the resident kernel (diagnostic, GPU).

Marks (thread 0 of each CTA, globaltimer ns): start, after load+ingest, one
per TV-L1 iteration (after the halo fetch), before the metric, before the
solve, then per primal-dual iteration: fetch done / primal done / dual
issued, and the end of the solve.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
H, W, epp, pd, tv, rate = bench.CONFIGS[cfgname]
pd = min(pd, int(os.environ.get("PROBE_PD", "50")))  # 256 timeline slots per CTA
sc = evr.SolverConfig(max_iterations=pd)
mc = evr.ManifoldConfig(denoise_iterations=tv)
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=2)
ctx = st.context()
evr.pipeline._prepare(st, mc, sc, evr.Thresholds())
ctx.call("evr_debug_timeline", 1, None, 0)
for p in bench.gen_packets(H, W, epp, 6, rate, 1):
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
buf = np.zeros(256 * 160, dtype=np.uint64)
ctx.call("evr_debug_timeline", -1, _lib.ptr(buf), buf.size)
tr = buf.reshape(-1, 256).astype(np.int64)
rows = [r for r in range(tr.shape[0]) if tr[r, 0] > 0]
t0 = min(tr[r, 0] for r in rows)
for r in [rows[0], rows[len(rows) // 2], rows[-1]]:
    m = (tr[r] - t0) / 1e3
    k = 2 + tv  # marks 0, 1, tv x TV, metric, solve-start
    tvd = np.diff(m[1:2 + tv])
    # per PD iteration: fetch done | primal issued (thread 0) | primal done | dual issued
    pdm = m[k + 2:k + 2 + 4 * pd].reshape(pd, 4)
    fetch = pdm[1:, 0] - pdm[:-1, 3]
    primal0 = pdm[:, 1] - pdm[:, 0]
    pbar = pdm[:, 2] - pdm[:, 1]
    primal = pdm[:, 2] - pdm[:, 0]
    dual = pdm[:, 3] - pdm[:, 2]
    print(f"{cfgname} f{'64' if prec == 0 else '32'} CTA {r:3d}: ingest {m[1]-m[0]:.2f} | TV/it {tvd.mean():.2f} "
          f"| metric {m[k] - m[k-1]:.2f} (+{m[k+1]-m[k]:.2f}) | PD/it {np.diff(pdm[:, 0]).mean():.2f} = "
          f"fetch {fetch.mean():.2f} + primal {primal.mean():.2f} (t0 {primal0.mean():.2f} bar {pbar.mean():.2f}) + dual {dual.mean():.2f} | end {m[k+2+4*pd]:.1f} us")

# neighbour handoff: fetch done (CTA r, iteration i) minus the later of the two
# neighbours' "dual issued" marks of iteration i-1 (thread 0 = column 0 both)
k = 2 + tv
eff = []
for r in rows[1:-1]:
    a = (tr[r] - t0)[k + 2:k + 2 + 4 * pd].reshape(pd, 4) / 1e3
    up = (tr[r - 1] - t0)[k + 2:k + 2 + 4 * pd].reshape(pd, 4) / 1e3
    dn = (tr[r + 1] - t0)[k + 2:k + 2 + 4 * pd].reshape(pd, 4) / 1e3
    own = a[:-1, 3]
    nb = np.maximum(up[:-1, 3], dn[:-1, 3])
    eff.append((a[1:, 0] - nb, a[1:, 0] - own, nb - own))
L = np.concatenate([e[0] for e in eff])
W8 = np.concatenate([e[1] for e in eff])
S = np.concatenate([e[2] for e in eff])
print(f"handoff after the later neighbour's put: median {np.median(L):.2f} us (p10 {np.percentile(L, 10):.2f}, p90 {np.percentile(L, 90):.2f}); "
      f"own wait {np.median(W8):.2f} us; neighbour lag behind own put {np.median(S):.2f} us")

# per CTA: the SM it ran on (slot 255) and its mean halo fetch per iteration
print("CTA smid TV/it PDfetch PD/it")
for r in rows:
    a = (tr[r] - t0)[k + 2:k + 2 + 4 * pd].reshape(pd, 4) / 1e3
    m = (tr[r] - t0) / 1e3
    tvd = np.diff(m[1:2 + tv]).mean()
    fetch = (a[1:, 0] - a[:-1, 3]).mean()
    print(f"{r:3d} {int(buf.reshape(-1, 256)[r, 255]):3d} {tvd:.2f} {fetch:.2f} {np.diff(a[:, 0]).mean():.2f}")
