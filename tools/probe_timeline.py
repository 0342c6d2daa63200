"""Probe: per-phase timeline of the resident kernel (diagnostic, GPU)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib
import bench

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
H, W, epp, pd, tv, rate = bench.CONFIGS[cfgname]
sc = evr.SolverConfig(max_iterations=pd)
mc = evr.ManifoldConfig(denoise_iterations=tv)
st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=2)
ctx = st.context()
evr.pipeline._prepare(st, mc, sc, evr.Thresholds())
ctx.call("evr_debug_timeline", 1, None, 0)
pk = bench.gen_packets(H, W, epp, 6, rate, 1)
for p in pk:
    evr.process_packet_arrays(st, p, mc, sc, evr.Thresholds(), want_frame=False)
nb = st.context()  # noqa
buf = np.zeros(256 * 160, dtype=np.uint64)
ctx.call("evr_debug_timeline", -1, _lib.ptr(buf), buf.size)
tr = buf.reshape(-1, 256).astype(np.int64)
rows = [r for r in range(tr.shape[0]) if tr[r, 0] > 0]
t0 = min(tr[r, 0] for r in rows)
nmark = 2 + tv + 1 + 1 + pd + 1
for r in [rows[0], rows[len(rows) // 2], rows[-1]]:
    m = tr[r, :nmark] - t0
    d = np.diff(m)
    print(f"CTA {r}: start {m[0]/1e3:.2f}us load+ingest {d[0]/1e3:.2f}us | TV iters mean {d[1:1+tv].mean()/1e3:.3f}us "
          f"max {d[1:1+tv].max()/1e3:.3f} | metric {d[1+tv]/1e3 + d[2+tv]/1e3:.2f}us | PD iters mean {d[3+tv:3+tv+pd].mean()/1e3:.3f}us "
          f"| end {m[-1]/1e3:.2f}us")
