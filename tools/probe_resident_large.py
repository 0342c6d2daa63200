import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1607_06283_b200 as evr
from paper_1607_06283_b200 import _lib
if "r1" in __import__("os").environ.get("EVR_LIBRARY", ""):
    _lib._SIGNATURES.pop("evr_time_iteration_kernel", None)  # round-1 library
import bench
H, W, epp, pd, tv, rate = bench.CONFIGS["C3"]
pk = bench.gen_packets(H, W, epp, 30, rate, 1)
mc, sc, th = evr.ManifoldConfig(denoise_iterations=tv), evr.SolverConfig(max_iterations=pd), evr.Thresholds()
for prec in (0, 1):
  for eng in (1, 3, 2):
    try:
        st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=eng)
        for p in pk[:5]:
            evr.process_packet_arrays(st, p, mc, sc, th, want_frame=False)
        import torch; torch.cuda.synchronize()
        t0 = time.perf_counter()
        for p in pk[5:25]:
            evr.process_packet_arrays(st, p, mc, sc, th, want_frame=False)
        dt = (time.perf_counter() - t0) / 20
        print(prec, eng, st.context().engine_detail()[:90], "%.3f ms" % (dt * 1e3))
    except Exception as e:
        print(prec, eng, "ERR", str(e)[:100])
