#!/usr/bin/env python
"""Throughput benchmark of the per-packet hot path (process_packet).

One step = one event packet through ingest -> normalize -> TV-L1 -> metric
-> manifold-TV/KL primal-dual -> re-anchor, on the BASELINE.json workload
that fits one GPU (configs[1], DAVIS346 346x260, 500-event packets, 50 PD +
50 TV-L1 iterations; synthetic generator U of SURVEY.md 8(d)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision f64|f32]
  python bench.py --impl reference ...   # the CPU reference path (C port)

Multi-GPU (torchrun, one rank per GPU): every rank reconstructs its own
independent stream (different seed), no collective on the data path
("scaling": "weak"); timing is the max over ranks.

Rank 0 prints ONE JSON line.  `value` is events/s with the packets resident
in HBM, timed with CUDA events on the context's stream, L2 flushed before
every step (outside the per-step event pair); `e2e` is the same metric
through the public API (process_packet_arrays) from pinned host events,
including the frame read-back.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (H, W, events_per_packet, pd_iters, tv_iters, event rate ev/s)
    "C1": (128, 128, 500, 50, 50, 1e5),
    "C2": (260, 346, 500, 50, 50, 1e6),
    "C3": (720, 1280, 1000, 100, 50, 1e6),
    "C4": (480, 640, 1000, 50, 50, 1e6),
    "C5": (2048, 2048, 1000, 50, 50, 1e6),
}
DESCR = {
    "C1": "DVS128 128x128, 500-event packets, manifold-TV + KL, 50 PD + 50 TV-L1 iters",
    "C2": "DAVIS346 346x260, 500-event packets, manifold-TV + KL, 50 PD + 50 TV-L1 iters",
    "C3": "1280x720 @ 1 Mev/s, 1000-event packets, 100 PD + 50 TV-L1 iters",
    "C4": "640x480 @ 1 Mev/s per stream, 1000-event packets, 50 PD + 50 TV-L1 iters",
    "C5": "2048x2048 @ 1 Mev/s, 1000-event packets, 50 PD + 50 TV-L1 iters",
}


def gen_packets(H, W, epp, n_packets, rate, seed):
    """Generator U: uniform pixels and polarities,
    t_i = i * 1e6 / rate microseconds."""
    from paper_1607_06283_b200 import make_event_array

    rng = np.random.default_rng(seed)
    n = epp * n_packets
    step = max(int(round(1e6 / rate)), 1)
    ev = make_event_array(rng.integers(0, W, n), rng.integers(0, H, n),
                          rng.choice([-1, 1], n), np.arange(n, dtype=np.int64) * step)
    return [ev[s:s + epp] for s in range(0, n, epp)]


def windows_for(packets, t_window=None, maxlen=10):
    """Adaptive surface window per packet (pipeline.py:128-132, :155)."""
    from collections import deque

    starts = deque(maxlen=maxlen)
    out = []
    for pk in packets:
        starts.append(int(pk["t"][0]))
        now = int(pk["t"][-1])
        out.append(float(t_window) if t_window else max(float(now - starts[0]), 1.0))
    return out


def algorithmic_bytes(H, W, w, pd, tv):
    """B_pkt = N * w * (11 * I_pd + 9 * I_tv)."""
    return H * W * w * (11 * pd + 9 * tv)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allmax(x, world, device="cuda"):
    """Max over ranks (the job's time is its slowest rank's)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ----------------------------------------------------------------------------


def cpu_port_run(H, W, epp, pd, tv, rate, n_packets, seed, budget_s):
    """The reference algorithm on host cores via the C port (oracle/), one
    packet per step; returns (seconds per packet list, threads)."""
    from oracle import oracle as O

    packets = gen_packets(H, W, epp, n_packets, rate, seed)
    s = O.OracleStream(H, W, O.make_config(max_iterations=pd, denoise_iterations=tv))
    times = []
    t_start = time.perf_counter()
    for pk in packets:
        t0 = time.perf_counter()
        s.process(np.ascontiguousarray(pk))
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return times, O.num_threads()


def run_reference(args):
    # CPU arm: rank 0 alone runs (no process group, no GPU work)
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    H, W, epp, pd, tv, rate = CONFIGS[args.config]
    os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    n = args.warmup + args.steps
    times, threads = cpu_port_run(H, W, epp, pd, tv, rate, n, seed=1, budget_s=1e9)
    timed = times[args.warmup:]
    sec = sum(timed)
    value = epp * len(timed) / sec
    line = {
        "impl": "reference", "metric": "events/s", "value": round(value, 3), "unit": "events/s",
        "n_gpus": args.gpus, "steps": len(timed), "warmup": args.warmup,
        "ms_per_step": round(1e3 * sec / len(timed), 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "frames_per_s": round(len(timed) / sec, 4),
        "config": {"workload": DESCR[args.config], "sensor": f"{W}x{H}",
                   "events_per_packet": epp, "pd_iterations": pd, "tv_iterations": tv,
                   "engine": "cpu (C port of the reference)", "precision": "f64",
                   "streams": "1 (rank 0 only)", "generator": "U(seed, W, H, 1 Mev/s)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "events/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{len(timed)} packets of the same workload, C port of "
                                   f"the reference (oracle/evr_oracle.c, OpenMP {threads} threads)"},
        "e2e": {"value": round(value, 3), "unit": "events/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    world, rank, local = dist_init(args)
    os.environ["EVR_DEVICE"] = str(local)
    import torch

    import paper_1607_06283_b200 as evr
    from paper_1607_06283_b200 import _lib

    torch.cuda.set_device(local)
    H, W, epp, pd, tv, rate = CONFIGS[args.config]
    prec = {"f64": 0, "f32": 1}[args.precision]
    engine = {"auto": 0, "streaming": 1, "resident": 2, "resident_gmem": 3,
              "resident_reg": 4}[args.engine]
    mc = evr.ManifoldConfig(denoise_iterations=tv)
    sc = evr.SolverConfig(max_iterations=pd)
    th = evr.Thresholds()
    n_total = args.warmup + args.steps
    packets = gen_packets(H, W, epp, 2 * n_total, rate, seed=1000 + rank)
    wins = windows_for(packets)

    st = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=engine)
    ctx = st.context()
    evr.pipeline._prepare(st, mc, sc, th)
    h = ctx.handle
    L = _lib.lib()
    stream = torch.cuda.ExternalStream(L.evr_stream(h), device=local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # packets resident in device memory (value leg)
    allev = np.concatenate(packets[:n_total])
    dev_ev = torch.from_numpy(allev.view(np.uint8)).to("cuda")
    base = dev_ev.data_ptr()

    def dev_packet(k):
        _lib.check(h, L.evr_process_packet_device(h, ctypes.c_void_p(base + 16 * epp * k), epp,
                                                  wins[k]), "packet")

    for k in range(args.warmup):
        dev_packet(k)
    torch.cuda.synchronize()
    L.evr_synchronize(h, None)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            k = args.warmup + i
            with torch.cuda.stream(stream):
                flush.zero_()  # > L2 (126 MB): every step starts cold
                starts[i].record(stream)
            dev_packet(k)
            with torch.cuda.stream(stream):
                ends[i].record(stream)
        torch.cuda.synchronize()
        L.evr_synchronize(h, None)
    barrier(world)
    launches = ctx.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_s = allmax(sum(step_ms) / 1e3, world)
    value = world * epp * args.steps / dev_s

    # end-to-end leg: public API from pinned host events, frame read back
    pinned = [torch.from_numpy(p.view(np.uint8)).pin_memory().numpy().view(evr.EVENT_DTYPE)
              for p in packets[n_total:]]
    st2 = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=engine)
    for k in range(args.warmup):
        evr.process_packet_arrays(st2, pinned[k], mc, sc, th)
    # (1) blocking: one process_packet_arrays call per step (H2D, solve, frame
    # D2H, one synchronize), L2 flushed before every call outside the timing
    e2e_times = []
    barrier(world)
    for i in range(args.steps):
        k = args.warmup + i
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, frame, _ = evr.process_packet_arrays(st2, pinned[k], mc, sc, th)
        e2e_times.append(time.perf_counter() - t0)
    barrier(world)
    blocking = world * epp * args.steps / allmax(sum(e2e_times), world)
    # (2) streaming (the headline e2e): stream_packets, the run_stream loop --
    # every step's events go up from pinned host memory and every step's
    # frame (H x W float64) comes back to the host; packet k+1 computes while
    # frame k is copied.  Timed from the first submit to the last frame on
    # the host.
    st3 = evr.init_state(evr.SensorGeometry(W, H), sc, precision=prec, engine=engine)
    for _ in evr.stream_packets(st3, pinned[:args.warmup], mc, sc, th):
        pass
    _lib.pinned_reserve((H, W), 6)  # setup: the stream's frame pool (cudaHostAlloc is ms)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    got = 0
    ticks = []
    for frame, res in evr.stream_packets(st3, pinned[args.warmup:n_total], mc, sc, th):
        got += int(frame is not None and res.iterations == pd)
        ticks.append(time.perf_counter())
    e2e_s = allmax(time.perf_counter() - t0, world)
    if os.environ.get("EVR_BENCH_DEBUG"):
        d = np.diff([t0] + ticks) * 1e3
        print("e2e stream ms/packet: first %.3f median %.3f max %.3f" % (d[0], np.median(d), d.max()),
              file=sys.stderr)
    assert got == args.steps
    e2e = world * epp * args.steps / e2e_s

    # roofline of the dominant kernel (one packet = one persistent launch on the
    # resident engine; whole-graph time on the streaming engine)
    w = 8 if prec == 0 else 4
    bpkt = algorithmic_bytes(H, W, w, pd, tv)
    kern_ms = statistics.mean(step_ms)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bpkt / (kern_ms * 1e-3) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        hit = tr.get(f"{args.config}/{args.precision}/{st.engine()}")
        traffic = hit["bytes_per_launch"] if hit else None
    except (OSError, ValueError, KeyError):
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))
        times, threads = cpu_port_run(H, W, epp, pd, tv, rate, 400, seed=1,
                                      budget_s=args.cpu_budget)
        times = times[1:] if len(times) > 1 else times
        cpu = {"value": round(epp * len(times) / sum(times), 3), "unit": "events/s",
               "cores": threads, "kind": "port",
               "sample": f"{len(times)} packets of the same workload (first packet excluded), "
                         f"C port of the reference (oracle/evr_oracle.c), OpenMP {threads} threads"}

    if rank == 0:
        line = {
            "metric": "events/s", "value": round(value, 1), "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dev_s * 1e3 / args.steps, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "frames_per_s": round(world * args.steps / dev_s, 2),
            "config": {"workload": DESCR[args.config], "sensor": f"{W}x{H}",
                       "events_per_packet": epp, "pd_iterations": pd, "tv_iterations": tv,
                       "engine": st.engine(), "precision": args.precision,
                       "streams": f"{world} independent (1 per GPU)",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "generator": "U(seed, W, H, 1 Mev/s)"},
            "e2e": {"value": round(e2e, 1), "unit": "events/s",
                    "h2d_bytes_per_step": 32 + 16 * epp, "d2h_bytes_per_step": 8 * H * W + 24,
                    "api": "stream_packets (run_stream loop, 2 packets in flight)",
                    "blocking_value": round(blocking, 1),
                    "blocking_api": "process_packet_arrays, one synchronous call per step"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": ctx.engine_detail() + (
                             " (one launch per packet)" if st.engine().startswith("resident")
                             else " (whole packet graph)"),
                         "algorithmic_bytes_per_launch": bpkt,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--engine", default="auto",
                    choices=["auto", "streaming", "resident", "resident_gmem", "resident_reg"])
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
