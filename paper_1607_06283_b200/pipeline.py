"""Per-event state machine on the device (reference: pipeline.py).

Drop-in for evrecon.pipeline: the same configuration dataclasses, state
fields and functions (init_state, apply_event, process_packet, run_stream),
with the packet work done by one CUDA context per stream:

  ingest (bit-exact scatter) -> normalize -> TV-L1 -> metric -> KL
  primal-dual solve -> f <- u re-anchor,

captured once as a CUDA graph and replayed per packet (include/evr.h,
evr_process_packet).  The state lives in device memory; the numpy views
``u``, ``f``, ``raw_timestamps`` and ``p`` are materialised on access.
Arrays handed out by (or assigned to) those attributes are treated as
caller-editable and are written back before the next device operation, so
the reference idioms (``state.f[y, x] = v`` then ``apply_event``) keep
working.  Array identity follows the reference: ``process_packet`` returns
the frame as the new ``state.u`` (a fresh array), re-anchors ``f`` to a
copy of it and replaces ``p``; ``apply_event`` and the ingest update ``f``
and ``raw_timestamps`` in place.
"""

from __future__ import annotations

import ctypes
import math
import os
import sys
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .events import Event, SensorGeometry, events_to_array
from .solve import SolveResult, SolverConfig, solver_config_struct
from .surface import MetricField, TimeSurface

# pipeline.py:32 -- trailing packets whose span sets the adaptive window
ADAPTIVE_WINDOW_PACKETS = 10

_PRECISIONS = {"f64": _lib.PREC_F64, "fp64": _lib.PREC_F64, "float64": _lib.PREC_F64,
               "f32": _lib.PREC_F32, "fp32": _lib.PREC_F32, "float32": _lib.PREC_F32}
_ENGINES = {"auto": _lib.ENGINE_AUTO, "streaming": _lib.ENGINE_STREAMING,
            "resident": _lib.ENGINE_RESIDENT}


def default_precision():
    """EVR_PRECISION=f64 (default, bit-exact) | f32."""
    return _PRECISIONS[os.environ.get("EVR_PRECISION", "f64").lower()]


def default_engine():
    """EVR_ENGINE=auto (default) | streaming | resident."""
    return _ENGINES[os.environ.get("EVR_ENGINE", "auto").lower()]


@dataclass
class PacketPolicy:
    """Events per frame and display decimation (pipeline.py:35-48)."""

    events_per_packet: int = 500
    frames_to_skip: int = 0

    def __post_init__(self):
        if self.events_per_packet < 1:
            raise ValueError(f"events_per_packet must be >= 1, got {self.events_per_packet}")
        if self.frames_to_skip < 0:
            raise ValueError(f"frames_to_skip must be >= 0, got {self.frames_to_skip}")


@dataclass
class Thresholds:
    """Log-intensity quanta (pipeline.py:51-68)."""

    pos: float = 0.15
    neg: float = 0.15

    def __post_init__(self):
        if self.pos <= 0 or self.neg <= 0:
            raise ValueError(f"thresholds must be positive, got {self.pos}, {self.neg}")

    @property
    def c_pos(self):
        return math.exp(self.pos)

    @property
    def c_neg(self):
        return math.exp(-self.neg)


@dataclass
class ManifoldConfig:
    """Time-surface parameters (pipeline.py:71-84)."""

    enabled: bool = True
    t_scale: float = 3.0
    t_window: float | None = None
    denoise_weight: float = 1.0
    denoise_iterations: int = 50


def device_config(manifold_cfg, solver_cfg, thresholds, engine=None):
    """evr_config for one (manifold, solver, thresholds) triple."""
    c = solver_config_struct(solver_cfg)
    c.manifold_enabled = 1 if manifold_cfg.enabled else 0
    c.t_scale = float(manifold_cfg.t_scale)
    c.denoise_weight = float(manifold_cfg.denoise_weight)
    c.denoise_iterations = int(manifold_cfg.denoise_iterations)
    c.engine = default_engine() if engine is None else int(engine)
    c.c_pos, c.c_neg = thresholds.c_pos, thresholds.c_neg
    return c


_FIELDS = ("u", "f", "raw_timestamps", "p")


class ReconstructionState:
    """Everything carried from packet to packet (pipeline.py:87-99), held in
    device memory.  Construct with init_state(); constructing it from arrays
    like the reference dataclass also works (uploaded on first use)."""

    def __init__(self, u=None, f=None, raw_timestamps=None, p=None, events_in_packet=0,
                 frame_index=0, packet_starts=None, *, precision=None, engine=None):
        self.events_in_packet = events_in_packet
        self.frame_index = frame_index
        self.packet_starts = (packet_starts if packet_starts is not None
                              else deque(maxlen=ADAPTIVE_WINDOW_PACKETS))
        self._precision = default_precision() if precision is None else precision
        self._engine = engine
        self._ctx = None
        self._shape = None
        self._mirror = {}
        self._exposed = set()
        self._cfg_struct = None
        for name, val in zip(_FIELDS, (u, f, raw_timestamps, p)):
            if val is not None:
                setattr(self, name, val)

    # ---- device context ----------------------------------------------------
    @property
    def shape(self):
        return self._shape

    @property
    def precision(self):
        return "f64" if self._precision == _lib.PREC_F64 else "f32"

    def _bind(self, shape):
        shape = (int(shape[0]), int(shape[1]))
        if self._shape is None:
            self._shape = shape
        elif shape != self._shape:
            raise ValueError(f"array shape {shape} != state shape {self._shape}")

    def context(self):
        if self._ctx is None:
            if self._shape is None:
                raise ValueError("state has no shape yet: use init_state(geometry, cfg)")
            self._ctx = _lib.Context(self._shape[0], self._shape[1], self._precision)
            # fields never assigned start as init_state would set them
            missing = [n for n in _FIELDS if n not in self._mirror]
            if missing:
                self._configure(ManifoldConfig(), SolverConfig(), Thresholds())
                self._ctx.call("evr_init_state")
            self._flush()
        return self._ctx

    def _configure(self, manifold_cfg, solver_cfg, thresholds):
        ctx = self._ctx
        c = device_config(manifold_cfg, solver_cfg, thresholds, self._engine)
        ctx.set_config(c)
        self._cfg_struct = c

    def _flush(self):
        """Write caller-visible (possibly edited) mirrors back to the device."""
        if not self._exposed:
            return
        args = {}
        for name in self._exposed:
            a = self._mirror[name]
            dtype = np.int64 if name == "raw_timestamps" else np.float64
            args[name] = np.ascontiguousarray(a, dtype=dtype)
        self._ctx.call("evr_set_state", _lib.ptr(args.get("u")), _lib.ptr(args.get("f")),
                       _lib.ptr(args.get("raw_timestamps")), _lib.ptr(args.get("p")))

    def _download(self, name, out=None):
        H, W = self._shape
        if out is None:
            out = np.empty((H, W, 3) if name == "p" else (H, W),
                           dtype=np.int64 if name == "raw_timestamps" else np.float64)
        ptrs = [None] * 4
        ptrs[_FIELDS.index(name)] = _lib.ptr(out)
        self._ctx.call("evr_get_state", *ptrs)
        return out

    def _after_device_write(self, replaced=(), in_place=()):
        """Device state changed: drop mirrors the reference would replace with
        new arrays, refresh in place those it mutates in place."""
        for name in replaced:
            self._mirror.pop(name, None)
            self._exposed.discard(name)
        for name in in_place:
            a = self._mirror.get(name)
            if a is not None:
                if a.flags.c_contiguous and a.dtype == (
                        np.int64 if name == "raw_timestamps" else np.float64):
                    self._download(name, out=a)
                else:
                    a[...] = self._download(name)

    def _get(self, name):
        a = self._mirror.get(name)
        if a is None:
            self.context()
            a = self._download(name)
            self._mirror[name] = a
        self._exposed.add(name)
        return a

    def _set(self, name, value):
        if name == "p":
            arr = np.asarray(value)
            if arr.ndim != 3 or arr.shape[2] != 3:
                raise ValueError(f"p must be (H, W, 3), got {arr.shape}")
            self._bind(arr.shape[:2])
        else:
            arr = np.asarray(value)
            if arr.ndim != 2:
                raise ValueError(f"{name} must be 2-D, got {arr.shape}")
            self._bind(arr.shape)
        self._mirror[name] = arr
        self._exposed.add(name)

    u = property(lambda s: s._get("u"), lambda s, v: s._set("u", v))
    f = property(lambda s: s._get("f"), lambda s, v: s._set("f", v))
    raw_timestamps = property(lambda s: s._get("raw_timestamps"),
                              lambda s, v: s._set("raw_timestamps", v))
    p = property(lambda s: s._get("p"), lambda s, v: s._set("p", v))

    def engine(self):
        return self.context().engine()

    def __repr__(self):
        return (f"ReconstructionState(shape={self._shape}, precision={self.precision}, "
                f"frame_index={self.frame_index}, events_in_packet={self.events_in_packet})")


def init_state(geometry, cfg: SolverConfig, *, precision=None, engine=None):
    """Neutral start u = f = box midpoint, raw = 0, p = 0 (pipeline.py:102-111)."""
    st = ReconstructionState(precision=precision, engine=engine)
    st._bind((geometry.height, geometry.width))
    st._ctx = _lib.Context(geometry.height, geometry.width, st._precision)
    st._configure(ManifoldConfig(), cfg, Thresholds())
    st._ctx.call("evr_init_state")
    return st


def _prepare(state, manifold_cfg, solver_cfg, thresholds):
    ctx = state.context()
    state._configure(manifold_cfg, solver_cfg, thresholds)
    state._flush()
    return ctx


def apply_event(state, event, thresholds, cfg: SolverConfig):
    """Multiplicative quantum + clamp at one pixel (pipeline.py:114-121), on
    the device ingest kernel."""
    ctx = _prepare(state, ManifoldConfig(), cfg, thresholds)
    ev = events_to_array([event])
    ctx.call("evr_ingest", _lib.ptr(ev), 1)
    state._after_device_write(in_place=("f", "raw_timestamps"))
    state.events_in_packet += 1
    return state


def _window(state, now, manifold_cfg):
    # pipeline.py:128-132
    if manifold_cfg.t_window is not None:
        return float(manifold_cfg.t_window)
    oldest = state.packet_starts[0] if state.packet_starts else now
    return max(float(now - oldest), 1.0)


def _device_early_stop(ctx):
    """convergence_tol > 0 folds rel_change and stops on the device on both
    engines (the resident column kernel's per-iteration fold; the fused
    streaming list's stop flag), so such packets take the one-round-trip
    path too."""
    return ctx.engine() in ("resident", "streaming")


def process_packet_arrays(state, events, manifold_cfg, solver_cfg, thresholds, trace=None,
                          debug_sink=None, want_frame=True):
    """process_packet for an EVENT_DTYPE array (no per-event Python work).

    Returns (state, frame or None, SolveResult or None).  ``want_frame=False``
    skips the frame download (the result's u/p are then None too).
    """
    n = len(events)
    if n == 0:  # pipeline.py:151-153
        return state, state.u.copy(), None
    events = events_to_array(events)
    ctx = _prepare(state, manifold_cfg, solver_cfg, thresholds)
    state.packet_starts.append(int(events["t"][0]))  # pipeline.py:155
    state.events_in_packet = n
    now = int(events["t"][-1])
    window = _window(state, now, manifold_cfg) if manifold_cfg.enabled else 1.0
    info = _lib.SolveInfo()
    split = (debug_sink is not None or trace is not None
             or (solver_cfg.convergence_tol > 0 and not _device_early_stop(ctx)))
    frame = None
    if not split:
        # one round trip: packet, solve and (pinned) frame download on the
        # context stream, then a single synchronize
        ctx.call("evr_process_packet_async", _lib.ptr(events), n, float(window))
        if want_frame:
            frame = _lib.pinned_empty(state.shape)
            ctx.call("evr_get_frame_async", _lib.ptr(frame))
        ctx.call("evr_synchronize", ctypes.byref(info))
    else:
        ctx.call("evr_packet_begin", _lib.ptr(events), n, float(window))
        if debug_sink is not None:
            H, W = state.shape
            t, tx, ty, G, sg = (np.empty((H, W)) for _ in range(5))
            ctx.call("evr_get_surface", _lib.ptr(t), None)
            ctx.call("evr_get_metric", _lib.ptr(tx), _lib.ptr(ty), _lib.ptr(G), _lib.ptr(sg))
            surface = TimeSurface(t=t, t_scale=manifold_cfg.t_scale) if manifold_cfg.enabled else None
            metric = MetricField(tx=tx, ty=ty, G=G, sqrtG=sg)
            state._after_device_write(in_place=("f", "raw_timestamps"))
            debug_sink(state.frame_index, surface, metric)
            state._flush()
        et = rt = None
        if trace is not None:
            et = np.zeros(solver_cfg.max_iterations)
            rt = np.zeros(solver_cfg.max_iterations)
        ctx.call("evr_packet_solve", ctypes.byref(info), _lib.ptr(et), _lib.ptr(rt))
        if trace is not None:
            for k in range(info.iterations):
                trace.append((k + 1, float(et[k]), float(rt[k])))
    state.frame_index += 1
    state._after_device_write(replaced=("u", "f", "p"), in_place=("raw_timestamps",))
    if not want_frame:
        return state, None, SolveResult(u=None, p=None, iterations=int(info.iterations),
                                        rel_change=float(info.rel_change))
    if frame is None:
        frame = _lib.pinned_empty(state.shape)
        ctx.call("evr_get_frame", _lib.ptr(frame))
    # frame aliases state.u, like the reference -- as a read-only snapshot:
    # an in-place edit would not reach the device state, so it raises
    # instead (assign state.u to change the warm start)
    frame.flags.writeable = False
    state._mirror["u"] = frame
    return state, frame, _LazyResult(state, frame, info)


class _LazyResult(SolveResult):
    """SolveResult whose dual p is fetched from the device on first read.

    In the reference result.p is state.p; it is served from the state while
    the state still holds this packet's solution."""

    def __new__(cls, state, frame, info, frame_index=None):
        self = super().__new__(cls, frame, None, int(info.iterations), float(info.rel_change))
        self._state = state
        self._frame_index = state.frame_index if frame_index is None else frame_index
        # device time of the packet (event upload .. frame download), when
        # it went through the frame pipeline (evr_frame_wait); else None
        self.packet_ms = float(info.packet_ms) if info.packet_ms > 0 else None
        return self

    @property
    def p(self):
        if self._state.frame_index != self._frame_index:
            raise RuntimeError("result.p is only available until the next packet is processed")
        return self._state.p


def stream_packets(state, packets, manifold_cfg, solver_cfg, thresholds, depth=2,
                   want_frames=True):
    """Pipelined process_packet over a sequence of packets (the run_stream
    loop, pipeline.py:228-256): yields ``(frame, SolveResult)`` per packet in
    stream order, with up to ``depth`` packets in flight on the device --
    packet k+1's events go up and its solve runs while frame k is copied to
    the host on a second stream (evr_frame_submit / evr_frame_wait).

    The state advances exactly as with one process_packet call per packet
    (the device executes the packets in order; frames are bit-identical).
    ``want_frames`` may be a bool or a callable ``(frame_index) -> bool``
    (decimation: frames not wanted come back as None).  A result's ``p`` is
    readable only while the state still holds that packet's solution (the
    last packet of the stream).  Packets that need the host-driven solve
    (``convergence_tol > 0`` on the streaming engine) run one at a time.
    """
    if not 1 <= depth <= 4:
        raise ValueError(f"depth must be in [1, 4], got {depth}")
    if solver_cfg.convergence_tol > 0 and not _device_early_stop(
            _prepare(state, manifold_cfg, solver_cfg, thresholds)):
        for pk in packets:
            idx = state.frame_index
            want = want_frames(idx) if callable(want_frames) else want_frames
            _, frame, res = process_packet_arrays(state, events_to_array(pk), manifold_cfg,
                                                  solver_cfg, thresholds, want_frame=bool(want))
            yield frame, res
        return
    ctx = _prepare(state, manifold_cfg, solver_cfg, thresholds)
    pending = deque()
    if want_frames:  # frames in flight + the one the caller holds
        _lib.pinned_reserve(state.shape, depth + 2)

    def finish():
        ticket, frame, idx = pending.popleft()
        info = _lib.SolveInfo()
        ctx.call("evr_frame_wait", ticket, ctypes.byref(info))
        if frame is not None:
            frame.flags.writeable = False  # a snapshot (see process_packet_arrays)
            if not pending and idx == state.frame_index:
                state._mirror["u"] = frame  # frame aliases state.u, like the reference
        return frame, _LazyResult(state, frame, info, frame_index=idx)

    it = iter(packets)
    try:
        while True:
            try:
                pk = next(it)
            except StopIteration:
                break
            except BaseException:
                # the packet source failed (e.g. StreamOrderError from
                # read_stream): the frames already computed go out first,
                # as the reference's run_stream delivers frame k before it
                # reads packet k+1
                while pending:
                    yield finish()
                raise
            events = events_to_array(pk)
            n = len(events)
            if n == 0:  # pipeline.py:151-153, after the packets before it
                while pending:
                    yield finish()
                yield state.u.copy(), None
                continue
            state._flush()
            state.packet_starts.append(int(events["t"][0]))  # pipeline.py:155
            state.events_in_packet = n
            now = int(events["t"][-1])
            window = _window(state, now, manifold_cfg) if manifold_cfg.enabled else 1.0
            want = want_frames(state.frame_index) if callable(want_frames) else want_frames
            ctx.call("evr_process_packet_async", _lib.ptr(events), n, float(window))
            frame = _lib.pinned_empty(state.shape) if want else None
            ticket = ctypes.c_int64(0)
            ctx.call("evr_frame_submit", _lib.ptr(frame), ctypes.byref(ticket))
            state.frame_index += 1
            state._after_device_write(replaced=("u", "f", "p"), in_place=("raw_timestamps",))
            pending.append((ticket.value, frame, state.frame_index))
            if len(pending) >= depth:
                yield finish()
        while pending:
            yield finish()
    finally:
        while pending:  # generator closed early (GeneratorExit): release the slots
            try:
                finish()
            except Exception:
                pending.clear()
                raise


def process_packet(state, events, manifold_cfg, solver_cfg, thresholds, trace=None,
                   debug_sink=None):
    """Integrate one packet and solve (pipeline.py:142-171); returns
    (state, frame, SolveResult) and mutates ``state`` in place."""
    if not isinstance(events, np.ndarray):
        events = list(events)
        if not events:
            return state, state.u.copy(), None
    return process_packet_arrays(state, events, manifold_cfg, solver_cfg, thresholds,
                                 trace=trace, debug_sink=debug_sink)


@dataclass
class StreamStats:
    """Per-run counters and per-packet timings (pipeline.py:174-203)."""

    events_consumed: int = 0
    packets: int = 0
    frames_emitted: int = 0
    wall_seconds: float = 0.0
    solve_ms: list = field(default_factory=list)
    iterations: list = field(default_factory=list)

    @property
    def events_per_sec(self):
        return self.events_consumed / self.wall_seconds if self.wall_seconds else 0.0

    @property
    def frames_per_sec(self):
        return self.packets / self.wall_seconds if self.wall_seconds else 0.0

    @property
    def mean_solve_ms(self):
        return float(np.mean(self.solve_ms)) if self.solve_ms else 0.0

    def summary(self):
        return (
            f"{self.packets} packets, {self.frames_emitted} frames emitted, "
            f"{self.events_consumed} events, "
            f"mean solve {self.mean_solve_ms:.2f} ms, "
            f"{self.events_per_sec:.0f} events/s, {self.frames_per_sec:.1f} frames/s"
        )


def _packets(events, epp):
    """Yield (packet, n_consumed) in stream order from a list/iterable of
    Event or from an EVENT_DTYPE array."""
    if isinstance(events, np.ndarray):
        for s in range(0, len(events), epp):
            chunk = events[s:s + epp]
            yield chunk, len(chunk)
        return
    packet = []
    for ev in events:
        packet.append(ev)
        if len(packet) == epp:
            yield packet, len(packet)
            packet = []
    if packet:
        yield packet, len(packet)


def run_stream(events, geometry, policy, manifold_cfg, solver_cfg, thresholds, sink=None,
               state=None, stats_every=0, log=sys.stderr, trace=None, debug_sink=None):
    """Packetise an event stream and reconstruct frames (pipeline.py:206-276).

    Every (frames_to_skip+1)-th frame goes to ``sink(index, frame)``; returns
    (state, StreamStats); pass the state back in to continue the stream.
    ``events`` may also be an EVENT_DTYPE array.
    """
    if state is None:
        state = init_state(geometry, solver_cfg)
    stats = StreamStats()
    stride = policy.frames_to_skip + 1
    t0 = time.perf_counter()
    if trace is not None:
        trace.write("packet,iteration,energy,rel_change\n")
    if trace is None and debug_sink is None:
        _run_pipelined(events, state, policy, manifold_cfg, solver_cfg, thresholds, sink,
                       stats, stride, stats_every, log, t0)
        stats.wall_seconds = time.perf_counter() - t0
        return state, stats
    for packet, n in _packets(events, policy.events_per_packet):
        stats.events_consumed += n
        rows = [] if trace is not None else None
        t_solve = time.perf_counter()
        # the frame is downloaded only when this packet will reach the sink
        emit = (state.frame_index % stride) == 0
        arr = events_to_array(packet)
        _, frame, result = process_packet_arrays(
            state, arr, manifold_cfg, solver_cfg, thresholds, trace=rows,
            debug_sink=debug_sink, want_frame=emit and sink is not None)
        if rows:
            for it, en, rel in rows:
                trace.write(f"{stats.packets},{it},{en:.10g},{rel:.6g}\n")
        ms = (time.perf_counter() - t_solve) * 1e3
        stats.packets += 1
        stats.solve_ms.append(ms)
        stats.iterations.append(result.iterations)
        if (state.frame_index - 1) % stride == 0:
            if sink is not None:
                sink(stats.frames_emitted, frame)
            stats.frames_emitted += 1
        if stats_every and stats.packets % stats_every == 0:
            elapsed = time.perf_counter() - t0
            rate = stats.events_consumed / elapsed if elapsed > 0 else 0.0
            print(f"packet {stats.packets}: {ms:.2f} ms/solve, "
                  f"{result.iterations} iterations, {rate:.0f} events/s", file=log)
    stats.wall_seconds = time.perf_counter() - t0
    return state, stats


def _run_pipelined(events, state, policy, manifold_cfg, solver_cfg, thresholds, sink, stats,
                   stride, stats_every, log, t0):
    """run_stream's packet loop over stream_packets: the device works on
    packet k+1 while frame k is read back and handed to the sink."""
    sizes = deque()

    def packets():
        for packet, n in _packets(events, policy.events_per_packet):
            sizes.append(n)
            yield events_to_array(packet)

    want = (lambda idx: idx % stride == 0) if sink is not None else False
    first_index = state.frame_index - stats.packets
    t_last = time.perf_counter()
    for frame, result in stream_packets(state, packets(), manifold_cfg, solver_cfg, thresholds,
                                        want_frames=want):
        n = sizes.popleft()
        stats.events_consumed += n
        now = time.perf_counter()
        # solve_ms as the reference records it (pipeline.py:239-249): the
        # packet's own processing time -- here its device time from event
        # upload to frame download (packets overlap in the pipeline, so
        # wall-clock deltas would be inter-arrival times instead)
        ms = result.packet_ms if result.packet_ms is not None else (now - t_last) * 1e3
        t_last = now
        stats.packets += 1
        stats.solve_ms.append(ms)
        stats.iterations.append(result.iterations)
        # decimation phase carried in the state (frame_index after the packet)
        if (first_index + stats.packets - 1) % stride == 0:
            if sink is not None:
                sink(stats.frames_emitted, frame)
            stats.frames_emitted += 1
        if stats_every and stats.packets % stats_every == 0:
            elapsed = now - t0
            rate = stats.events_consumed / elapsed if elapsed > 0 else 0.0
            print(f"packet {stats.packets}: {ms:.2f} ms/solve, "
                  f"{result.iterations} iterations, {rate:.0f} events/s", file=log)
