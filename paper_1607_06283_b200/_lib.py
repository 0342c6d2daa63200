"""ctypes binding of the C ABI (include/evr.h) implemented by libevr.so.

There is deliberately no fallback: if the shared library is missing, was
built for another architecture, or no CUDA device is visible, every entry
point raises.  The product path is the sm_100a CUDA library or nothing.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EVR_LIBRARY", os.path.join(_HERE, "libevr.so"))

EVR_OK = 0
EVR_ERR_INVALID = -1
EVR_ERR_CUDA = -2
EVR_ERR_OOM = -3
EVR_ERR_RANGE = -4
EVR_ERR_UNSUPPORTED = -5

PREC_F64 = 0
PREC_F32 = 1
ENGINE_AUTO = 0
ENGINE_STREAMING = 1
ENGINE_RESIDENT = 2
ENGINE_NAMES = {ENGINE_AUTO: "auto", ENGINE_STREAMING: "streaming", ENGINE_RESIDENT: "resident"}

# evr_event (include/evr.h): 16-byte packed camera event
EVENT_DTYPE = np.dtype([("t", "<i8"), ("x", "<i4"), ("y", "<i2"), ("polarity", "<i2")])
assert EVENT_DTYPE.itemsize == 16


class Config(ctypes.Structure):
    """evr_config: SolverConfig + ManifoldConfig + Thresholds quanta."""

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
        ("engine", ctypes.c_int32),
        ("c_pos", ctypes.c_double),
        ("c_neg", ctypes.c_double),
    ]


class SolveInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("packet_ms", ctypes.c_float),
                ("rel_change", ctypes.c_double)]


class EvrError(RuntimeError):
    """A failure reported by the CUDA library."""

    def __init__(self, code, message):
        super().__init__(f"evr error {code}: {message}")
        self.code = code


_P = ctypes.c_void_p
_i32, _i64, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_double

_SIGNATURES = {
    "evr_version": ([], ctypes.c_char_p),
    "evr_device_count": ([_P], _i32),
    "evr_create": ([_P, _i32, _i32, _i32, _i32], _i32),
    "evr_destroy": ([_P], None),
    "evr_last_error": ([_P], ctypes.c_char_p),
    "evr_set_config": ([_P, _P], _i32),
    "evr_active_engine": ([_P, _P], _i32),
    "evr_engine_detail": ([_P, ctypes.c_char_p, _i32], _i32),
    "evr_init_state": ([_P], _i32),
    "evr_set_state": ([_P, _P, _P, _P, _P], _i32),
    "evr_get_state": ([_P, _P, _P, _P, _P], _i32),
    "evr_ingest": ([_P, _P, _i64], _i32),
    "evr_process_packet": ([_P, _P, _i64, _d, _P], _i32),
    "evr_process_packet_async": ([_P, _P, _i64, _d], _i32),
    "evr_process_packet_device": ([_P, _P, _i64, _d], _i32),
    "evr_packet_begin": ([_P, _P, _i64, _d], _i32),
    "evr_packet_solve": ([_P, _P, _P, _P], _i32),
    "evr_synchronize": ([_P, _P], _i32),
    "evr_get_frame": ([_P, _P], _i32),
    "evr_get_frame_async": ([_P, _P], _i32),
    "evr_frame_submit": ([_P, _P, _P], _i32),
    "evr_set_tile_k": ([_P, _i32], _i32),
    "evr_time_iteration_kernel": ([_P, _i32, _i32, _P, _P], _i32),
    "evr_frame_wait": ([_P, _i64, _P], _i32),
    "evr_host_alloc": ([ctypes.c_size_t, _P], _i32),
    "evr_host_free": ([_P], _i32),
    "evr_sim_create": ([_P, _i32], _i32),
    "evr_sim_destroy": ([_P], None),
    "evr_sim_last_error": ([_P], ctypes.c_char_p),
    "evr_sim_generate": ([_P, _P, _P, _i32, _i32, _i32, _d, _d, _P], _i32),
    "evr_sim_events": ([_P, _P, _i64], _i32),
    "evr_sim_device_events": ([_P, _P, _P], _i32),
    "evr_get_surface": ([_P, _P, _P], _i32),
    "evr_get_metric": ([_P, _P, _P, _P, _P], _i32),
    "evr_get_frame_u8": ([_P, _d, _d, _P], _i32),
    "evr_event_buffer": ([_P, _i64, _P], _i32),
    "evr_debug_timeline": ([_P, _i32, _P, _i64], _i32),
    "evr_group_create": ([_P, _i32, _P, _i32, _i32, _i32], _i32),
    "evr_group_destroy": ([_P], None),
    "evr_group_last_error": ([_P], ctypes.c_char_p),
    "evr_group_band": ([_P, _i32, _P, _P, _P], _i32),
    "evr_group_set_config": ([_P, _P], _i32),
    "evr_group_init_state": ([_P], _i32),
    "evr_group_set_state": ([_P, _P, _P, _P, _P], _i32),
    "evr_group_get_state": ([_P, _P, _P, _P, _P], _i32),
    "evr_group_process_packet": ([_P, _P, _i64, _d, _P], _i32),
    "evr_group_get_frame": ([_P, _P], _i32),
    "evr_group_launch_count": ([_P], _i64),
    "evr_parse_events": ([_P, _i64, _i32, _i32, _i64, _P, _P, _i64, _P, _P, _P, _P], _i32),
    "evr_stream": ([_P], _P),
    "evr_launch_count": ([_P], _i64),
    "evr_op_grad": ([_P, _P, _P, _P], _i32),
    "evr_op_div": ([_P, _P, _P, _P], _i32),
    "evr_op_normalize": ([_P, _P, _d, _d, _d, _P], _i32),
    "evr_op_denoise": ([_P, _P, _d, _i32, _d, _P], _i32),
    "evr_op_metric": ([_P, _P, _P, _P, _P, _P], _i32),
    "evr_op_coeffs": ([_P, _P, _P, _P, _P], _i32),
    "evr_op_surface_gradient": ([_P, _P, _P, _P, _P, _P], _i32),
    "evr_op_surface_gradient_adjoint": ([_P, _P, _P, _P, _P, _P], _i32),
    "evr_op_prox_data": ([_P, _P, _P, _P, _d, _d, _d, _d, _P], _i32),
    "evr_op_prox_dual": ([_P, _P, _P, _P], _i32),
    "evr_op_energy": ([_P, _P, _P, _P, _P, _P, _P, _d, _P], _i32),
    "evr_op_pd_solve": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _i32),
    "evr_op_to_gray": ([_P, _P, _d, _d, _P], _i32),
    "evr_op_rof_solve": ([_P, _P, _P, _P, _P, _P, _d, _i32, _P], _i32),
    "evr_op_l1_solve": ([_P, _P, _P, _P, _P, _P, _d, _i32, _P], _i32),
    "evr_op_tgv_solve": ([_P, _P, _P, _P, _P, _P, _d, _d, _d, _i32, _d, _d, _i32, _P, _P], _i32),
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return sorted(_SIGNATURES)


def load(path=None):
    """Load libevr.so and declare every C ABI signature (no device work)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ImportError(
                f"CUDA library {p} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)"
            )
        lib = ctypes.CDLL(p)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def ptr(a):
    """Data pointer of a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


def check(ctx, rc, what=""):
    if rc == EVR_OK:
        return
    msg = lib().evr_last_error(ctx).decode() if ctx else "no context"
    if rc in (EVR_ERR_INVALID,):
        raise ValueError(msg)
    if rc == EVR_ERR_RANGE:
        raise IndexError(msg)
    raise EvrError(rc, f"{what}: {msg}" if what else msg)


def device_count():
    n = ctypes.c_int(0)
    rc = lib().evr_device_count(ctypes.byref(n))
    return n.value if rc == EVR_OK else 0


class _PinnedBlock:
    """A page-locked host block (evr_host_alloc); goes back to the pool when
    the last array viewing it is collected."""

    __slots__ = ("addr", "nbytes")

    def __init__(self, addr, nbytes):
        self.addr, self.nbytes = addr, nbytes

    def __del__(self):
        try:
            with _pinned_lock:
                _pinned_free.setdefault(self.nbytes, []).append(self.addr)
        except Exception:  # interpreter shutdown
            pass


_pinned_free: dict = {}
_pinned_lock = threading.Lock()


def pinned_reserve(shape, count, dtype=np.float64):
    """Grow the pinned pool to at least `count` free blocks of this size
    (cudaHostAlloc is milliseconds: keep it out of a stream's hot loop)."""
    nbytes = max(1, int(np.prod(shape)) * np.dtype(dtype).itemsize)
    with _pinned_lock:
        have = len(_pinned_free.get(nbytes, ()))
    for _ in range(count - have):
        out = ctypes.c_void_p()
        if lib().evr_host_alloc(nbytes, ctypes.byref(out)) != 0:
            raise MemoryError(f"evr_host_alloc({nbytes}) failed")
        with _pinned_lock:
            _pinned_free.setdefault(nbytes, []).append(out.value)


def pinned_empty(shape, dtype=np.float64):
    """np.empty in page-locked host memory, from a size-keyed pool, so frame
    downloads run at full link speed without a staging copy."""
    dtype = np.dtype(dtype)
    nbytes = max(1, int(np.prod(shape)) * dtype.itemsize)
    with _pinned_lock:
        addrs = _pinned_free.get(nbytes)
        addr = addrs.pop() if addrs else None
    if addr is None:
        out = ctypes.c_void_p()
        rc = lib().evr_host_alloc(nbytes, ctypes.byref(out))
        if rc != 0:
            raise MemoryError(f"evr_host_alloc({nbytes}) failed ({rc})")
        addr = out.value
    buf = (ctypes.c_char * nbytes).from_address(addr)
    buf._block = _PinnedBlock(addr, nbytes)  # lives as long as any view of buf
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


class Context:
    """Owns one evr_ctx (one sensor shape, one device, one precision)."""

    def __init__(self, height, width, precision=PREC_F64, device=None):
        if device is None:
            device = int(os.environ.get("EVR_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        L = lib()
        if device_count() < 1:
            raise RuntimeError("no CUDA device visible: the evr hot path runs on the GPU only")
        h = ctypes.c_void_p()
        rc = L.evr_create(ctypes.byref(h), int(device), int(height), int(width), int(precision))
        if rc != EVR_OK:
            raise EvrError(rc, f"evr_create({height}x{width}, device {device}) failed")
        self._h = h
        self.height, self.width = int(height), int(width)
        self.precision = int(precision)
        self.device = int(device)
        self._cfg_key = None

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().evr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name, *args):
        rc = getattr(lib(), name)(self._h, *args)
        check(self._h, rc, name)

    def set_config(self, cfg: Config):
        key = bytes(cfg)
        if key != self._cfg_key:
            self.call("evr_set_config", ctypes.byref(cfg))
            self._cfg_key = key

    def engine(self):
        e = ctypes.c_int(0)
        self.call("evr_active_engine", ctypes.byref(e))
        return ENGINE_NAMES.get(e.value, str(e.value))

    def engine_detail(self):
        buf = ctypes.create_string_buffer(256)
        self.call("evr_engine_detail", buf, len(buf))
        return buf.value.decode()

    def launch_count(self):
        return int(lib().evr_launch_count(self._h))
