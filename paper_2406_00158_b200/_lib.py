"""ctypes binding of libdrk.so, the C ABI declared in include/drk.h.

There is deliberately no fallback: if the library is missing or fails to load, importing
anything that launches work raises ``DrkLibraryError`` with the reason.  The package is
a device runtime; computing on the host instead would silently change what is measured.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DRK_LIB") or os.path.join(_HERE, "libdrk.so")  # DRK_LIB: kernel experiments
CSRC_DIR = os.path.join(_HERE, "csrc")

# dtype codes (include/drk.h)
F32, F64, I32, I64 = 0, 1, 2, 3
ADD, MUL, MIN, MAX = 0, 1, 2, 3
GEN_UNIFORM, GEN_MOD = 0, 1
E_ARG, E_DTYPE, E_SCRATCH, E_JIT, E_COMM = 1001, 1002, 1003, 1004, 1005

DTYPE_CODE = {
    np.dtype(np.float32): F32,
    np.dtype(np.float64): F64,
    np.dtype(np.int32): I32,
    np.dtype(np.int64): I64,
}
CODE_DTYPE = {v: k for k, v in DTYPE_CODE.items()}


class DrkLibraryError(RuntimeError):
    """libdrk.so could not be loaded (not built, or built for another platform)."""


class DrkError(RuntimeError):
    """A libdrk call failed; ``code`` is the cudaError_t or DRK_E_* value."""

    def __init__(self, code: int, func: str, msg: str):
        self.code = code
        self.func = func
        super().__init__(f"{func} failed ({code}): {msg}")


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_sz = ctypes.c_size_t
_dbl = ctypes.c_double
_cp = ctypes.c_char_p

# name -> (restype, argtypes); must cover every function declared in include/drk.h
SIGNATURES = {
    "drk_version": (_int, []),
    "drk_last_error": (_cp, []),
    "drk_device_count": (_int, [ctypes.POINTER(_int)]),
    "drk_memcpy_async": (_int, [_vp, _vp, _sz, _int, _vp]),
    "drk_memset_async": (_int, [_vp, _int, _sz, _int, _vp]),
    "drk_readback": (_int, [_vp, _vp, _sz, _int, _vp]),
    "drk_mapped_ptr": (_int, [_vp, ctypes.POINTER(_vp)]),
    "drk_stream_synchronize": (_int, [_int, _vp]),
    "drk_enable_peer_access": (_int, [_int, _int]),
    "drk_copy": (_int, [_int, _vp, _vp, _i64, _int, _vp]),
    "drk_fill": (_int, [_int, _vp, _i64, _vp, _int, _vp]),
    "drk_iota": (_int, [_int, _vp, _i64, _i64, _int, _vp]),
    "drk_scale": (_int, [_int, _vp, _vp, _i64, _vp, _int, _vp]),
    "drk_add": (_int, [_int, _vp, _vp, _vp, _i64, _int, _vp]),
    "drk_triad": (_int, [_int, _vp, _vp, _vp, _i64, _vp, _int, _vp]),
    "drk_black_scholes": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "drk_black_scholes_ex": (_int, [_int, _int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "drk_generate": (_int, [_int, _vp, _i64, _u64, _u64, _int, _dbl, _dbl, _int, _vp]),
    "drk_reduce_scratch_bytes": (_sz, []),
    "drk_acc_dtype": (_int, [_int, _int]),
    "drk_reduce": (_int, [_int, _int, _vp, _i64, _vp, _vp, _int, _vp]),
    "drk_dot": (_int, [_int, _vp, _vp, _i64, _vp, _vp, _int, _vp]),
    "drk_scan_scratch_bytes": (_sz, [_int, _int, _i64]),
    "drk_scan": (_int, [_int, _int, _int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "drk_reduce_batch": (_int, [_int, _int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), _vp, _vp, _int, _vp]),
    "drk_reduce_batch_ex": (_int, [_int, _int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), _vp, _vp, _u64, _vp,
                                   _int, _vp]),
    "drk_dot_batch_ex": (_int, [_int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), _vp, _vp,
                                _u64, _vp, _int, _vp]),
    "drk_wait_flags": (_int, [_vp, _int, _u64, _int, _vp]),
    "drk_reduce_fused": (_int, [_int, _int, _int, _int, ctypes.POINTER(_int), ctypes.POINTER(_vp), ctypes.POINTER(_int),
                                ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_int),
                                _vp, _vp, _vp, _vp, _vp, _u64, ctypes.POINTER(_vp)]),
    "drk_ipc_alloc": (_int, [_sz, _int, ctypes.POINTER(_vp)]),
    "drk_ipc_free": (_int, [_vp]),
    "drk_ipc_handle": (_int, [_vp, _vp]),
    "drk_ipc_open": (_int, [_vp, _int, ctypes.POINTER(_vp)]),
    "drk_ipc_close": (_int, [_vp]),
    "drk_mailbox_allgather": (_int, [_vp, ctypes.POINTER(_vp), _int, _int, _vp, _u64, _u64, _vp, _vp, _int, _vp]),
    "drk_graph_begin": (_int, [_int, _vp]),
    "drk_graph_end": (_int, [_int, _vp, ctypes.POINTER(_vp)]),
    "drk_graph_launch": (_int, [_vp, _int, _vp]),
    "drk_graph_destroy": (_int, [_vp]),
    "drk_reduce_multi": (_int, [_int, _int, _int, _int, ctypes.POINTER(_int), ctypes.POINTER(_vp), ctypes.POINTER(_int),
                                ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_vp),
                                ctypes.POINTER(_vp), _u64, ctypes.POINTER(_vp)]),
    "drk_dot_batch": (_int, [_int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), _vp, _vp,
                             _int, _vp]),
    "drk_scan_batch_scratch_bytes": (_sz, [_int, _int, _int, ctypes.POINTER(_i64)]),
    "drk_scan_batch": (_int, [_int, _int, _int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                              _vp, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "drk_scan_ex": (_int, [_int, _int, _int, _int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "drk_scan_view": (_int, [_int, _int, _int, _int, ctypes.POINTER(_u64), _int, _int, _vp, _i64, _vp, _vp, _vp, _vp,
                             _vp, _vp, _sz, _int, _vp]),
    "drk_scan_view_ex": (_int, [_int, _int, _int, _int, _int, ctypes.POINTER(_u64), _int, _int, _vp, _i64, _vp, _vp,
                                _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "drk_jit_scan_view": (_int, [_vp, _int, _int, _int, _int, _int, _int, _int, _int, _int, ctypes.POINTER(_u64),
                                 _int, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _int, _vp]),
    "drk_carry_fold": (_int, [_int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _int, _vp, _vp, _vp, _int,
                              _vp]),
    "drk_partial_dtype": (_int, [_int, _int]),
    "drk_reduce_fold": (_int, [_int, _int, ctypes.POINTER(_vp), _int, _vp, _vp, _vp, _int, _vp]),
    "drk_comm_available": (_int, []),
    "drk_comm_version": (_int, []),
    "drk_comm_create": (_int, [_int, ctypes.POINTER(_int), ctypes.POINTER(_vp)]),
    "drk_comm_destroy": (_int, [_vp]),
    "drk_comm_allgather": (_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, ctypes.POINTER(_vp)]),
    "drk_comm_reduce": (_int, [_vp, _int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, ctypes.POINTER(_int),
                               _int, _vp, ctypes.POINTER(_vp), _vp, ctypes.POINTER(_vp)]),
    "drk_sort_keys": (_int, [_int, _vp, _vp, _i64, _vp, ctypes.POINTER(_sz), _int, _vp]),
    "drk_sort_pairs": (_int, [_int, _vp, _vp, _vp, _vp, _i64, _vp, ctypes.POINTER(_sz), _int, _vp]),
    "drk_gather": (_int, [_int, _vp, _vp, _vp, _i64, _int, _vp]),
    "drk_sort_bounds": (_int, [_int, _vp, _i64, _vp, _int, _vp, _int, _vp]),
    "drk_tune": (_int, [_cp, _int]),
    "drk_scan_set_trace": (_int, [_vp]),
    "drk_launch_count": (_i64, []),
    "drk_note_launch": (_i64, []),
    "drk_jit_compile": (_int, [_cp, _cp, _cp, ctypes.POINTER(_vp), ctypes.c_char_p, _sz]),
    "drk_jit_cubin": (_int, [_cp, _cp, _cp, _vp, ctypes.POINTER(_sz), ctypes.c_char_p, _sz]),
    "drk_jit_load": (_int, [_vp, ctypes.POINTER(_vp)]),
    "drk_jit_launch": (_int, [_vp, _cp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp, _sz, _int, _vp]),
    "drk_jit_occupancy": (_int, [_vp, _cp, ctypes.c_uint, ctypes.c_uint, _int,
                                 ctypes.POINTER(_int), ctypes.POINTER(_int)]),
    "drk_jit_last_error": (_cp, []),
    "drk_jit_scan_scratch_bytes": (_sz, [_i64, _int]),
    "drk_jit_scan": (_int, [_vp, _cp, _int, _int, _int, _int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                            _int, _vp]),
}

_lock = threading.Lock()
_lib = None
_load_error = None


def load():
    """The loaded library; raises DrkLibraryError if it cannot be loaded."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            _load_error = (
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2406_00158_b200/csrc`"
            )
            raise DrkLibraryError(_load_error)
        try:
            lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        except OSError as exc:  # pragma: no cover - depends on the host
            _load_error = f"cannot load {LIB_PATH}: {exc}"
            raise DrkLibraryError(_load_error) from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        # DRK_TUNE="name=value,...": launch-parameter overrides for kernel experiments
        for kv in filter(None, os.environ.get("DRK_TUNE", "").split(",")):
            k, v = kv.split("=")
            lib.drk_tune(k.strip().encode(), int(v))
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().drk_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, func: str) -> None:
    if rc != 0:
        lib = load()
        msg = lib.drk_last_error() or b""
        if func.startswith("drk_jit"):
            msg = (lib.drk_jit_last_error() or b"") or msg
        raise DrkError(rc, func, msg.decode(errors="replace"))


_FUNCS = {}


def fn(name: str):
    """The bound entry point `name` (cached): hot paths call it directly and check rc."""
    f = _FUNCS.get(name)
    if f is None:
        f = _FUNCS[name] = getattr(load(), name)
    return f


def call(name: str, *args) -> None:
    """Call an int-returning entry point and raise DrkError on failure."""
    fn = _FUNCS.get(name)
    if fn is None:
        fn = _FUNCS[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        check(rc, name)


def device_count() -> int:
    n = _int(0)
    call("drk_device_count", ctypes.byref(n))
    return n.value


def launch_count() -> int:
    return int(load().drk_launch_count())


CARRY_MAX = 64  # drk.h DRK_CARRY_MAX: predecessors one drk_carry_fold call folds
SCAN_CHAINED = 1  # drk.h DRK_SCAN_CHAINED
SCAN_SEGS = 16  # drk.h DRK_SCAN_SEGS
RED_SEGS = 16  # drk.h DRK_RED_SEGS
FOLD_MAX = 64  # drk.h DRK_FOLD_MAX: partials one drk_reduce_fold folds
COMM_MAX_DEV = 16  # drk.h DRK_COMM_MAX_DEV
COMM_MAX_RANKS = 32  # drk.h DRK_COMM_MAX_RANKS
VIEW_PRODUCT, VIEW_AFFINE = 1, 2  # drk.h DRK_VIEW_*
BS_FAST = 1  # drk.h DRK_BS_FAST
JIT_WORDS = 16  # drk_device.cuh DRK_JIT_WORDS: 8-byte words of a fused scan loader

# sort / gather / bounds also take unsigned keys (drk.h DRK_U32 / DRK_U64)
SORT_DTYPE_CODE = {**DTYPE_CODE, np.dtype(np.uint32): 4, np.dtype(np.uint64): 5}


def sort_dtype_code(dtype) -> int:
    try:
        return SORT_DTYPE_CODE[np.dtype(dtype)]
    except KeyError:
        raise TypeError(f"dtype {np.dtype(dtype)} cannot be sorted on the device "
                        "(supported: float32, float64, int32, int64, uint32, uint64)") from None


def dtype_code(dtype) -> int:
    try:
        return DTYPE_CODE[np.dtype(dtype)]
    except KeyError:
        raise TypeError(
            f"dtype {np.dtype(dtype)} has no device kernels (supported: float32, float64, int32, int64)"
        ) from None


_ACC = {}


def acc_dtype(dtype, op: int) -> np.dtype:
    """Accumulator dtype of the device kernels for (dtype, op) (cached drk_acc_dtype)."""
    key = (np.dtype(dtype), op)
    r = _ACC.get(key)
    if r is None:
        r = _ACC[key] = CODE_DTYPE[load().drk_acc_dtype(dtype_code(dtype), op)]
    return r


def scalar_buffer(value, dtype) -> ctypes.Array:
    """A host buffer holding `value` converted to `dtype` (for by-pointer scalars)."""
    arr = np.asarray([value]).astype(np.dtype(dtype), copy=False)
    buf = (ctypes.c_char * arr.nbytes).from_buffer_copy(arr.tobytes())
    return buf
