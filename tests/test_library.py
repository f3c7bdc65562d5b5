"""The C ABI: libdrk.so loads on a CPU-only host, exports every function declared in
include/drk.h, and validates arguments before touching a device."""

import ctypes
import os
import re

import pytest

from paper_2406_00158_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "drk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(drk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for f in ("drk_dot", "drk_reduce", "drk_scan", "drk_triad", "drk_copy", "drk_fill", "drk_black_scholes",
              "drk_generate", "drk_jit_compile", "drk_jit_launch"):
        assert f in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_the_header():
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_host_side_queries_without_gpu():
    lib = _lib.load()
    assert lib.drk_version() >= 1
    assert lib.drk_reduce_scratch_bytes() > 0
    assert lib.drk_scan_scratch_bytes(_lib.F32, _lib.ADD, 1 << 30) > (1 << 30) // 5120 * 16
    assert lib.drk_acc_dtype(_lib.F32, _lib.ADD) == _lib.F64
    assert lib.drk_acc_dtype(_lib.I32, _lib.ADD) == _lib.I64
    assert lib.drk_acc_dtype(_lib.I32, _lib.MIN) == _lib.I32
    assert lib.drk_acc_dtype(_lib.F64, _lib.MUL) == _lib.F64


def test_argument_errors_before_any_launch():
    lib = _lib.load()
    rc = lib.drk_copy(_lib.F32, None, None, 16, 0, None)
    assert rc == _lib.E_ARG and "null" in _lib.last_error()
    rc = lib.drk_scan(_lib.F32, _lib.ADD, 1, 1, 1, 4, None, None, None, None, None, None, 0, 0, None)
    assert rc == _lib.E_ARG and "init" in _lib.last_error()
    rc = lib.drk_dot(7, 1, 1, 4, 1, 1, 0, None)
    assert rc == _lib.E_DTYPE
    with pytest.raises(_lib.DrkError):
        _lib.call("drk_reduce", _lib.F32, _lib.ADD, None, 4, None, None, 0, None)


def test_zero_length_is_a_no_op():
    lib = _lib.load()
    assert lib.drk_triad(_lib.F32, None, None, None, 0, _lib.scalar_buffer(3.0, "float32"), 0, None) == 0


def test_device_count_is_zero_or_more():
    assert _lib.device_count() >= 0


def test_round2_entries_validate_before_any_launch():
    """The round-2 entries (multi-device / fused reduce, device fold, communicator, graphs,
    completion words, Black-Scholes tiers) reject bad arguments before touching a device."""
    lib = _lib.load()
    vp = ctypes.c_void_p
    one = (ctypes.c_int * 1)(1)
    assert lib.drk_reduce_multi(5, _lib.F32, _lib.ADD, 1, one, (vp * 1)(), one, (vp * 1)(), None,
                                (ctypes.c_int64 * 1)(4), (vp * 1)(), None, 1, (vp * 1)()) == _lib.E_ARG
    assert "kind" in _lib.last_error()
    assert lib.drk_reduce_multi(0, _lib.F32, _lib.ADD, 1, one, (vp * 1)(), (ctypes.c_int * 1)(17), (vp * 1)(),
                                None, (ctypes.c_int64 * 1)(4), (vp * 1)(1), None, 1, (vp * 1)(1)) == _lib.E_ARG
    assert lib.drk_reduce_fused(0, _lib.F32, _lib.ADD, 1, one, (vp * 1)(), one, (vp * 1)(), None,
                                (ctypes.c_int64 * 1)(4), (ctypes.c_int * 1)(0), None, None, None, None, None, 1,
                                (vp * 1)()) == _lib.E_ARG
    assert lib.drk_reduce_fold(_lib.F32, _lib.ADD, None, _lib.FOLD_MAX + 1, None, None, None, 0, None) == _lib.E_ARG
    h = ctypes.c_void_p()
    assert lib.drk_comm_create(0, None, ctypes.byref(h)) == _lib.E_ARG
    assert lib.drk_comm_create(2, (ctypes.c_int * 2)(0, 0), ctypes.byref(h)) == _lib.E_ARG
    assert "duplicate" in _lib.last_error()
    assert lib.drk_graph_launch(None, 0, None) == _lib.E_ARG
    assert lib.drk_graph_destroy(None) == 0
    assert lib.drk_wait_flags(None, 1, 1, 0, None) == _lib.E_ARG
    assert lib.drk_wait_flags(None, 0, 1, 0, None) == 0
    assert lib.drk_black_scholes_ex(_lib.F32, 4, 1, 1, 1, 1, 1, 1, 16, 0, None) == _lib.E_ARG
    assert "flags" in _lib.last_error()
    assert lib.drk_partial_dtype(_lib.F32, _lib.ADD) == _lib.F32
    assert lib.drk_partial_dtype(_lib.I32, _lib.ADD) == _lib.I64
    assert lib.drk_partial_dtype(_lib.I32, _lib.MIN) == _lib.I32


def test_ipc_entries_validate_before_any_launch():
    lib = _lib.load()
    vp = ctypes.c_void_p
    p = vp()
    assert lib.drk_ipc_alloc(0, 0, ctypes.byref(p)) == _lib.E_ARG
    assert lib.drk_ipc_handle(None, None) == _lib.E_ARG
    assert lib.drk_ipc_open(None, 0, ctypes.byref(p)) == _lib.E_ARG
    assert lib.drk_ipc_close(None) == 0 and lib.drk_ipc_free(None) == 0
    assert lib.drk_mailbox_allgather(None, None, 2, 0, None, 1, 1, None, None, 0, None) == _lib.E_ARG
    boxes = (vp * 2)(1, 1)
    assert lib.drk_mailbox_allgather(1, boxes, 2, 2, 1, 1, 1, 1, 1, 0, None) == _lib.E_ARG
    assert "range" in _lib.last_error()
