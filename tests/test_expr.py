"""Tracer dtype rules against numpy itself, traceability errors, AOT catalogue matching,
and NVRTC compilation of generated kernels (compile only: no GPU needed)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import _lib, codegen, expr, kernels, views
from paper_2406_00158_b200 import bench as B

DTYPES = [np.float32, np.float64, np.int32, np.int64]
OPS = [
    lambda a, b: a + b, lambda a, b: a - b, lambda a, b: a * b, lambda a, b: a / b,
    lambda a, b: np.maximum(a, b), lambda a, b: a > b, lambda a, b: np.where(a > b, a, b),
]
SCALARS = [2, 3.5, True, np.float32(1.5), np.int64(3)]


def sym(dt, slot=0):
    return expr.Sym(expr.leaf(slot, dt))


@given(st.sampled_from(DTYPES), st.sampled_from(DTYPES), st.integers(0, len(OPS) - 1))
@settings(max_examples=120)
def test_binary_dtype_matches_numpy(da, db, k):
    op = OPS[k]
    a, b = np.ones(3, dtype=da), np.ones(3, dtype=db)
    want = np.asarray(op(a, b)).dtype
    got = op(sym(da), sym(db, 1))
    assert got.dtype == want


@given(st.sampled_from(DTYPES), st.sampled_from(SCALARS), st.integers(0, 5))
@settings(max_examples=120)
def test_weak_scalar_dtype_matches_numpy(da, s, k):
    op = OPS[k]
    a = np.ones(3, dtype=da)
    with np.errstate(all="ignore"):
        want = np.asarray(op(a, s)).dtype
        got = op(sym(da), s)
    assert got.dtype == want


@pytest.mark.parametrize("fn,dt", [
    (np.sqrt, np.float32), (np.sqrt, np.int32), (np.exp, np.float64), (np.floor_divide, np.int64),
    (np.abs, np.int32), (np.square, np.float32), (np.negative, np.int64),
])
def test_ufunc_dtype(fn, dt):
    a = np.ones(3, dtype=dt)
    x = sym(dt)
    if fn is np.floor_divide:
        assert fn(x, 3).dtype == fn(a, 3).dtype
    else:
        assert fn(x).dtype == fn(a).dtype


def test_triad_traces_to_two_roundings():
    node = expr.trace(lambda t: (t[1] + 3.0 * t[2], None, None),
                      (expr.leaf(0, np.float32), expr.leaf(1, np.float32), expr.leaf(2, np.float32)))
    assert node[0].op == "add" and node[0].dtype == np.float32
    assert node[0].args[1].op == "multiply" and node[0].args[1].args[0].value == 3.0


@pytest.mark.parametrize("fn", [
    lambda x: x if x > 0 else -x,
    lambda x: float(x),
    lambda x: np.asarray(x),
    lambda x: [v for v in x],
    lambda x: x[0],
])
def test_untraceable_functions_raise(fn):
    with pytest.raises(expr.TraceError):
        expr.trace(fn, expr.leaf(0, np.float64))


def test_trace_cache_respects_closures():
    out = []
    for alpha in (2.0, 3.0):
        f = lambda x, a=alpha: x * a  # noqa: E731
        g = (lambda a: (lambda x: x * a))(alpha)
        n1 = expr.trace_cached(f, expr.leaf(0, np.float64), ("k",))
        n2 = expr.trace_cached(g, expr.leaf(0, np.float64), ("k",))
        out.append((n1.args[1].value, n2.args[1].value))
    assert out == [(2.0, 2.0), (3.0, 3.0)]


def _lowered(meta_rt, dtypes, n=16):
    vecs = [sr.DistributedVector(meta_rt[1], n, dtype=d) for d in dtypes]
    z = views.zip(*vecs)
    return views.lower(z.segments()[0])


@pytest.mark.parametrize("fn,kernel", [
    (lambda t: (t[1] + 3.0 * t[2], None, None), "drk_triad"),
    (lambda t: (3.0 * t[2] + t[1], None, None), "drk_triad"),
    (lambda t: (t[1] * 2.0, None, None), "drk_scale"),
    (lambda t: (t[1] + t[2], None, None), "drk_add"),
    (lambda t: (t[1], None, None), "drk_copy"),
    (lambda t: (0.5, None, None), "drk_fill"),
    (lambda t: (np.sqrt(t[1]), None, None), None),
])
def test_catalogue_matching(meta_rt, fn, kernel):
    lw = _lowered(meta_rt, [np.float32] * 3)
    res = expr.trace(fn, lw.value)
    m = kernels.match_map(res[0], lw.leaves, np.float32)
    assert (m[0] if m else None) == kernel


def test_black_scholes_catalogue(meta_rt):
    lw = _lowered(meta_rt, [np.float32] * 6)
    res = expr.trace(lambda t: (B.black_scholes_call(t[1], t[2], t[3], t[4], t[5]),) + (None,) * 5, lw.value)
    name, args = kernels.match_map(res[0], lw.leaves, np.float32)
    assert name == "drk_black_scholes_ex" and args(0, 1, [0] * 6, None)[1] == 0  # fp64 internal
    res = expr.trace(lambda t: (B.black_scholes_call_fast(t[1], t[2], t[3], t[4], t[5]),) + (None,) * 5, lw.value)
    name, args = kernels.match_map(res[0], lw.leaves, np.float32)
    assert name == "drk_black_scholes_ex" and args(0, 1, [0] * 6, None)[1] == _lib.BS_FAST


def test_codegen_compiles_map_reduce_scan(meta_rt):
    lw = _lowered(meta_rt, [np.float32, np.float64, np.int32])
    res = expr.trace(lambda t: (np.where(t[0] > 0.5, np.sqrt(t[1]), t[2] // 3), t[2] % 7 + 1, None), lw.value)
    writes = [(lw.target[0], res[0]), (lw.target[1], res[1])]
    src = codegen._map_source(writes, lw.leaves)[0]
    assert len(codegen.cubin_for(src, "map.cu")) > 1000
    op = sr.BinaryOp(lambda a, b: a + b + 1)
    opname, opsrc = codegen._op_struct(None, op, np.dtype(np.int64))
    assert "OpC" in opsrc
    mod_src = f'#include "drk_device.cuh"\n{opsrc}\nextern "C" __global__ void k(const drk::ScanParams<long long, ' \
              f'const long long*> p) {{ drk::scan_kernel_body<drk::PlainLoad<long long>, long long, OpC, 256, 10, 1>(p); }}'
    assert len(codegen.cubin_for(mod_src, "scan.cu")) > 1000


def test_match_binary():
    assert codegen.match_binary(lambda a, b: a + b, np.dtype(np.int64)) == 0
    assert codegen.match_binary(lambda a, b: b * a, np.dtype(np.float64)) == 1
    assert codegen.match_binary(lambda a, b: np.minimum(a, b), np.dtype(np.float64)) == 2
    assert codegen.match_binary(lambda a, b: a + b + 1, np.dtype(np.int64)) is None


# ----------------------------------------------------------------------------------------
# trace cache: a cached trace must never outlive the state it was traced from


class _Params:
    alpha = 2.0


def _consts(node):
    return sorted((n.value, n.dtype.str) for n in node.walk() if n.op == "const")


def test_trace_cache_sees_attribute_mutation(meta_rt):
    p = _Params()
    x = sr.DistributedVector(meta_rt[2], 10, dtype=np.float64)
    v = views.transform(x, lambda t: t * p.alpha)
    seg = v.segments()[0]
    assert _consts(views.lower(seg).value) == [(2.0, "<f8")]
    p.alpha = 3.0
    assert _consts(views.lower(v.segments()[0]).value) == [(3.0, "<f8")]
    assert expr._fn_key(lambda t: t * p.alpha) is None  # reaches an object attribute


def test_trace_cache_keys_closure_by_type_and_value():
    leaf = expr.leaf(0, np.int32)
    out = []
    for a in (2, 2.0, np.float64(2.0), 0.0, -0.0):
        fn = (lambda a_: (lambda t: t * a_))(a)
        node = expr.trace_cached(fn, leaf, ("k",))
        out.append((node.dtype.str, _consts(node)))
    assert out[0][0] == "<i4"          # int32 * 2 stays int32
    assert out[1][0] == "<f8"          # int32 * 2.0 -> float64 (NEP 50), not the cached int32 trace
    assert out[2][0] == "<f8"
    assert out[3][1] != out[4][1] or repr(out[3][1]) != repr(out[4][1])


def test_trace_cache_follows_globals_and_helpers():
    g = {"np": np, "K": 2}
    exec("def helper(t):\n    return t * K\n\ndef f(t):\n    return helper(t) + 1\n", g)
    leaf = expr.leaf(0, np.float64)
    a = expr.trace_cached(g["f"], leaf, ("g",))
    g["K"] = 5
    b = expr.trace_cached(g["f"], leaf, ("g",))
    assert (5, "<f8") not in [(c[0], c[1]) for c in _consts(a)]
    assert any(c[0] == 5 for c in _consts(b))
    g["state"] = [1]
    exec("def h(t):\n    return t * state[0]\n", g)
    assert expr._fn_key(g["h"]) is None  # a list can change under the cache


def test_trace_cache_keys_stay_hashable_for_numpy_functions():
    fn = lambda t: np.sqrt(t) * np.float32(1.5)  # noqa: E731
    assert expr._fn_key(fn) is not None


# ----------------------------------------------------------------------------------------
# fused view scans (compile only; the GPU parity tests run them)


def _scan_view_source(monkeypatch, node, leaves, T, opcode, combiner=None):
    got = {}

    def fake_compile(src, name):
        got["src"] = src
        return codegen.Module(None)

    monkeypatch.setattr(codegen, "compile_module", fake_compile)
    codegen._SCAN_VIEW_PLANS.clear()
    view = kernels.ScanView(node, leaves, [0] * len(leaves), 100)
    mod, words, geom = codegen.scan_view_plan(view, T, opcode, combiner)
    return got["src"], words, geom


@pytest.mark.parametrize("T", [np.float32, np.int64])
def test_scan_view_nvrtc_compiles(meta_rt, monkeypatch, T):
    lw = _lowered(meta_rt, [T, np.float64])
    node = expr.cast(expr.trace(lambda t: np.sqrt(t[0] * t[1] + 1.5) * 2, lw.value), T)
    src, words, geom = _scan_view_source(monkeypatch, node, lw.leaves, np.dtype(T), 0)
    assert "drk_scan_l2_l" in src and "drk_scan_1p" in src
    same = np.dtype(T).itemsize == 8  # the float64 leaf is staged with a same-size value only
    assert len(words) <= 16 and geom[1] == (2 if same else 0)
    assert len(codegen.cubin_for(src, "scan_view.cu")) > 1000


def test_scan_view_nvrtc_staged_single_leaf(meta_rt, monkeypatch):
    lw = _lowered(meta_rt, [np.float32, np.float32])
    node = expr.trace(lambda t: np.where(t[0] > 0.5, t[0] * 3.0, -t[0]).astype(np.float32), lw.value)
    src, words, geom = _scan_view_source(monkeypatch, node, lw.leaves, np.dtype(np.float32), 0)
    assert geom == (20, 1, 4, 8, 20) and "compute" in src
    assert len(codegen.cubin_for(src, "scan_view.cu")) > 1000


def test_scan_view_custom_combiner_compiles(meta_rt, monkeypatch):
    lw = _lowered(meta_rt, [np.float64, np.float64])
    node = expr.trace(lambda t: t[0] * 0.5, lw.value)
    op = sr.BinaryOp(lambda a, b: np.maximum(a, b) + 0.25 * b)
    src, words, _ = _scan_view_source(monkeypatch, node, lw.leaves, np.dtype(np.float64), None, op)
    assert "OpC" in src
    assert len(codegen.cubin_for(src, "scan_view.cu")) > 1000


def test_scan_view_catalogue(meta_rt):
    lw = _lowered(meta_rt, [np.float32, np.float32])
    f32 = np.dtype(np.float32)
    prod = expr.trace(lambda t: t[0] * t[1], lw.value)
    assert kernels.match_scan_view(prod, lw.leaves, 0, f32)[0] == 1
    aff = expr.trace(lambda t: 2.5 * t[0] + 1.0, lw.value)
    m = kernels.match_scan_view(aff, lw.leaves, 0, f32)
    assert m[0] == 2 and m[1] == ("leaf", 0) and m[4] == 1
    sub = expr.trace(lambda t: t[1] - 3.0, lw.value)
    m = kernels.match_scan_view(sub, lw.leaves, 0, f32)
    assert m[0] == 2 and codegen.const_bits(-3.0, f32) == m[3]
    assert kernels.match_scan_view(prod, lw.leaves, 1, f32) is None  # multiply-scan: NVRTC
    li = _lowered(meta_rt, [np.int32, np.int32])
    mixed = expr.trace(lambda t: t[0] * 2.5, li.value)  # int32 * 2.5 -> float64
    assert kernels.match_scan_view(mixed, li.leaves, 0, f32) is None


def test_trace_cache_sees_globals_of_nested_functions():
    g = {"np": np, "K": 2}
    exec("def f(t):\n    return (lambda u: u * K)(t)\n", g)
    leaf = expr.leaf(0, np.float64)
    a = expr.trace_cached(g["f"], leaf, ("n",))
    g["K"] = 7
    b = expr.trace_cached(g["f"], leaf, ("n",))
    assert any(c[0] == 2 for c in _consts(a)) and any(c[0] == 7 for c in _consts(b))
