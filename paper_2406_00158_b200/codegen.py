"""CUDA code generation for traced expressions outside the AOT kernel catalogue.

A lowered segment (views.lower) is a list of leaves plus an expression DAG (expr.Node).
When kernels.match_map / run_reduce find no hand-written libdrk kernel for it, this
module writes a small functor in CUDA C++ — loads of the leaves, the expression in SSA
form with numpy's loop dtypes and rounding (no FMA contraction: NVRTC runs with
-fmad=false and adds/multiplies use the _rn intrinsics), stores of the outputs — and
instantiates the same map / reduce / scan templates the AOT library uses
(csrc/drk_device.cuh).  NVRTC compiles it for sm_100a once; modules are cached in memory
by the expression's *shape* (constants are kernel parameters, so `x * 2.5` and `x * 3.0`
share one kernel) and cubins on disk under _jitcache/.

This is the path that keeps arbitrary user lambdas on the device — the reference
evaluates them with numpy on the host (views.py:164-181, algorithms.py:101-111, 153-162,
216-231).  Nothing here ever evaluates an element on the host.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import threading

import numpy as np

from . import _lib, expr

_HERE = os.path.dirname(os.path.abspath(__file__))
CACHE_DIR = os.environ.get("DRK_JIT_CACHE", os.path.join(_HERE, "_jitcache"))
BLOCK = 256

_CTYPE = {
    "f4": "float", "f8": "double", "i4": "int", "i8": "long long", "u4": "unsigned int",
    "u8": "unsigned long long", "b1": "bool", "i2": "short", "u2": "unsigned short", "i1": "signed char",
    "u1": "unsigned char",
}


class JitError(TypeError):
    """An expression could not be compiled to a device kernel."""


def ctype(dt) -> str:
    dt = np.dtype(dt)
    key = dt.kind + str(dt.itemsize)
    if key not in _CTYPE:
        raise JitError(f"dtype {dt} has no device representation")
    return _CTYPE[key]


# ----------------------------------------------------------------------------------------
# module cache


class Module:
    def __init__(self, handle):
        self.handle = handle


_lock = threading.Lock()
_modules: dict = {}


_HEADER_DIGEST = None


def _header_digest() -> bytes:
    """Hash of the device header the generated sources include: a cubin cached on disk is
    reused only when both the source and drk_device.cuh are unchanged."""
    global _HEADER_DIGEST
    if _HEADER_DIGEST is None:
        h = hashlib.sha256()
        for fn in ("drk_device.cuh", "drk_erf_table.inc", "drk_log_table.inc"):
            with open(os.path.join(_lib.CSRC_DIR, fn), "rb") as fh:
                h.update(fh.read())
        _HEADER_DIGEST = h.digest()
    return _HEADER_DIGEST


def compile_module(source: str, name: str) -> Module:
    digest = hashlib.sha256(_header_digest() + source.encode()).hexdigest()[:32]
    with _lock:
        mod = _modules.get(digest)
        if mod is not None:
            return mod
        lib = _lib.load()
        cubin = None
        path = os.path.join(CACHE_DIR, digest + ".cubin")
        if os.path.exists(path):
            with open(path, "rb") as fh:
                cubin = fh.read()
        if cubin is None:
            log = ctypes.create_string_buffer(1 << 16)
            size = ctypes.c_size_t(0)
            rc = lib.drk_jit_cubin(source.encode(), name.encode(), _lib.CSRC_DIR.encode(), None,
                                   ctypes.byref(size), log, len(log))
            if rc != 0:
                raise JitError(f"NVRTC failed for {name}:\n{log.value.decode(errors='replace')}\n--- source ---\n"
                               f"{source}")
            buf = ctypes.create_string_buffer(size.value)
            rc = lib.drk_jit_cubin(source.encode(), name.encode(), _lib.CSRC_DIR.encode(), buf,
                                   ctypes.byref(size), log, len(log))
            _lib.check(rc, "drk_jit_cubin")
            cubin = buf.raw[: size.value]
            try:
                os.makedirs(CACHE_DIR, exist_ok=True)
                tmp = path + f".{os.getpid()}"
                with open(tmp, "wb") as fh:
                    fh.write(cubin)
                os.replace(tmp, path)
            except OSError:
                pass
        handle = ctypes.c_void_p()
        cbuf = ctypes.create_string_buffer(cubin, len(cubin))
        _lib.check(lib.drk_jit_load(cbuf, ctypes.byref(handle)), "drk_jit_load")
        mod = Module(handle)
        _modules[digest] = mod
        return mod


def cubin_for(source: str, name: str) -> bytes:
    """Compile only (no device needed) — used by tests on CPU-only hosts."""
    lib = _lib.load()
    log = ctypes.create_string_buffer(1 << 16)
    size = ctypes.c_size_t(0)
    rc = lib.drk_jit_cubin(source.encode(), name.encode(), _lib.CSRC_DIR.encode(), None, ctypes.byref(size), log,
                           len(log))
    if rc != 0:
        raise JitError(log.value.decode(errors="replace"))
    buf = ctypes.create_string_buffer(size.value)
    _lib.check(lib.drk_jit_cubin(source.encode(), name.encode(), _lib.CSRC_DIR.encode(), buf, ctypes.byref(size),
                                 log, len(log)), "drk_jit_cubin")
    return buf.raw[: size.value]


# ----------------------------------------------------------------------------------------
# parameter words


class Words:
    """Kernel parameter block: 8-byte words (pointers, int64, constant bit patterns)."""

    def __init__(self):
        self.values = []

    def add(self, v) -> int:
        self.values.append(v)
        return len(self.values) - 1

    def pack(self) -> bytes:
        return b"".join(struct.pack("<Q", v & 0xFFFFFFFFFFFFFFFF) for v in self.values)


def const_bits(value, dtype) -> int:
    """The constant's bit pattern in dtype, zero-extended to 64 bits (read by bits_as<T>)."""
    a = np.zeros(1, dtype=np.uint64)
    raw = np.asarray([value]).astype(np.dtype(dtype)).tobytes()
    a.view(np.uint8)[: len(raw)] = np.frombuffer(raw, dtype=np.uint8)
    return int(a[0])


# ----------------------------------------------------------------------------------------
# expression emitter


_BIN_ARITH = {"add": "add", "subtract": "sub", "multiply": "mul"}
_CMP = {"greater": ">", "greater_equal": ">=", "less": "<", "less_equal": "<=", "equal": "==", "not_equal": "!="}
_UN_MATH = {
    "sqrt", "exp", "exp2", "expm1", "log", "log2", "log10", "log1p", "sin", "cos", "tan", "arcsin", "arccos",
    "arctan", "sinh", "cosh", "tanh", "arcsinh", "arccosh", "arctanh", "floor", "ceil", "trunc", "rint", "cbrt",
    "fabs", "erf",
}


class Emitter:
    """Emits SSA statements for an expression; leaves and constants come from callbacks."""

    def __init__(self, leaf_expr, words: Words, const_mode="param"):
        self.leaf_expr = leaf_expr  # slot -> C expression of the leaf value
        self.words = words
        self.lines = []
        self.names = {}
        self.consts = {}
        self.const_mode = const_mode
        self.n = 0

    def tmp(self, ctyp, code) -> str:
        name = f"v{self.n}"
        self.n += 1
        self.lines.append(f"const {ctyp} {name} = {code};")
        return name

    def const_word(self, node) -> int:
        key = id(node)
        if key not in self.consts:
            self.consts[key] = self.words.add(const_bits(node.value, node.dtype))
        return self.consts[key]

    def emit(self, node) -> str:
        key = id(node)
        if key in self.names:
            return self.names[key]
        name = self._emit(node)
        self.names[key] = name
        return name

    def _emit(self, node) -> str:
        op, dt = node.op, node.dtype
        T = ctype(dt)
        if op == "leaf":
            return self.tmp(T, f"({T})({self.leaf_expr(node.value)})")
        if op == "const":
            if self.const_mode == "inline":
                return self.tmp(T, _literal(node.value, dt))
            return self.tmp(T, f"drk::bits_as<{T}>(p.w[{self.const_word(node)}])")
        if op == "cast":
            a = self.emit(node.args[0])
            if dt.kind == "b":
                return self.tmp(T, f"({a} != 0)")
            return self.tmp(T, f"({T})({a})")
        args = [self.emit(a) for a in node.args]
        ins = node.loop[:-1] if node.loop else [a.dtype for a in node.args]
        L = ctype(ins[0]) if ins else T
        if op in _BIN_ARITH:
            return self.tmp(T, f"drk::Arith<{L}>::{_BIN_ARITH[op]}({args[0]}, {args[1]})")
        if op == "true_divide":
            return self.tmp(T, f"({args[0]} / {args[1]})")
        if op == "floor_divide":
            f = "np_floordiv" if np.dtype(ins[0]).kind == "f" else "np_ifloordiv"
            return self.tmp(T, f"drk::{f}<{L}>({args[0]}, {args[1]})")
        if op == "remainder":
            f = "np_fmodpy" if np.dtype(ins[0]).kind == "f" else "np_imod"
            return self.tmp(T, f"drk::{f}<{L}>({args[0]}, {args[1]})")
        if op == "fmod":
            if np.dtype(ins[0]).kind == "f":
                return self.tmp(T, f"drk::m_fmod({args[0]}, {args[1]})")
            return self.tmp(T, f"({args[1]} == 0 ? ({L})0 : ({L})({args[0]} % {args[1]}))")
        if op == "power":
            if np.dtype(ins[0]).kind == "f":
                return self.tmp(T, f"drk::m_pow({args[0]}, {args[1]})")
            return self.tmp(T, f"drk::np_ipow<{L}>({args[0]}, {args[1]})")
        if op == "minimum":
            return self.tmp(T, f"drk::np_min<{L}>({args[0]}, {args[1]})")
        if op == "maximum":
            return self.tmp(T, f"drk::np_max<{L}>({args[0]}, {args[1]})")
        if op in ("fmin", "fmax"):
            if np.dtype(ins[0]).kind == "f":
                return self.tmp(T, f"drk::m_{op}({args[0]}, {args[1]})")
            f = "np_min" if op == "fmin" else "np_max"
            return self.tmp(T, f"drk::{f}<{L}>({args[0]}, {args[1]})")
        if op in _CMP:
            return self.tmp(T, f"({args[0]} {_CMP[op]} {args[1]})")
        if op == "logical_and":
            return self.tmp(T, f"(({args[0]} != 0) && ({args[1]} != 0))")
        if op == "logical_or":
            return self.tmp(T, f"(({args[0]} != 0) || ({args[1]} != 0))")
        if op == "logical_xor":
            return self.tmp(T, f"(({args[0]} != 0) != ({args[1]} != 0))")
        if op in ("bitwise_and", "bitwise_or", "bitwise_xor"):
            sym = {"bitwise_and": "&", "bitwise_or": "|", "bitwise_xor": "^"}[op]
            return self.tmp(T, f"({T})({args[0]} {sym} {args[1]})")
        if op in ("left_shift", "right_shift"):
            sym = "<<" if op == "left_shift" else ">>"
            return self.tmp(T, f"({T})({args[0]} {sym} {args[1]})")
        if op in ("arctan2", "hypot", "copysign"):
            return self.tmp(T, f"drk::m_{op}({args[0]}, {args[1]})")
        if op == "negative":
            if dt.kind in "iu":
                return self.tmp(T, f"drk::Arith<{T}>::sub(({T})0, {args[0]})")
            return self.tmp(T, f"(-{args[0]})")
        if op == "positive":
            return args[0]
        if op == "absolute":
            return self.tmp(T, f"drk::np_abs({args[0]})")
        if op == "square":
            return self.tmp(T, f"drk::Arith<{T}>::mul({args[0]}, {args[0]})")
        if op == "reciprocal":
            if dt.kind == "f":
                return self.tmp(T, f"(({T})1 / {args[0]})")
            return self.tmp(T, f"({args[0]} == 0 ? ({T})0 : ({T})(1 / {args[0]}))")
        if op == "sign":
            return self.tmp(T, f"drk::np_sign<{T}>({args[0]})")
        if op == "logical_not":
            return self.tmp(T, f"(!({args[0]} != 0))")
        if op == "invert":
            if dt.kind == "b":
                return self.tmp(T, f"(!{args[0]})")
            return self.tmp(T, f"({T})(~{args[0]})")
        if op in ("isnan", "isinf", "isfinite"):
            return self.tmp(T, f"drk::np_{op}({args[0]})")
        if op in _UN_MATH:
            if np.dtype(ins[0]).kind != "f":
                raise JitError(f"{op} on {ins[0]}")
            return self.tmp(T, f"drk::m_{op}({args[0]})")
        if op == "where":
            return self.tmp(T, f"({args[0]} ? {args[1]} : {args[2]})")
        if op == "call:black_scholes":  # the reference's fp64-internal pricing (drk::BSRef)
            return self.tmp(T, f"drk::BSRef<{T}>::price({', '.join(args)})")
        if op == "call:black_scholes_fast":
            return self.tmp(T, f"drk::BSMath<{T}>::price({', '.join(args)})")
        raise JitError(f"no device code for operation {op}")


def _literal(value, dt) -> str:
    dt = np.dtype(dt)
    if dt.kind == "b":
        return "true" if value else "false"
    if dt.kind == "f":
        v = float(value)
        if np.isnan(v):
            return "(0.0/0.0)" if dt.itemsize == 8 else "(0.0f/0.0f)"
        if np.isinf(v):
            return ("(1.0/0.0)" if v > 0 else "(-1.0/0.0)") if dt.itemsize == 8 else (
                "(1.0f/0.0f)" if v > 0 else "(-1.0f/0.0f)")
        return v.hex() if dt.itemsize == 8 else f"((float){v.hex()})"
    return f"({ctype(dt)})({int(value)}LL)"


# ----------------------------------------------------------------------------------------
# map


def _vector_width(dtypes) -> int:
    sizes = [np.dtype(d).itemsize for d in dtypes]
    return max(1, 16 // min(sizes)) if sizes else 4


def _map_source(writes, leaves):
    """(source, words builder info) for a multi-output map functor."""
    nout = len(writes)
    used = sorted(expr.leaves_used(tuple(n for _, n in writes)))
    array_slots = [k for k in used if leaves[k].kind in ("array", "host")]
    out_dt = [np.dtype(t.dtype) for t, _ in writes]
    E = _vector_width([leaves[k].dtype for k in array_slots] + out_dt)
    # word layout: outs, then one word per used leaf (ptr or index base), then constants
    words = Words()
    out_w = [words.add(0) for _ in range(nout)]
    leaf_w = {k: words.add(0) for k in used}
    lines = []

    def leaf_expr_vec(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + gi)"
        return f"r.a{k}[e]"

    def leaf_expr_scalar(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + i)"
        return f"(({ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}])[i]"

    ev = Emitter(leaf_expr_vec, words)
    outs_v = [ev.emit(n) for _, n in writes]
    body_vec = ev.lines
    es = Emitter(leaf_expr_scalar, words)
    es.consts = ev.consts  # share constant words
    outs_s = [es.emit(n) for _, n in writes]
    body_scalar = es.lines
    regs = "\n".join(f"    {ctype(leaves[k].dtype)} a{k}[E];" for k in array_slots) or "    int unused;"
    loads = "\n".join(
        f"    drk::ldv<{ctype(leaves[k].dtype)}, E>((const {ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}] + i, r.a{k});"
        for k in array_slots)
    ocl = "\n".join(f"    {ctype(out_dt[j])} o{j}[E];" for j in range(nout))
    assign = "\n".join(f"      o{j}[e] = ({ctype(out_dt[j])})({outs_v[j]});" for j in range(nout))
    stores = "\n".join(f"    drk::stv<{ctype(out_dt[j])}, E>(({ctype(out_dt[j])}*)p.w[{out_w[j]}] + i, o{j});"
                       for j in range(nout))
    sstores = "\n".join(f"    (({ctype(out_dt[j])}*)p.w[{out_w[j]}])[i] = ({ctype(out_dt[j])})({outs_s[j]});"
                        for j in range(nout))
    nwords = len(words.values)
    U = 4 if len(array_slots) <= 4 else 2
    src = f'''#include "drk_device.cuh"
struct F {{
  struct Params {{ unsigned long long w[{nwords}]; }};
  static constexpr int E = {E};
  struct Regs {{
{regs}
  }};
  static __device__ __forceinline__ void load(const Params& p, long long i, Regs& r) {{
{loads}
  }}
  static __device__ __forceinline__ void store(const Params& p, long long i, const Regs& r) {{
{ocl}
#pragma unroll
    for (int e = 0; e < E; ++e) {{
      const long long gi = i + e;
      (void)gi;
      {(chr(10) + "      ").join(body_vec)}
{assign}
    }}
{stores}
  }}
  static __device__ __forceinline__ void scalar(const Params& p, long long i) {{
    {(chr(10) + "    ").join(body_scalar)}
{sstores}
  }}
}};
struct MArgs {{ F::Params p; long long n; }};
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_map_vec(const MArgs a) {{
  drk::map_vec_body<F, {BLOCK}, {U}>(a.p, a.n);
}}
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_map_striped(const MArgs a) {{
  drk::map_striped_body<F, {BLOCK}, 4>(a.p, a.n);
}}
'''
    return src, words, out_w, leaf_w, E, U, array_slots


_GRID_CACHE = {}


def _grid(mod, kernel, work, device):
    key = (id(mod), kernel, device)
    cap = _GRID_CACHE.get(key)
    if cap is None:
        per, sms = ctypes.c_int(0), ctypes.c_int(0)
        _lib.call("drk_jit_occupancy", mod.handle, kernel.encode(), BLOCK, 0, device, ctypes.byref(per),
                  ctypes.byref(sms))
        cap = max(1, per.value) * max(1, sms.value) * 8
        _GRID_CACHE[key] = cap
    return int(max(1, min(cap, work)))


_MAP_PLANS = {}
_REDUCE_PLANS = {}
_PLAN_MAX = 2048


def _leaf_sig(leaves, used):
    return tuple((k, leaves[k].kind, leaves[k].dtype.str) for k in sorted(used))


def run_map(writes, leaves, ptrs, n, launch):
    mod, kernel, grid, buf, nbytes = map_launch(writes, leaves, ptrs, n, launch.device)
    from .kernels import launch_jit

    launch_jit(mod, kernel, grid, BLOCK, 0, buf, nbytes, launch, n)


def map_launch(writes, leaves, ptrs, n, device):
    """(module, kernel, grid, packed argument buffer, its size) of the generated map kernel
    for these writes (compiled and cached on first use)."""
    key = (tuple((np.dtype(t.dtype).str, node.key()) for t, node in writes),
           _leaf_sig(leaves, expr.leaves_used(tuple(n_ for _, n_ in writes))))
    plan = _MAP_PLANS.get(key)
    if plan is None:
        src, words, out_w, leaf_w, E, U, array_slots = _map_source(writes, leaves)
        plan = (compile_module(src, "drk_map.cu"), list(words.values), out_w, leaf_w, E, U, array_slots)
        if len(_MAP_PLANS) >= _PLAN_MAX:
            _MAP_PLANS.clear()
        _MAP_PLANS[key] = plan
    mod, wvals, out_w, leaf_w, E, U, array_slots = plan
    words = Words()
    words.values = list(wvals)
    for j, (tgt, _) in enumerate(writes):
        words.values[out_w[j]] = tgt.ptr()
    for k, w in leaf_w.items():
        words.values[w] = ptrs[k] if leaves[k].kind != "index" else leaves[k].base
    vec_ok = all(ptrs[k] % 16 == 0 for k in array_slots) and all(t.ptr() % 16 == 0 for t, _ in writes)
    blob = words.pack() + struct.pack("<q", n)
    buf = ctypes.create_string_buffer(blob, len(blob))
    if vec_ok:
        kernel = "drk_map_vec"
        grid = (n // E + BLOCK * U - 1) // (BLOCK * U) + 1
    else:
        kernel = "drk_map_striped"
        grid = _grid(mod, kernel, (n + BLOCK * 4 - 1) // (BLOCK * 4), device)
    return mod, kernel, int(min(grid, 0x7FFFFFFF)), buf, len(blob)


# ----------------------------------------------------------------------------------------
# reduce


def _op_struct(opcode, combiner, dtype):
    """C++ operator struct: a libdrk op, or a traced custom combiner over `dtype`."""
    if opcode is not None:
        return {_lib.ADD: "drk::OpAdd", _lib.MUL: "drk::OpMul", _lib.MIN: "drk::OpMin", _lib.MAX: "drk::OpMax"}[opcode], ""
    node = expr.trace_binary(combiner.fn, dtype)
    T = ctype(dtype)
    em = Emitter(lambda k: "a" if k == 0 else "b", Words(), const_mode="inline")
    res = em.emit(node)
    body = "\n      ".join(em.lines)
    src = f'''struct OpC {{
  static constexpr int code = -1;
  static constexpr bool widens = false;
  static __device__ __forceinline__ {T} apply({T} a, {T} b) {{
      {body}
      return ({T})({res});
  }}
  template <class X> static __device__ __forceinline__ X apply(X a, X b) {{ return (X)apply(({T})a, ({T})b); }}
}};
'''
    return "OpC", src


def match_binary(fn, dtype):
    """If fn(a, b) traces to exactly one of add/multiply/minimum/maximum of its two
    arguments, return that op code (so a Python lambda uses the AOT kernels)."""
    try:
        node = expr.trace_binary(fn, dtype)
    except expr.TraceError:
        return None
    if node.op in ("add", "multiply", "minimum", "maximum") and node.dtype == np.dtype(dtype):
        a, b = node.args
        if {(a.op, a.value), (b.op, b.value)} == {("leaf", 0), ("leaf", 1)} and all(
                x.dtype == np.dtype(dtype) for x in (a, b)):
            if node.op in ("minimum", "maximum") and not (a.value == 0):
                return None  # np.minimum(b, a) picks b on ties/NaN: keep operand order exact
            return {"add": _lib.ADD, "multiply": _lib.MUL, "minimum": _lib.MIN, "maximum": _lib.MAX}[node.op]
    return None


def run_reduce(node, leaves, ptrs, n, opcode, combiner, launch, slot, result_ptr=None):
    V = np.dtype(node.dtype)
    fk = expr._fn_key(combiner.fn) if (opcode is None and combiner is not None) else None
    cacheable = opcode is not None or fk is not None
    key = (node.key(), _leaf_sig(leaves, expr.leaves_used(node)), opcode, fk)
    plan = _REDUCE_PLANS.get(key) if cacheable else None
    if plan is None:
        plan = _reduce_plan(node, leaves, opcode, combiner, V)
        if cacheable:
            if len(_REDUCE_PLANS) >= _PLAN_MAX:
                _REDUCE_PLANS.clear()
            _REDUCE_PLANS[key] = plan
    mod, wvals, leaf_w, E, array_slots, opcode = plan
    words = Words()
    words.values = list(wvals)
    for k, w in leaf_w.items():
        words.values[w] = ptrs[k] if leaves[k].kind != "index" else leaves[k].base
    vec_ok = all(ptrs[k] % 16 == 0 for k in array_slots)
    st = launch.state
    scratch = st.reduce_scratch.data_ptr()
    res = result_ptr if result_ptr is not None else st.host_result_dev_ptr(slot)
    blob = (words.pack() + struct.pack("<qi4x", n, 1 if vec_ok else 0)
            + struct.pack("<QQQ", scratch, scratch + 128, scratch + 128 + 4096 * 8)
            + struct.pack("<QQ", res, 0))
    buf = ctypes.create_string_buffer(blob, len(blob))
    work = (n // E if vec_ok else n) // (BLOCK * 4) + 1
    grid = min(_grid(mod, "drk_reduce", work, launch.device) // 8, 4096)
    from .kernels import launch_jit

    launch_jit(mod, "drk_reduce", max(1, grid), BLOCK, 0, buf, len(blob), launch, n)
    return opcode


def _reduce_plan(node, leaves, opcode, combiner, V):
    if opcode is None and combiner is not None:
        code = match_binary(combiner.fn, V)
        if code is not None:
            opcode = code
    opname, opsrc = _op_struct(opcode, combiner, V)
    used = sorted(expr.leaves_used(node))
    array_slots = [k for k in used if leaves[k].kind in ("array", "host")]
    E = _vector_width([leaves[k].dtype for k in array_slots] + [V])
    words = Words()
    leaf_w = {k: words.add(0) for k in used}

    def lv(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + gi)"
        return f"a{k}[e]"

    def ls(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + i)"
        return f"(({ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}])[i]"

    ev = Emitter(lv, words)
    rv = ev.emit(node)
    es = Emitter(ls, words)
    es.consts = ev.consts
    rs = es.emit(node)
    T = ctype(V)
    regs = "\n".join(f"    {ctype(leaves[k].dtype)} a{k}[E];\n    drk::ldv<{ctype(leaves[k].dtype)}, E>("
                     f"(const {ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}] + i, a{k});" for k in array_slots)
    if not words.values:
        words.add(0)
    nwords = len(words.values)
    A = _acc_ctype(V, opcode)
    nl = "\n      "
    nl4 = "\n    "
    src = f'''#include "drk_device.cuh"
{opsrc}
struct LD {{
  typedef {T} V;
  struct Params {{ unsigned long long w[{nwords}]; }};
  static constexpr int E = {E};
  static __device__ __forceinline__ void load(const Params& p, long long i, V (&v)[E]) {{
{regs}
#pragma unroll
    for (int e = 0; e < E; ++e) {{
      const long long gi = i + e;
      (void)gi;
      {nl.join(ev.lines)}
      v[e] = (V)({rv});
    }}
  }}
  static __device__ __forceinline__ V one(const Params& p, long long i) {{
    {nl4.join(es.lines)}
    return (V)({rs});
  }}
}};
struct RArgs {{ LD::Params p; long long n; int vec_ok; drk::ReduceScratch s; {A}* result; int* has; }};
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_reduce(const RArgs a) {{
  drk::reduce_body<LD, {opname}, {BLOCK}, 4>(a.p, a.n, a.vec_ok, a.s, a.result, a.has);
}}
'''
    mod = compile_module(src, "drk_reduce.cu")
    return (mod, list(words.values), leaf_w, E, array_slots, opcode)


def _acc_ctype(V, opcode):
    if opcode is None:
        return ctype(V)
    return ctype(_lib.acc_dtype(V, opcode)) if V in _lib.DTYPE_CODE else ctype(V)


def acc_dtype(V, opcode):
    if opcode is None or np.dtype(V) not in _lib.DTYPE_CODE:
        return np.dtype(V)
    return _lib.acc_dtype(V, opcode)


# ----------------------------------------------------------------------------------------
# scan with a custom operator


def _scan_items(dt):
    return 20 if np.dtype(dt).itemsize == 4 else 10


def scan_module(dtype, combiner):
    T = ctype(dtype)
    opname, opsrc = _op_struct(None, combiner, dtype)
    items = _scan_items(dtype)
    src = f'''#include "drk_device.cuh"
{opsrc}
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_scan(
    const drk::ScanParams<{T}, const {T}*> p) {{
  drk::scan_kernel_body<drk::PlainLoad<{T}>, {T}, {opname}, {BLOCK}, {items}, 1>(p);
}}
'''
    return compile_module(src, "drk_scan.cu"), items


def custom_scan(rt, in_segs, out_segs, live, op, exclusive, init, carry=None):
    """Aligned scan with an operator that is not a numpy ufunc (algorithms.py:216-231, the
    Python fold of `_accumulate`).  If the traced operator is exactly add / multiply /
    minimum / maximum of its arguments, the libdrk scans run.  Otherwise each segment is
    scanned by a generated kernel that applies the traced combiner — reading a plain vector
    directly, or a view fused into the scan (no materialised input).  One GPU: the carry
    chains on the device.  Several GPUs: every segment's total is reduced on its GPU with
    the same combiner, the host folds the totals in segment order exactly like the
    reference's driver loop (algorithms.py:256-262), and each segment is scanned with its
    carry."""
    from .algorithms import BinaryOp, _scan_impl
    from .kernels import Launch, ScanView, run_reduce, run_scan_view, stage_leaves, _dealias
    from .runtime import await_pending
    from .views import Target, lower

    T = None
    for k in live:
        tgt = lower(out_segs[k]).target
        if not isinstance(tgt, Target):
            raise TypeError("scan output segments must be writable vector storage")
        T = np.dtype(tgt.dtype)
    code = match_binary(op.fn, T)
    if code is not None:
        ufunc = {_lib.ADD: np.add, _lib.MUL: np.multiply, _lib.MIN: np.minimum, _lib.MAX: np.maximum}[code]
        return _scan_impl(_SegList(in_segs), out_segs_view(out_segs), BinaryOp(op.fn, op.identity, ufunc), exclusive,
                          init, carry)
    mod, items = scan_module(T, op)
    tile = BLOCK * items
    work = []
    for k in live:
        lw = lower(in_segs[k])
        tgt = lower(out_segs[k]).target
        st = rt.state_of(out_segs[k].rank)
        launch = Launch(st)
        node = lw.value
        if isinstance(node, tuple):
            raise TypeError("scan needs scalar elements; apply a transform to the zip first")
        plain = node.op == "leaf" and lw.leaves[node.value].kind == "array" and node.dtype == T
        if plain and lw.leaves[node.value].device == st.index:
            await_pending(st, [lw.leaves[node.value].handle, tgt.handle])
            node_t = node
            leaves = lw.leaves
            ptrs = [lf.ptr() if lf.kind == "array" else 0 for lf in leaves]
            src = leaves[node.value].ptr()
        else:
            node_t = expr.cast(node, T)
            leaves = _dealias([(tgt, node_t)], lw.leaves, lw.length, launch)
            await_pending(st, [tgt.handle])
            ptrs = stage_leaves(leaves, launch)
            src = ScanView(node_t, leaves, ptrs, lw.length)
        work.append((k, st, launch, src, tgt, node_t, leaves, ptrs))
    partials = [None] * len(in_segs)
    lib = _lib.load()

    def scan_one(j, st, launch, src, tgt, init_v, carry_v, carry_dev, slots):
        if isinstance(src, ScanView):
            run_scan_view(T, None, exclusive, src, tgt.ptr(), tgt.length, launch, combiner=op, init=init_v,
                          carry_value=carry_v, carry_dev=carry_dev, seg_total_slot=slots[0],
                          carry_out_slot=slots[1], scratch_index=j % 2)
            return
        n = tgt.length
        scratch = st.scan_scratch(int(lib.drk_jit_scan_scratch_bytes(n, tile)), j % 2)
        init_buf = _lib.scalar_buffer(init_v, T) if exclusive else None
        carry_buf = _lib.scalar_buffer(carry_v, T) if carry_v is not None else None
        _lib.call("drk_jit_scan", mod.handle, b"drk_scan", T.itemsize, tile, tile * T.itemsize,
                  1 if exclusive else 0, src, tgt.ptr(), n,
                  ctypes.addressof(init_buf) if init_buf is not None else None,
                  ctypes.addressof(carry_buf) if carry_buf is not None else None, carry_dev,
                  st.result_dev_ptr(slots[0]) if slots[0] is not None else None,
                  st.result_dev_ptr(slots[1]) if slots[1] is not None else None,
                  scratch.data_ptr(), scratch.numel(), st.index, st.handle)

    from . import algorithms

    if len({id(w[1]) for w in work}) == 1 and not algorithms._FORCE_MULTI_DEVICE_SCAN:
        st = work[0][1]
        st.ensure_results(2 * len(work) + 2)
        prev = None
        for j, (k, _st, launch, src, tgt, *_r) in enumerate(work):
            scan_one(j, st, launch, src, tgt, init, carry if j == 0 else None,
                     st.result_dev_ptr(prev) if prev is not None else None, (2 * j, 2 * j + 1))
            prev = 2 * j + 1
        raw = st.fetch_results(2 * len(work))
        for j, (k, *_r) in enumerate(work):
            partials[k] = np.frombuffer(raw[16 * j: 16 * j + T.itemsize].tobytes(), dtype=T)[0].item()
        return partials
    # several GPUs: totals on every GPU (in parallel), driver fold, carried scans
    count = {}
    for w in work:
        count[id(w[1])] = count.get(id(w[1]), 0) + 1
    for w in work:
        w[1].ensure_results(count[id(w[1])])
    slot_of, used = {}, {}
    for k, st, launch, src, tgt, node_t, leaves, ptrs in work:
        slot = used.get(id(st), 0)
        used[id(st)] = slot + 1
        slot_of[k] = slot
        run_reduce(node_t, leaves, tgt.length, None, op, launch, slot, ptrs=ptrs)
    fetched = {}
    for w in work:
        if id(w[1]) not in fetched:
            fetched[id(w[1])] = w[1].fetch_host_results(count[id(w[1])])
    for k, st, *_r in work:
        raw = fetched[id(st)]
        partials[k] = np.frombuffer(raw[8 * slot_of[k]: 8 * slot_of[k] + T.itemsize].tobytes(), dtype=T)[0].item()
    prefix = carry
    for j, (k, st, launch, src, tgt, *_r) in enumerate(work):
        off = prefix
        if partials[k] is not None:
            prefix = partials[k] if prefix is None else op.fn(prefix, partials[k])
        scan_one(j, st, launch, src, tgt, init, off, None, (None, None))
    for w in work:
        w[1].synchronize()
    return partials


# ----------------------------------------------------------------------------------------
# scan of a fused view (NVRTC loader for the L2 / single-pass scan templates)


_SCAN_VIEW_PLANS = {}


def scan_view_plan(view, T, opcode, combiner=None):
    """(module, words, geometry) of the fused scan of `view` (kernels.ScanView: node already
    cast to the output dtype T) with a libdrk operator or a traced custom combiner.  The
    module defines drk_scan_l2_s / drk_scan_l2_l / drk_scan_1p over a generated loader whose
    parameters are JitWords: one word per used leaf (pointer or index base), then constants
    (kernel parameters, so expressions differing only in constants share one module).
    geometry = (items, nl, subs_small, subs_large, items_1p) for drk_jit_scan_view."""
    T = np.dtype(T)
    node, leaves = view.node, view.leaves
    fk = expr._fn_key(combiner.fn) if combiner is not None else None
    cacheable = combiner is None or fk is not None
    used = sorted(expr.leaves_used(node))
    key = (node.key(), _leaf_sig(leaves, used), T.str, opcode, fk)
    plan = _SCAN_VIEW_PLANS.get(key) if cacheable else None
    if plan is None:
        plan = _scan_view_plan(node, leaves, T, opcode, combiner, used)
        if cacheable:
            if len(_SCAN_VIEW_PLANS) >= _PLAN_MAX:
                _SCAN_VIEW_PLANS.clear()
            _SCAN_VIEW_PLANS[key] = plan
    mod, wvals, leaf_w, geom = plan
    words = list(wvals)
    for k, w in leaf_w.items():
        words[w] = view.ptrs[k] if leaves[k].kind != "index" else leaves[k].base
    return mod, words, geom


def scan_geometry(T, nl):
    """drk_device.cuh ScanGeom: (items, subs_small, subs_large) of the L2 scan for values of
    dtype T and nl staged leaves."""
    four = np.dtype(T).itemsize == 4
    if nl >= 2:
        return (12 if four else 6), 3, 7
    return (20 if four else 10), 4, 8


def _scan_view_plan(node, leaves, T, opcode, combiner, used):
    if opcode is None and combiner is not None:
        code = match_binary(combiner.fn, T)
        if code is not None:
            opcode = code
            combiner = None
    opname, opsrc = _op_struct(opcode, combiner, T)
    array_slots = [k for k in used if leaves[k].kind in ("array", "host")]
    # staged (TMA through the ring, values computed in shared memory) when the view reads one
    # or two arrays of the value's element size; otherwise a register loader
    staged = 1 <= len(array_slots) <= 2 and all(leaves[k].dtype.itemsize == T.itemsize for k in array_slots)
    nl = len(array_slots) if staged else 0
    raw_of = {k: r for r, k in enumerate(array_slots)}
    words = Words()
    leaf_w = {k: words.add(0) for k in used}

    def lv(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + gi)"
        if staged:
            return f"drk::bits_as<{ctype(leaves[k].dtype)}>(raw[{raw_of[k]}][e])"
        return f"a{k}[e]"

    def ls(k):
        if leaves[k].kind == "index":
            return f"(long long)(p.w[{leaf_w[k]}] + i)"
        return f"(({ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}])[i]"

    ev = Emitter(lv, words)
    rv = ev.emit(node)
    es = Emitter(ls, words)
    es.consts = ev.consts
    rs = es.emit(node)
    if len(words.values) > _lib.JIT_WORDS:
        raise JitError(f"fused scan needs {len(words.values)} parameter words (max {_lib.JIT_WORDS})")
    V = ctype(T)
    items, subs_small, subs_large = scan_geometry(T, nl)
    items_1p = _scan_items(T)
    nl_ = "\n      "
    nl4 = "\n    "
    if staged:
        leaf_sel = " : ".join(f"k == {r} ? p.w[{leaf_w[k]}]" for r, k in enumerate(array_slots)) + " : 0ull"
        body = f'''  typedef typename drk::RawOf<V>::type R;
  static constexpr int NL = {nl};
  static __device__ __forceinline__ const void* leaf(const Params& p, int k) {{ return (const void*)({leaf_sel}); }}
  template <int E>
  static __device__ __forceinline__ void compute(const Params& p, const R (&raw)[NL][E], long long gi0, V (&v)[E]) {{
#pragma unroll
    for (int e = 0; e < E; ++e) {{
      const long long gi = gi0 + e;
      (void)gi;
      {nl_.join(ev.lines)}
      v[e] = (V)({rv});
    }}
  }}'''
    else:
        loads = "\n".join(f"    {ctype(leaves[k].dtype)} a{k}[E];\n    drk::ldv_hint<{ctype(leaves[k].dtype)}, E>("
                          f"(const {ctype(leaves[k].dtype)}*)p.w[{leaf_w[k]}] + i, a{k}, pol);" for k in array_slots)
        body = f'''  static constexpr int NL = 0;
  static constexpr int E = 16 / sizeof(V);
  static __device__ __forceinline__ void load16(const Params& p, long long i, V (&v)[E], unsigned long long pol) {{
{loads}
#pragma unroll
    for (int e = 0; e < E; ++e) {{
      const long long gi = i + e;
      (void)gi;
      {nl_.join(ev.lines)}
      v[e] = (V)({rv});
    }}
  }}'''
    params = f"drk::ScanParams<typename drk::WideAcc<{V}, {opname}>::type, drk::JitWords>"
    src = f'''#include "drk_device.cuh"
{opsrc}
struct LD {{
  typedef {V} V;
  typedef drk::JitWords Params;
  static constexpr bool bulk = false;
{body}
  static __device__ __forceinline__ V one(const Params& p, long long i) {{
    {nl4.join(es.lines)}
    return (V)({rs});
  }}
}};
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_scan_l2_s(const {params} p) {{
  drk::scan_l2_body<LD, {opname}, {BLOCK}, {items}, {subs_small}, 3>(p);
}}
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_scan_l2_l(const {params} p) {{
  drk::scan_l2_body<LD, {opname}, {BLOCK}, {items}, {subs_large}, 3>(p);
}}
extern "C" __global__ void __launch_bounds__({BLOCK}) drk_scan_1p(const {params} p) {{
  drk::scan_kernel_body<LD, {V}, {opname}, {BLOCK}, {items_1p}, 3>(p);
}}
'''
    mod = compile_module(src, "drk_scan_view.cu")
    return (mod, list(words.values), leaf_w, (items, nl, subs_small, subs_large, items_1p))


class _SegList:
    """A segmented range given by an explicit segment list."""

    def __init__(self, segs):
        self._segs = list(segs)
        self.is_segmented = True

    def segments(self):
        return list(self._segs)

    def __len__(self):
        return sum(len(s) for s in self._segs)

    @property
    def runtime(self):
        for s in self._segs:
            rt = getattr(s, "runtime", None)
            if rt is not None:
                return rt
        return None


def out_segs_view(out_segs):
    return _SegList(out_segs)
