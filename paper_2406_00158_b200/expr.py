"""Expression IR and tracer: how a Python element function becomes a device kernel.

The reference applies user functions to numpy arrays (views.py:164-181
`_apply_elementwise`, algorithms.py:101-111).  Here a function is called once on
*symbols* — proxies that record every arithmetic operation, numpy ufunc (and
scipy.special.erf) and ``np.where``/``np.clip`` applied to them — producing an
expression over the segment's leaves.  Result dtypes follow numpy exactly because every
operation asks numpy itself for the ufunc loop (``ufunc.resolve_dtypes``, NEP 50 weak
Python scalars included), so ``3.0 * float32`` stays float32 and ``int32 / int32`` is
float64.  The expression is then matched against the ahead-of-time kernel catalogue or
compiled (codegen.py) — never evaluated on the host.

Functions that branch on element values (``if x > 0``), have side effects only (return
None), or materialise their input (``np.asarray(x)``) cannot be traced; they raise
``TraceError`` (a TypeError) instead of silently running elsewhere.
"""

from __future__ import annotations

import numpy as np

try:  # scipy.special.erf is a ufunc; the reference's norm_cdf uses it (bench.py:19,102-103)
    import scipy.special as _sps

    _ERF = _sps.erf
except Exception:  # pragma: no cover
    _sps = None
    _ERF = None


class TraceError(TypeError):
    """The function cannot be lowered to a device expression."""


# ----------------------------------------------------------------------------------------
# IR


class Node:
    """One expression node.

    op: "leaf" (value = leaf slot), "const" (value = Python scalar), "index" (value = 0,
    the element's global index offset is supplied per segment), "cast", a ufunc name
    ("add", "sqrt", ...), "where", or "call:<name>" for registered device functions.
    ``loop`` is the tuple of numpy loop dtypes the operation computes in (inputs..., out).
    """

    __slots__ = ("op", "args", "dtype", "value", "loop", "_key")

    def __init__(self, op, args=(), dtype=None, value=None, loop=None):
        self.op = op
        self.args = tuple(args)
        self.dtype = np.dtype(dtype) if dtype is not None else None
        self.value = value
        self.loop = tuple(np.dtype(d) for d in loop) if loop else None
        self._key = None

    def key(self) -> tuple:
        """Structural identity (constants included)."""
        if self._key is None:
            val = self.value
            if self.op == "const":
                val = (type(val).__name__, repr(val))
            self._key = (
                self.op,
                self.dtype.str if self.dtype is not None else None,
                val,
                tuple(a.key() for a in self.args),
                tuple(d.str for d in self.loop) if self.loop else None,
            )
        return self._key

    def shape_key(self) -> tuple:
        """Structural identity with constants abstracted (kernel cache key)."""
        if self.op == "const":
            return ("const", self.dtype.str)
        return (
            self.op,
            self.dtype.str if self.dtype is not None else None,
            self.value if self.op in ("leaf", "index") else None,
            tuple(a.shape_key() for a in self.args),
            tuple(d.str for d in self.loop) if self.loop else None,
        )

    def walk(self):
        yield self
        for a in self.args:
            yield from a.walk()

    def __repr__(self):
        if self.op == "leaf":
            return f"in{self.value}:{self.dtype}"
        if self.op == "const":
            return f"{self.value!r}:{self.dtype}"
        if self.op == "index":
            return "index"
        return f"{self.op}({', '.join(map(repr, self.args))}):{self.dtype}"


_LEAVES = {}


def leaf(slot: int, dtype) -> Node:
    """Interned leaf node (so structural keys of repeated lowerings are cached)."""
    dt = np.dtype(dtype)
    key = (slot, dt.str)
    n = _LEAVES.get(key)
    if n is None:
        n = _LEAVES[key] = Node("leaf", (), dt, slot)
    return n


def const(value, dtype) -> Node:
    return Node("const", (), dtype, value)


def cast(node: Node, dtype) -> Node:
    dtype = np.dtype(dtype)
    if node.dtype == dtype:
        return node
    if node.op == "const":
        return const(_convert_scalar(node.value, dtype), dtype)
    return Node("cast", (node,), dtype)


def _convert_scalar(value, dtype):
    arr = np.array(value)
    if dtype.kind in "iu" and arr.dtype.kind in "iu":
        info = np.iinfo(dtype)
        if not info.min <= int(value) <= info.max:
            raise OverflowError(f"Python integer {value} out of bounds for {dtype}")
    return np.array(value).astype(dtype).item() if dtype.kind != "b" else bool(value)


# ----------------------------------------------------------------------------------------
# symbols

UNARY_UFUNCS = {
    "negative", "positive", "absolute", "sqrt", "exp", "exp2", "expm1", "log", "log2", "log10",
    "log1p", "sin", "cos", "tan", "arcsin", "arccos", "arctan", "sinh", "cosh", "tanh", "arcsinh",
    "arccosh", "arctanh", "floor", "ceil", "trunc", "rint", "square", "reciprocal", "sign",
    "logical_not", "invert", "isnan", "isinf", "isfinite", "cbrt", "fabs", "erf",
}
BINARY_UFUNCS = {
    "add", "subtract", "multiply", "true_divide", "divide", "floor_divide", "remainder", "mod",
    "fmod", "power", "minimum", "maximum", "fmin", "fmax", "greater", "greater_equal", "less",
    "less_equal", "equal", "not_equal", "logical_and", "logical_or", "logical_xor", "bitwise_and",
    "bitwise_or", "bitwise_xor", "arctan2", "hypot", "copysign", "left_shift", "right_shift",
}
_ALIASES = {"divide": "true_divide", "mod": "remainder"}


def _ufunc_name(uf) -> str | None:
    if _ERF is not None and uf is _ERF:
        return "erf"
    name = getattr(uf, "__name__", None)
    if name is None:
        return None
    name = _ALIASES.get(name, name)
    if name in UNARY_UFUNCS or name in BINARY_UFUNCS:
        if name == "erf":
            return None
        return name
    return None


def _ufunc_obj(name):
    if name == "erf":
        return _ERF
    return getattr(np, name)


def _operand(x):
    """(node or None, python scalar or None) for an operand of an operation."""
    if isinstance(x, Sym):
        return x.node, None
    if isinstance(x, (bool, int, float)) and not isinstance(x, np.generic):
        return None, x
    if isinstance(x, np.generic):
        return const(x.item(), x.dtype), None
    if isinstance(x, np.ndarray) and x.ndim == 0:
        return const(x.item(), x.dtype), None
    raise TraceError(
        f"cannot trace an operation with a {type(x).__name__} operand; element functions may only "
        "combine their arguments with scalars"
    )


def _weak_type(v):
    if isinstance(v, bool):
        return np.dtype(np.bool_)  # Python bools are not weak under NEP 50
    if isinstance(v, int):
        return int
    return float


_LOOPS = {}


def _resolve(uf, name, descr):
    key = (name, tuple(d.str if isinstance(d, np.dtype) else d.__name__ for d in descr))
    loop = _LOOPS.get(key)
    if loop is None:
        try:
            loop = uf.resolve_dtypes(tuple(descr) + (None,))
        except Exception as exc:
            raise TraceError(f"numpy has no {name} loop for {descr}: {exc}") from None
        _LOOPS[key] = loop
    return loop


def apply_ufunc(name: str, *xs):
    """Record ufunc `name` applied to operands (Syms / scalars) with numpy's loop dtypes."""
    uf = _ufunc_obj(name)
    if uf is None:
        raise TraceError(f"ufunc {name} unavailable")
    nodes, descr = [], []
    for x in xs:
        node, scalar = _operand(x)
        nodes.append((node, scalar))
        descr.append(node.dtype if node is not None else _weak_type(scalar))
    # numpy special-cases float ** {2, 0.5, -1, 1, 0} (fast_scalar_power)
    if name == "power" and nodes[0][0] is not None and nodes[1][0] is None and nodes[0][0].dtype.kind == "f":
        p = nodes[1][1]
        if p == 2:
            return apply_ufunc("square", xs[0])
        if p == 0.5:
            return apply_ufunc("sqrt", xs[0])
        if p == 1:
            return xs[0]
        if p == -1:
            return apply_ufunc("reciprocal", xs[0])
    loop = _resolve(uf, name, descr)
    args = []
    for (node, scalar), dt in zip(nodes, loop[:-1]):
        if node is None:
            args.append(const(_convert_scalar(scalar, dt), dt))
        else:
            args.append(cast(node, dt))
    out = loop[-1]
    # all-constant operations fold on the host (they are not element work)
    if all(a.op == "const" for a in args):
        with np.errstate(all="ignore"):
            val = uf(*[np.array(a.value, dtype=a.dtype) for a in args])
        return Sym(const(np.asarray(val).item(), out))
    return Sym(Node(name, args, out, loop=loop))


def where(cond, a, b):
    cn, cs = _operand(cond)
    if cn is None:
        return a if cs else b
    cond_node = cast(cn, np.bool_) if cn.dtype != np.bool_ else cn
    an, asc = _operand(a)
    bn, bsc = _operand(b)
    descr_a = an.dtype if an is not None else _weak_type(asc)
    descr_b = bn.dtype if bn is not None else _weak_type(bsc)
    # np.where's output dtype: result_type with weak Python scalars
    probe = [np.zeros(1, dtype=d) if isinstance(d, np.dtype) else d(0) for d in (descr_a, descr_b)]
    out = np.result_type(*probe)
    args = [cond_node]
    for node, scalar in ((an, asc), (bn, bsc)):
        args.append(cast(node, out) if node is not None else const(_convert_scalar(scalar, out), out))
    return Sym(Node("where", args, out, loop=(np.bool_, out, out, out)))


class Sym:
    """A traced value.  Behaves like a numpy array under arithmetic and ufuncs."""

    __slots__ = ("node",)
    __array_priority__ = 1000

    def __init__(self, node: Node):
        self.node = node

    dtype = property(lambda self: self.node.dtype)
    ndim = 1
    shape = property(lambda self: (-1,))

    def astype(self, dtype, copy=True):
        return Sym(cast(self.node, np.dtype(dtype)))

    # arithmetic
    def __add__(self, o): return apply_ufunc("add", self, o)
    def __radd__(self, o): return apply_ufunc("add", o, self)
    def __sub__(self, o): return apply_ufunc("subtract", self, o)
    def __rsub__(self, o): return apply_ufunc("subtract", o, self)
    def __mul__(self, o): return apply_ufunc("multiply", self, o)
    def __rmul__(self, o): return apply_ufunc("multiply", o, self)
    def __truediv__(self, o): return apply_ufunc("true_divide", self, o)
    def __rtruediv__(self, o): return apply_ufunc("true_divide", o, self)
    def __floordiv__(self, o): return apply_ufunc("floor_divide", self, o)
    def __rfloordiv__(self, o): return apply_ufunc("floor_divide", o, self)
    def __mod__(self, o): return apply_ufunc("remainder", self, o)
    def __rmod__(self, o): return apply_ufunc("remainder", o, self)
    def __pow__(self, o): return apply_ufunc("power", self, o)
    def __rpow__(self, o): return apply_ufunc("power", o, self)
    def __neg__(self): return apply_ufunc("negative", self)
    def __pos__(self): return apply_ufunc("positive", self)
    def __abs__(self): return apply_ufunc("absolute", self)
    def __invert__(self): return apply_ufunc("invert", self)
    def __and__(self, o): return apply_ufunc("bitwise_and", self, o)
    def __rand__(self, o): return apply_ufunc("bitwise_and", o, self)
    def __or__(self, o): return apply_ufunc("bitwise_or", self, o)
    def __ror__(self, o): return apply_ufunc("bitwise_or", o, self)
    def __xor__(self, o): return apply_ufunc("bitwise_xor", self, o)
    def __rxor__(self, o): return apply_ufunc("bitwise_xor", o, self)
    def __lshift__(self, o): return apply_ufunc("left_shift", self, o)
    def __rshift__(self, o): return apply_ufunc("right_shift", self, o)
    def __lt__(self, o): return apply_ufunc("less", self, o)
    def __le__(self, o): return apply_ufunc("less_equal", self, o)
    def __gt__(self, o): return apply_ufunc("greater", self, o)
    def __ge__(self, o): return apply_ufunc("greater_equal", self, o)
    def __eq__(self, o): return apply_ufunc("equal", self, o)
    def __ne__(self, o): return apply_ufunc("not_equal", self, o)
    __hash__ = object.__hash__

    # things a traced function may not do
    def __bool__(self):
        raise TraceError(
            "element function branches on element values; data-dependent control flow cannot be "
            "traced into a device kernel (use np.where / np.minimum / np.maximum instead)"
        )

    def __float__(self):
        raise TraceError("element function converts an element to a Python float; not traceable")

    def __int__(self):
        raise TraceError("element function converts an element to a Python int; not traceable")

    __index__ = __int__

    def __len__(self):
        raise TraceError("element function takes len() of an element array; not traceable")

    def __iter__(self):
        raise TraceError("element function iterates over an element array; not traceable")

    def __getitem__(self, i):
        raise TraceError("element function indexes into an element array; not traceable")

    def __array__(self, dtype=None, copy=None):
        raise TraceError(
            "element function materialises its input as a numpy array (np.asarray); device "
            "kernels cannot run host numpy code"
        )

    def tolist(self):
        raise TraceError("element function calls tolist(); not traceable")

    item = tolist

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        if method != "__call__":
            raise TraceError(f"ufunc method {ufunc.__name__}.{method} is not traceable")
        if kwargs.get("out") is not None:
            raise TraceError("ufunc out= arguments are not traceable")
        dtype = kwargs.pop("dtype", None)
        kwargs.pop("casting", None)
        if kwargs:
            raise TraceError(f"ufunc keyword arguments {sorted(kwargs)} are not traceable")
        name = _ufunc_name(ufunc)
        if name is None:
            raise TraceError(f"ufunc {getattr(ufunc, '__name__', ufunc)} has no device implementation")
        r = apply_ufunc(name, *inputs)
        return r.astype(dtype) if dtype is not None else r

    def __array_function__(self, func, types, args, kwargs):
        impl = _ARRAY_FUNCTIONS.get(func)
        if impl is None:
            raise TraceError(f"numpy function {func.__name__} is not traceable")
        return impl(*args, **kwargs)

    def __repr__(self):
        return f"Sym({self.node!r})"


def _np_where(cond, x=None, y=None):
    if x is None or y is None:
        raise TraceError("np.where(cond) without values is not traceable")
    return where(cond, x, y)


def _np_clip(a, a_min=None, a_max=None, **kw):
    r = a
    if a_min is not None:
        r = apply_ufunc("maximum", r, a_min)
    if a_max is not None:
        r = apply_ufunc("minimum", r, a_max)
    return r


def _np_asarray(a, dtype=None, **kw):
    if isinstance(a, Sym):
        return a.astype(dtype) if dtype is not None else a
    raise TraceError("np.asarray on a non-element value is not traceable")


_ARRAY_FUNCTIONS = {
    np.where: _np_where,
    np.clip: _np_clip,
    np.copy: lambda a, **k: a,
    np.square: lambda a: apply_ufunc("square", a),
}


# ----------------------------------------------------------------------------------------
# registered device functions (named kernels usable inside traced functions)

class DeviceFunction:
    """A function with a hand-written device implementation (e.g. the Black-Scholes call
    price): calling it on symbols records a ``call:<name>`` node; the AOT catalogue or the
    code generator supplies the body."""

    def __init__(self, name, arity, result_dtype, host_impl):
        self.name = name
        self.arity = arity
        self.result_dtype = result_dtype  # callable(list of dtypes) -> dtype
        self.host_impl = host_impl        # used for non-symbol arguments (device evaluation)

    def __call__(self, *args):
        if any(isinstance(a, Sym) for a in args):
            if len(args) != self.arity:
                raise TypeError(f"{self.name} takes {self.arity} arguments")
            nodes = []
            dts = []
            for a in args:
                node, scalar = _operand(a)
                if node is None:
                    node = const(float(scalar), np.float64)
                nodes.append(node)
                dts.append(node.dtype)
            out = np.dtype(self.result_dtype(dts))
            nodes = [cast(n, out) for n in nodes]
            return Sym(Node("call:" + self.name, nodes, out, loop=tuple([out] * (self.arity + 1))))
        return self.host_impl(*args)


# ----------------------------------------------------------------------------------------
# tracing entry points

def symbolize(value):
    """Turn a lowered value (Node or nested tuple of Nodes) into call arguments."""
    if isinstance(value, tuple):
        return tuple(symbolize(v) for v in value)
    return Sym(value)


def to_nodes(result):
    """Normalise a traced result: Sym -> Node, scalars -> const nodes, tuples recursively,
    None kept (it means "leave this element alone")."""
    if result is None:
        return None
    if isinstance(result, Sym):
        return result.node
    if isinstance(result, (tuple, list)):
        return tuple(to_nodes(r) for r in result)
    if isinstance(result, (bool, int, float)) and not isinstance(result, np.generic):
        if isinstance(result, bool):
            return const(result, np.bool_)
        if isinstance(result, int):
            return const(result, np.int64)
        return const(result, np.float64)
    if isinstance(result, np.generic):
        return const(result.item(), result.dtype)
    if isinstance(result, np.ndarray) and result.ndim == 0:
        return const(result.item(), result.dtype)
    raise TraceError(f"element function returned {type(result).__name__}; expected element values")


_TRACES = {}
_TRACE_CACHE_MAX = 4096


class _Uncacheable(Exception):
    pass


# modules whose attributes a traced function may read without defeating the cache: their
# contents are functions/ufuncs/constants, not user state
_STABLE_MODULES = ("numpy", "math", "operator", "scipy", "cmath", "builtins")


def _freeze(v, depth):
    """A hashable, type-exact snapshot of a value a traced function can see, or
    _Uncacheable.  Keyed by type and exact value: 2 and 2.0, 0.0 and -0.0, np.float64(0.5)
    and 0.5 all differ (their traces differ under numpy's promotion rules)."""
    import types

    if v is None or isinstance(v, (bool, str, bytes)):
        return (type(v), v)
    if isinstance(v, (int, float, complex)) and not isinstance(v, np.generic):
        return (type(v), repr(v))  # repr separates -0.0 from 0.0 and keeps the type exact
    if isinstance(v, np.generic):
        return (type(v), v.dtype.str, v.tobytes())
    if isinstance(v, np.dtype):
        return ("dtype", v.str)
    if isinstance(v, type):
        return ("type", v)  # classes (np.float32, int ...) are used as dtypes/constructors
    if isinstance(v, (tuple, frozenset)):
        return (type(v), tuple(_freeze(x, depth) for x in v))
    if isinstance(v, np.ufunc) or v is _ERF:
        return ("ufunc", v)
    if isinstance(v, types.BuiltinFunctionType):
        return ("builtin", v)
    if isinstance(v, types.ModuleType):
        if v.__name__.split(".")[0] in _STABLE_MODULES:
            return ("module", v.__name__)
        raise _Uncacheable(v.__name__)
    if isinstance(v, DeviceFunction):
        return ("devfn", id(v), v.name)
    if isinstance(v, types.FunctionType):
        if depth > 4:
            raise _Uncacheable("helper nesting")
        return ("fn", _fn_key_strict(v, depth + 1))
    if isinstance(v, functools_partial()):
        return ("partial", _freeze(v.func, depth + 1), _freeze(tuple(v.args), depth),
                _freeze(tuple(sorted((v.keywords or {}).items())), depth))
    # objects with mutable state (instances, lists, dicts, arrays, modules of user code):
    # the function may read anything through them, so its trace is not cached
    raise _Uncacheable(type(v).__name__)


def functools_partial():
    import functools

    return functools.partial


_CODE = type(_freeze.__code__)


def _all_names(code, out):
    """Names a code object and the code objects nested in it (inner lambdas, comprehensions)
    may look up as globals."""
    out.update(code.co_names)
    for c in code.co_consts:
        if type(c) is _CODE:
            _all_names(c, out)
    return out


def _fn_key_strict(fn, depth=0):
    code = getattr(fn, "__code__", None)
    if code is None:
        raise _Uncacheable("no code")
    cells = tuple(_freeze(c.cell_contents, depth) for c in (fn.__closure__ or ()))
    g = fn.__globals__
    glob = tuple((nm, _freeze(g[nm], depth)) for nm in sorted(_all_names(code, set())) if nm in g)
    defaults = _freeze(tuple(fn.__defaults__ or ()), depth)
    kwdefaults = _freeze(tuple(sorted((fn.__kwdefaults__ or {}).items())), depth)
    return (code, defaults, kwdefaults, cells, glob)


def _fn_key(fn):
    """A hashable identity of a function's behaviour: its code, defaults, closure contents
    and the globals it names, each frozen by type and exact value (helper functions
    recursively).  None — no caching, the function is traced on every call like the
    reference calls it every time — when it can reach mutable state (an object attribute,
    a list, an array, a user module) whose value could change between calls."""
    code = getattr(fn, "__code__", None)
    if (code is not None and not code.co_names and fn.__closure__ is None and fn.__defaults__ is None
            and not fn.__kwdefaults__ and not any(type(c) is _CODE for c in code.co_consts)):
        return (code,)  # a pure function of its argument (lambda t: t[0] * t[1]): the code alone
    if isinstance(fn, functools_partial()):
        try:
            return ("partial", _freeze(fn, 0))
        except (_Uncacheable, TypeError, ValueError):
            return None
    try:
        key = _fn_key_strict(fn)
        hash(key)
        return key
    except (_Uncacheable, TypeError, ValueError):
        return None


def trace_cached(fn, value, value_key, fk=None):
    """trace() memoised on (function identity, lowered value structure)."""
    if fk is None:
        fk = _fn_key(fn)
    if fk is None:
        return trace(fn, value)
    key = (fk, value_key)
    out = _TRACES.get(key)
    if out is None:
        out = trace(fn, value)
        if len(_TRACES) >= _TRACE_CACHE_MAX:
            _TRACES.clear()
        _TRACES[key] = out
    return out


def trace(fn, value):
    """Call fn once on symbols for `value` and return the result as nodes."""
    args = symbolize(value)
    try:
        with np.errstate(all="ignore"):
            out = fn(args)
    except TraceError:
        raise
    except (TypeError, ValueError, AttributeError, IndexError, KeyError) as exc:
        raise TraceError(f"element function is not traceable into a device kernel: "
                         f"{type(exc).__name__}: {exc}") from exc
    return to_nodes(out)


def trace_binary(fn, dtype):
    """Trace a binary operator fn(a, b) over elements of `dtype` (custom reduce/scan ops)."""
    a, b = Sym(leaf(0, dtype)), Sym(leaf(1, dtype))
    try:
        with np.errstate(all="ignore"):
            out = fn(a, b)
    except TraceError:
        raise
    except (TypeError, ValueError, AttributeError) as exc:
        raise TraceError(f"binary operator is not traceable: {type(exc).__name__}: {exc}") from exc
    node = to_nodes(out)
    if not isinstance(node, Node):
        raise TraceError("binary operator must return one value")
    return cast(node, dtype)


def leaves_used(node) -> set:
    if node is None:
        return set()
    if isinstance(node, tuple):
        s = set()
        for n in node:
            s |= leaves_used(n)
        return s
    return {n.value for n in node.walk() if n.op == "leaf"}


def uses_index(node) -> bool:
    if node is None:
        return False
    if isinstance(node, tuple):
        return any(uses_index(n) for n in node)
    return any(n.op == "index" for n in node.walk())
