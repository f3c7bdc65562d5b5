"""Deterministic synthetic data: splitmix64 streams and CRC-32 checksums.

Host functions restate the reference's generator (/root/reference/pkg/src/segrange/
repro.py:21-53): draw i of stream `seed` mixes ``seed + (i+1) * 0x9E3779B97F4A7C15``;
unit doubles are ``(bits >> 11) * 2^-53``.  ``fill_*`` functions are the device twin
(libdrk ``drk_generate``): they write the same values straight into a distributed
vector's segments, bit-identical to generating on the host and casting with
``astype``, so 2^30-element inputs never cross PCIe.
"""

from __future__ import annotations

import zlib

import numpy as np

from . import _lib

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws [start, start+count) of the splitmix64 stream for seed."""
    if count < 0:
        raise ValueError("count must be non-negative")
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        return z ^ (z >> np.uint64(31))


def unit_doubles(seed: int, start: int, count: int) -> np.ndarray:
    return (splitmix64(seed, start, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_doubles(seed: int, start: int, count: int, lo: float, hi: float) -> np.ndarray:
    return lo + (hi - lo) * unit_doubles(seed, start, count)


def canonical_bytes(arr: np.ndarray) -> bytes:
    a = np.ascontiguousarray(arr)
    return a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()


def checksum(arr) -> str:
    """CRC-32 of the little-endian bytes, 8 hex digits (repro.py:43-53)."""
    if np.isscalar(arr) or (isinstance(arr, np.ndarray) and arr.ndim == 0):
        arr = np.asarray([arr])
    return format(zlib.crc32(canonical_bytes(np.asarray(arr))) & 0xFFFFFFFF, "08x")


# ---- device twins ----------------------------------------------------------------------

def _generate(vec, seed, start, kind, a, b):
    rt = vec.runtime
    rt._check_compute()
    code = _lib.dtype_code(vec.dtype)
    used = {}
    for h, d in zip(vec.storage, vec.distribution.descriptors):
        if not d.length:
            continue
        st = rt.state_of(d.rank)
        _lib.call("drk_generate", code, h.data_ptr(), d.length, seed & 0xFFFFFFFFFFFFFFFF,
                  start + d.global_offset, kind, float(a), float(b), st.index, st.handle)
        used[st.index] = st
    for st in used.values():
        st.synchronize()
    return vec


def fill_unit(vec, seed: int, start: int = 0):
    """vec[i] = dtype(unit_doubles(seed, start, n)[i])."""
    return _generate(vec, seed, start, _lib.GEN_UNIFORM, 0.0, 1.0)


def fill_uniform(vec, seed: int, start: int, lo: float, hi: float):
    """vec[i] = dtype(uniform_doubles(seed, start, n, lo, hi)[i])."""
    return _generate(vec, seed, start, _lib.GEN_UNIFORM, lo, hi)


def fill_mod(vec, seed: int, start: int, modulus: int, offset: int):
    """vec[i] = dtype(int64(splitmix64(seed, start, n)[i] % modulus) + offset)."""
    return _generate(vec, seed, start, _lib.GEN_MOD, float(modulus), float(offset))
