"""CUDA code generation + NVRTC for traced expressions outside the AOT catalogue."""

from __future__ import annotations


class JitUnavailable(TypeError):
    pass


def run_map(writes, leaves, ptrs, n, launch):
    raise JitUnavailable(f"no device kernel for this element expression yet: {[w[1] for w in writes]}")


def run_reduce(node, leaves, ptrs, n, opcode, combiner, launch, slot):
    raise JitUnavailable(f"no device kernel for this reduction yet: {node}")


def custom_scan(rt, in_segs, out_segs, live, op, exclusive, init, carry=None):
    raise JitUnavailable("no device kernel for a scan with a custom operator yet")
