"""Cross-GPU combine of reduce on the device (Runtime(reduce_combine="device" | "nccl" |
"fused")).

The reference folds per-segment partials on the driver in ascending order
(algorithms.py:146-149).  The device folds (drk_reduce_fold from peer memory, and the NCCL
all-gather + per-GPU fold of drk_comm_reduce) run the same fold in numpy's reduce dtype, so
every golden reduce / dot case must give the host fold's value bit for bit, and the golden
value within the parity tolerance.  On one GPU the NCCL communicator has one rank; the
segment-order bookkeeping (several segments per GPU, padded slots) is the same code that
runs across GPUs.
"""

import numpy as np
import pytest

from conftest import dec, golden

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import _lib, algorithms as A, bench as B, views
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu

CASES = golden().cases
REL = {"float32": 1e-5, "float64": 1e-12}
MODES = ("device", "nccl", "fused")


def _close(got, exp, dtype):
    rel = REL[dtype]
    return abs(got) <= rel if exp == 0 else abs(got - exp) <= rel * abs(exp)


@pytest.fixture(scope="module")
def pools():
    made = {}

    def get(mode, p):
        key = (mode, p)
        if key not in made:
            made[key] = sr.Runtime(p, reduce_combine=mode)
        return made[key]

    yield get
    for rt in made.values():
        rt.close()


def _sel(*ops):
    cs = [c for c in CASES if c["op"] in ops and "raises" not in c]
    return pytest.mark.parametrize("case", cs, ids=[c["id"] for c in cs])


def _run(case, rt):
    dt = np.dtype(case["dtype"])
    if case["op"] == "reduce":
        x = O.generate(case["inputs"][0], dt)
        return A.reduce(sr.DistributedVector.from_numpy(rt, x), dec(case["init"]), getattr(A, case["ufunc"]))
    if case["op"] == "dot":
        x, y = [O.generate(d, dt) for d in case["inputs"]]
        return B.dot_product(sr.DistributedVector.from_numpy(rt, x), sr.DistributedVector.from_numpy(rt, y))
    x = O.generate(case["inputs"][0], dt)
    v = sr.DistributedVector.from_numpy(rt, x)
    return A.reduce(views.take(views.drop(v, case["drop"]), case["take"]), 0, A.add)


@pytest.mark.parametrize("mode", MODES)
@_sel("reduce", "dot", "reduce_view")
def test_device_fold_matches_host_fold(case, mode, pools):
    if mode == "nccl" and not _lib.load().drk_comm_available():
        pytest.fail("libnccl.so.2 is not loadable on a GPU box")
    host = _run(case, pools("host", case["p"]))
    got = _run(case, pools(mode, case["p"]))
    assert type(got) is type(host)
    assert np.array_equal(np.asarray(got), np.asarray(host)), (got, host)  # bit for bit (NaN-safe)
    exp = dec(case["result"])
    if np.dtype(case["dtype"]).kind == "i" or case.get("ufunc") in ("minimum", "maximum"):
        assert got == exp
    else:
        assert _close(got, exp, case["dtype"]), (got, exp)


@pytest.mark.parametrize("mode", MODES)
def test_init_promotion_falls_back_to_host(mode, pools):
    """An init that changes numpy's result dtype (float init over int32, a float64 scalar
    over float32 partials) folds on the host, like the reference."""
    rt = pools(mode, 3)
    xi = np.arange(1, 101, dtype=np.int32)
    vi = sr.DistributedVector.from_numpy(rt, xi)
    r = A.reduce(vi, 0.5, A.add)
    assert r == 5050.5 and isinstance(r, float)
    xf = (np.arange(1000, dtype=np.float32) * np.float32(0.1)).astype(np.float32)
    vf = sr.DistributedVector.from_numpy(rt, xf)
    host = A.reduce(sr.DistributedVector.from_numpy(pools("host", 3), xf), np.float64(0.25), A.add)
    assert A.reduce(vf, np.float64(0.25), A.add) == host


@pytest.mark.parametrize("mode", MODES)
def test_many_segments_and_custom_ops(mode, pools):
    """17 segments (more than one batched launch holds), empty trailing segments, and a
    custom operator (host fold) through a device-combine runtime."""
    rt = pools(mode, 17)
    x = O.mod_ints(5, 0, 10_007, 2001, -1000).astype(np.int32)
    v = sr.DistributedVector.from_numpy(rt, x)
    assert A.reduce(v, 0, A.add) == int(x.astype(np.int64).sum())
    assert A.reduce(v, 7, A.minimum) == min(7, int(x.min()))
    small = sr.DistributedVector.from_numpy(rt, np.arange(5, dtype=np.int64))  # 12 empty segments
    assert A.reduce(small, 10, A.add) == 20
    assert A.reduce(v, 0, lambda a, b: a + b) == int(x.astype(np.int64).sum())


def test_nccl_allgather_one_rank(pools):
    """drk_comm_allgather on a one-GPU communicator copies the words (the all-gather the
    combine is built on)."""
    import ctypes

    import torch

    rt = pools("nccl", 2)
    st = rt.device_states[0]
    src = torch.arange(8, dtype=torch.int64, device=st.device)
    dst = torch.zeros(8, dtype=torch.int64, device=st.device)
    torch.cuda.synchronize()
    vp = ctypes.c_void_p
    _lib.call("drk_comm_allgather", rt.comm(), (vp * 1)(src.data_ptr()), (vp * 1)(dst.data_ptr()), 8,
              (vp * 1)(st.handle))
    st.synchronize()
    assert torch.equal(src, dst)


def test_wait_flags_reports_a_missing_completion(pools):
    """drk_wait_flags on an idle stream whose completion word never arrives returns an error
    instead of spinning forever."""
    rt = pools("host", 2)
    st = rt.device_states[0]
    fh, _ = st.flag_ptrs()
    st.synchronize()
    rc = _lib.load().drk_wait_flags(fh, 1, (1 << 62) + 12345, st.index, st.handle)
    assert rc == _lib.E_ARG and "idle" in _lib.last_error()
