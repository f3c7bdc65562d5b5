"""The L2 scan's experiment knobs (drk_tune; all off by default, DESIGN.md §3 "Small and mid
sizes") keep the scan exact when forced on: the two-launch schedule (scan_2p_*: a reduce-and-
publish launch, then a scan launch with every aggregate published), the early look-back
snapshot (scan_lb_snap) and the output-store L2 policies (scan_rescan_pol bits 2-3).  Checked
against the oracle on int32 data (bit-exact) at sizes that take the L2 kernel with 80 KB and
160 KB tiles, plain and exclusive, one segment and several."""

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import _lib, algorithms as A
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu

KNOBS = {
    "two_launch": {"scan_2p_lo_kb": 1, "scan_2p_hi_kb": 1 << 22},
    "lb_snapshot": {"scan_lb_snap": 1},
    "store_evict_normal": {"scan_rescan_pol": 4},
    "store_evict_last": {"scan_rescan_pol": 8},
}


@pytest.fixture(scope="module")
def rt1():
    with sr.Runtime(1) as rt:
        yield rt


@pytest.fixture(scope="module")
def rt3():
    with sr.Runtime(3) as rt:
        yield rt


@pytest.fixture(params=sorted(KNOBS))
def knob(request):
    lib = _lib.load()
    old = {k: lib.drk_tune(k.encode(), v) for k, v in KNOBS[request.param].items()}
    yield request.param
    for k, v in old.items():
        lib.drk_tune(k.encode(), v)


def _data(n, seed):
    return ((np.arange(n, dtype=np.int64) * 2654435761 + seed) % 2001 - 1000).astype(np.int32)


@pytest.mark.parametrize("n", [(1 << 22) + 4099, (1 << 25) + 77])
@pytest.mark.parametrize("exclusive", [False, True])
def test_knob_scan_exact(rt1, knob, n, exclusive):
    x = _data(n, 11)
    v = sr.DistributedVector.from_numpy(rt1, x)
    out = sr.DistributedVector(rt1, n, init=0, dtype=np.int32)
    if exclusive:
        A.exclusive_scan(v, out, 7)
    else:
        A.inclusive_scan(v, out)
    exp, _ = O.scan(x, 1, exclusive=exclusive, init=7 if exclusive else None)
    assert np.array_equal(out.to_numpy(), exp)


def test_knob_scan_segments(rt3, knob):
    n = 3 * (1 << 22) + 5
    x = _data(n, 3)
    v = sr.DistributedVector.from_numpy(rt3, x)
    out = sr.DistributedVector(rt3, n, init=0, dtype=np.int32)
    A.inclusive_scan(v, out)
    exp, _ = O.scan(x, 3)
    assert np.array_equal(out.to_numpy(), exp)
