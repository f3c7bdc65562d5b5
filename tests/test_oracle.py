"""The oracle (oracle/segrange_port.py) is pinned to the real reference: every golden
case produced by tests/golden/make_golden.py (which ran segrange itself) must be
reproduced bit-for-bit by the CPU restatement."""

import numpy as np
import pytest

from conftest import dec, golden
from oracle import segrange_port as O

CASES = golden().cases
SORT_KEYS = {"none": None, "abs": np.abs, "neg": np.negative}


def _ids(cases):
    return [c["id"] for c in cases]


def _run(case):
    dt = np.dtype(case["dtype"])
    ins = [O.generate(d, dt) for d in case["inputs"]]
    op = case["op"]
    if op == "dot":
        return O.dot(ins[0], ins[1], case["p"]), None
    if op == "reduce":
        init = dec(case["init"])
        return O.reduce(ins[0], case["p"], init, getattr(np, case["ufunc"])), None
    if op == "triad":
        return None, O.triad(ins[0], ins[1], case["alpha"], case["p"])
    if op in ("inclusive_scan", "exclusive_scan"):
        uf = getattr(np, case.get("ufunc", "add"))
        out, parts = O.scan(ins[0], case["p"], dt, op == "exclusive_scan", dec(case["init"]), uf)
        return parts, out
    if op == "black_scholes":
        return None, O.black_scholes_prices(ins, dt, case["p"])
    if op == "copy":
        return None, ins[0].copy()
    if op == "reduce_view":
        n, p = case["n"], case["p"]
        lens = O.trimmed_lengths(O.block_lengths(n, p), case["drop"], case["drop"] + case["take"])
        x = ins[0][case["drop"]: case["drop"] + case["take"]]
        return O.reduce(x, len(lens), 0, np.add, lengths=lens), None
    if op == "dot_nonaligned":
        lens = O.realigned_lengths(*case["parts"])
        return O.reduce(ins[0] * ins[1], len(lens), 0.0, np.add, lengths=lens), None
    if op == "scan_view":
        out, _ = O.scan(ins[0] * 3 - 1, case["p"], dt)
        return None, out
    if op == "copy_transform":
        return None, (ins[0] * 7 - 3) if dt.kind == "i" else (ins[0] * 2.5 + 1)
    if op == "sort":
        return None, O.sample_sort(ins[0], case["p"], SORT_KEYS[case["key"]])
    raise AssertionError(op)


@pytest.mark.parametrize("case", [c for c in CASES if "raises" not in c], ids=_ids([c for c in CASES if "raises" not in c]))
def test_oracle_matches_reference(case):
    g = golden()
    scalar, array = _run(case)
    if "input_checksums" in case:
        dt = np.dtype(case["dtype"])
        assert [O.checksum(O.generate(d, dt)) for d in case["inputs"]] == case["input_checksums"]
    if "result" in case:
        exp = dec(case["result"])
        assert type(scalar) is type(exp) and scalar == exp
    if "partials" in case:
        assert scalar == [dec(p) for p in case["partials"]]
    if "checksum" in case:
        assert O.checksum(array) == case["checksum"]
        if case.get("array"):
            ref = g.arrays[case["id"]]
            assert ref.dtype == array.dtype and np.array_equal(ref, array)


def test_overflow_case_recorded():
    c = [c for c in CASES if "raises" in c]
    assert c and c[0]["raises"] == "AggregateTaskError:OverflowError"


def test_known_answers():
    kat = golden().meta["kat"]
    assert dec(kat["dot_123_456"]) == 32.0
    assert [str(int(v)) for v in O.splitmix64(42, 0, 5)] == kat["splitmix_seed42_first5"]
    assert O.checksum(np.array([1.5, -2.25])) == kat["checksum_15_m225"]
    assert float(O.black_scholes(100.0, 100.0, 0.0, 0.2, 1.0)) == dec(kat["bs_atm"])
    assert abs(dec(kat["bs_atm"]) - 7.9656) < 1e-3
    assert float(O.black_scholes(110.0, 100.0, 0.0, 0.0, 1.0)) == 10.0


def test_textbook_splitmix():
    # reference tests/test_bench.py:15-36: vectorised stream == scalar textbook splitmix64
    mask = (1 << 64) - 1
    for seed in (0, 1, 42, 2**63):
        state, want = seed & mask, []
        for _ in range(20):
            state = (state + 0x9E3779B97F4A7C15) & mask
            z = state
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
            want.append(z ^ (z >> 31))
        assert O.splitmix64(seed, 0, 20).tolist() == want


def test_hand_examples():
    out, parts = O.scan(np.array([1, 2, 3, 4], dtype=np.int64), 2)
    assert out.tolist() == [1, 3, 6, 10] and parts == [3, 7]
    out, _ = O.scan(np.array([1, 2, 3, 4], dtype=np.int64), 3, exclusive=True, init=0)
    assert out.tolist() == [0, 1, 3, 6]
    out, _ = O.scan(np.array([1, 1], dtype=np.int64), 5, exclusive=True, init=10)
    assert out.tolist() == [10, 11]
    assert O.reduce(np.arange(1, 101, dtype=np.int64), 7) == 5050
