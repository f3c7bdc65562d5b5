"""The piecewise fp64 erf behind the reference-precision Black-Scholes kernel
(drk_device.cuh erf_pw, table csrc/drk_erf_table.inc fitted by tools/fit/fit_erf_pw.py).

CPU: the table header matches the committed fit, and the host restatement of the kernel's
operation sequence (tools/fit/erf_pw_check.c) stays within its accuracy bounds against glibc's
long-double erfl.  GPU: the device function (reached through a traced scipy.special.erf on
float64) is bit-identical to that restatement."""

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIT = os.path.join(ROOT, "tools", "fit")
INC = os.path.join(ROOT, "paper_2406_00158_b200", "csrc", "drk_erf_table.inc")


def _harness(tmp_path, n, dump=None):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    exe = str(tmp_path / "erf_pw_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(FIT, "erf_pw_check.c"), "-lm"], check=True)
    args = [exe, os.path.join(FIT, "pw8_8.txt"), str(n)] + ([dump] if dump else [])
    return json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)


def test_table_header_matches_fit():
    rows, deg = {}, None
    for line in open(os.path.join(FIT, "pw8_8.txt")):
        f = line.split()
        if f[0] == "DEG":
            deg = int(f[1])
        elif f[0] == "I":
            v = [float.fromhex(t) for t in f[3:]]
            rows[int(f[1])] = v[2:] + [v[1], v[0]]  # coefficients, lo, hi: the kernel's order
    src = open(INC).read()
    body = src.split("k_erf_p[DRK_ERF_NPAIR][DRK_ERF_ROWS] = {", 1)[1].split("};", 1)[0].strip().splitlines()
    pairs = [[[float.fromhex(t) for t in cell.split(", ")] for cell in line.strip().strip(",")[2:-2].split("}, {")]
             for line in body]
    assert len(pairs) == (deg + 3 + 1) // 2 and all(len(p) == 64 for p in pairs)
    for i, want in rows.items():
        got = [x for j in range(len(pairs)) for x in pairs[j][i]][: len(want)]
        assert got == want, i
    assert "#define DRK_ERF_HI_LIMIT 0x4017c000" in src


def test_host_restatement_accuracy(tmp_path):
    s = _harness(tmp_path, 400_000)
    assert s["special_bad"] == 0
    assert s["correctly_rounded"] >= 0.96
    assert s["max_ulp"] < 1.5 and s["boundary_max_ulp"] < 1.0


@pytest.mark.gpu
def test_device_erf_matches_restatement(tmp_path):
    from scipy.special import erf
    import paper_2406_00158_b200 as sr

    dump = str(tmp_path / "erf.bin")
    _harness(tmp_path, 1 << 18, dump)
    x, host, _ = np.fromfile(dump).reshape(-1, 3).T
    rt = sr.Runtime(1)
    try:
        special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e300, -1e300, 5.875, -5.86, 0.125, 0.375])
        xs = np.concatenate([x, special])
        v = sr.DistributedVector.from_numpy(rt, xs)
        out = sr.DistributedVector(rt, len(xs), dtype=np.float64)
        sr.transform(v, out, lambda t: erf(t))
        dev = out.to_numpy()
    finally:
        rt.close()
    np.testing.assert_array_equal(dev[: len(x)].view(np.int64), host.view(np.int64))
    sp = dev[len(x):]
    assert sp[0] == 0.0 and not np.signbit(sp[0]) and sp[1] == 0.0 and np.signbit(sp[1])
    assert sp[2] == 1.0 and sp[3] == -1.0 and np.isnan(sp[4])
    assert sp[5] == 5e-324 * 1.1283791670955126 or sp[5] == erf(5e-324)
    assert sp[6] == 1.0 and sp[7] == -1.0 and sp[8] == 1.0 - 2.0**-53  # erfc(5.875) = 9.7e-17 > 2^-54
    np.testing.assert_allclose(sp[9:], erf(special[9:]), rtol=3e-16)
