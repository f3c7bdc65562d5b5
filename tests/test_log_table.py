"""The table-driven fp64 log behind the reference-precision Black-Scholes kernel
(drk_device.cuh log_tab, table csrc/drk_log_table.inc from tools/fit/fit_log_tab.py): the header
matches the committed fit, and the host restatement of the kernel's operation sequence
(tools/fit/log_tab_check.c) stays within its accuracy bounds against glibc's logl."""

import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIT = os.path.join(ROOT, "tools", "fit")
INC = os.path.join(ROOT, "paper_2406_00158_b200", "csrc", "drk_log_table.inc")


def test_table_header_matches_fit():
    rows, poly, ln2 = {}, None, None
    for line in open(os.path.join(FIT, "log_6.txt")):
        f = line.split()
        if f[0] == "T":
            rows[int(f[1])] = [float.fromhex(v) for v in f[2:]]
        elif f[0] == "P":
            poly = [float.fromhex(v) for v in f[1:]]
        elif f[0] == "LN2":
            ln2 = [float.fromhex(v) for v in f[1:]]
    src = open(INC).read()
    pairs = src.split("k_log_tab[128] = {", 1)[1].split("};", 1)[0].strip().splitlines()
    lo = src.split("k_log_lo[128] = {", 1)[1].split("}", 1)[0].split(", ")
    consts = src.split("k_log_c[2 + DRK_LOG_NP] = {", 1)[1].split("}", 1)[0].split(", ")
    assert len(pairs) == 128
    for i, line in enumerate(pairs):
        a, b = line.strip().strip(",").strip("{}").split(", ")
        assert [float.fromhex(a), float.fromhex(b), float.fromhex(lo[i])] == rows[i]
    assert [float.fromhex(v) for v in consts] == ln2 + poly
    # c = 1 on the intervals touching 1 (arguments near 1 keep full relative accuracy)
    assert rows[79][:2] == [1.0, 0.0] and rows[80][:2] == [1.0, 0.0]


def test_host_restatement_accuracy(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    exe = str(tmp_path / "log_tab_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(FIT, "log_tab_check.c"), "-lm"], check=True)
    s = json.loads(subprocess.run([exe, os.path.join(FIT, "log_6.txt"), "400000"], check=True, capture_output=True,
                                  text=True).stdout)
    assert s["special_bad"] == 0 and s["correctly_rounded"] >= 0.998 and s["max_ulp"] < 0.75
