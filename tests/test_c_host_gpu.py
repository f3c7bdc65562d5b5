"""The C ABI used from plain C (examples/c_host.c): dot, triad, a two-segment scan with the
carry passed on the device, the device fold of the dot partials and the radix sort, checked
by the C program itself against host loops."""

import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_c_host_program():
    exe = os.path.join(ROOT, "examples", "c_host")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True, capture_output=True)
    out = subprocess.run([exe, "22"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["triad_mismatches"] == 0 and res["scan_mismatches"] == 0
    assert res["sort_errors"] == 0 and res["device_fold_ok"]
    assert res["launches"] >= 8
