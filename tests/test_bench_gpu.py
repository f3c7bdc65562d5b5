"""bench.py on the GPU: the single-process multi-GPU (shp) mode in its shared-GPU test mode
(every GPU's segment on GPU 0), and the named C1 workload; one JSON line each."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=e)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_shp_two_gpus_shared_mode():
    steps = 3
    d = _bench("--gpus", "2", "--steps", str(steps), "--warmup", "3", "--log2n", "20", "--no-e2e", "--no-cpu",
               env={"DRK_BENCH_SHARE_GPU": "1"})
    assert d["n_gpus"] == 2 and d["config"]["mode"].startswith("shp")
    assert d["config"]["global_elements"] == 2 << 20 and d["config"]["devices"] == [0]
    assert d["workloads"]["triad"]["launches"] == 2 * steps  # both locales' kernels
    assert d["gpu_launches"] >= 4 * steps and d["checks"]["dot_mean_ok"]
    assert d["value"] > 0 and d["elements_per_s"] > 0


def test_bench_c1_named_workload():
    d = _bench("--workloads", "dot", "--log2n", "24", "--segments", "2", "--steps", "20", "--warmup", "5",
               "--no-cpu", "--e2e-log2n", "24")
    assert d["n_gpus"] == 1 and d["config"]["segments_per_gpu"] == 2
    assert d["workloads"]["dot"]["bytes_per_launch"] == 8 << 24  # one batched launch for both segments
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4 << 24


def test_bench_fused_scan_workloads():
    d = _bench("--workloads", "scan_affine,scan_product", "--log2n", "24", "--steps", "5", "--warmup", "3",
               "--no-cpu", "--no-e2e")
    assert d["workloads"]["scan_affine"]["launches"] == 5 and d["workloads"]["scan_product"]["launches"] == 5
    assert d["workloads"]["scan_product"]["kernel"] == "drk_scan_view:product"
