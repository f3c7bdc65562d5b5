"""bench.py contract pieces that run without a GPU: the reference arm prints one JSON
line with the driver's keys (the CPU path of the reference, via the oracle port)."""

import json
import os

import pytest
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--cpu-log2n", "16", "--log2n", "16"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["config"]["same_size_as_gpu_arm"] and d["config"]["elements_per_step"] == 1 << 16
    assert d["cpu_baseline"]["cpu"] and d["elements_per_s"] > 0


# ----------------------------------------------------------------------------------------
# multi-GPU launch plumbing (bench.py --gpus N)


def test_launch_mode_shp_without_torchrun():
    import bench

    assert bench.launch_mode(4, env={}) == ("shp", 4)
    assert bench.launch_mode(1, env={"WORLD_SIZE": "1"}) == ("shp", 1)
    assert bench.launch_mode(8, env={"WORLD_SIZE": "8", "RANK": "3"}) == ("spmd", 8)


def test_shp_layout():
    import bench

    assert bench.shp_layout(4, 1, 8) == ([0, 1, 2, 3], 4)
    assert bench.shp_layout(2, 3, 2) == ([0, 1], 6)        # segment k on GPU k mod 2
    assert bench.shp_layout(2, 1, 1, share=True) == ([0], 2)
    with pytest.raises(SystemExit):
        bench.shp_layout(4, 1, 1)                           # never silently fewer GPUs


def test_parse_defaults():
    import bench

    a = bench.parse([])
    assert (a.gpus, a.segments, a.log2n, a.share_gpu) == (1, 1, 30, False)
    a = bench.parse(["--gpus", "8", "--segments", "2", "--share-gpu"])
    assert (a.gpus, a.segments, a.share_gpu) == (8, 2, True)
