"""drbench CLI (reference cli.py / tests/test_bench.py TestCli): usage errors on any host,
runs and CSV on the GPU."""

import pytest

from paper_2406_00158_b200 import bench as B
from paper_2406_00158_b200.cli import run


def test_unknown_bench_usage_error(capsys):
    assert run(["--bench", "nope", "--size", "10"]) == 2


def test_missing_bench_flag(capsys):
    assert run([]) == 2


def test_bad_reps_value(capsys):
    assert run(["--bench", "dot", "--reps", "0"]) == 2


def test_gemm_is_not_offered(capsys):
    assert run(["--bench", "gemm"]) == 2


@pytest.mark.gpu
def test_successful_run_exits_zero(capsys):
    code = run(["--bench", "dot", "--size", "1000", "--locales", "2", "--reps", "2", "--seed", "7", "--check"])
    out = capsys.readouterr().out
    assert code == 0 and out.count("rep=") == 2 and "verified=yes" in out


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(B.BENCH_NAMES))
def test_each_bench_verifies(name, capsys):
    assert run(["--bench", name, "--size", "3000", "--locales", "3", "--reps", "2", "--seed", "5", "--check"]) == 0


@pytest.mark.gpu
def test_float32_and_strict(capsys):
    assert run(["--bench", "stream", "--size", "2000", "--locales", "2", "--mode", "strict", "--dtype", "float32",
                "--check"]) == 0


@pytest.mark.gpu
def test_csv_written(tmp_path, capsys):
    path = tmp_path / "r.csv"
    assert run(["--bench", "reduce", "--size", "500", "--locales", "2", "--check", "--csv", str(path)]) == 0
    lines = path.read_text().strip().split("\n")
    assert lines[0] == "bench,size,locales,rep,seconds,checksum,verified"
    assert all(l.split(",")[6] == "true" for l in lines[1:])


@pytest.mark.gpu
def test_checksums_identical_across_locale_counts(capsys):
    sums = {B.run_spec(B.BenchSpec(name="inclusive_scan", size=4096, locales=p, reps=1, seed=3)).checksum
            for p in (1, 2, 4, 7)}
    assert len(sums) == 1


@pytest.mark.gpu
def test_verification_failure_exits_one(capsys, monkeypatch):
    monkeypatch.setitem(B.BENCHES, "dot", lambda spec, rt: B.BenchResult(spec, [0.0], "deadbeef", verified=False))
    assert run(["--bench", "dot", "--size", "10", "--locales", "1", "--check"]) == 1
    assert "FAILED" in capsys.readouterr().err


def test_gpu_columns_extend_the_reference_schema():
    spec = B.BenchSpec(name="dot", size=1 << 20, locales=2, reps=2)
    res = B.BenchResult(spec, [0.002, 0.001], "0badf00d", verified=True,
                        extra={"device_seconds": [0.001, 0.0005], "bytes_per_element": 8, "devices": 1})
    rows = B.csv_rows([res], gpu_columns=True)
    head = rows[0].split(",")
    assert rows[0].startswith(B.CSV_HEADER + ",")  # the reference's seven columns first
    assert head[7:] == B.GPU_COLUMNS.split(",")
    f = rows[2].split(",")
    assert f[:7] == ["dot", str(1 << 20), "2", "1", "0.001000000", "0badf00d", "true"]
    assert abs(float(f[8]) - 8 * (1 << 20) / 0.0005 / 1e9) < 1e-3
    assert abs(float(f[9]) - (1 << 20) / 0.0005) / float(f[9]) < 1e-6
    assert abs(float(f[10]) - float(f[8]) / B.hbm_peak_gbs()) < 1e-4
    assert B.csv_rows([res])[0] == B.CSV_HEADER  # default: the reference schema unchanged


@pytest.mark.gpu
def test_csv_gpu_columns_written(tmp_path, capsys):
    path = tmp_path / "g.csv"
    assert run(["--bench", "stream", "--size", "100000", "--locales", "2", "--check", "--csv", str(path),
                "--gpu-columns"]) == 0
    lines = path.read_text().strip().split("\n")
    assert lines[0] == B.CSV_HEADER + "," + B.GPU_COLUMNS
    for l in lines[1:]:
        f = l.split(",")
        assert f[6] == "true" and float(f[7]) > 0 and float(f[8]) > 0 and int(f[11]) >= 1
    assert "GB/s" in capsys.readouterr().out
