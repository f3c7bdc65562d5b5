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
