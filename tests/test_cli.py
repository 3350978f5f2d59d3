"""CLI front end (reference tests/test_cli.py contract: CSV header, exit codes)."""

import json

import pytest

from paper_2104_11471_b200.cli import CSV_HEADER, main


def _run(capsys, *argv):
    code = main(list(argv))
    captured = capsys.readouterr()
    return code, captured.out, captured.err


def test_plan_dump_schedules(capsys):
    code, out, _ = _run(capsys, "plan", "--sizes", "131072", "16")
    assert code == 0
    first, second = (json.loads(line) for line in out.strip().splitlines())
    assert first["schedule_x"] == [8192, 16]
    assert second["schedule_x"] == [16]
    assert [p["kind"] for p in first["b200_passes"]] == ["strip", "rowT"]


def test_plan_2d(capsys):
    code, out, _ = _run(capsys, "plan", "--sizes", "512", "--dims", "2", "--ny", "512", "--batch", "4")
    d = json.loads(out)
    assert code == 0 and d["schedule_y"] == [512] and len(d["b200_passes"]) == 2


def test_rejects_non_power_of_two(capsys):
    code, _, err = _run(capsys, "plan", "--sizes", "96")
    assert code == 2 and "96" in err


def test_double_mode_is_usage_error(capsys):
    code, _, err = _run(capsys, "plan", "--sizes", "256", "--mode", "double")
    assert code == 2


def test_fragmap_not_applicable(capsys):
    code, _, err = _run(capsys, "fragmap")
    assert code == 2 and "TMEM" in err


@pytest.mark.gpu
def test_verify_small_size_passes(capsys):
    code, out, _ = _run(capsys, "verify", "--sizes", "16", "256", "4096", "--seed", "1", "--batch", "4")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0] == CSV_HEADER
    kind, n, ny, batch, metric, value = lines[1].split(",")
    assert (kind, n, ny, batch, metric) == ("1d", "16", "", "4", "relative_error")
    assert float(value) < 0.0015


@pytest.mark.gpu
def test_verify_2d_row_format(capsys):
    code, out, _ = _run(capsys, "verify", "--sizes", "64", "--dims", "2", "--ny", "64")
    assert code == 0
    assert out.strip().splitlines()[1].startswith("2d,64,64,1,")


@pytest.mark.gpu
def test_verify_envelope_failure_exits_nonzero(capsys):
    code, _, err = _run(capsys, "verify", "--sizes", "256", "--envelope", "0.0001")
    assert code == 1 and "exceeds" in err


@pytest.mark.gpu
def test_bench_reports_positive_throughput(capsys):
    code, out, _ = _run(capsys, "bench", "--sizes", "65536", "--batch", "8", "--min-time", "0.01")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0] == CSV_HEADER
    kind, n, _, batch, metric, value = lines[1].split(",")
    assert (kind, n, batch, metric) == ("1d", "65536", "8", "tflops") and float(value) > 0
