"""CLI surface (paper_2307_05389_b200.cli), modelled on the reference's
tests/test_cli.py: binary endpoint wire format, exit codes, bench table
schema.  Cases that never reach a kernel run on CPU; round trips are gpu."""

import subprocess
import sys

import numpy as np
import pytest

from paper_2307_05389_b200.bench import CSV_HEADER, BenchConfig, BenchRow, emit_table, generate_data
from paper_2307_05389_b200.cli import main


def le(a):
    return a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()


def run_endpoint(tmp_path, payload, args):
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    src.write_bytes(payload)
    return main(["downsample", *args, "--input", str(src), "--output", str(dst)]), dst


def read_indices(path):
    return np.fromfile(path, dtype=np.dtype(np.uint64).newbyteorder("<"))


def test_features_report(capsys):
    assert main(["features"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].startswith("device: ")
    assert lines[1:] == ["levels: sm_100a", "selected: sm_100a"]
    assert main(["bench", "features"]) == 0


def test_endpoint_truncated_stream(tmp_path, capsys):
    code, _ = run_endpoint(tmp_path, b"\x00" * 79,
                           ["--algo", "minmax", "--dtype", "f64", "--count", "10", "--n-out", "2"])
    assert code == 1
    assert capsys.readouterr().err.strip() == "truncated input stream"


def test_endpoint_core_error_text_verbatim(tmp_path, capsys):
    code, _ = run_endpoint(tmp_path, le(np.zeros(10)),
                           ["--algo", "minmax", "--dtype", "f64", "--count", "10", "--n-out", "3"])
    assert code == 1
    assert capsys.readouterr().err.strip() == "n_out must be a multiple of 2"


def test_endpoint_unknown_algorithm(tmp_path, capsys):
    code, _ = run_endpoint(tmp_path, le(np.zeros(4)),
                           ["--algo", "mean", "--dtype", "f64", "--count", "4", "--n-out", "2"])
    assert code == 1
    assert capsys.readouterr().err.strip() == "unknown algorithm: 'mean'"


def test_endpoint_identity_needs_no_gpu(tmp_path):
    # len <= n_out returns arange(len) before any kernel (algorithms.py:126-127)
    code, dst = run_endpoint(tmp_path, le(np.arange(6, dtype=np.float32)),
                             ["--algo", "m4", "--dtype", "f32", "--count", "6", "--n-out", "8"])
    assert code == 0
    assert read_indices(dst).tolist() == list(range(6))


def test_endpoint_missing_input_file_exits_1(tmp_path, capsys):
    code = main(["downsample", "--algo", "minmax", "--dtype", "f64", "--count", "4", "--n-out", "2",
                 "--input", str(tmp_path / "absent.bin")])
    assert code == 1
    assert "absent.bin" in capsys.readouterr().err


@pytest.mark.parametrize("argv", [
    ["downsample", "--dtype", "f64", "--count", "4", "--n-out", "2"],
    ["downsample", "--algo", "minmax", "--dtype", "f128", "--count", "4", "--n-out", "2"],
    ["downsample", "--algo", "minmax", "--dtype", "f64", "--x-dtype", "f16", "--count", "4", "--n-out", "2"],
    ["bench", "--sizes", "1e6"],
    ["nonsense"],
])
def test_invocation_errors_exit_2(argv):
    with pytest.raises(SystemExit) as exc:
        main(argv)
    assert exc.value.code == 2


def test_bench_unknown_algorithm_exits_1(capsys):
    assert main(["bench", "--algos", "median", "--quiet"]) == 1
    assert "unknown algorithm: median" in capsys.readouterr().err


def test_bench_table_schema():
    rows = [BenchRow("f64", "m4", True, 100, 1.5, 0.25), BenchRow("f32", "minmax", False, 100, error="boom")]
    assert emit_table(rows).splitlines() == [CSV_HEADER, "f32,minmax,false,100,,", "f64,m4,true,100,1.500000,0.250000"]
    md = emit_table(rows, "markdown").splitlines()
    assert md[0] == "| dtype | n | minmax (sequential) | m4 (parallel) |"
    with pytest.raises(ValueError, match="repeats must be >= 3"):
        BenchConfig(repeats=2).validate()
    a, b = generate_data("i8", 5000, 3), generate_data("i8", 5000, 3)
    assert np.array_equal(a, b) and a.min() == -128 and a.max() == 127


@pytest.mark.gpu
def test_bench_csv_to_file(tmp_path, capsys):
    out = tmp_path / "rows.csv"
    assert main(["bench", "--dtypes", "f32", "--sizes", "600", "--n-out", "50", "--algos", "minmax",
                 "--parallel", "false", "--repeats", "3", "--quiet", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 2
    dtype, algo, par, n, med, std = lines[1].split(",")
    assert (dtype, algo, par, n) == ("f32", "minmax", "false", "600")
    assert float(med) > 0 and float(std) >= 0
    assert capsys.readouterr().out == ""
