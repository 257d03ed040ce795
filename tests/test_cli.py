"""The chainscan-compatible command line (test_bench_cli.py's shape):
usage errors on CPU; records, formats, fault injection and exit codes on
the device."""

import csv
import io
import json

import numpy as np
import pytest

from paper_1604_04815_b200.cli import main
from paper_1604_04815_b200.records import CSV_COLUMNS, EXTENDED_COLUMNS


def test_csv_columns_pinned():
    # test_bench_cli.py:27-32
    assert CSV_COLUMNS == [
        "algorithm", "dtype", "op", "n", "workers", "warp_width", "k",
        "warps_per_block", "runs", "best_seconds", "mean_seconds", "geps",
        "validated", "in_place",
    ]
    assert EXTENDED_COLUMNS[:len(CSV_COLUMNS)] == CSV_COLUMNS


@pytest.mark.parametrize("argv", [["--runs", "0"], ["--n", "-5"], ["--workers", "0"],
                                  ["--algo", "blelloch"], ["simulate"]])
def test_usage_errors_exit_2(argv, capsys):
    assert main(argv) == 2
    assert "error" in capsys.readouterr().err


def test_argparse_rejects_bad_dtype():
    with pytest.raises(SystemExit) as e:
        main(["--dtype", "u8"])
    assert e.value.code == 2


@pytest.mark.gpu
def test_records_csv_json_and_validation(capsys):
    assert main(["--n", "1000", "--n", "100000", "--runs", "2", "--dtype", "i64", "--op", "max"]) == 0
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))
    assert rows[0] == CSV_COLUMNS and len(rows) == 3
    rec = dict(zip(rows[0], rows[1]))
    assert rec["algorithm"] == "chained" and rec["dtype"] == "i64" and rec["op"] == "max"
    assert rec["validated"] == "true" and rec["in_place"] == "false" and int(rec["n"]) == 1000
    assert main(["--n", "4097", "--format", "json", "--extended", "--timing", "device", "--in-place"]) == 0
    js = json.loads(capsys.readouterr().out)
    assert js[0]["validated"] == "true" and js[0]["in_place"] == "true" and js[0]["impl"] == "lscan-b200"
    assert js[0]["geps"] == pytest.approx(js[0]["n"] / js[0]["best_seconds"] * 1e-9)
    for tok in ("f32", "f64"):
        assert main(["--n", "300001", "--dtype", tok, "--exclusive"]) == 0


@pytest.mark.gpu
def test_inject_slot_fault_exits_1(capsys):
    # test_bench_cli.py:215-224
    assert main(["--n", "50000", "--inject-slot-fault", "2"]) == 1
    out = capsys.readouterr()
    assert "validation failed" in out.err
    assert "false" in out.out


@pytest.mark.gpu
def test_output_io_error_exits_3(tmp_path):
    assert main(["--n", "1000", "--output", str(tmp_path / "missing" / "x.csv")]) == 3
    path = tmp_path / "r.csv"
    assert main(["--n", "1000", "--output", str(path)]) == 0
    assert path.read_text().splitlines()[0] == ",".join(CSV_COLUMNS)


def test_host_check_agrees_with_oracle_rule(oracle_lib):
    # records.host_check is the reference's rule (bench.py:95-114): on correct
    # results and on perturbed ones it agrees with the oracle's validate_output
    from paper_1604_04815_b200.records import host_check
    for tok in ("i32", "i64", "f32", "f64"):
        x = oracle_lib.generate_input(5000, tok, [4, len(tok) + ord(tok[0])])
        y = oracle_lib.sequential_scan(x)
        assert host_check(x, y) is None and oracle_lib.validate_output(x, y) is None
        bad = y.copy()
        bad[1234] = bad[1234] + (1 if tok[0] == "i" else np.float32(0.05))
        assert "1234" in host_check(x, bad) and oracle_lib.validate_output(x, bad) is not None
        ex = np.concatenate([[0], y[:-1]]).astype(x.dtype)
        assert host_check(x, ex, exclusive=True) is None
        assert host_check(x, y, exclusive=True) is not None


def test_host_check_compares_bits_for_max_min():
    # stricter than np.array_equal: a -0 / +0 swap or a different NaN payload fails
    from paper_1604_04815_b200.records import host_check
    x = np.array([-0.0, 0.0, -1.0, np.nan, 2.0], dtype=np.float32)
    y = np.maximum.accumulate(x)
    assert host_check(x, y, "max") is None
    swapped = y.copy()
    swapped[1] = -0.0  # max(-0, +0) is +0 (numpy keeps the right operand on ties)
    assert swapped[1] == y[1] and host_check(x, swapped, "max") is not None
    payload = y.copy()
    payload.view(np.uint32)[3] ^= 1  # another NaN
    assert np.isnan(payload[3]) and host_check(x, payload, "max") is not None
    assert host_check(x, np.minimum.accumulate(x), "min") is None


def test_reference_geometry_flags_validated(capsys):
    # WarpGeometry's rules (warp.py:42-82) and CHAINSCAN_WORKERS (cli.py:99-110)
    assert main(["--warp-width", "3", "--n", "8"]) == 2
    assert main(["--warp-width", "128", "--n", "8"]) == 2
    assert main(["--k", "0", "--n", "8"]) == 2
    assert main(["--warps-per-block", "33", "--n", "8"]) == 2
    with pytest.raises(SystemExit) as e:
        main(["--algo", "bogus"])
    assert e.value.code == 2
    capsys.readouterr()


@pytest.mark.gpu
@pytest.mark.parametrize("plant", ["sign_of_zero", "nan_payload"])
def test_planted_tie_error_exits_1(monkeypatch, capsys, plant):
    # the device result is bit-exact on zeros and NaNs (exit 0); the same run
    # with one planted -0/+0 swap or NaN payload change must exit 1
    import paper_1604_04815_b200.cli as C
    base = np.array([0.0, -0.0, 0.0, 0.5, -2.0, np.nan, 1.0, -0.0] * 1000, dtype=np.float32)
    base.view(np.uint32)[5::8] |= 0x1234  # NaN payloads
    monkeypatch.setattr(C, "generate_input", lambda n, tok, seed: base[:n].copy())
    assert main(["--n", "8000", "--dtype", "f32", "--op", "max", "--runs", "1"]) == 0
    real = C.chained_scan

    def planted(problem, config=None):
        y = real(problem, config)
        if plant == "sign_of_zero":
            z = np.nonzero(y == 0)[0][0]
            y.view(np.uint32)[z] ^= 0x80000000
        else:
            k = np.nonzero(np.isnan(y))[0][0]
            y.view(np.uint32)[k] ^= 1
        return y

    monkeypatch.setattr(C, "chained_scan", planted)
    assert main(["--n", "8000", "--dtype", "f32", "--op", "max", "--runs", "1"]) == 1
    assert "validation failed" in capsys.readouterr().err
