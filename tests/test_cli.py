"""The chainscan-compatible command line (test_bench_cli.py's shape):
usage errors on CPU; records, formats, fault injection and exit codes on
the device."""

import csv
import io
import json

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
