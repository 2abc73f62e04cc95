"""The C++ host API (include/rocp_b200/rocp.hpp) driven like the reference's
own doctest suites (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_api")


def test_cpp_api_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2007_10798_b200")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_api_suite():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=240)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_bench_cli_reports(tmp_path):
    """The reference CLI's `bench` subcommand: the two CSV reports in the reference schema."""
    cli = os.path.join(ROOT, "paper_2007_10798_b200", "_lib", "rocp_bench")
    csv, upd = tmp_path / "r.csv", tmp_path / "u.csv"
    r = subprocess.run([cli, "--dims", "10", "9", "30", "--rank", "3", "--batch", "4", "--trials", "2",
                        "--seed", "5", "--sir-db", "20", "--csv", str(csv), "--updates-csv", str(upd)],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr
    rows = csv.read_text().splitlines()
    assert rows[0] == "trial,algorithm,fitness,init_seconds,stream_seconds,updates,seconds_per_update"
    assert [l.split(",")[0] for l in rows[1:]] == ["0", "1", "mean", "std"]
    assert all(l.split(",")[1] == "rocp" for l in rows[1:])
    assert int(rows[1].split(",")[5]) == 6  # 30 slices, init 6, batches of 4
    assert 0.5 < float(rows[1].split(",")[2]) <= 1.0
    u = upd.read_text().splitlines()
    assert u[0] == "trial,algorithm,update,seconds" and len(u) == 1 + 2 * 6
    bad = subprocess.run([cli, "--dims", "6", "6", "12", "--algorithms", "batch_cold"], capture_output=True,
                         text=True, timeout=60)
    assert bad.returncode == 1 and "baseline" in bad.stderr
