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
