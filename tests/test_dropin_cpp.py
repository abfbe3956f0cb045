"""The C++ drop-in headers (include/blockmask/*.hpp) against the reference's own test cases.

CPU: the test program compiles and links against libbbm with the reference's C++20 dialect (the
headers are a drop-in for proj/include/blockmask). GPU: the program runs on the B200 and every
case passes (tests/cpp/test_dropin.cpp cites the reference test each case mirrors).
"""
import os
import subprocess

import pytest

from tests.conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2409_15097_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lbbm", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True,
                   capture_output=True, text=True)
    return exe


def test_dropin_headers_compile_and_link(tmp_path):
    assert os.path.exists(build(tmp_path))


def test_dropin_headers_fail_loudly_without_device(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode != 0 and "FAIL" in r.stdout  # no CPU fallback behind the headers


@pytest.mark.gpu
def test_dropin_reference_cases_pass_on_gpu(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
