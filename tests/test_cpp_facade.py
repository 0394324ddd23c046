"""The C++ facade (include/randnla_b200/randnla.hpp) compiles against the C
ABI, and (on a GPU) passes the reference's own unit checks restated in C++."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1505_07570_b200", "_lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")


def build(tmp_path):
    exe = str(tmp_path / "test_facade")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe, "-L", LIBDIR,
                    "-lrnla_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_reference_checks(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "facade ok" in out.stdout
