"""The C++ facade (include/randnla_b200/randnla.hpp) compiles against the C
ABI, and (on a GPU) passes the reference's own unit checks and its hot-path
acceptance criteria 3, 5, 6 and 10 restated in C++ (tests/cpp/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1505_07570_b200", "_lib")
SOURCES = {"facade": os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"),
           "acceptance": os.path.join(ROOT, "tests", "cpp", "test_acceptance.cpp")}


def build(tmp_path, name):
    exe = str(tmp_path / f"test_{name}")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SOURCES[name], "-o",
                    exe, "-L", LIBDIR, "-lrnla_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


@pytest.mark.parametrize("name", sorted(SOURCES))
def test_facade_compiles_and_links(tmp_path, name):
    assert os.path.exists(build(tmp_path, name))


@pytest.mark.gpu
def test_facade_runs_reference_checks(tmp_path):
    exe = build(tmp_path, "facade")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
def test_facade_acceptance_criteria_3_5_6_10(tmp_path):
    exe = build(tmp_path, "acceptance")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "acceptance ok" in out.stdout
