"""The C++ drop-in facade (include/dba/dba_b200.hpp) compiles against the C ABI
and behaves like the reference's dba:: API (host parts on CPU, the solve on GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2112_01349_b200")
EXE = os.path.join(ROOT, "build", "facade_test")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_main.cpp"), "-L", LIBDIR, "-ldbag",
                    f"-Wl,-rpath,{LIBDIR}", "-o", EXE], check=True)
    return EXE


def test_facade_host_parts():
    out = subprocess.run([build(), "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
def test_facade_solve_on_gpu():
    out = subprocess.run([build(), "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "facade gpu ok" in out.stdout
