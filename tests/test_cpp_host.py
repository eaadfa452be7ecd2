"""The C++ host mirror (include/pairamg_b200.hpp) compiles against the C ABI
(CPU) and, on a GPU, runs the reference usage flow end to end."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "example")


def build_example():
    from paper_2303_02352_b200 import build

    build.build()
    pkg = os.path.join(ROOT, "paper_2303_02352_b200")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "example.cpp"), "-o", EXE, "-L", pkg, "-lpairamg_b200",
           f"-Wl,-rpath,{pkg}"]
    subprocess.run(cmd, check=True)
    return EXE


def test_cpp_header_compiles():
    assert os.path.exists(build_example())


@pytest.mark.gpu
def test_cpp_example_runs():
    exe = build_example()
    r = subprocess.run([exe, "24"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "operator complexity" in r.stdout and "iterations" in r.stdout
