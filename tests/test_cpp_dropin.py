"""The C++ host API (include/pathgcn_b200.hpp) as a reference user would
call it: compile here (CPU), run the known-answer checks on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def compile_dropin():
    from oracle.oracle import build_oracle
    from paper_2204_02662_b200 import _lib

    so = _lib.build()
    build_oracle()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    pkg = os.path.dirname(so)
    orc = os.path.join(ROOT, "oracle")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC, "-o", OUT,
           f"-L{pkg}", "-lpathgcn_b200", f"-L{orc}", "-l:liboracle.so", f"-Wl,-rpath,{pkg}:{orc}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return OUT


def test_cpp_header_compiles():
    assert os.path.exists(compile_dropin())


@pytest.mark.gpu
def test_cpp_dropin_runs():
    exe = compile_dropin()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout and r.stdout.count("[PASS]") >= 22
