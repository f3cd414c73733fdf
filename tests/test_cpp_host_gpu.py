"""The C++ host mirror (include/pnn_b200/tensor_ops.hpp) -- what a C++ user of
the reference switches to -- compiled with g++ against libpnn_b200.so and run
on the B200, checked bit for bit against the oracle restatement."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_host_ops_test(out_dir) -> str:
    pkg = os.path.join(REPO, "paper_2105_00053_b200")
    obj = os.path.join(out_dir, "posit_oracle.o")
    exe = os.path.join(out_dir, "host_ops_test")
    subprocess.run(["gcc", "-std=c11", "-O2", "-c", os.path.join(REPO, "oracle", "posit_oracle.c"), "-o", obj],
                   check=True)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "tests", "cpp", "host_ops_test.cpp"), obj, "-L", pkg, "-lpnn_b200",
                    f"-Wl,-rpath,{pkg}", "-o", exe], check=True)
    return exe


def test_cpp_host_ops(cuda, tmp_path):
    exe = build_host_ops_test(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:] + r.stdout[-1000:]
    assert "host_ops_test: ok" in r.stdout
