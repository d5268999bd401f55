"""The C++ boundary: tests/native/shim_check.cpp is compiled against include/expmc_b200.hpp and
linked to the in-tree libexpmc_b200.so, then run -- host-only checks on the CPU container,
the full set (run_level / mlmc_driver / exception types through the C-ABI) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1904_12754_b200", "_lib")


def _build(tmp_path):
    exe = tmp_path / "shim_check"
    subprocess.run(["/usr/bin/g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "shim_check.cpp"), "-L", LIBDIR, "-lexpmc_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return str(exe)


def test_cpp_shim_host(tmp_path):
    r = subprocess.run([_build(tmp_path), "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_shim_gpu(gpu, tmp_path):
    r = subprocess.run([_build(tmp_path), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
