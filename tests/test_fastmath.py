"""The sampler's table-driven fp64 log (csrc/fastmath.cuh) against a long-double reference on the
sampler's argument distribution x = 1 - u (u = k 2^-53), near 1 and near 0.  The host build
runs the identical fma sequence as the device (tests/test_gpu_parity.py covers the device)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fast_log_within_one_ulp(tmp_path):
    exe = tmp_path / "fastlog_check"
    csrc = os.path.join(ROOT, "paper_1904_12754_b200", "csrc")
    subprocess.run(["/usr/bin/g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", csrc,
                    os.path.join(ROOT, "tests", "native", "fastlog_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "3000000"], check=True, capture_output=True, text=True).stdout.split()
    worst, checked = float(out[0]), int(out[1])
    assert checked > 4_000_000
    assert worst <= 1.0, out


def test_holding_test_rewrites_host(tmp_path):
    """walker.cuh S-mode (1 - u > S, S <- S / (1 - u)) decides every event like the reference's
    u < -expm1(-rate*remaining) / remaining -= -log1p(-u)/rate sequence on the same draws, and
    ed_walker.cuh's closed-form first-hold threshold never claims a hold the full event would
    reject (tests/native/hold_check.cpp)."""
    exe = tmp_path / "hold_check"
    csrc = os.path.join(ROOT, "paper_1904_12754_b200", "csrc")
    subprocess.run(["/usr/bin/g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", csrc,
                    os.path.join(ROOT, "tests", "native", "hold_check.cpp"), "-o", str(exe)], check=True)
    mism, events, viol, checks = map(int, subprocess.run([str(exe), "400000"], check=True, capture_output=True,
                                                         text=True).stdout.split())
    assert events > 1_000_000 and mism == 0
    assert checks > 500_000 and viol == 0
