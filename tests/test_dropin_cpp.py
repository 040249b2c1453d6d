"""The C++ drop-in (include/msc_b200/dropin.hpp) exercised against the
unmodified reference: tests/cpp/dropin_test.cpp, built by
__graft_entry__.build() (tests/cpp/Makefile) where /root/reference exists.

* CPU: the binary links (reference objects + libmscg.so) and, without a GPU,
  fails loudly with the library's "no CUDA device" error (no CPU fallback).
* GPU: every check passes (apply vs dense B^-1 and vs the reference, ILUT
  factors bit-identical, the reference's own gmres driving the GPU
  preconditioner, identical SingularMatrixError).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")


def _binary():
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
        else:
            pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    return BIN


def test_dropin_fails_loudly_without_gpu():
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present")
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "no CUDA device" in (r.stdout + r.stderr)


@pytest.mark.gpu
def test_dropin_against_reference():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 8
