"""A C++ consumer of the drop-in boundary: tests/native/backend_native.cpp is compiled against
include/mbatch/backend.hpp (the reference's operator API) and linked with libmbx.so, then runs
the reference's backend test cases (proj/tests/backend_test.cpp:33-57, :96-103, :134-237), the
flush scope and the batched decision read-back.  CPU: host-only dry contexts (shapes, offsets,
gather bytes, error texts); GPU: values too."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2305_10611_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "backend_native")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "native", "backend_native.cpp"), "-L" + LIBDIR, "-lmbx",
                           "-Wl,-rpath," + LIBDIR, "-o", exe])
    return exe


def test_native_consumer_dry(tmp_path):
    exe = _build(tmp_path)
    p = subprocess.run([exe], env=dict(os.environ, MBX_DEVICE="-1"), capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout


@pytest.mark.gpu
def test_native_consumer_gpu(tmp_path):
    exe = _build(tmp_path)
    p = subprocess.run([exe], env=dict(os.environ, MBX_DEVICE="0"), capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout, p.stdout
