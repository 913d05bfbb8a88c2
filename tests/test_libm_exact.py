"""The device activations (paper_2305_10611_b200/csrc/libm_fp32.cuh) compiled for the host must
equal the libm the reference links (glibc expf / tanhf) on every one of the 2^32 float inputs.
The same header is what the sm_100a kernels execute (explicit _rn intrinsics, no contraction), so
this is what makes the FP32 path bit-exact."""
import json
import os
import subprocess

from conftest import ROOT


def test_expf_tanhf_exhaustive(tmp_path):
    exe = tmp_path / "libm_exhaustive"
    src = os.path.join(ROOT, "tests", "native", "libm_exhaustive.cpp")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-pthread", "-o", str(exe), src])
    out = json.loads(subprocess.check_output([str(exe)], timeout=600))
    assert out["range"] == [0, 1 << 32]
    assert out["expf_mismatch"] == 0, out
    assert out["tanhf_mismatch"] == 0, out
