"""Every generated per-plan kernel (tensor-core gate / levels configurations, bit-exact gate
kernel, pointwise kernels) compiles for sm_100a with NVRTC, for every zoo model at the reference's
sizes and at the BASELINE sizes — checked on a GPU-less host (dry contexts compile without
loading: MBX_JIT_IN_DRY).  Runs in a subprocess so the environment switch takes effect."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("treelstm", 512), ("treelstm", 256), ("birnn", 512), ("nestedrnn", 512), ("mvrnn", 128),
         ("rnn", 64), ("drnn", 64), ("stackrnn", 64), ("fig5", 32)]


@pytest.mark.parametrize("prec", ["fp32", "bf16x3"])
def test_generated_kernels_compile(prec):
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_2305_10611_b200 import mbx\n"
        "for name, h in %r:\n"
        "    c = mbx.Context(-1, %r); m = mbx.Model(c, name, h); m.close(); c.close()\n"
        "print('ok')\n" % (ROOT, CASES, prec))
    env = dict(os.environ, MBX_JIT_IN_DRY="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]
