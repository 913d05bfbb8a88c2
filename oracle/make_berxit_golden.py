"""Generates tests/golden/berxit.json.gz from the Berxit CPU restatement (oracle/berxit_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  PARITY UNPINNED: the reference has no Berxit model
(proj/src/zoo.cpp:305-317), so these vectors are the oracle's own outputs — they freeze the
restatement (tests/test_berxit.py re-derives them on the CPU) and let the GPU tests and bench.py
check every instance of a BERT-base batch without running the slow oracle on the GPU box.

    python oracle/make_berxit_golden.py     # ~1 min on 16 cores
"""
import ctypes
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from test_berxit import BerxitOracle, SMALL  # noqa: E402
from paper_2305_10611_b200 import mbx  # noqa: E402  (config struct / defaults only)

RUNS = [("bert-base", {}, 64, 1), ("bert-base", {}, 8, 2), ("small", SMALL, 13, 1)]


def main():
    o = BerxitOracle()
    runs = []
    for name, kw, batch, seed in RUNS:
        c = mbx.berxit_config(**kw)
        p = o.params(c, seed)
        x = o.inputs(c, seed, range(batch))
        lg, ex = o.run(c, p, x, threads=os.cpu_count() or 1)
        runs.append({"name": name, "config": {f: getattr(c, f) for f, _ in c._fields_}, "batch": batch,
                     "seed": seed, "exit_layer": ex.tolist(), "logits": lg.astype(np.float64).tolist()})
        print(name, batch, seed, np.bincount(ex, minlength=c.layers).tolist())
    with gzip.open(os.path.join(ROOT, "tests", "golden", "berxit.json.gz"), "wt") as f:
        json.dump({"generator": "oracle/berxit_oracle.cpp (parity unpinned)", "runs": runs}, f)


if __name__ == "__main__":
    main()
