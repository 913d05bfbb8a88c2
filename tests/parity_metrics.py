"""Tolerance metrics of SURVEY §8a, shared by the GPU parity tests, smoke() and bench.py.

Per element:  |gpu - ref| <= rel * max(|ref|, 1e-6)   ("passes"), reported as the largest
per-element relative error (max_rel, same 1e-6 floor) and the fraction of elements passing
(frac_pass).  A secondary normwise figure ||gpu - ref|| / ||ref|| is kept beside it.
"""
import numpy as np

FLOOR = 1e-6


def elementwise(got, want, rel):
    got = np.asarray(got, np.float64).ravel()
    want = np.asarray(want, np.float64).ravel()
    assert got.shape == want.shape, (got.shape, want.shape)
    if want.size == 0:
        return {"n": 0, "max_rel": 0.0, "frac_pass": 1.0, "normwise": 0.0, "max_abs": 0.0, "fails": 0}
    err = np.abs(got - want)
    denom = np.maximum(np.abs(want), FLOOR)
    r = err / denom
    ok = err <= rel * denom
    nw = float(np.linalg.norm(got - want) / max(1e-30, np.linalg.norm(want)))
    return {"n": int(want.size), "max_rel": float(np.max(r)), "frac_pass": float(np.mean(ok)), "normwise": nw,
            "max_abs": float(np.max(err)), "fails": int(np.sum(~ok))}


def merge(stats):
    """Combines per-output stats into one (max of maxima, element-weighted pass fraction)."""
    stats = [s for s in stats if s["n"]]
    if not stats:
        return elementwise([], [], 1.0)
    n = sum(s["n"] for s in stats)
    return {"n": n, "max_rel": max(s["max_rel"] for s in stats),
            "frac_pass": sum(s["frac_pass"] * s["n"] for s in stats) / n,
            "normwise": max(s["normwise"] for s in stats), "max_abs": max(s["max_abs"] for s in stats),
            "fails": sum(s["fails"] for s in stats)}
