"""Randomised bit-identity stress of the large-d fast paths (intra-CTA
hand-over, GEMM beside the sweep) against the serial global-memory path:
random lengths / dimensions / orders, single pairs and small batches."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("STRESS_SEED", "5")))
cases = int(os.environ.get("STRESS_CASES", "40"))


def walk(n, d, scale):
    return np.cumsum(rng.normal(0.0, scale / np.sqrt(n), size=(n, d)), axis=0)


def run(x, y, order):
    r = sk.propagate(x, y, order, sk.PropagateOptions(strict_corner=False))
    return np.float64(r.value).view(np.int64).item()


bad = 0
for c in range(cases):
    d = int(rng.choice([17, 20, 33, 64, 130]))
    lx, ly = int(rng.integers(40, 900)), int(rng.integers(40, 900))
    order = int(rng.choice([4, 8, 12]))
    x, y = walk(lx, d, 1.0), walk(ly, d, 1.0)
    os.environ.pop("SK_NO_INTRA", None)
    os.environ.pop("SK_NO_OVERLAP", None)
    a = run(x, y, order)
    os.environ["SK_NO_INTRA"] = "1"
    os.environ["SK_NO_OVERLAP"] = "1"
    b = run(x, y, order)
    if a != b:
        bad += 1
        print(f"MISMATCH case {c}: d={d} lx={lx} ly={ly} N={order}", flush=True)
print(f"{cases} cases, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
