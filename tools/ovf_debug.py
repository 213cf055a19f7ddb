"""Diagnostics: error reporting of one overflowing pair under the streaming and
segment-DAG schedules (argv[1]: segment columns)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle.oracle import Restatement  # noqa: E402  (input generation only)
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

R = Restatement()
rng = R.rng(2024)
for (lx, ly, d) in [(70, 100, 3), (130, 97, 2), (66, 200, 8), (90, 64, 40), (41, 150, 16)]:
    for _ in range(10):
        rng.random_series(lx if _ < 5 else ly, d, 1.0)
x = rng.random_series(80, 1, 1.0)
y = rng.random_series(90, 1, 1.0)
x[40:] *= 3e4
y[50:] *= 3e4
for mode in ("stream", "seg"):
    if mode == "stream":
        os.environ["SK_STREAM"] = "1"
    else:
        os.environ.pop("SK_STREAM")
        os.environ["SK_FORCE_SEGMENTS"] = "1"
        os.environ["SK_SEG_COLS"] = sys.argv[1]
    for strict in (True, False):
        try:
            v = sk.propagate(x, y, 8, sk.PropagateOptions(strict_corner=strict)).value
            print(mode, strict, v, flush=True)
        except Exception as e:  # noqa: BLE001
            print(mode, strict, type(e).__name__, e, flush=True)

# the same sequence as tests/test_gpu_parity.py::test_segment_dag_matches_streaming
if len(sys.argv) > 2:
    rng = R.rng(2024)
    cases = []
    for (lx, ly, d, order) in [(70, 100, 3, 8), (130, 97, 2, 12), (66, 200, 8, 20), (90, 64, 40, 8), (41, 150, 16, 5)]:
        xs = np.stack([rng.random_series(lx, d, 1.0) for _ in range(5)])
        ys = np.stack([rng.random_series(ly, d, 1.0) for _ in range(5)])
        cases.append((xs, ys, order))
    for mode in ("stream", "seg"):
        if mode == "stream":
            os.environ["SK_STREAM"] = "1"
            os.environ.pop("SK_FORCE_SEGMENTS", None)
        else:
            os.environ.pop("SK_STREAM")
            os.environ["SK_FORCE_SEGMENTS"] = "1"
        for xs, ys, order in cases:
            if "pw" in sys.argv[2]:
                sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(order))
            if "ad" in sys.argv[2]:
                sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12), want_max_abs_rho=True)
            if "gr" in sys.argv[2]:
                sk.propagate_grid(xs[0], ys[0], order)
        try:
            print("after", sys.argv[2], mode, sk.propagate(x, y, 8).value, flush=True)
        except Exception as e:  # noqa: BLE001
            print("after", sys.argv[2], mode, type(e).__name__, e, flush=True)
