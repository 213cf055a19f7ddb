"""cfg 1 host-phase trace (run with SK_TRACE=1; the last block is a warm call)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

x, y = sk.TimeSeries(sk.brownian(1000, 2, 1)), sk.TimeSeries(sk.brownian(1000, 2, 2))
pol = sk.TruncationPolicy.adaptive(1e-12)
for _ in range(5):
    sk.propagate_with_policy(x, y, pol)
print("---- traced call", file=sys.stderr)
t = time.perf_counter()
sk.propagate_with_policy(x, y, pol)
print("wall", time.perf_counter() - t, file=sys.stderr)
