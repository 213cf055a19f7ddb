"""cfg 3 (one pair l=10^6, d=4, N=8, prefix knots) sweep time for A/B of
variant builds (SIGKER_B200_LIB)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

x, y = sk.brownian(1_000_000, 4, 1), sk.brownian(1_000_000, 4, 2)
loose = sk.PropagateOptions(strict_corner=False)
sk.stats_enable(True)
sk.stats_reset()
t = time.perf_counter()
r = sk.propagate(x, y, 8, loose, diag=True)
wall = time.perf_counter() - t
s = sk.stats_get()
print(f"[{os.path.basename(os.environ.get('SIGKER_B200_LIB', 'default'))}] cfg3: e2e {wall:.2f} s, "
      f"sweep {s['sweep_ms'] / 1e3:.2f} s, K={r.value!r}", flush=True)
