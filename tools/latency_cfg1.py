"""cfg 1 latency (one pair l=1000, d=2) through the public API: adaptive and
fixed order, with the library's device time of the sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

x, y = sk.brownian(1000, 2, 1), sk.brownian(1000, 2, 2)
pol = sk.TruncationPolicy.adaptive(1e-12)
for name, fn in (("adaptive", lambda: sk.propagate_with_policy(x, y, pol)), ("fixed 8", lambda: sk.propagate(x, y, 8)),
                 ("adaptive, no corner check",
                  lambda: sk.propagate_with_policy(x, y, pol, sk.PropagateOptions(strict_corner=False)))):
    for _ in range(3):
        fn()
    sk.stats_enable(True)
    sk.stats_reset()
    t = time.perf_counter()
    for _ in range(20):
        fn()
    wall = (time.perf_counter() - t) / 20
    s = sk.stats_get()
    sk.stats_enable(False)
    print(f"{name}: {wall * 1e3:.3f} ms e2e, sweep {s['sweep_ms'] / 20:.3f} ms, {s['sweep_launches'] / 20:.1f} sweeps "
          f"+ {s['aux_launches'] / 20:.1f} aux per call, literal re-sweeps {s['literal_rechecks']}", flush=True)
