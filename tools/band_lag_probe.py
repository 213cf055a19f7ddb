"""Step time of a lone band and the hand-over lag per band on one pair:
x of length 4096, y of 32 B + 1 points (B bands), d = 8, N = 8.  The sweep
time is ~ (cols + 31) t_step + (B - 1) lag t_step."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

loose = sk.PropagateOptions(strict_corner=False)
L = int(os.environ.get("PROBE_LEN", "4096"))
d = int(os.environ.get("PROBE_DIM", "8"))
x = sk.brownian(L, d, 1)
base = None
for B in (1, 2, 4, 8, 16, 32, 64, 128):
    y = sk.brownian(32 * B + 1, d, 2)
    sk.propagate(x, y, 8, loose)
    sk.stats_enable(True)
    sk.stats_reset()
    for _ in range(5):
        sk.propagate(x, y, 8, loose)
    ms = sk.stats_get()["sweep_ms"] / 5
    sk.stats_enable(False)
    if base is None:
        base = ms
        t_step = ms * 1e3 / (L - 1 + 31)
    lag = (ms - base) * 1e3 / t_step / max(1, B - 1)
    print(f"bands {B:4d}: sweep {ms:.3f} ms, step {t_step * 1e3:.0f} ns (lone band), lag/band {lag:.1f} steps",
          flush=True)
