"""Single-pair latency through the public API (the reference acceptance
suite's criterion-6 shapes: Brownian d=2, order 7, lengths 129..4097 and
beyond), median of 9 after a warm-up, with the sweep's device time.
`--shapes lx:ly,...` times rectangular pairs instead: one band (ly = 33)
gives the per-column step time, one column (lx = 2..33) the per-band lag."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402


def timed(lx, ly, order=7):
    rng = np.random.default_rng(606)
    x = np.cumsum(rng.standard_normal((lx, 2)) / np.sqrt(max(lx, ly)), axis=0)
    y = np.cumsum(rng.standard_normal((ly, 2)) / np.sqrt(max(lx, ly)), axis=0)
    sk.propagate(x, y, order)
    walls, sweeps = [], []
    for _ in range(9):
        sk.stats_enable(True)
        sk.stats_reset()
        t0 = time.perf_counter()
        sk.propagate(x, y, order)
        walls.append(time.perf_counter() - t0)
        sweeps.append(sk.stats_get()["sweep_ms"])
    return np.median(walls) * 1e3, np.median(sweeps)


if "--shapes" in sys.argv:
    for spec in sys.argv[sys.argv.index("--shapes") + 1].split(","):
        lx, ly = map(int, spec.split(":"))
        w, s = timed(lx, ly)
        print(f"lx {lx:6d} ly {ly:6d}: wall {w:8.3f} ms  sweep {s:8.3f} ms", flush=True)
    sys.exit(0)
lengths = [int(a) for a in sys.argv[1:]] or [129, 257, 513, 1025, 2049, 4097, 8193, 16385]
for L in lengths:
    w, s = timed(L, L)
    tiles = (L - 1) ** 2
    print(f"len {L:6d}: wall {w:8.3f} ms  sweep {s:8.3f} ms  {tiles / (s / 1e3):.3e} tiles/s in the sweep  "
          f"{(s * 1e6) / (2 * L):.1f} ns per wavefront step", flush=True)
