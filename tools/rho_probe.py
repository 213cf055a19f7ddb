"""Large-d (fused rho producer) timing probe: cfg 4 (one pair l=16384,
d=512) and a batch (32 pairs l=2048, d=64), fixed N=8, corner check off.
SIGKER_B200_LIB selects a variant build of the C-ABI library."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

loose = sk.PropagateOptions(strict_corner=False)


def run(name, fn, tiles, flops_per_tile, reps=3):
    fn()
    sk.stats_enable(True)
    sk.stats_reset()
    t = time.perf_counter()
    for _ in range(reps):
        v = fn()
    wall = (time.perf_counter() - t) / reps
    s = sk.stats_get()
    sk.stats_enable(False)
    sw = s["sweep_ms"] / reps
    print(f"{name}: wall {wall * 1e3:.2f} ms, sweep {sw:.2f} ms, {tiles / (sw / 1e3):.3e} tiles/s, "
          f"{tiles * flops_per_tile / (sw / 1e3) / 1e12 / 37.11 * 100:.1f}% of FP64 peak, value {v!r}", flush=True)


x, y = sk.brownian(16384, 512, 1), sk.brownian(16384, 512, 2)
run(f"cfg4 [{os.environ.get('SIGKER_B200_LIB', 'default')}]", lambda: sk.propagate(x, y, 8, loose).value, 16383 ** 2,
    4 * 81 + 2 * 512)
xs = sk.brownian_family(2048, 64, range(100, 132))
ys = sk.brownian_family(2048, 64, range(200, 232))
run("batch 32 x 2048^2 d=64", lambda: sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(8), loose).values[0],
    32 * 2047 ** 2, 4 * 81 + 2 * 64)
