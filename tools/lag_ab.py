"""A/B of variant builds (SIGKER_B200_LIB) on the latency-bound sweeps: one
pair chains where every band waits on the band below (cfg 1, a d=8 pair at
l=16384, cfg 4), plus cfg 2 and a small Gram as throughput guards.  Device
time of the sweep launches from the library's CUDA events."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

pol = sk.TruncationPolicy.adaptive(1e-12)
loose = sk.PropagateOptions(strict_corner=False)


def timed(fn, reps):
    fn()
    sk.stats_enable(True)
    sk.stats_reset()
    t = time.perf_counter()
    for _ in range(reps):
        r = fn()
    wall = (time.perf_counter() - t) / reps
    s = sk.stats_get()
    sk.stats_enable(False)
    return r, wall * 1e3, s["sweep_ms"] / reps


tag = os.path.basename(os.environ.get("SIGKER_B200_LIB", "default"))
x, y = sk.brownian(1000, 2, 1), sk.brownian(1000, 2, 2)
r, w, d = timed(lambda: sk.propagate_with_policy(x, y, pol), 20)
print(f"[{tag}] cfg1: e2e {w:.3f} ms, sweep {d:.3f} ms, K={r.value!r}", flush=True)
for L, dim in ((4096, 8), (16384, 8), (65536, 4)):
    x, y = sk.brownian(L, dim, 1), sk.brownian(L, dim, 2)
    r, w, d = timed(lambda: sk.propagate(x, y, 8, loose), 5)
    print(f"[{tag}] pair l={L} d={dim}: e2e {w:.2f} ms, sweep {d:.2f} ms, K={r.value!r}", flush=True)
x, y = sk.brownian(16384, 512, 1), sk.brownian(16384, 512, 2)
r, w, d = timed(lambda: sk.propagate(x, y, 8, loose), 3)
print(f"[{tag}] cfg4: e2e {w:.2f} ms, sweep {d:.2f} ms, K={r.value!r}", flush=True)
xs = sk.brownian_family(4096, 8, [2 * p + 1 for p in range(256)])
ys = sk.brownian_family(4096, 8, [2 * p + 2 for p in range(256)])
r, w, d = timed(lambda: sk.pairwise(xs, ys, pol), 3)
print(f"[{tag}] cfg2: sweep {d:.2f} ms", flush=True)
fam = sk.brownian_family(4096, 16, range(1000, 1064))
r, w, d = timed(lambda: sk.gram_matrix(fam, sk.GramOptions(policy=pol)), 2)
print(f"[{tag}] gram m=64: sweep {d:.1f} ms", flush=True)
