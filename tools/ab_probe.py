"""A/B timing of variant builds (SIGKER_B200_LIB) on the throughput sweeps:
a cfg-5-shaped Gram (first M members of the north-star family; one sweep
launch) and BASELINE cfg 2 (256 pairs, l = 4096, d = 8), device time of the
sweep launches from the library's CUDA events.  Prints one line per case."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

m = int(os.environ.get("AB_M", "128"))
fam = sk.brownian_family(4096, 16, range(1000, 1000 + m))
xs = sk.brownian_family(4096, 8, [2 * p + 1 for p in range(256)])
ys = sk.brownian_family(4096, 8, [2 * p + 2 for p in range(256)])
pol = sk.TruncationPolicy.adaptive(1e-12)
# AB_LOOSE=1: corner check off (timing-only experiment builds whose values are wrong)
loose = os.environ.get("AB_LOOSE") == "1"
popt = sk.PropagateOptions(strict_corner=not loose)


def timed(fn, reps):
    fn()
    sk.stats_enable(True)
    sk.stats_reset()
    for _ in range(reps):
        fn()
    s = sk.stats_get()
    sk.stats_enable(False)
    return s["sweep_ms"] / reps, s["tile_flops"] / (s["sweep_ms"] / 1e3) / 1e12 / 37.11


g_ms, g_fr = timed(lambda: sk.gram_matrix(fam, sk.GramOptions(policy=pol, strict_corner=not loose)), 2)
c_ms, c_fr = timed(lambda: sk.pairwise(xs, ys, pol, popt), 5)
print(f"[{os.path.basename(os.environ.get('SIGKER_B200_LIB', 'default'))}] gram m={m}: {g_ms:.1f} ms "
      f"({g_fr:.1%} FP64); cfg2: {c_ms:.2f} ms ({c_fr:.1%})", flush=True)

if os.environ.get("AB_D16"):
    x16 = sk.brownian_family(4096, 16, [1000 + p for p in range(256)])
    y16 = sk.brownian_family(4096, 16, [1300 + p for p in range(256)])
    for want in (False, True):
        ms, fr = timed(lambda: sk.pairwise(x16, y16, pol, want_max_abs_rho=want), 3)
        print(f"  d=16 256 pairs, exact max|rho| {want}: {ms:.2f} ms ({fr:.1%})", flush=True)
    for want in (False, True):
        ms, fr = timed(lambda: sk.pairwise(xs, ys, pol, want_max_abs_rho=want), 3)
        print(f"  d=8 256 pairs, exact max|rho| {want}: {ms:.2f} ms ({fr:.1%})", flush=True)
