"""Diagnostics: BASELINE.json configs through the public API (host inputs),
with sweep-kernel device time from the library's CUDA-event accounting.

  cfg1  single pair  l=1000,  d=2   adaptive
  cfg3  single pair  l=L,     d=4   (default L = 1_000_000), sigma-scaled Brownian
  cfg4  single pair  l=16384, d=512 (table path)
  cfg5  Gram m x m,  l=4096,  d=16  adaptive (default m = 128: a sample of the 1024 Gram)
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402


def brownian(n, length, dim, seed, sigma=1.0):
    """n series datagen::brownian(length, dim, seed + k) -- the reference's
    generator, bit for bit (SURVEY.md section 8d inputs), times sigma."""
    return sigma * sk.brownian_family(length, dim, [seed + k for k in range(n)])


def timed(fn):
    sk.stats_enable(True)
    sk.stats_reset()
    t0 = time.perf_counter()
    r = fn()
    wall = time.perf_counter() - t0
    s = sk.stats_get()
    sk.stats_enable(False)
    return r, wall, s


def report(name, tiles, wall, s, extra=""):
    sw = s["sweep_ms"] / 1e3
    tf = s["tile_flops"] / max(sw, 1e-12) / 1e12
    print(f"{name}: wall {wall:.3f} s, sweep {sw:.3f} s ({s['sweep_launches']} launches), "
          f"{tiles / wall:.3e} tile-updates/s end-to-end, {tiles / max(sw, 1e-12):.3e} in the sweep, "
          f"{tf:.2f} TF/s = {100 * tf / 37.11:.1f}% of FP64 peak {extra}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg1", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--len3", type=int, default=1_000_000)
    ap.add_argument("--sigma3", type=float, default=1.0)
    ap.add_argument("--m5", type=int, default=128)
    ap.add_argument("--warm", action="store_true", help="cfg5: one small Gram first (kernel loading, allocations)")
    a = ap.parse_args()
    pol = sk.TruncationPolicy.adaptive(1e-12)
    for cfg in a.configs:
        if cfg == "cfg1":
            x, y = brownian(1, 1000, 2, 1)[0], brownian(1, 1000, 2, 2)[0]  # seeds 1 / 2
            sk.propagate_with_policy(x, y, pol)
            r, wall, s = timed(lambda: sk.propagate_with_policy(x, y, pol))
            report("cfg1 l=1000 d=2", 999 * 999, wall, s, f"K={r.value!r} N={r.order}")
        elif cfg == "cfg3":
            L = a.len3
            x = brownian(1, L, 4, 1, a.sigma3)[0]
            y = brownian(1, L, 4, 2, a.sigma3)[0]
            r, wall, s = timed(lambda: sk.propagate_with_policy(x, y, pol, sk.PropagateOptions(strict_corner=False)))
            report(f"cfg3 l={L} d=4 sigma={a.sigma3}", (L - 1) ** 2, wall, s, f"K={r.value!r} N={r.order}")
        elif cfg == "cfg4":
            x, y = brownian(1, 16384, 512, 1)[0], brownian(1, 16384, 512, 2)[0]
            sk.propagate_with_policy(x, y, pol, sk.PropagateOptions(strict_corner=False))
            r, wall, s = timed(lambda: sk.propagate_with_policy(x, y, pol, sk.PropagateOptions(strict_corner=False)))
            report("cfg4 l=16384 d=512", 16383 ** 2, wall, s, f"K={r.value!r} N={r.order} (large-d path: table mode where it fits, see DESIGN 4.3)")
        elif cfg == "cfg5":
            m = a.m5
            fam = brownian(m, 4096, 16, 1000)  # (m, l, d): gram_matrix's no-copy path
            if a.warm:
                sk.gram_matrix(fam[:8], sk.GramOptions(policy=pol))
            r, wall, s = timed(lambda: sk.gram_matrix(fam, sk.GramOptions(policy=pol)))
            npairs = m * (m + 1) // 2
            report(f"cfg5 Gram m={m} l=4096 d=16", npairs * 4095 ** 2, wall, s,
                   f"{npairs / wall:.1f} kernel-evals/s end-to-end, orders {r.min_order}..{r.max_order}")


if __name__ == "__main__":
    main()
