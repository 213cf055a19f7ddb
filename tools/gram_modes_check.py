"""Diagnostics: a BASELINE-config-5-shaped Gram (m x l=4096, d=16, adaptive)
under the segment-DAG and the streaming schedules -- identical bits expected
(exercises column-buffer slot reuse at scale: slots < pairs)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 96
rng = np.random.default_rng(5)
fam = list(np.cumsum(rng.standard_normal((m, 4096, 16)) / 64.0, axis=1))
pol = sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12))
sk.gram_matrix(fam[:4], pol)
out = {}
for mode in ("seg", "stream"):
    if mode == "stream":
        os.environ["SK_STREAM"] = "1"
    sk.stats_enable(True)
    sk.stats_reset()
    t0 = time.perf_counter()
    r = sk.gram_matrix(fam, pol)
    wall = time.perf_counter() - t0
    s = sk.stats_get()
    out[mode] = np.asarray(r.values)
    npairs = m * (m + 1) // 2
    print(f"{mode}: wall {wall:.2f} s, sweep {s['sweep_ms'] / 1e3:.2f} s, {npairs / wall:.0f} evals/s, "
          f"{100 * s['tile_flops'] / s['sweep_ms'] / 1e9 / 37.11:.1f}% of roof, orders {r.min_order}..{r.max_order}",
          flush=True)
print("identical:", np.array_equal(out["seg"].view(np.int64), out["stream"].view(np.int64)))
