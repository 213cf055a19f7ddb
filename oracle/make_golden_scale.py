#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- BASELINE-scale goldens (tests/golden/scale.json)
from the UNMODIFIED reference (oracle/_ref/libsigker_ref.so) and, where the
reference throws or is infeasible, from the check-free C restatement
(oracle/sigker_oracle.c, pinned bit-exactly to the reference by
tests/test_oracle.py).  Run here, where /root/reference exists:

    python oracle/make_golden_scale.py [--jobs 7]

Inputs are the SURVEY.md section 8(d) datagen recipes (datagen.cpp:78-88,
seeds as listed there); the GPU tests regenerate them bit-identically.  About
20 minutes of one-off CPU time on 7 cores.

  cfg4  x = brownian(16384,512,1), y = (...,2): the reference's order, the
        check-free restatement's K (wavefront.cpp:35-59,70-192 without
        tile_series.cpp:70-75), its worst corner mismatch, the tile where the
        reference throws, and the reference's own throw (code, tile, message).
  cfg3  x = s*brownian(L,4,1), y = s*brownian(L,4,2), L = 1,000,000, s in
        {1, 8}: prefix knots K(a, a), a in {4096, 16384, 65536} -- the
        reference's propagate on x[:a+1], y[:a+1] (s = 1), the restatement
        (s = 8, where the reference's corner check throws).  Tile (i, j)
        depends only on tiles (i' <= i, j' <= j), so K(a, a) of the full run
        equals propagate on the prefixes at the full run's order.
  cfg5  family x_i = brownian(4096,16,1000+i), i < 1024: 64 entries (8 per
        eighth of the upper-triangle pair range, one diagonal each) via the
        reference's propagate_with_policy (adaptive 1e-12), as gram.cpp:51-66
        evaluates each entry.
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "scale.json")
L3 = 1_000_000
KNOTS3 = (4096, 16384, 65536)
M5, LEN5, DIM5 = 1024, 4096, 16


def f(x):
    return float(repr(float(x))) if np.isfinite(x) else repr(float(x))


def cs_order_bound(x, y, ref):
    """N via Cauchy-Schwarz: max|rho| <= max|dx|*max|dy|; estimate_order is
    monotone in max|rho| and never below 8, so N(bound) == 8 proves N == 8."""
    dx, dy = np.diff(x, axis=0), np.diff(y, axis=0)
    ub = float(np.sqrt((dx * dx).sum(1).max()) * np.sqrt((dy * dy).sum(1).max())) * (1 + 1e-12)
    n, _ = ref.estimate_order(ub, x.shape[0], 1e-12)
    return ub, n


def pair_index(m, i, j):
    return i * m - i * (i - 1) // 2 + (j - i)


def cfg5_samples():
    """8 entries per eighth of the upper-triangle range (row-major, i <= j), the
    first of each a diagonal entry -- so every shard of an 8-way split and every
    1/8 bench slice holds sampled entries."""
    rng = np.random.default_rng(2502)
    total = M5 * (M5 + 1) // 2
    starts = np.zeros(M5 + 1, dtype=np.int64)
    for i in range(M5):
        starts[i + 1] = starts[i] + (M5 - i)
    out = []
    for s in range(8):
        lo, hi = total * s // 8, total * (s + 1) // 8
        rows = [i for i in range(M5) if lo <= starts[i] < hi]
        i = int(rng.choice(rows))
        out.append((i, i))
        picked = set()
        while len(picked) < 7:
            t = int(rng.integers(lo, hi))
            i = int(np.searchsorted(starts, t, side="right") - 1)
            j = i + int(t - starts[i])
            if i != j:
                picked.add((i, j))
        out.extend(sorted(picked))
    return out


# ------------------------------------------------------------------ jobs
def job(spec):
    from oracle.oracle import OracleError, Reference, Restatement
    ref, R = Reference(), Restatement()
    kind = spec[0]
    t0 = time.time()
    if kind == "cfg4_restatement":
        x, y = ref.brownian(16384, 512, 1), ref.brownian(16384, 512, 2)
        v, _, mc, tile = R.propagate_probe(x, y, 8, check_corner=False)
        res = {"value": f(v), "max_corner_rel": f(mc), "first_corner_tile": list(tile)}
    elif kind == "cfg4_maxrho":
        x, y = ref.brownian(16384, 512, 1), ref.brownian(16384, 512, 2)
        mr = ref.max_abs_rho(x, y)
        n, c = ref.estimate_order(mr, 16384, 1e-12)
        res = {"max_abs_rho": f(mr), "order": n, "converged": c}
    elif kind == "cfg4_reference":
        x, y = ref.brownian(16384, 512, 1), ref.brownian(16384, 512, 2)
        try:
            v, _ = ref.propagate(x, y, 8, threads=1)
            res = {"value": f(v)}
        except OracleError as e:
            res = {"code": e.code, "tile_k": e.tile_k, "tile_l": e.tile_l, "message": str(e)}
    elif kind == "cfg3_reference":
        _, sigma, a = spec
        x, y = sigma * ref.brownian(L3, 4, 1)[: a + 1], sigma * ref.brownian(L3, 4, 2)[: a + 1]
        try:
            v, _ = ref.propagate(x, y, 8, threads=1)
            res = {"value": f(v)}
        except OracleError as e:
            res = {"code": e.code, "tile_k": e.tile_k, "tile_l": e.tile_l, "message": str(e)}
    elif kind == "cfg3_restatement":
        _, sigma = spec
        a = max(KNOTS3)
        x, y = sigma * ref.brownian(L3, 4, 1)[: a + 1], sigma * ref.brownian(L3, 4, 2)[: a + 1]
        v, kv, mc, tile = R.propagate_probe(x, y, 8, knots=KNOTS3, check_corner=False)
        res = {"knots": list(KNOTS3), "values": [f(t) for t in kv], "max_corner_rel": f(mc),
               "first_corner_tile": list(tile)}
    elif kind == "cfg3_order":
        _, sigma = spec
        x, y = sigma * ref.brownian(L3, 4, 1), sigma * ref.brownian(L3, 4, 2)
        ub, n = cs_order_bound(x, y, ref)
        res = {"cs_bound": f(ub), "order": n}
    elif kind == "cfg5_entry":
        _, i, j = spec
        x, y = ref.brownian(LEN5, DIM5, 1000 + i), ref.brownian(LEN5, DIM5, 1000 + j)
        # gram.cpp:51-66: x = member i (columns), y = member j (rows)
        try:
            v, n, c = ref.propagate_with_policy(x, y, adaptive=True, tol=1e-12)
            res = {"value": f(v), "order": n, "max_abs_rho": f(ref.max_abs_rho(x, y))}
        except OracleError as e:
            res = {"code": e.code, "tile_k": e.tile_k, "tile_l": e.tile_l, "message": str(e)}
        if i < 64 and j < 64:
            _, _, mc, _ = R.propagate_probe(x, y, res.get("order", 8), check_corner=False)
            res["max_corner_rel"] = f(mc)
    else:
        raise ValueError(kind)
    res["cpu_s"] = round(time.time() - t0, 1)
    return spec, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=7)
    ap.add_argument("--only", default="", help="comma list of job kinds")
    a = ap.parse_args()
    samples = cfg5_samples()
    specs = [("cfg3_reference", 1.0, 65536), ("cfg3_restatement", 1.0), ("cfg3_restatement", 8.0),
             ("cfg4_restatement",), ("cfg4_reference",), ("cfg4_maxrho",),
             ("cfg3_reference", 1.0, 16384), ("cfg3_reference", 8.0, 16384), ("cfg3_reference", 1.0, 4096),
             ("cfg3_reference", 8.0, 4096), ("cfg3_order", 1.0), ("cfg3_order", 8.0)]
    specs += [("cfg5_entry", i, j) for (i, j) in samples]
    if a.only:
        keep = set(a.only.split(","))
        specs = [s for s in specs if s[0] in keep]
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    t0 = time.time()
    with mp.Pool(a.jobs) as pool:
        for spec, res in pool.imap_unordered(job, specs):
            print(f"[{time.time() - t0:7.1f}s] {spec}: {res}", flush=True)
            kind = spec[0]
            if kind.startswith("cfg4"):
                out.setdefault("cfg4", {"recipe": ["brownian", 16384, 512, 1, 2, 1.0]})[kind[5:]] = res
            elif kind == "cfg3_reference":
                d = out.setdefault("cfg3", {"length": L3, "dim": 4, "seeds": [1, 2]})
                d.setdefault(f"sigma{spec[1]:g}", {}).setdefault("reference", {})[str(spec[2])] = res
            elif kind in ("cfg3_restatement", "cfg3_order"):
                d = out.setdefault("cfg3", {"length": L3, "dim": 4, "seeds": [1, 2]})
                d.setdefault(f"sigma{spec[1]:g}", {})[kind[5:]] = res
            else:
                d = out.setdefault("cfg5", {"m": M5, "length": LEN5, "dim": DIM5, "seed0": 1000, "entries": []})
                d["entries"] = [e for e in d["entries"] if (e["i"], e["j"]) != (spec[1], spec[2])]
                d["entries"].append(dict(i=spec[1], j=spec[2], linear=pair_index(M5, spec[1], spec[2]), **res))
                d["entries"].sort(key=lambda e: e["linear"])
            json.dump(out, open(OUT, "w"), indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
