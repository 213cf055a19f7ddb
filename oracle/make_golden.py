#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- regenerates tests/golden/*.json from the
UNMODIFIED reference engine (oracle/_ref/libsigker_ref.so, built from
/root/reference/proj/src by oracle/Makefile).  Run here (where
/root/reference exists):  python oracle/make_golden.py

Inputs are stored by recipe (datagen seed / Rng seed) or inline when small;
outputs are the reference's own results, printed with repr() (round-trip
exact).  Cases follow the reference's tests and SURVEY.md section 8c /
Appendix B.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.oracle import OracleError, Reference, Restatement  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def f(x):
    return float(repr(float(x))) if np.isfinite(x) else repr(float(x))


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    R = Restatement()
    t0 = time.time()

    # ---- datagen / RNG streams (datagen.cpp:12-88)
    dg = {"rng": [], "brownian": [], "fbm": []}
    for seed in (0, 1, 42, 900, 2 ** 40 + 7):
        dg["rng"].append({"seed": seed, "uniform": [f(v) for v in ref.rng_stream(seed, 12, False)],
                          "gaussian": [f(v) for v in ref.rng_stream(seed, 12, True)]})
    for (length, dim, seed) in ((2, 1, 1), (33, 2, 3), (1000, 2, 1), (4096, 8, 1), (257, 16, 1000)):
        b = ref.brownian(length, dim, seed)
        dg["brownian"].append({"length": length, "dim": dim, "seed": seed, "first": [f(v) for v in b[:3].ravel()],
                               "last": [f(v) for v in b[-1]], "sum": f(b.sum())})
    for (length, dim, h, seed) in ((51, 2, 0.3, 1), (129, 3, 0.1, 2)):
        b = ref.fbm(length, dim, h, seed)
        dg["fbm"].append({"length": length, "dim": dim, "hurst": h, "seed": seed, "last": [f(v) for v in b[-1]],
                          "sum": f(b.sum())})
    json.dump(dg, open(os.path.join(OUT, "datagen.json"), "w"), indent=1)

    # ---- single tiles: step_tile (wavefront.cpp:223-237)
    tiles = []
    rng = R.rng(31)
    for trial in range(40):
        order = [0, 1, 2, 7, 8, 12, 16, 24, 40, 64][trial % 10]
        a = np.array([(2.0 * rng.uniform01() - 1.0) / (r * r + 1.0) for r in range(order + 1)])
        b = np.array([(2.0 * rng.uniform01() - 1.0) / (r * r + 1.0) for r in range(order + 1)])
        a[0] = b[0] = 2.0 * rng.uniform01() - 1.0
        delta = 6.0 * rng.uniform01() - 3.0
        oa, ob = ref.step_tile(delta, a, b, order)
        tiles.append({"order": order, "delta": f(delta), "alpha": [f(v) for v in a], "beta": [f(v) for v in b],
                      "out_alpha": [f(v) for v in oa], "out_beta": [f(v) for v in ob]})
    json.dump({"tiles": tiles}, open(os.path.join(OUT, "step_tile.json"), "w"))

    # ---- estimate_order grid (truncation.cpp:41-55)
    est = []
    for rho in (0.0, 1e-3, 0.2, 0.4109, 0.411, 0.9, 1.0, 2.5, 7.0, 30.0, 1e3, 1e6):
        for tol in (1e-2, 1e-6, 1e-10, 1e-12, 1e-14):
            o, c = ref.estimate_order(rho, 16, tol)
            est.append({"rho": rho, "tol": tol, "order": o, "converged": c})
    json.dump({"cases": est}, open(os.path.join(OUT, "estimate_order.json"), "w"))

    # ---- small propagate cases with grids (random_series, tests/helpers.hpp:17-33)
    small = []
    rng = R.rng(2024)
    shapes = [(2, 2, 1), (3, 2, 1), (5, 9, 2), (9, 5, 3), (12, 13, 2), (40, 70, 3), (70, 40, 4), (97, 33, 8),
              (33, 97, 16), (50, 45, 40), (21, 21, 3)]
    for (lx, ly, d) in shapes:
        for order in (1, 7, 8, 13, 16, 17, 24):
            x = rng.random_series(lx, d, 1.0)
            y = rng.random_series(ly, d, 1.0)
            v, pk, g = ref.propagate(x, y, order, grid=True)
            case = {"x": [f(t) for t in x.ravel()], "y": [f(t) for t in y.ravel()], "dim": d, "order": order,
                    "value": f(v), "peak_live": pk}
            if lx * ly <= 512:
                case["grid"] = [f(t) for t in g]
            small.append(case)
    json.dump({"cases": small}, open(os.path.join(OUT, "propagate_small.json"), "w"))

    # ---- error contract cases
    errs = []
    one = np.array([[0.0], [1.0]])
    for (name, x, y, order) in (("overflow_1_1", [[0.0], [400.0]], [[0.0], [400.0]], 24),
                                ("overflow_2_3", [[0.0], [1.0], [401.0]], [[0.0], [0.5], [1.0], [401.0]], 8),
                                ("nonfinite", [[0.0], [340.0], [680.0], [1020.0], [1360.0], [1700.0], [2040.0]],
                                 [[0.0], [340.0], [680.0], [1020.0], [1360.0], [1700.0], [2040.0]], 24)):
        x, y = np.array(x, float), np.array(y, float)
        try:
            v, _ = ref.propagate(x, y, order)
            errs.append({"name": name, "x": x.ravel().tolist(), "y": y.ravel().tolist(), "order": order,
                         "value": f(v)})
        except OracleError as e:
            errs.append({"name": name, "x": x.ravel().tolist(), "y": y.ravel().tolist(), "order": order,
                         "code": e.code, "tile_k": e.tile_k, "tile_l": e.tile_l, "message": str(e)})
    # a scaled-volatility Brownian pair on which the reference's corner check throws
    for (length, sigma) in ((4097, 3.0), (1025, 8.0), (1025, 12.0)):
        x = sigma * ref.brownian(length, 4, 1)
        y = sigma * ref.brownian(length, 4, 2)
        try:
            v, n, _ = ref.propagate_with_policy(x, y, adaptive=True)
            errs.append({"name": f"sigma{sigma}", "recipe": ["brownian", length, 4, 1, 2, sigma], "value": f(v),
                         "order": n})
        except OracleError as e:
            mr = ref.max_abs_rho(x, y)
            n, _ = ref.estimate_order(mr, length, 1e-12)
            try:
                vf, _ = R.propagate(x, y, n, check_corner=False)
                vf = f(vf)
            except OracleError as e2:
                vf = f"raises {e2.code} at ({e2.tile_k}, {e2.tile_l})"
            errs.append({"name": f"sigma{sigma}", "recipe": ["brownian", length, 4, 1, 2, sigma], "code": e.code,
                         "order": n, "checkfree_value": vf, "message": str(e)})
    json.dump({"cases": errs}, open(os.path.join(OUT, "errors.json"), "w"), indent=1)

    # ---- BASELINE-shaped known answers
    known = []
    def brown_pair(length, dim, s1, s2, sigma=1.0):
        return sigma * ref.brownian(length, dim, s1), sigma * ref.brownian(length, dim, s2)
    for (label, length, dim, s1, s2, sigma) in (("cfg1", 1000, 2, 1, 2, 1.0), ("cfg2_pair0", 4096, 8, 1, 2, 1.0),
                                                ("cfg3_shape_sigma2", 4097, 4, 1, 2, 2.0),
                                                ("cfg4_shape", 2049, 512, 1, 2, 1.0)):
        x, y = brown_pair(length, dim, s1, s2, sigma)
        mr = ref.max_abs_rho(x, y)
        v, n, c = ref.propagate_with_policy(x, y, adaptive=True)
        known.append({"label": label, "recipe": ["brownian", length, dim, s1, s2, sigma], "max_abs_rho": f(mr),
                      "order": n, "value": f(v)})
        print(label, v, n, time.time() - t0, flush=True)
    xf, yf = ref.fbm(513, 2, 0.1, 1), ref.fbm(513, 2, 0.1, 2)
    v, n, c = ref.propagate_with_policy(xf, yf, adaptive=True)
    known.append({"label": "fbm_H0.1", "recipe": ["fbm", 513, 2, 0.1, 1, 2], "max_abs_rho": f(ref.max_abs_rho(xf, yf)),
                  "order": n, "value": f(v)})
    json.dump({"cases": known}, open(os.path.join(OUT, "known_answers.json"), "w"), indent=1)

    # ---- Gram (gram.cpp:16-98)
    grams = []
    fam = np.stack([ref.brownian(33, 2, s) for s in (1, 2, 3)])
    r = ref.gram(fam, adaptive=True, threads=4)
    grams.append({"label": "brownian33x3", "recipe": ["brownian", 33, 2, [1, 2, 3]], "adaptive": True,
                  "values": [f(v) for v in r["values"].ravel()], "orders": r["orders"].ravel().tolist(),
                  "max_product": f(r["max_product"]), "peak_live": r["peak_live"]})
    fam = np.stack([ref.brownian(4096, 16, 1000 + i) for i in range(4)])
    r = ref.gram(fam, adaptive=True, threads=8, compute_bound=True)
    grams.append({"label": "cfg5_block4", "recipe": ["brownian", 4096, 16, [1000, 1001, 1002, 1003]],
                  "adaptive": True, "values": [f(v) for v in r["values"].ravel()],
                  "orders": r["orders"].ravel().tolist(), "max_product": f(r["max_product"]),
                  "bound": f(r["bound"]), "peak_live": r["peak_live"]})
    print("gram", time.time() - t0, flush=True)
    rng = R.rng(4)
    fam = np.stack([rng.random_series(6, 2, 0.9) for _ in range(4)])
    for order in (8, 12, 16, 64):
        r = ref.gram(fam, adaptive=False, order=order, compute_bound=True)
        grams.append({"label": f"random6x4_N{order}", "inline": fam.ravel().tolist(), "shape": list(fam.shape),
                      "adaptive": False, "order": order, "values": [f(v) for v in r["values"].ravel()],
                      "orders": r["orders"].ravel().tolist(), "max_product": f(r["max_product"]),
                      "bound": f(r["bound"])})
    fam = np.array([[[0.0], [1.0]], [[0.0], [1e4]]])
    r = ref.gram(fam, adaptive=False, order=8)
    grams.append({"label": "failure_entry", "inline": fam.ravel().tolist(), "shape": list(fam.shape),
                  "adaptive": False, "order": 8, "values": [f(v) for v in r["values"].ravel()],
                  "n_failures": r["n_failures"]})
    json.dump({"cases": grams}, open(os.path.join(OUT, "gram.json"), "w"), indent=1)

    # ---- Gram error bound / Bessel (truncation.cpp:28-39,57-87)
    misc = {"bessel_i0": [[x, f(ref.bessel_i0(x))] for x in (0.0, 0.5, 2.0, 2.0 * np.sqrt(2.0), 10.0, 50.0)],
            "gram_error_bound": [[m, l, x, n, f(ref.gram_error_bound(m, l, x, n))]
                                 for (m, l, x, n) in ((3, 5, 0.0, 7), (1, 2, 1.0, 7), (2, 6, 0.8, 9), (2, 8, 1.0, 24),
                                                      (4, 33, 0.01, 8))]}
    json.dump(misc, open(os.path.join(OUT, "truncation_misc.json"), "w"), indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
