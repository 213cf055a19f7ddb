"""GPU parity at BASELINE.json scale, against tests/golden/scale.json
(oracle/make_golden_scale.py: the unmodified reference where it runs, the
check-free restatement -- pinned bit-exactly to the reference by
tests/test_oracle.py -- where the reference throws).  Inputs are the
reference's own datagen streams (datagen.cpp:78-88, SURVEY.md section 8d
seeds), regenerated bit-identically.

Tolerance (BASELINE.json north_star): |K_gpu - K_ref| / |K_ref| <= 1e-10 in
fp64, the relative error proper, with the identical truncation order."""
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale.json")
TOL = 1e-10


@pytest.fixture(scope="module")
def scale():
    with open(GOLD) as f:
        return json.load(f)


def relerr(a, b):
    return abs(a - b) / abs(b)


def test_cfg4_full_size(sk, restatement, scale):
    """cfg 4: l = 16384, d = 512 (x = brownian(16384,512,1), y = (...,2)), the
    large-d path.  Adaptive order and exact max|rho| equal the reference's;
    with the corner check off K matches the check-free restatement of
    wavefront.cpp:35-59,70-192; with it on (the reference's default) the call
    raises InconsistentBoundaryError at the tile where the reference throws."""
    g = scale["cfg4"]
    x, y = restatement.brownian(16384, 512, 1), restatement.brownian(16384, 512, 2)
    pol = sk.TruncationPolicy.adaptive(1e-12)
    r = sk.propagate_with_policy(x, y, pol, sk.PropagateOptions(strict_corner=False))
    assert r.order == g["maxrho"]["order"]
    assert relerr(r.value, g["restatement"]["value"]) <= TOL, (r.value, g["restatement"]["value"])
    assert sk.IncrementTable(x, y).max_abs_rho() == g["maxrho"]["max_abs_rho"]
    assert g["reference"]["code"] == 3  # the reference itself throws here
    k, l = g["restatement"]["first_corner_tile"]
    with pytest.raises(sk.InconsistentBoundaryError) as e:
        sk.propagate_with_policy(x, y, pol)
    assert f"tile ({k}, {l})" in str(e.value), str(e.value)


@pytest.mark.parametrize("sigma", [1.0, 8.0])
def test_cfg3_million_point_pair_prefix_knots(sk, restatement, scale, sigma):
    """cfg 3: ONE pair of l = 1,000,000, d = 4, x = s*brownian(1e6,4,1),
    y = s*brownian(1e6,4,2), s = 1 and the rough s = 8.  Tile (i, j) depends
    only on tiles (i' <= i, j' <= j), so the full run's knots K(a, a) equal
    the reference's propagate on the length-(a+1) prefixes (s = 1: the
    reference itself; s = 8: the check-free restatement, identical to the
    reference wherever the reference also ran, a <= 16384)."""
    g = scale["cfg3"][f"sigma{sigma:g}"]
    L = scale["cfg3"]["length"]
    x, y = sigma * restatement.brownian(L, 4, 1), sigma * restatement.brownian(L, 4, 2)
    pol = sk.TruncationPolicy.adaptive(1e-12)
    # order: the Cauchy-Schwarz proof of the golden (N = 8) and the C-ABI's own
    r = sk.propagate(x, y, g["order"]["order"], sk.PropagateOptions(strict_corner=False), diag=True)
    assert g["order"]["order"] == 8
    assert np.isfinite(r.value) and r.diag[-1] == r.value
    knots = g["restatement"]["knots"]
    for q, a in enumerate(knots):
        expect = g["restatement"]["values"][q]
        if sigma == 1.0:
            assert g["reference"][str(a)]["value"] == expect  # restatement == reference, bit for bit
        assert relerr(r.diag[a - 1], expect) <= TOL, (a, r.diag[a - 1], expect)
    for a, ref in g["reference"].items():
        if "value" in ref:
            assert relerr(r.diag[int(a) - 1], ref["value"]) <= TOL, a


def test_cfg5_full_gram_sampled_entries(sk, restatement, scale):
    """cfg 5: the full N = 1024 Gram (l = 4096, d = 16, member i =
    brownian(4096,16,1000+i), adaptive) on one GPU; 64 entries (8 per eighth of
    the pair range, 8 diagonal) against the reference's propagate_with_policy
    (gram.cpp:51-66), same orders.  Strict corner mode (default): no run may
    need more than a handful of literal re-sweeps (measured: 26 of 524,800
    pairs cross the 1e-11 screen; each then decides exactly as the reference).
    Symmetry and K(x,x) >= 1 over all entries."""
    g = scale["cfg5"]
    m = g["m"]
    fam = [restatement.brownian(g["length"], g["dim"], g["seed0"] + i) for i in range(m)]
    sk.stats_enable(True)
    sk.stats_reset()
    r = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)))
    st = sk.stats_get()
    sk.stats_enable(False)
    assert st["literal_rechecks"] <= 64, st["literal_rechecks"]
    V = np.asarray(r.values).reshape(m, m)
    O = np.asarray(r.orders).reshape(m, m)
    assert not r.failures and np.all(np.isfinite(V))
    assert np.array_equal(V, V.T)
    assert np.all(np.diag(V) >= 1.0)
    worst = 0.0
    for e in g["entries"]:
        i, j = e["i"], e["j"]
        assert O[i, j] == e["order"], (i, j)
        err = relerr(V[i, j], e["value"])
        worst = max(worst, err)
        assert err <= TOL, (i, j, V[i, j], e["value"], err)
    assert len(g["entries"]) == 64 and sum(e["i"] == e["j"] for e in g["entries"]) == 8
    print(f"cfg5: 64 sampled entries, worst relative error {worst:.2e}, {r.wall_seconds:.1f} s")
