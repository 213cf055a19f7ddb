"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle
(oracle/sigker_oracle.c, pinned bit-exactly to the reference by
tests/test_oracle.py) and the golden fixtures generated from the reference.

Tolerance (BASELINE.json north_star): |K_gpu - K_ref| <= 1e-10 * max(1, |K_ref|)
in fp64 with the identical truncation order per pair.  Orders <= 16 run the
factorial-scaled register solver (re-associated sums); orders above 16 run
the literal kernel, bit-identical to the reference, and are checked for
equality.  max|rho| is bit-exact by construction and checked for equality."""
import json
import math
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def brown_pair(R, recipe):
    kind = recipe[0]
    if kind == "brownian":
        _, length, dim, s1, s2, sigma = recipe
        return sigma * R.brownian(length, dim, s1), sigma * R.brownian(length, dim, s2)
    _, length, dim, h, s1, s2 = recipe
    return R.fbm(length, dim, h, s1), R.fbm(length, dim, h, s2)


# ------------------------------------------------------------ single pairs
def test_single_tile_bessel(sk):
    x = np.array([[0.0], [1.0]])
    assert rel(sk.propagate(x, x, 24).value, 2.2795853023360673) < 1e-14
    for rho in (-4.0, -1.0, 0.5, 1.0, 4.0):
        y = np.array([[0.0], [rho]])
        expect = sum(rho ** i / math.factorial(i) ** 2 for i in range(25))
        assert rel(sk.propagate(x, y, 24).value, expect) < 1e-14


def test_constant_series_is_exactly_one(sk):
    for length in (2, 3, 9, 40):
        x = np.tile([[0.4, -1.0]], (length, 1))
        r = sk.propagate(x, x, 12)
        assert r.value == 1.0
        assert r.tiles_processed == (length - 1) ** 2


def test_golden_small_cases(sk):
    for c in load("propagate_small.json")["cases"]:
        d = c["dim"]
        x = np.array(c["x"]).reshape(-1, d)
        y = np.array(c["y"]).reshape(-1, d)
        if "grid" in c:
            r = sk.propagate_grid(x, y, c["order"])
            g = np.array(c["grid"])
            if c["order"] > 16:
                assert r.grid.tolist() == c["grid"]
            else:
                assert np.max(np.abs(r.grid - g) / np.maximum(1.0, np.abs(g))) < TOL
        else:
            r = sk.propagate(x, y, c["order"])
        if c["order"] > 16:
            assert r.value == c["value"], (c["order"], x.shape, y.shape)
        else:
            assert rel(r.value, c["value"]) < TOL, (c["order"], x.shape, y.shape)
        assert r.peak_live_series == c["peak_live"]


@pytest.mark.parametrize("order", [1, 2, 7, 8, 12, 16, 17, 24])
@pytest.mark.parametrize("shape", [(2, 2, 1), (5, 9, 2), (40, 70, 3), (70, 40, 4), (97, 33, 8), (33, 97, 16),
                                   (130, 66, 5), (66, 130, 11)])
def test_random_series_orders(sk, restatement, order, shape):
    lx, ly, d = shape
    rng = restatement.rng(1000 * order + lx + 7 * ly)
    x = rng.random_series(lx, d, 1.0)
    y = rng.random_series(ly, d, 1.0)
    v_ref, pk_ref = restatement.propagate(x, y, order)
    r = sk.propagate(x, y, order)
    if order > 16:
        assert r.value == v_ref
    else:
        assert rel(r.value, v_ref) < TOL
    assert r.peak_live_series == pk_ref


def test_step_tile_bit_exact(sk):
    for t in load("step_tile.json")["tiles"]:
        oa, ob = sk.step_tile(t["delta"], np.array(t["alpha"]), np.array(t["beta"]), t["order"])
        assert oa.tolist() == t["out_alpha"]
        assert ob.tolist() == t["out_beta"]


def test_step_tile_fast_solver(sk):
    """The register solver of the sweep on single tiles (orders 1..16)."""
    for t in load("step_tile.json")["tiles"]:
        if not 1 <= t["order"] <= 16:
            continue
        oa, ob = sk.step_tile(t["delta"], np.array(t["alpha"]), np.array(t["beta"]), t["order"], fast=True)
        scale = max(1.0, max(abs(v) for v in t["out_alpha"] + t["out_beta"]))
        assert np.max(np.abs(oa - np.array(t["out_alpha"]))) < 1e-13 * scale
        assert np.max(np.abs(ob - np.array(t["out_beta"]))) < 1e-13 * scale


def test_step_tile_examples(sk):
    """test_wavefront.cpp:86-105."""
    order = 16
    u = np.zeros(order + 1)
    u[0] = 1.0
    up, right = sk.step_tile(1.0, u, u, order)
    for i in range(order + 1):
        expect = 1.0 / math.factorial(i) ** 2
        assert abs(up[i] - expect) <= 1e-14 * expect and abs(right[i] - expect) <= 1e-14 * expect
    pu, pr = sk.step_tile(0.0, np.array([1.0, 0.5, -0.1]), np.array([1.0, 0.25, 0.0]), 2)
    assert abs(pu[0] - 1.25) < 1e-15 and pu[1] == 0.5 and pu[2] == -0.1
    assert abs(pr[0] - 1.4) < 1e-15 and pr[1] == 0.25


def test_known_answers(sk, restatement):
    for c in load("known_answers.json")["cases"]:
        x, y = brown_pair(restatement, c["recipe"])
        assert sk.IncrementTable(x, y).max_abs_rho() == c["max_abs_rho"], c["label"]
        r = sk.propagate_with_policy(x, y, sk.TruncationPolicy.adaptive(1e-12))
        assert r.order == c["order"], c["label"]
        assert r.order_converged
        assert rel(r.value, c["value"]) < TOL, (c["label"], r.value, c["value"])


def test_adaptive_order_10_at_unit_rho(sk):
    """test_wavefront.cpp:226-234."""
    x = np.array([[0.0], [1.0]])
    fixed = sk.propagate_with_policy(x, x, sk.TruncationPolicy.fixed(24))
    adaptive = sk.propagate_with_policy(x, x, sk.TruncationPolicy.adaptive(1e-12))
    assert fixed.order == 24 and adaptive.order == 10 and adaptive.order_converged
    assert abs(adaptive.value - fixed.value) < 1e-10


# ----------------------------------------------------------------- errors
def test_error_contract(sk):
    for c in load("errors.json")["cases"]:
        if "x" not in c:
            continue
        x = np.array(c["x"]).reshape(-1, 1)
        y = np.array(c["y"]).reshape(-1, 1)
        if "code" in c:
            with pytest.raises(sk.NumericOverflowError) as e:
                sk.propagate(x, y, c["order"])
            assert (e.value.tile_k, e.value.tile_l) == (c["tile_k"], c["tile_l"]), c["name"]
            assert "rescale" in str(e.value)
        else:
            assert rel(sk.propagate(x, y, c["order"]).value, c["value"]) < TOL


def test_inconsistent_boundary_contract(sk, restatement):
    """Scaled-volatility Brownian pairs near the reference's corner check
    (tile_series.cpp:70-75).  Strict mode (the C++ API default) must decide
    exactly as the reference does: raise InconsistentBoundaryError where the
    reference raises -- at the tile where the reference's sweep throws (the
    restatement, bit-identical to the reference, locates it) -- and return the
    reference's value where it returns one.  The register kernels screen the
    corner at 1e-11 and hand screened pairs to the literal (bit-identical)
    kernel, so a returned value is then the reference's bits.  With the check
    off the value is the check-free restatement's."""
    for c in load("errors.json")["cases"]:
        if "recipe" not in c:
            continue
        x, y = brown_pair(restatement, c["recipe"])
        loose = sk.PropagateOptions(strict_corner=False)
        r = sk.propagate(x, y, c["order"], loose)
        expect = c.get("checkfree_value", c.get("value"))
        assert rel(r.value, expect) < TOL, (c["name"], r.value, expect)
        sk.stats_enable(True)
        sk.stats_reset()
        if "code" in c:
            _, _, _, tile = restatement.propagate_probe(x, y, c["order"])
            with pytest.raises(sk.InconsistentBoundaryError) as e:
                sk.propagate(x, y, c["order"])
            assert f"tile ({tile[0]}, {tile[1]})" in str(e.value), (c["name"], str(e.value), tile)
            assert sk.stats_get()["literal_rechecks"] == 1
        else:
            v = sk.propagate(x, y, c["order"]).value
            if sk.stats_get()["literal_rechecks"]:
                assert v == c["value"], c["name"]
            else:
                assert rel(v, c["value"]) < TOL, c["name"]
        sk.stats_enable(False)


def test_strict_corner_screen_spares_clean_pairs(sk, restatement):
    """Brownian inputs sit far below the 1e-11 screen: strict mode re-sweeps
    nothing and equals the unchecked result bit for bit."""
    xs = np.stack([restatement.brownian(700, 4, 70 + k) for k in range(6)])
    ys = np.stack([restatement.brownian(650, 4, 80 + k) for k in range(6)])
    sk.stats_enable(True)
    sk.stats_reset()
    strict = sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12))
    assert sk.stats_get()["literal_rechecks"] == 0
    sk.stats_enable(False)
    loose = sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12), sk.PropagateOptions(strict_corner=False))
    assert strict.values.tolist() == loose.values.tolist()


def test_strict_corner_screen_in_batches_and_grams(sk, restatement):
    """The literal re-sweep inside pairwise and gram: a throwing pair is a
    per-pair InconsistentBoundaryError in pairwise (raised, as the reference
    would on that pair) and aborts gram_matrix (gram.cpp:74-77 lets it
    through); a screened pair that the reference accepts keeps its value."""
    throw = load("errors.json")["cases"]
    hot = [c for c in throw if c.get("name") == "sigma12.0"][0]
    x, y = brown_pair(restatement, hot["recipe"])
    with pytest.raises(sk.InconsistentBoundaryError):
        sk.pairwise(np.stack([x, x]), np.stack([y, x]), sk.TruncationPolicy.adaptive(1e-12))
    with pytest.raises(sk.InconsistentBoundaryError):
        sk.gram_matrix([x, y], sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)))


def test_overflow_inside_batch_is_per_pair(sk, restatement):
    rng = restatement.rng(5)
    xs = np.stack([rng.random_series(6, 1, 1.0) for _ in range(4)])
    ys = np.stack([rng.random_series(6, 1, 1.0) for _ in range(4)])
    xs[2, 3:, 0] += 500.0
    ys[2, 4:, 0] += 500.0
    res = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(12))
    assert math.isnan(res.values[2])
    assert [f[0] for f in res.failures] == [2]
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        restatement.propagate(xs[2], ys[2], 12)
    assert (res.failures[0][1], res.failures[0][2]) == (e.value.tile_k, e.value.tile_l)
    for k in (0, 1, 3):
        assert rel(res.values[k], restatement.propagate(xs[k], ys[k], 12)[0]) < TOL


# ---------------------------------------------------------------- batches
def test_pairwise_mixed_orders(sk, restatement):
    """Rough (fBm) and smooth pairs in one batch: per-pair adaptive orders,
    one sweep launch per distinct order."""
    xs, ys, expect = [], [], []
    for k, h in enumerate((0.1, 0.2, 0.3, 0.5, 0.7, 0.15)):
        x = restatement.fbm(129, 2, h, 10 + k)
        y = restatement.fbm(129, 2, h, 20 + k)
        xs.append(x)
        ys.append(y)
        expect.append(restatement.propagate_with_policy(x, y, 1e-12))
    res = sk.pairwise(np.stack(xs), np.stack(ys), sk.TruncationPolicy.adaptive(1e-12), want_max_abs_rho=True)
    assert len(set(res.orders.tolist())) > 1
    for k, (v, n, conv) in enumerate(expect):
        assert res.orders[k] == n
        assert res.max_abs_rho[k] == restatement.max_abs_rho(xs[k], ys[k])
        if n > 16:
            assert res.values[k] == v
        else:
            assert rel(res.values[k], v) < TOL


def test_slot_reuse_and_groups_are_deterministic(sk, restatement, monkeypatch):
    """Force tiny unit groups / column-buffer slots so pairs recycle slots
    (band 0 of pair p waits for the last band of pair p - slots)."""
    rng = restatement.rng(77)
    xs = np.stack([rng.random_series(70, 3, 1.0) for _ in range(11)])
    ys = np.stack([rng.random_series(100, 3, 1.0) for _ in range(11)])
    base = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(8)).values
    monkeypatch.setenv("SK_FORCE_GROUP", "2")
    monkeypatch.setenv("SK_FORCE_SLOTS", "3")
    forced = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(8)).values
    assert forced.tolist() == base.tolist()
    for k in range(11):
        assert rel(base[k], restatement.propagate(xs[k], ys[k], 8)[0]) < TOL


@pytest.mark.parametrize("seg_cols", ["32", "96"])
def test_segment_dag_matches_streaming(sk, restatement, monkeypatch, seg_cols):
    """The segment-DAG schedule (units = band segments, dependency counters,
    lane state carried between segments) computes exactly what the streaming
    schedule computes: values, orders, max|rho|, errors, knot grids -- across
    register / literal / table kernels, ragged shapes and slot reuse."""
    rng = restatement.rng(2024)
    cases = []
    for (lx, ly, d, order) in [(70, 100, 3, 8), (130, 97, 2, 12), (66, 200, 8, 20), (90, 64, 40, 8), (41, 150, 16, 5),
                               (2, 300, 2, 8), (3, 170, 1, 6), (50, 90, 40, 20), (60, 120, 12, 10)]:
        xs = np.stack([rng.random_series(lx, d, 1.0) for _ in range(5)])
        ys = np.stack([rng.random_series(ly, d, 1.0) for _ in range(5)])
        cases.append((xs, ys, order))

    # a pair that overflows inside the sweep
    x = rng.random_series(80, 1, 1.0)
    y = rng.random_series(90, 1, 1.0)
    x[40:] *= 3e4
    y[50:] *= 3e4

    def bits(v):
        return np.ascontiguousarray(v, dtype=np.float64).view(np.int64).tolist()

    def run_all():
        out = []
        for xs, ys, order in cases:
            r = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(order))
            out.append(bits(r.values))
            a = sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12), want_max_abs_rho=True)
            out.append((bits(a.values), list(a.orders), bits(a.max_abs_rho)))
            g = sk.propagate_grid(xs[0], ys[0], order)
            out.append(bits(g.grid))
        # an overflow inside the sweep: first failing tile, as streaming reports it
        for strict in (True, False):
            try:
                out.append(bits([sk.propagate(x, y, 8, sk.PropagateOptions(strict_corner=strict)).value]))
            except sk.NumericOverflowError as e:
                out.append(("overflow", e.tile_k, e.tile_l))
            except sk.InconsistentBoundaryError as e:
                out.append(("corner", str(e)))
        return out

    monkeypatch.setenv("SK_STREAM", "1")
    ref = run_all()
    monkeypatch.delenv("SK_STREAM")
    monkeypatch.setenv("SK_FORCE_SEGMENTS", "1")
    monkeypatch.setenv("SK_SEG_COLS", seg_cols)

    def check(got):
        assert len(got) == len(ref)
        for k, (a, b) in enumerate(zip(got, ref)):
            assert a == b, (k, str(a)[:300], str(b)[:300])

    check(run_all())
    monkeypatch.setenv("SK_FORCE_SLOTS", "2")
    monkeypatch.setenv("SK_FORCE_GROUP", "1")
    check(run_all())


def test_thread_safety_and_determinism(sk, restatement):
    rng = restatement.rng(123)
    pairs = [(rng.random_series(60, 2, 1.0), rng.random_series(45, 2, 1.0)) for _ in range(8)]
    ref = [sk.propagate(x, y, 10).value for x, y in pairs]
    out = [None] * len(pairs)

    def work(k):
        x, y = pairs[k]
        out[k] = sk.propagate(x, y, 10).value

    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(pairs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out == ref


def test_large_dim_table_path(sk, restatement):
    rng = restatement.rng(77)
    for d in (17, 40, 100):
        x = rng.random_series(50, d, 1.0)
        y = rng.random_series(45, d, 1.0)
        for order in (8, 20):
            v_ref, _ = restatement.propagate(x, y, order)
            got = sk.propagate(x, y, order).value
            assert (got == v_ref) if order > 16 else rel(got, v_ref) < TOL
        assert sk.IncrementTable(x, y).max_abs_rho() == restatement.max_abs_rho(x, y)


def test_cfg4_shape_dmma_table_path(sk, restatement):
    """BASELINE config 4's shape (d = 512, the DMMA rho-table path) at a
    length the oracle finishes in seconds: adaptive single pair and a ragged
    batch, against the restatement (same orders; 1e-10 at N <= 16, bit-exact
    on the literal kernel above)."""
    x = restatement.brownian(257, 512, 41)
    y = restatement.brownian(193, 512, 42)
    v_ref, n_ref, _ = restatement.propagate_with_policy(x, y, 1e-12, check_corner=False)
    r = sk.propagate_with_policy(x, y, sk.TruncationPolicy.adaptive(1e-12), sk.PropagateOptions(strict_corner=False))
    assert r.order == n_ref
    assert (r.value == v_ref) if n_ref > 16 else rel(r.value, v_ref) < TOL
    xs = np.stack([restatement.brownian(130, 512, 50 + k) for k in range(3)])
    ys = np.stack([restatement.brownian(97, 512, 60 + k) for k in range(3)])
    res = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(8), sk.PropagateOptions(strict_corner=False))
    assert not res.failures
    for k in range(3):
        v, _ = restatement.propagate(xs[k], ys[k], 8, check_corner=False)
        assert rel(res.values[k], v) < TOL, k


def test_max_abs_rho_bit_exact(sk, restatement):
    rng = restatement.rng(99)
    for d in (1, 2, 3, 5, 8, 13, 16, 33):
        x = rng.random_series(37, d, 1.7)
        y = rng.random_series(29, d, 1.7)
        assert sk.IncrementTable(x, y).max_abs_rho() == restatement.max_abs_rho(x, y)


def test_prefix_knots_diag(sk, restatement):
    """K at knots (a, a) of a long pair equals the kernel of the length-(a+1)
    prefixes: the verification route for l = 10^6."""
    x = restatement.brownian(2049, 4, 1)
    y = restatement.brownian(2049, 4, 2)
    r = sk.propagate(x, y, 8, diag=True)
    assert r.diag[-1] == r.value
    for a in (1, 2, 31, 32, 33, 64, 100, 513):
        v_ref, _ = restatement.propagate(x[: a + 1], y[: a + 1], 8)
        assert rel(r.diag[a - 1], v_ref) < TOL, a


def test_w_fault_negative_control(sk, restatement):
    x = restatement.brownian(33, 2, 1)
    y = restatement.brownian(33, 2, 2)
    good = sk.propagate(x, y, 8).value
    sk.set_w_fault_for_testing(True)
    try:
        bad = sk.propagate(x, y, 8).value
        bad_lit = sk.propagate(x, y, 20).value
    finally:
        sk.set_w_fault_for_testing(False)
    assert rel(bad, good) > 1e-6
    assert rel(bad_lit, sk.propagate(x, y, 20).value) > 1e-6


# -------------------------------------------------------------------- gram
def test_gram_golden(sk, restatement):
    for c in load("gram.json")["cases"]:
        if "inline" in c:
            fam = list(np.array(c["inline"]).reshape(c["shape"]))
        else:
            _, length, dim, seeds = c["recipe"]
            fam = [restatement.brownian(length, dim, s) for s in seeds]
        pol = sk.TruncationPolicy.adaptive(1e-12) if c["adaptive"] else sk.TruncationPolicy.fixed(c["order"])
        opts = sk.GramOptions(policy=pol, compute_bound="bound" in c)
        r = sk.gram_matrix(fam, opts)
        for got, ref in zip(r.values.tolist(), c["values"]):
            if isinstance(ref, str) or (isinstance(ref, float) and math.isnan(ref)):
                assert math.isnan(got)
            elif c.get("order", 8) > 16:
                assert got == ref
            else:
                assert rel(got, ref) < TOL, c["label"]
        if "orders" in c:
            assert r.orders.tolist() == c["orders"], c["label"]
        if "max_product" in c:
            assert r.max_abs_increment_product == c["max_product"], c["label"]
        if "bound" in c and not isinstance(c["bound"], str):
            assert r.bound == pytest.approx(c["bound"], rel=1e-12)
        if "n_failures" in c:
            assert len(r.failures) == c["n_failures"]
            assert (r.failures[0].row, r.failures[0].col) == (1, 1)


def test_gram_shards_reassemble(sk, restatement):
    rng = restatement.rng(3)
    fam = [rng.random_series(20, 2, 1.0) for _ in range(9)]
    full = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.fixed(14)))
    assembled = np.full(81, np.nan)
    for s in range(4):
        part = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.fixed(14)), shard=s, nshards=4)
        m = ~np.isnan(part.values)
        assert np.isnan(assembled[m]).all()
        assembled[m] = part.values[m]
    assert assembled.tolist() == full.values.tolist()
    vals = full.values.reshape(9, 9)
    assert np.array_equal(vals, vals.T)
    assert (np.diag(vals) >= 1.0 - 1e-10).all()


# ------------------------------------------------------- multi-GPU strips
def test_strip_protocol_emulated_on_one_gpu(sk, restatement):
    """The long-pair strip pipeline of 1, 2 and 3 virtual GPUs emulated in one
    launch (block-cyclic column buffers and exchange areas per virtual GPU, the
    hand-off every `block` bands -- block = 1: at every band boundary -- with
    system-scope release/acquire, the last GPU handing to the first):
    bit-identical to the plain sweep."""
    from paper_2502_20392_b200.distributed import propagate_split_emulated, strip_bands
    for d in (4, 12, 40):  # register kernel with shared-memory / direct top-row hand-up, large-d path
        x = restatement.brownian(300, d, 5)
        y = restatement.brownian(400, d, 6)
        for order in (8, 20):
            plain = sk.propagate(x, y, order).value
            nb = strip_bands(400, order)
            assert nb >= 3
            for block in range(1, nb):
                for gpus in (1, 2, 3):
                    if -(-nb // block) < gpus:
                        continue
                    assert propagate_split_emulated(x, y, order, block, gpus=gpus) == plain, (d, order, block, gpus)


def test_gram_over_a_device_list_matches_one_call(sk, restatement):
    """GramOptions.devices: one host thread per listed GPU, each a sub-shard
    (here the same GPU twice -- independent pairs, no cross-kernel waits);
    the merged matrix equals the single-call one bit for bit."""
    rng = restatement.rng(404)
    fam = [rng.random_series(40 + 3 * k, 2, 1.0) for k in range(9)]
    pol = sk.TruncationPolicy.adaptive(1e-12)
    one = sk.gram_matrix(fam, sk.GramOptions(policy=pol, compute_bound=True))
    two = sk.gram_matrix(fam, sk.GramOptions(policy=pol, compute_bound=True, devices=[0, 0]))
    assert np.asarray(two.values).view(np.int64).tolist() == np.asarray(one.values).view(np.int64).tolist()
    assert list(two.orders) == list(one.orders)
    assert two.max_abs_increment_product == one.max_abs_increment_product
    assert two.orders_converged == one.orders_converged


def test_gram_device_list_merges_entry_failures(sk, restatement):
    """Entries that overflow (NumericOverflowError -> NaN + a failures record,
    gram.cpp:74-77) merge from the device-list sub-shards exactly as one call
    reports them: same NaN cells, same (i, j, message) records in order."""
    rng = restatement.rng(405)
    fam = [rng.random_series(30 + 2 * k, 1, 1.0) for k in range(7)]
    fam[4] = fam[4] * 3e3  # |delta| > 1.25e5 against itself and the larger series
    pol = sk.TruncationPolicy.fixed(8)
    one = sk.gram_matrix(fam, sk.GramOptions(policy=pol, strict_corner=False))
    two = sk.gram_matrix(fam, sk.GramOptions(policy=pol, strict_corner=False, devices=[0, 0]))
    assert one.failures, "the scaled series must overflow somewhere"
    assert [(f.row, f.col, f.message) for f in two.failures] == [(f.row, f.col, f.message) for f in one.failures]
    assert all(f.row <= f.col for f in one.failures)
    assert (4, 4) in [(f.row, f.col) for f in one.failures]
    assert np.isnan(np.asarray(two.values)).tolist() == np.isnan(np.asarray(one.values)).tolist()
    for f in one.failures:
        assert "rescale" in f.message


def test_baseline_size_batch_properties(sk, restatement):
    """BASELINE config 2 at full size (256 pairs, l = 4096, d = 8, adaptive)
    through the throughput schedule: four pairs against the restatement, and
    size-independent properties over all 256 -- symmetry K(x,y) = K(y,x) and
    batch == single-pair evaluation."""
    xs = np.stack([restatement.brownian(4096, 8, 2 * p + 1) for p in range(256)])
    ys = np.stack([restatement.brownian(4096, 8, 2 * p + 2) for p in range(256)])
    pol = sk.TruncationPolicy.adaptive(1e-12)
    fwd = sk.pairwise(xs, ys, pol)
    rev = sk.pairwise(ys, xs, pol)
    assert not fwd.failures and list(fwd.orders) == [8] * 256
    assert np.max(np.abs(fwd.values - rev.values) / np.maximum(1.0, np.abs(fwd.values))) < 1e-12
    for p in (0, 77, 255):
        assert rel(sk.propagate_with_policy(xs[p], ys[p], pol).value, fwd.values[p]) < 1e-13
    for p in (0, 1, 128, 255):
        v_ref, _ = restatement.propagate(xs[p], ys[p], 8)
        assert rel(fwd.values[p], v_ref) < TOL, p


def test_long_pair_prefix_identity_at_scale(sk, restatement):
    """A 65537 x 65537 pair (4.3e9 tiles, the long-pair schedule): knots K(a, a)
    from the one run equal separate runs on the length-(a+1) prefixes."""
    x = restatement.brownian(65537, 4, 11)
    y = restatement.brownian(65537, 4, 12)
    r = sk.propagate(x, y, 8, diag=True)
    assert r.diag[-1] == r.value and np.all(np.isfinite(r.diag))
    for a in (4096, 16384, 40000):
        assert rel(r.diag[a - 1], sk.propagate(x[: a + 1], y[: a + 1], 8).value) < 1e-12, a


def test_long_pair_devices_single_gpu_is_plain_propagate(sk, restatement):
    """propagate_long_pair_devices with one device is the ordinary sweep; with
    several distinct GPUs it runs the strip pipeline over peer access (not
    reachable on a one-GPU box -- the protocol itself is pinned by
    test_strip_protocol_emulated_on_one_gpu)."""
    from paper_2502_20392_b200 import _capi, distributed as skd
    x = restatement.brownian(300, 3, 5)
    y = restatement.brownian(260, 3, 6)
    v, dg = skd.propagate_long_pair_devices(x, y, 8, devices=[0], diag=True)
    r = sk.propagate(x, y, 8, diag=True)
    assert v == r.value and np.array_equal(dg, r.diag)
    st = _capi.SkStatus()
    assert _capi.load().sk_enable_peer_access(0, __import__("ctypes").byref(st)) == 0  # own device: no-op


def _fd_knots(x, y, R):
    """Independent check: K_st = rho K on the tile grid by an implicit
    trapezoidal finite-difference march (R cells per tile), Richardson
    extrapolated from R and 2R, sampled at the knots."""
    dx, dy = np.diff(x, axis=0), np.diff(y, axis=0)
    rho = dy @ dx.T  # rows (y) x cols (x)

    def march(r):
        rows, cols = rho.shape
        K = np.ones((cols * r + 1, rows * r + 1))
        h2 = 1.0 / (r * r)
        for a in range(cols * r):
            for b in range(rows * r):
                q = 0.25 * rho[b // r, a // r] * h2
                K[a + 1, b + 1] = (K[a + 1, b] + K[a, b + 1] - K[a, b] + q * (K[a, b] + K[a + 1, b] + K[a, b + 1])) / (1 - q)
        return K[::r, ::r]

    c, f = march(R), march(2 * R)
    return f + (f - c) / 3.0


def test_grid_against_finite_differences(sk, restatement):
    """test_wavefront.cpp:168-198: the knot grid against an FD solve (R = 16,
    extrapolated) and the grid's boundary / self-grid symmetry contract."""
    rng = restatement.rng(808)
    x = rng.random_series(6, 2, 0.9)
    y = rng.random_series(5, 2, 0.9)
    g = sk.propagate_grid(x, y, 24)
    G = np.asarray(g.grid).reshape(g.grid_rows, g.grid_cols)
    assert G.shape == (6, 5) and np.all(G[0] == 1.0) and np.all(G[:, 0] == 1.0)
    fd = _fd_knots(x, y, 16)
    assert np.max(np.abs(G - fd)) < 2e-4
    s = sk.propagate_grid(x, x, 24)
    S = np.asarray(s.grid).reshape(s.grid_rows, s.grid_cols)
    assert np.max(np.abs(S - S.T)) < 1e-12


def test_large_d_fused_rho_matches_table(sk, restatement, monkeypatch):
    """d > 16: the rho table (GEMM into HBM, used where it fits the memory
    budget) and the fused producer warps (rho formed in shared memory, O(l)
    memory) run the same DMMA k-order or the same sequential dot, so every
    output is bit-identical -- values, orders, max|rho|, knot grids, literal
    orders, error tiles, strict-corner decisions; both against the oracle.
    The table mode's intra-CTA hand-over (consecutive bands of a single pair
    in one CTA, alpha through shared memory) and the GEMM running beside the
    sweep match the serial, global-memory path too."""
    rng = restatement.rng(4242)

    def bits(v):
        return np.ascontiguousarray(v, dtype=np.float64).view(np.int64).tolist()

    x1, y1 = restatement.brownian(300, 40, 7), restatement.brownian(260, 40, 8)
    xs = np.stack([rng.random_series(90, 33, 1.0) for _ in range(5)])
    ys = np.stack([rng.random_series(150, 33, 1.0) for _ in range(5)])
    xo = rng.random_series(70, 20, 1.0)
    yo = rng.random_series(80, 20, 1.0)
    xo[35:] *= 8e3
    yo[40:] *= 8e3

    def run_all():
        out = [bits([sk.propagate(x1, y1, 8).value]), bits([sk.propagate(x1, y1, 20).value])]
        a = sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12), want_max_abs_rho=True)
        out.append((bits(a.values), list(a.orders), bits(a.max_abs_rho)))
        out.append(bits(sk.propagate_grid(xs[0], ys[0], 8).grid))
        try:
            out.append(bits([sk.propagate(xo, yo, 8).value]))
        except sk.NumericOverflowError as e:
            out.append(("overflow", e.tile_k, e.tile_l))
        return out

    monkeypatch.setenv("SK_RHO_FUSED", "0")
    # single pairs: consecutive bands hand over inside a CTA, and the GEMM
    # runs beside the sweep (bands start on published row blocks)
    table = run_all()
    monkeypatch.setenv("SK_NO_INTRA", "1")
    monkeypatch.setenv("SK_NO_OVERLAP", "1")
    table_global = run_all()  # every hand-over through global memory, GEMM first
    monkeypatch.delenv("SK_NO_INTRA")
    monkeypatch.delenv("SK_NO_OVERLAP")
    monkeypatch.setenv("SK_RHO_FUSED", "1")
    fused = run_all()
    assert table_global == table
    assert fused == table
    v_ref, _ = restatement.propagate(x1, y1, 20)
    assert sk.propagate(x1, y1, 20).value == v_ref
    assert rel(sk.propagate(x1, y1, 8).value, restatement.propagate(x1, y1, 8)[0]) < TOL


def test_large_d_intra_and_overlap_across_pairs(sk, restatement, monkeypatch):
    """d > 16, streaming, one pair per group but several pairs per launch
    (SK_FORCE_GROUP=1): intra-CTA claims straddle the pairs' band ranges and
    the GEMM beside the sweep publishes row blocks per pair.  Band counts not
    multiples of four, tall and wide pairs; bit-identical to the serial,
    global-memory path, and to the oracle within tolerance."""
    rng = restatement.rng(777)
    xs = np.stack([rng.random_series(97, 24, 1.0) for _ in range(3)])
    ys = np.stack([rng.random_series(161, 24, 1.0) for _ in range(3)])

    def bits(v):
        return np.ascontiguousarray(v, dtype=np.float64).view(np.int64).tolist()

    def run():
        a = sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(8), want_max_abs_rho=True)
        b = sk.pairwise(ys, xs, sk.TruncationPolicy.fixed(8))
        return bits(a.values), bits(a.max_abs_rho), bits(b.values)

    monkeypatch.setenv("SK_RHO_FUSED", "0")
    monkeypatch.setenv("SK_STREAM", "1")
    monkeypatch.setenv("SK_FORCE_GROUP", "1")
    fast = run()
    monkeypatch.setenv("SK_NO_INTRA", "1")
    monkeypatch.setenv("SK_NO_OVERLAP", "1")
    serial = run()
    assert fast == serial
    for k in range(3):
        ref, _ = restatement.propagate(xs[k], ys[k], 8)
        assert rel(np.array(fast[0], dtype=np.int64).view(np.float64)[k], ref) < TOL


def test_large_d_fast_paths_randomised(sk, monkeypatch):
    """Random large-d single pairs (d 17..130, lengths 40..900, orders 4/8/12):
    the intra-CTA hand-over and the GEMM beside the sweep are bit-identical
    to the serial global-memory path (tools/large_d_stress.py at scale)."""
    rng = np.random.default_rng(5)
    opts = sk.PropagateOptions(strict_corner=False)
    for _ in range(30):
        d = int(rng.choice([17, 20, 33, 64, 130]))
        lx, ly = int(rng.integers(40, 900)), int(rng.integers(40, 900))
        order = int(rng.choice([4, 8, 12]))
        x = np.cumsum(rng.normal(0.0, 1.0 / np.sqrt(lx), size=(lx, d)), axis=0)
        y = np.cumsum(rng.normal(0.0, 1.0 / np.sqrt(ly), size=(ly, d)), axis=0)
        monkeypatch.delenv("SK_NO_INTRA", raising=False)
        monkeypatch.delenv("SK_NO_OVERLAP", raising=False)
        a = sk.propagate(x, y, order, opts).value
        monkeypatch.setenv("SK_NO_INTRA", "1")
        monkeypatch.setenv("SK_NO_OVERLAP", "1")
        b = sk.propagate(x, y, order, opts).value
        assert np.float64(a).view(np.int64) == np.float64(b).view(np.int64), (d, lx, ly, order)


@pytest.mark.parametrize("kernel", ["register", "runtime"])
def test_literal_kernels_bit_identical_to_the_reference(sk, restatement, monkeypatch, kernel):
    """The literal kernels -- the order-8 register-resident one the strict
    re-sweeps use, and the runtime-order one -- repeat the reference's
    arithmetic bit for bit (values, knot grids, max|rho|) across the delta
    paths (inline d <= 8, per-chunk d = 9..16, large d through the producer
    ring and the table)."""
    monkeypatch.setenv("SK_FORCE_LITERAL", "1")
    if kernel == "runtime":
        monkeypatch.setenv("SK_NO_LIT_REG", "1")
    rng = restatement.rng(8088)
    for d in (1, 2, 5, 8, 13, 16, 40):
        x = rng.random_series(70, d, 1.0)
        y = rng.random_series(90, d, 1.0)
        v_ref, _, g_ref = restatement.propagate(x, y, 8, grid=True)
        assert sk.propagate(x, y, 8).value == v_ref, d
        g = sk.propagate_grid(x, y, 8)
        assert np.asarray(g.grid).tolist() == g_ref.tolist(), d
        res = sk.pairwise(np.stack([x, x]), np.stack([y, y[::-1].copy()]), sk.TruncationPolicy.fixed(8),
                          want_max_abs_rho=True)
        assert res.values[0] == v_ref
        assert res.values[1] == restatement.propagate(x, y[::-1].copy(), 8)[0]
        assert res.max_abs_rho[0] == restatement.max_abs_rho(x, y)
        if d == 40:
            monkeypatch.setenv("SK_RHO_FUSED", "1")
            assert sk.propagate(x, y, 8).value == v_ref
            monkeypatch.delenv("SK_RHO_FUSED")


def test_gram_max_product_with_and_without_per_pair_maxima(sk, restatement):
    """GramResult.max_abs_increment_product (gram.cpp:89-96) is the exact
    maximum over the family whether or not the per-entry maxima are asked for
    (without them one launch-wide running max lets tiles skip the exact dot);
    with them every entry is its pair's exact max|rho|."""
    fam = [restatement.brownian(300 + 7 * k, 16, 90 + k) for k in range(6)]
    fam[3] = fam[3] * 2.5
    pol = sk.TruncationPolicy.adaptive(1e-12)
    a = sk.gram_matrix(fam, sk.GramOptions(policy=pol))
    b = sk.gram_matrix(fam, sk.GramOptions(policy=pol, pair_max_abs_rho=True))
    assert a.pair_max_abs_rho is None
    assert a.max_abs_increment_product == b.max_abs_increment_product
    assert np.asarray(a.values).tobytes() == np.asarray(b.values).tobytes()
    L = max(s.shape[0] for s in fam)
    padded = [np.concatenate([s, np.repeat(s[-1:], L - s.shape[0], axis=0)]) for s in fam]
    P = np.asarray(b.pair_max_abs_rho).reshape(6, 6)
    best = 0.0
    for i in range(6):
        for j in range(i, 6):
            mr = restatement.max_abs_rho(padded[i], padded[j])
            assert P[i, j] == mr and P[j, i] == mr
            best = max(best, mr)
    assert a.max_abs_increment_product == best
