"""Tile totals only where the final tile can fall (sk_sweep.cuh kFlagAllTotals).

Throughput sweeps skip the per-tile total except in the chunks that can hold a
pair's final tile; a pair that ends flagged or non-finite is swept again with
every total formed and checked.  Values, orders, max|rho| and the reported
error (kind and tile) must be exactly those of the every-tile-checked sweep
(SK_ALL_TOTALS=1), on both schedules, for pairwise, single pairs and Gram."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(v):
    return np.ascontiguousarray(v, dtype=np.float64).view(np.int64).tolist()


def outcome(fn):
    try:
        return ("ok", bits([fn().value]))
    except Exception as e:  # noqa: BLE001 -- the error kind and tile are the contract
        return (type(e).__name__, getattr(e, "tile_k", None), getattr(e, "tile_l", None), str(e))


def test_final_tile_totals_match_every_tile_totals(sk, restatement, monkeypatch):
    rng = restatement.rng(2024)
    cases = []
    for (lx, ly, d, order, npairs) in [(300, 200, 2, 7, 3), (130, 97, 4, 12, 2), (66, 260, 8, 16, 1),
                                       (90, 64, 40, 8, 1), (41, 150, 12, 5, 3), (2, 300, 2, 8, 1),
                                       (400, 20, 1, 1, 1), (257, 129, 16, 10, 2), (520, 530, 3, 8, 2)]:
        xs = np.stack([rng.random_series(lx, d, 1.0) for _ in range(npairs)])
        ys = np.stack([rng.random_series(ly, d, 1.0) for _ in range(npairs)])
        cases.append((xs, ys, order))
    # failures: a delta overflow mid-pair, a series that overflows to inf with
    # every |delta| below the guard (non-finite total, no other flag), and
    # sigma-scaled pairs where the corner check can fire
    x = rng.random_series(80, 1, 1.0)
    y = rng.random_series(90, 1, 1.0)
    x[40:] *= 3e4
    y[50:] *= 3e4
    ramp_x = (np.arange(40, dtype=np.float64) * 31.6).reshape(-1, 1)
    ramp_y = (np.arange(45, dtype=np.float64) * 31.6).reshape(-1, 1)
    bx = restatement.brownian(300, 2, 5) * 6.0
    by = restatement.brownian(280, 2, 6) * 6.0
    fam = [restatement.brownian(70, 3, 40 + s) for s in range(5)]
    fam[2] = fam[2] * 40.0

    def run_all():
        out = []
        for xs, ys, order in cases:
            out.append(bits(sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(order)).values))
            a = sk.pairwise(xs, ys, sk.TruncationPolicy.adaptive(1e-12), want_max_abs_rho=True)
            out.append((bits(a.values), list(a.orders), bits(a.max_abs_rho)))
        for strict in (True, False):
            opt = sk.PropagateOptions(strict_corner=strict)
            for (u, v) in ((x, y), (ramp_x, ramp_y), (bx, by)):
                out.append(outcome(lambda: sk.propagate(u, v, 8, opt)))
        for strict in (True, False):
            try:
                p = sk.pairwise(np.stack([ramp_x[:40], ramp_x[:40] * 1e-3]), np.stack([ramp_y[:40], ramp_y[:40]]),
                                sk.TruncationPolicy.fixed(8), sk.PropagateOptions(strict_corner=strict))
                out.append((bits(p.values), p.failures))
            except Exception as e:  # noqa: BLE001
                out.append((type(e).__name__, str(e)))
        try:
            g = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.fixed(8)))
            out.append((bits(g.values), [(f.row, f.col) for f in g.failures]))
        except Exception as e:  # noqa: BLE001
            out.append((type(e).__name__, str(e)))
        return out

    for sched in ({"SK_STREAM": "1"}, {"SK_FORCE_SEGMENTS": "1", "SK_SEG_COLS": "64"}, {}):
        for k, v in sched.items():
            monkeypatch.setenv(k, v)
        monkeypatch.setenv("SK_ALL_TOTALS", "1")
        ref = run_all()
        monkeypatch.delenv("SK_ALL_TOTALS")
        got = run_all()
        assert len(got) == len(ref)
        for k, (a, b) in enumerate(zip(got, ref)):
            assert a == b, (sched, k, str(a)[:300], str(b)[:300])
        for k in sched:
            monkeypatch.delenv(k)
    # the non-finite case really is one: the reference's NumericOverflowError
    assert outcome(lambda: sk.propagate(ramp_x, ramp_y, 8, sk.PropagateOptions(strict_corner=False)))[0] \
        == "NumericOverflowError"


def test_failing_pair_is_swept_again(sk, restatement):
    """A flagged pair costs a second, fully checked sweep; a clean one does not."""
    x = (np.arange(40, dtype=np.float64) * 31.6).reshape(-1, 1)
    sk.stats_enable(True)
    sk.stats_reset()
    with pytest.raises(sk.NumericOverflowError):
        sk.propagate(x, x, 8, sk.PropagateOptions(strict_corner=False))
    assert sk.stats_get()["sweep_launches"] == 2
    sk.stats_reset()
    sk.propagate(restatement.brownian(100, 2, 1), restatement.brownian(100, 2, 2), 8)
    assert sk.stats_get()["sweep_launches"] == 1


def test_staged_upload_of_pageable_inputs(sk, restatement, monkeypatch):
    """Large pageable inputs go through pinned staging (sk_capi.cu h2d, 8 host
    threads, 4 MB chunks); the result is bit-identical to a plain copy.  The
    byte count is not a multiple of the chunk; the second call reuses the
    staging buffers."""
    rng = np.random.default_rng(99)
    npairs, length, d = 2047, 1023, 7
    xs = np.cumsum(rng.standard_normal((npairs, length, d)) / 32.0, axis=1)
    ys = np.cumsum(rng.standard_normal((npairs, length, d)) / 32.0, axis=1)
    assert xs.nbytes % (4 << 20) != 0 and xs.nbytes > (16 << 20)
    pol = sk.TruncationPolicy.adaptive(1e-12)
    a = sk.pairwise(xs, ys, pol)
    b = sk.pairwise(xs[::-1].copy(), ys[::-1].copy(), pol)
    monkeypatch.setenv("SK_NO_STAGING", "1")
    ref = sk.pairwise(xs, ys, pol)
    assert bits(a.values) == bits(ref.values)
    assert bits(b.values) == bits(ref.values[::-1])
    k = 1234
    want = restatement.propagate(xs[k], ys[k], int(ref.orders[k]))[0]
    assert abs(ref.values[k] - want) <= 1e-10 * max(1.0, abs(want))
