"""Paired bands (sk_sweep.cuh sweep_pair_kernel): for latency-bound streaming
launches each band runs on two warps, the alpha warp (waits, staging, alpha',
totals, checks, outputs) and the beta warp (beta').  The split evaluates the
same expressions in the same order as the one-warp band, so every output --
values, knot grids, error tiles -- must be bit-identical to the one-warp
streaming schedule, and the product must match the oracle like every other
path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10


def bits(v):
    return np.ascontiguousarray(v, dtype=np.float64).view(np.int64).tolist()


def test_paired_bands_bit_identical_to_one_warp_bands(sk, restatement, monkeypatch):
    rng = restatement.rng(77)
    cases = []
    # inline products (d <= 8), per-chunk products (d = 9..16), rho table (d > 16);
    # ragged shapes, one band, one column, orders 1..16
    for (lx, ly, d, order, npairs) in [(300, 200, 2, 7, 1), (130, 97, 4, 12, 2), (66, 260, 8, 16, 1),
                                       (90, 64, 40, 8, 1), (41, 150, 12, 5, 3), (2, 300, 2, 8, 1),
                                       (400, 20, 1, 1, 1), (170, 3, 3, 3, 2), (257, 129, 16, 10, 1)]:
        xs = np.stack([rng.random_series(lx, d, 1.0) for _ in range(npairs)])
        ys = np.stack([rng.random_series(ly, d, 1.0) for _ in range(npairs)])
        cases.append((xs, ys, order))
    x = rng.random_series(80, 1, 1.0)
    y = rng.random_series(90, 1, 1.0)
    x[40:] *= 3e4
    y[50:] *= 3e4

    def run_all():
        out = []
        for xs, ys, order in cases:
            out.append(bits(sk.pairwise(xs, ys, sk.TruncationPolicy.fixed(order)).values))
            out.append(bits(sk.propagate_grid(xs[0], ys[0], order).grid))
            out.append(bits([sk.propagate(xs[0], ys[0], order, diag=True).value]))
        for strict in (True, False):
            try:
                out.append(bits([sk.propagate(x, y, 8, sk.PropagateOptions(strict_corner=strict)).value]))
            except sk.NumericOverflowError as e:
                out.append(("overflow", e.tile_k, e.tile_l))
            except sk.InconsistentBoundaryError as e:
                out.append(("corner", str(e)))
        return out

    monkeypatch.setenv("SK_STREAM", "1")
    monkeypatch.setenv("SK_PAIRED", "0")
    sk.stats_enable(True)
    sk.stats_reset()
    ref = run_all()
    assert sk.stats_get()["paired_launches"] == 0
    monkeypatch.setenv("SK_PAIRED", "1")
    sk.stats_reset()
    got = run_all()
    assert sk.stats_get()["paired_launches"] > 0
    assert len(got) == len(ref)
    for k, (a, b) in enumerate(zip(got, ref)):
        assert a == b, (k, str(a)[:300], str(b)[:300])
    # slot reuse inside one paired launch (more pairs than slots)
    monkeypatch.setenv("SK_FORCE_SLOTS", "1")
    monkeypatch.setenv("SK_FORCE_GROUP", "1")
    got2 = run_all()
    for k, (a, b) in enumerate(zip(got2, ref)):
        assert a == b, (k, str(a)[:300], str(b)[:300])


def test_paired_bands_chosen_for_a_single_long_pair(sk, restatement, monkeypatch):
    """With SK_PAIRED=1 the schedule picks paired bands for one long pair and
    matches the oracle (the reference's algorithm) at the parity tolerance."""
    monkeypatch.setenv("SK_PAIRED", "1")
    x = restatement.brownian(1500, 2, 11)
    y = restatement.brownian(1200, 2, 12)
    sk.stats_enable(True)
    sk.stats_reset()
    got = sk.propagate(x, y, 8).value
    assert sk.stats_get()["paired_launches"] == 1
    want = restatement.propagate(x, y, 8)[0]
    assert abs(got - want) <= TOL * max(1.0, abs(want)), (got, want)
