"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle
(oracle/sigker_oracle.c restatement, itself pinned to the reference and the
golden fixtures).  Tolerance: |K_gpu - K_ref| / max(1, |K_ref|) <= 1e-10 in
fp64 (BASELINE.json north_star), identical truncation order per pair."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def test_single_tile_bessel(sk):
    x = np.array([[0.0], [1.0]])
    r = sk.propagate(x, x, 24)
    assert rel(r.value, 2.2795853023360673) < 1e-14


def test_config1_brownian_adaptive(sk, restatement):
    x = restatement.brownian(1000, 2, 1)
    y = restatement.brownian(1000, 2, 2)
    r = sk.propagate_with_policy(x, y, sk.TruncationPolicy.adaptive(1e-12))
    assert r.order == 8
    assert rel(r.value, 1.2640724761915605) < TOL


@pytest.mark.parametrize("order", [1, 2, 7, 8, 12, 16, 17, 24])
@pytest.mark.parametrize("shape", [(2, 2, 1), (5, 9, 2), (40, 70, 3), (70, 40, 4), (97, 33, 8), (33, 97, 16)])
def test_random_series_orders(sk, restatement, order, shape):
    lx, ly, d = shape
    rng = restatement.rng(1000 * order + lx)
    x = rng.random_series(lx, d, 1.0)
    y = rng.random_series(ly, d, 1.0)
    v_ref, pk_ref = restatement.propagate(x, y, order)
    r = sk.propagate(x, y, order)
    assert rel(r.value, v_ref) < TOL
    assert r.peak_live_series == pk_ref


def test_large_dim_table_path(sk, restatement):
    rng = restatement.rng(77)
    x = rng.random_series(50, 40, 1.0)
    y = rng.random_series(45, 40, 1.0)
    v_ref, _ = restatement.propagate(x, y, 8)
    assert rel(sk.propagate(x, y, 8).value, v_ref) < TOL


def test_grid_matches_oracle(sk, restatement):
    rng = restatement.rng(321)
    x = rng.random_series(12, 2, 1.0)
    y = rng.random_series(13, 2, 1.0)
    _, _, g_ref = restatement.propagate(x, y, 14, grid=True)
    r = sk.propagate_grid(x, y, 14)
    assert r.grid.shape == g_ref.shape
    assert np.max(np.abs(r.grid - g_ref) / np.maximum(1.0, np.abs(g_ref))) < TOL


def test_overflow_guard(sk):
    x = np.array([[0.0], [400.0]])
    with pytest.raises(sk.NumericOverflowError) as e:
        sk.propagate(x, x, 24)
    assert e.value.tile_k == 1 and e.value.tile_l == 1
    assert "rescale" in str(e.value)
