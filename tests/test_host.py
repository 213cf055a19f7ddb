"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/sigker_b200.h declares, the host arithmetic
(estimate_order, shard ranges, live-series counter, error bound) matches the
reference (golden fixtures / oracle), argument validation follows the
reference's std::invalid_argument contract, and -- without a GPU -- compute
entry points fail loudly instead of falling back to the CPU."""
import ctypes
import json
import math
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sigker_b200.h")).read()
    return sorted(set(re.findall(r"\b(sk_[a-z_0-9]+)\s*\(", txt)))


def test_capi_exports_every_declared_symbol():
    from paper_2502_20392_b200 import _capi
    lib = _capi.load()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTED) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sk_[a-z_0-9]+)$", out, re.M))
    assert set(declared) <= exported
    assert lib.sk_abi_version() == 3


def test_estimate_order_matches_reference_table():
    from paper_2502_20392_b200 import sigker as sk
    for c in json.load(open(os.path.join(GOLD, "estimate_order.json")))["cases"]:
        e = sk.estimate_order(c["rho"], 16, c["tol"])
        assert (e.order, e.converged) == (c["order"], c["converged"])


def test_estimate_order_validation():
    from paper_2502_20392_b200 import sigker as sk
    with pytest.raises(ValueError):
        sk.estimate_order(1.0, 16, 0.0)
    with pytest.raises(ValueError):
        sk.estimate_order(-1.0, 16, 1e-12)
    with pytest.raises(ValueError):
        sk.estimate_order(float("inf"), 16, 1e-12)


def test_truncation_policy_contract():
    from paper_2502_20392_b200 import sigker as sk
    with pytest.raises(ValueError):
        sk.TruncationPolicy.fixed(0)
    with pytest.raises(ValueError):
        sk.TruncationPolicy.fixed(65)
    with pytest.raises(ValueError):
        sk.TruncationPolicy.adaptive(0.0)
    assert sk.TruncationPolicy().order == 7
    assert sk.TruncationPolicy.adaptive(1e-10).mode == "adaptive"


def test_bessel_and_bound_match_reference():
    from paper_2502_20392_b200 import sigker as sk
    m = json.load(open(os.path.join(GOLD, "truncation_misc.json")))
    for x, v in m["bessel_i0"]:
        assert sk.bessel_i0(x) == v
    for (mm, length, mx, n, v) in m["gram_error_bound"]:
        got = sk.gram_error_bound(sk.ErrorBoundInputs(mm, length, mx, n))
        assert got == pytest.approx(v, rel=1e-13, abs=0.0)


@pytest.mark.parametrize("rows,cols", [(1, 1), (1, 5), (5, 1), (4, 4), (32, 8), (8, 33), (63, 64), (200, 77)])
def test_peak_live_closed_form(restatement, rows, cols):
    from paper_2502_20392_b200 import sigker as sk
    assert sk._peak_live(rows, cols) == restatement.peak_live(rows, cols)


def test_peak_live_closed_form_dense(restatement):
    from paper_2502_20392_b200 import sigker as sk
    for rows in range(1, 48):
        for cols in range(1, 48):
            assert sk._peak_live(rows, cols) == restatement.peak_live(rows, cols), (rows, cols)


def test_time_series_contract():
    from paper_2502_20392_b200 import sigker as sk
    with pytest.raises(ValueError):
        sk.TimeSeries([1.0, 2.0, 3.0], 2)
    with pytest.raises(ValueError):
        sk.TimeSeries([1.0, float("nan")], 1)
    with pytest.raises(ValueError):
        sk.TimeSeries([], 1)
    t = sk.pad_to_length(sk.TimeSeries([[0.0, 1.0], [2.0, 3.0]]), 4)
    assert t.length() == 4 and t.values()[-1].tolist() == [2.0, 3.0]
    with pytest.raises(ValueError):
        sk.pad_to_length(t, 2)
    tab = sk.IncrementTable(np.array([[0.0], [1.0], [3.0]]), np.array([[0.0], [2.0]]))
    assert tab.rho(1, 0) == 4.0
    with pytest.raises(ValueError):
        tab.rho(2, 0)


def test_all_finite_scan():
    """sk_all_finite (the TimeSeries check) on the threaded and the serial path:
    one non-finite value anywhere -- first, last, chunk seams -- is found."""
    from paper_2502_20392_b200 import _capi, sigker as sk
    lib = _capi.load()
    for n in (1, 7, (1 << 20) + 3, 5 * (1 << 20) + 11):
        v = np.random.default_rng(n).standard_normal(n)
        assert lib.sk_all_finite(v.ctypes.data, n) == 1
        for pos in sorted({0, n - 1, n // 2, min(n - 1, 1 << 20), min(n - 1, (1 << 20) - 1)}):
            for bad in (np.nan, np.inf, -np.inf):
                w = v.copy()
                w[pos] = bad
                assert lib.sk_all_finite(w.ctypes.data, n) == 0, (n, pos, bad)
    big = np.zeros((1 << 21, 2))
    big[-1, 1] = np.inf
    with pytest.raises(ValueError):
        sk.TimeSeries(big)
    assert lib.sk_all_finite(np.full(4, 1.7976931348623157e308).ctypes.data, 4) == 1


def test_propagate_argument_validation():
    """wavefront.cpp:72-77: checked before any device work."""
    from paper_2502_20392_b200 import sigker as sk
    x = np.array([[0.0], [1.0]])
    with pytest.raises(ValueError):
        sk.propagate(x, np.array([[0.0, 0.0], [1.0, 1.0]]), 8)
    with pytest.raises(ValueError):
        sk.propagate(x, x, 0)
    with pytest.raises(ValueError):
        sk.propagate(x, x, 65)
    with pytest.raises(ValueError):
        sk.propagate(np.array([[1.0]]), x, 8)
    with pytest.raises(ValueError):
        sk.gram_matrix([])
    with pytest.raises(ValueError):
        sk.gram_matrix([x, np.array([[0.0, 1.0], [1.0, 2.0]])])


def test_no_cpu_fallback_without_gpu():
    from paper_2502_20392_b200 import sigker as sk
    if sk.device_count() > 0:
        pytest.skip("a GPU is visible")
    x = np.array([[0.0], [1.0]])
    with pytest.raises(sk.DeviceError):
        sk.propagate(x, x, 8)
    with pytest.raises(sk.DeviceError):
        sk.gram_matrix([x, x])


def test_shard_ranges_partition_the_upper_triangle():
    from paper_2502_20392_b200.distributed import shard_mask, shard_range
    for m in (1, 2, 5, 17, 64):
        total = m * (m + 1) // 2
        for n in (1, 2, 3, 8):
            bounds = [shard_range(m, s, n) for s in range(n)]
            assert bounds[0][0] == 0 and bounds[-1][1] == total
            assert all(bounds[s][1] == bounds[s + 1][0] for s in range(n - 1))
            assert max(b - a for a, b in bounds) - min(b - a for a, b in bounds) <= 1
            cover = sum(shard_mask(m, s, n).astype(int) for s in range(n))
            assert (cover == 1).all()


def _gram_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from oracle.oracle import Restatement
        from paper_2502_20392_b200 import sigker as sk
        from paper_2502_20392_b200.distributed import gram_matrix_distributed, shard_mask
        R = Restatement()
        rng = R.rng(11)
        family = [rng.random_series(7, 2, 1.0) for _ in range(6)]
        family.append(np.array([[0.0, 0.0], [1e4, 0.0]] + [[1e4, 0.0]] * 5))  # overflow entries

        def oracle_shard(fam, opt, shard, nshards):
            # stands in for the GPU shard computation on this CPU-only box
            arr = np.stack([s.values() for s in fam])
            vals, ords, mp, _ = R.gram(arr, adaptive=opt.policy.mode == "adaptive", order=opt.policy.order)
            mask = shard_mask(len(fam), shard, nshards)
            res = sk.GramResult(size=len(fam), values=np.where(mask, vals, np.nan).ravel(),
                                orders=np.where(mask, ords, 0).ravel(), adaptive=False)
            res.failures = [sk.GramEntryError(i, j, "overflow") for i in range(len(fam))
                            for j in range(i, len(fam)) if mask[i, j] and np.isnan(vals[i, j])]
            res.max_abs_increment_product = mp
            return res

        opts = sk.GramOptions(policy=sk.TruncationPolicy.fixed(12))
        r = gram_matrix_distributed(family, opts, compute=oracle_shard)
        full, ords, _, _ = R.gram(np.stack(family), adaptive=False, order=12)
        expect_fail = [(i, j) for i in range(7) for j in range(i, 7) if np.isnan(full[i, j])]
        ok = np.array_equal(np.isnan(r.values), np.isnan(full.ravel())) and \
            np.array_equal(np.nan_to_num(r.values), np.nan_to_num(full.ravel())) and \
            (r.orders == 12).all() and [(f.row, f.col) for f in r.failures] == expect_fail and \
            len(expect_fail) > 0
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_distributed_gram_assembly_gloo():
    """world_size 2 over gloo: shard ranges + all-reduce assembly reproduce
    the single-process Gram (CPU; the shard computation is injected)."""
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randint(0, 2000)
    procs = [ctx.Process(target=_gram_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


def test_strip_partition_and_error_order():
    from paper_2502_20392_b200.distributed import first_error, strip_bands, strip_ranges
    assert strip_bands(1_000_001, 8) == (1_000_000 + 31) // 32
    for bands in (2, 7, 31250):
        for world in (1, 2, 3, 8):
            if bands < world:
                continue
            r = strip_ranges(bands, world)
            assert r[0][0] == 0 and r[-1][1] == bands
            assert all(r[g][1] == r[g + 1][0] and r[g][0] < r[g][1] for g in range(world - 1))
    # earliest tile in (diagonal, row) order wins across strips
    recs = [None, (2, 10, 40, "a"), (3, 30, 19, "b"), (2, 20, 30, "c")]
    assert first_error(recs)[3] == "b"          # diagonal 47 < 48
    recs = [(2, 10, 40, "a"), (2, 20, 30, "c")]  # same diagonal: lower row first
    assert first_error(recs)[3] == "c"
    assert first_error([None, None]) is None


def test_block_cyclic_strip_plan():
    """The block-cyclic long-pair layout (sk_strip_plan / distributed.py):
    every band is owned by exactly one GPU, blocks are dealt round-robin, a
    GPU's exchange rounds are the blocks >= 1 it owns, block sizes never
    exceed the resident band workers, and the host model (tools/strip_sim.py)
    scales where the contiguous layout of round 1 does not."""
    from paper_2502_20392_b200.distributed import BAND_WORKERS, block_owner, strip_bands, strip_block, strip_plan
    for ly, world in ((400, 1), (400, 3), (1_000_001, 8), (65_537, 2), (33, 1)):
        bands = strip_bands(ly, 8)
        for block in (1, 2, 5, strip_block(bands, world)):
            if -(-bands // block) < world:
                continue
            owned = [0] * world
            for b in range(bands):
                owned[block_owner(b, world, block)] += 1
            nblocks = -(-bands // block)
            for g in range(world):
                o, rounds, in_rounds = strip_plan(ly, 8, world, g, block)
                mine = list(range(g, nblocks, world))
                assert o == owned[g]
                assert rounds == len(mine)
                assert in_rounds == (max(mine) // world + 1 if any(k >= 1 for k in mine) else 0)
    bands = strip_bands(1_000_001, 8)
    for world in (1, 2, 4, 8):
        assert strip_block(bands, world) <= BAND_WORKERS
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import strip_sim
    # more bands per GPU than resident workers: contiguous strips starve
    kw = dict(dt_ns=100_000.0, workers=100)
    t1 = strip_sim.simulate(49_999, 2_000, 1, **kw)
    t4c = strip_sim.simulate(49_999, 2_000, 4, "cyclic", block=100, **kw)
    t4s = strip_sim.simulate(49_999, 2_000, 4, "contiguous", **kw)
    assert t4c < 0.5 * t4s
    assert t1 / (4 * t4c) > 0.8


def test_segment_dag_model():
    """The segment-DAG schedule's dependency rules (tools/segment_dag_sim.py
    mirrors csrc/sk_sweep.cuh): every unit runs once, after its inputs, for
    ragged shapes including one-column pairs (the band above starts later than
    the band below ends) and slot reuse."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("segsim", os.path.join(ROOT, "tools", "segment_dag_sim.py"))
    sim = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sim)
    for rows in (1, 31, 32, 33, 64, 65, 100, 300):
        for cols in (1, 2, 3, 31, 32, 33, 100):
            for L in (32, 64, 96, 256):
                for slots in (1, 2, 5):
                    sim.simulate(rows, cols, 5, slots, 32, L)


def test_long_pair_devices_rejects_a_shared_gpu():
    """Strips wait on each other: two strips on one GPU are refused up front
    (no GPU needed to reach the check)."""
    from paper_2502_20392_b200 import distributed as skd
    x = np.cumsum(np.ones((40, 2)), axis=0)
    with pytest.raises(ValueError, match="distinct"):
        skd.propagate_long_pair_devices(x, x, 8, devices=[0, 0])


# ------------------------------------------------------------- bench plumbing
def test_bench_step_ranges_tile_the_gram():
    """bench.py's step split: for every world size the ranks' ranges tile
    each slice, and the slices tile the upper triangle, in row-major order
    (sk_gram_shard_range arithmetic)."""
    import bench
    for ws in (1, 2, 3, 8):
        covered = []
        for step in range(bench.SLICES):
            parts = [bench.step_range(step, r, ws) for r in range(ws)]
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            covered.append((parts[0][0], parts[-1][1]))
        assert covered[0][0] == 0 and covered[-1][1] == bench.TOTAL_PAIRS
        for (a, b), (c, d) in zip(covered, covered[1:]):
            assert b == c
    lib = __import__("paper_2502_20392_b200._capi", fromlist=["load"]).load()
    import ctypes
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    for shard, n in ((0, 32), (5, 64), (63, 64)):
        lib.sk_gram_shard_range(bench.M, shard, n, ctypes.byref(lo), ctypes.byref(hi))
        assert (lo.value, hi.value) == bench.pair_range(bench.TOTAL_PAIRS, shard, n)
    assert bench.pair_of(0) == (0, 0) and bench.pair_of(bench.M) == (1, 1)
    assert bench.pair_of(bench.TOTAL_PAIRS - 1) == (bench.M - 1, bench.M - 1)


def test_bench_spawns_ranks_and_assembles_over_gloo():
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run; --cpu-smoke runs the multi-rank split, all-reduce
    assembly and max-over-ranks timing over gloo with the C restatement as
    the per-rank computation."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--cpu-smoke"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["world_size"] == 2 and line["assembled_equals_single_process"]


def test_bench_refuses_more_gpus_than_visible():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "GPU(s) visible" in out.stderr


def test_block_cyclic_kernel_indexing_model():
    """The sweep kernel's strip indexing (sk_sweep.cuh: unit -> band decode,
    column-buffer slot, exchange-area rounds), restated in Python: every band
    is swept by exactly one GPU, in increasing order on that GPU; a GPU's
    concurrently live blocks never share a column buffer; and at every block
    boundary the producer writes exactly the exchange slot its consumer reads,
    in the consumer GPU's area."""
    from paper_2502_20392_b200.distributed import strip_plan
    for ly, G, S in ((400, 2, 3), (400, 3, 1), (1_000_001, 8, 1302), (999, 4, 7), (33, 1, 1)):
        bands = (ly - 1 + 31) // 32
        nblocks = -(-bands // S)
        if nblocks < G:
            continue
        seen = []
        for g in range(G):
            owned, rounds, in_rounds = strip_plan(ly, 8, G, g, S)
            decoded = []
            for bi in range(owned):  # sweep_kernel streaming decode
                b = (g + G * (bi // S)) * S + bi % S
                decoded.append(b)
                blk = b // S
                assert blk % G == g and b < bands
                assert blk // G < rounds  # column-buffer slot (round) exists
                if b > 0 and b % S == 0:  # bottom band of a block: reads this GPU's area
                    assert blk // G < in_rounds
                if b + 1 < bands and (b + 1) % S == 0:  # top band: writes GPU (blk+1) mod G's area
                    consumer = (blk + 1) % G
                    _, _, c_in = strip_plan(ly, 8, G, consumer, S)
                    assert (blk + 1) // G < c_in
            assert decoded == sorted(decoded)
            seen += decoded
        assert sorted(seen) == list(range(bands))
