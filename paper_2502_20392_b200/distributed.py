"""Multi-GPU Gram matrix: row-block sharding over torch.distributed ranks
(one process per GPU).

The upper-triangle pair list (i <= j, row-major -- gram.cpp:39-42) is cut
into `world_size` contiguous ranges of equal pair count (sk_gram_shard_range;
all pairs cost the same because gram_matrix pads the family to one length).
Every rank evaluates its range on its own GPU with no communication during
compute; one all-reduce then assembles the matrix (entries outside a rank's
range contribute 0, failed entries stay NaN because NaN + 0 = NaN).  Over
NVLink the assembly moves 8 m^2 bytes (8 MB at m = 1024), negligible next to
the compute, so the collective is plain NCCL (backend of the process group).
"""
from __future__ import annotations

import ctypes
import math
from typing import Callable, Optional, Sequence

import numpy as np

from . import _capi
from . import sigker as sk


def shard_range(m: int, shard: int, nshards: int):
    """[first, last) row-major upper-triangle pair indices of `shard`."""
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    rc = _capi.load().sk_gram_shard_range(m, shard, nshards, ctypes.byref(lo), ctypes.byref(hi))
    if rc != 0:
        raise ValueError(f"shard {shard} out of range [0, {nshards})")
    return lo.value, hi.value


def shard_mask(m: int, shard: int, nshards: int) -> np.ndarray:
    """m x m boolean mask of the (mirrored) entries `shard` owns."""
    lo, hi = shard_range(m, shard, nshards)
    mask = np.zeros((m, m), dtype=bool)
    t = 0
    for i in range(m):
        row_len = m - i
        a, b = max(lo, t), min(hi, t + row_len)
        if a < b:
            js = np.arange(i + (a - t), i + (b - t))
            mask[i, js] = True
            mask[js, i] = True
        t += row_len
    return mask


def gram_matrix_distributed(family: Sequence, options: Optional[sk.GramOptions] = None, group=None,
                            compute: Optional[Callable] = None, device=None, shard: int = 0,
                            nshards: int = 1) -> sk.GramResult:
    """gram_matrix over all ranks of `group` (default: the world group).

    The upper-triangle pairs of shard `shard` of `nshards` (default: the whole
    Gram) are split over the ranks: rank r evaluates sub-shard
    shard * world + r of nshards * world, so the ranks' ranges tile the shard
    exactly.  `compute(family, options, shard, nshards) -> GramResult`
    evaluates one sub-shard; it defaults to the GPU path (sk.gram_matrix).
    Every rank returns the assembled GramResult (entries outside the shard
    NaN, as gram_matrix leaves them)."""
    import torch
    import torch.distributed as dist

    options = options or sk.GramOptions()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    compute = compute or (lambda fam, opt, s, n: sk.gram_matrix(fam, opt, shard=s, nshards=n))
    if isinstance(family, np.ndarray) and family.ndim == 3:
        fam = family  # an (m, length, dim) block: gram_matrix's no-copy path
        m, length = family.shape[0], max(2, family.shape[1])
    else:
        fam = [sk._as_series(s) for s in family]
        m, length = len(fam), max(2, max(s.length() for s in fam))
    err = None
    try:
        local = compute(fam, options, shard * world + rank, nshards * world)
    except sk.InconsistentBoundaryError as e:  # gram.cpp:74-77 lets it propagate
        err, local = str(e), None
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
            else torch.device("cpu")
    flag = torch.tensor([1.0 if err else 0.0], dtype=torch.float64, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if flag.item() > 0:
        raise sk.InconsistentBoundaryError(err or "inconsistent boundary on another rank")
    mask = shard_mask(m, shard * world + rank, nshards * world)
    vals = np.where(mask, np.asarray(local.values).reshape(m, m), 0.0)
    ords = np.where(mask, np.asarray(local.orders).reshape(m, m), 0).astype(np.float64)
    pmax = np.zeros((m, m)) if local.pair_max_abs_rho is None else \
        np.where(mask, np.asarray(local.pair_max_abs_rho).reshape(m, m), 0.0)
    buf = torch.from_numpy(np.stack([vals, ords, pmax])).to(device)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    stats = torch.tensor([local.max_abs_increment_product, 0.0 if local.orders_converged else 1.0],
                         dtype=torch.float64, device=device)
    dist.all_reduce(stats, op=dist.ReduceOp.MAX, group=group)
    failures = [None] * world
    dist.all_gather_object(failures, [(f.row, f.col, f.message) for f in local.failures], group=group)
    out = buf.cpu().numpy()
    if nshards > 1:
        outside = ~shard_mask(m, shard, nshards)
        out[0][outside] = np.nan
    r = sk.GramResult(size=m, values=out[0].ravel(), orders=out[1].ravel().astype(np.int32),
                      adaptive=local.adaptive, orders_converged=stats[1].item() == 0.0,
                      wall_seconds=local.wall_seconds)
    r.failures = [sk.GramEntryError(a, b, msg) for lst in failures for (a, b, msg) in lst]
    r.failures.sort(key=lambda e: (e.row, e.col))
    computed = r.orders[r.orders > 0]
    r.min_order = int(computed.min()) if computed.size else 0
    r.max_order = int(computed.max()) if computed.size else 0
    r.max_abs_increment_product = float(stats[0].item())
    r.pair_max_abs_rho = out[2].ravel() if local.pair_max_abs_rho is not None else None
    n_ok = int(np.sum(~np.isnan(r.values)))
    r.peak_live_series = sk._peak_live(length - 1, length - 1) if n_ok else 0
    if options.compute_bound:
        r.bound = sk.gram_error_bound(sk.ErrorBoundInputs(m, length, r.max_abs_increment_product, r.min_order))
    else:
        r.bound = math.nan
    return r


# ------------------------------------------------------------ long pairs
# Resident band workers of one B200 at the register kernels' 12 one-warp CTAs
# per SM: the block size of the cyclic strip layout.
BAND_WORKERS = 12 * 148


def strip_ranges(bands: int, world: int):
    """Contiguous, balanced band ranges [b0, b1), one per rank (round 1's
    layout; kept for the error-order helpers and comparisons)."""
    return [(bands * g // world, bands * (g + 1) // world) for g in range(world)]


def strip_block(bands: int, world: int, workers: int = BAND_WORKERS) -> int:
    """Block size of the block-cyclic layout: the bands split into
    world x rounds equal blocks, rounds = ceil(bands / (world x workers)),
    so a GPU's block never exceeds its resident band workers."""
    rounds = max(1, -(-bands // (world * workers)))
    return max(1, -(-bands // (world * rounds)))


def strip_plan(ly: int, order: int, world: int, rank: int, block: int):
    """(owned bands, column-buffer rounds, exchange rounds received) of rank
    `rank` in the block-cyclic layout (sk_strip_plan)."""
    o, r, i = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    if _capi.load().sk_strip_plan(ly, int(order), world, rank, block, ctypes.byref(o), ctypes.byref(r),
                                  ctypes.byref(i)) != 0:
        raise ValueError("strip_plan: bad arguments")
    return o.value, r.value, i.value


def block_owner(band: int, world: int, block: int) -> int:
    return (band // block) % world


def first_error(records):
    """The reference's 1-thread throw order (wavefront.cpp:133-173): among
    per-strip first failures (code, tile_k, tile_l, message), the earliest
    tile in (diagonal, row) order wins."""
    best = None
    for rec in records:
        if rec is None:
            continue
        code, k, l, msg = rec
        key = (k - 1 + l - 1, l - 1)
        if best is None or key < best[0]:
            best = (key, rec)
    return None if best is None else best[1]


def _raise_first(recs):
    err = first_error(recs)
    if err is not None:
        code, k, l, msg = err
        if code == _capi.SK_NUMERIC_OVERFLOW:
            raise sk.NumericOverflowError(msg, k, l)
        if code == _capi.SK_INCONSISTENT_BOUNDARY:
            raise sk.InconsistentBoundaryError(msg)
        raise RuntimeError(msg)


def propagate_long_pair_distributed(x, y, order: int, options: Optional[sk.PropagateOptions] = None,
                                    group=None, diag: bool = False, block: Optional[int] = None):
    """K(1,1) of ONE long pair over the ranks of `group` (one process per GPU,
    SURVEY.md section 8e), block-cyclic: the 32-row bands are cut into blocks
    of `block` bands (default strip_block) dealt round-robin over the ranks;
    at every block boundary the top band streams its alpha series straight
    into the next rank's exchange area over NVLink (CUDA IPC peer mapping,
    system-scope release/acquire; the last rank hands to rank 0).  Every rank
    returns (value, diag-or-None); diag holds this rank's knots K(a, a)
    (NaN elsewhere)."""
    import torch.distributed as dist

    x, y = sk._as_series(x), sk._as_series(y)
    if x.dim() != y.dim():
        raise ValueError("propagate: series dimensions differ")
    lib = _capi.load()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lx, ly, d = x.length(), y.length(), x.dim()
    bands = strip_bands(ly, order)
    block = block or strip_block(bands, world)
    nblocks = -(-bands // block)
    if nblocks < world:
        raise ValueError(f"{nblocks} blocks of {block} bands cannot feed {world} GPUs")
    _, _, in_rounds = strip_plan(ly, order, world, rank, block)
    sends = any(k + 1 < nblocks for k in range(rank, nblocks, world))
    st = _capi.SkStatus()
    in_a, in_p, out_a, out_p = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    handles = None
    if world > 1 and in_rounds > 0:
        sk._check(lib.sk_exchange_alloc(lx, int(order), in_rounds, ctypes.byref(in_a), ctypes.byref(in_p),
                                        ctypes.byref(st)), st)
        ha, hp = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
        sk._check(lib.sk_ipc_handle(in_a, ha, ctypes.byref(st)), st)
        sk._check(lib.sk_ipc_handle(in_p, hp, ctypes.byref(st)), st)
        handles = (bytes(ha), bytes(hp))
    all_handles = [None] * world
    dist.all_gather_object(all_handles, handles, group=group)
    nxt = (rank + 1) % world
    try:
        if world > 1 and sends:
            ha, hp = all_handles[nxt]
            sk._check(lib.sk_ipc_open(ctypes.create_string_buffer(ha, 64), ctypes.byref(out_a), ctypes.byref(st)), st)
            sk._check(lib.sk_ipc_open(ctypes.create_string_buffer(hp, 64), ctypes.byref(out_p), ctypes.byref(st)), st)
        dist.barrier(group=group)
        value = ctypes.c_double(float("nan"))
        dg = np.full(min(lx, ly) - 1, np.nan) if diag else None
        xv, yv = x.values(), y.values()
        rc = lib.sk_propagate_strip(sk._ptr(xv), lx, sk._ptr(yv), ly, d, int(order), sk._flags(options), world, rank,
                                    block, in_a if in_a.value else None, in_p if in_p.value else None,
                                    out_a if out_a.value else None, out_p if out_p.value else None,
                                    ctypes.byref(value), sk._ptr(dg) if dg is not None else None, ctypes.byref(st))
        rec = None if rc == 0 else (int(st.code), int(st.tile_k), int(st.tile_l), st.message.decode(errors="replace"))
        recs = [None] * world
        owner_last = (nblocks - 1) % world
        dist.all_gather_object(recs, (rec, value.value if rank == owner_last else None), group=group)
    finally:
        dist.barrier(group=group)
        if out_a.value:
            lib.sk_ipc_close(out_a)
        if out_p.value:
            lib.sk_ipc_close(out_p)
        if in_a.value:
            lib.sk_exchange_free(in_a, in_p)
    _raise_first([r for r, _ in recs])
    final = [v for _, v in recs if v is not None][0]
    return final, dg


def propagate_split_emulated(x, y, order: int, block: int, options: Optional[sk.PropagateOptions] = None,
                             gpus: int = 1):
    """One-GPU test of the strip protocol: a single launch over all bands of
    `gpus` virtual GPUs in the block-cyclic layout, every `block` bands handed
    over through an exchange area exactly as between GPUs
    (sk_propagate_split)."""
    x, y = sk._as_series(x), sk._as_series(y)
    lib = _capi.load()
    st = _capi.SkStatus()
    value = ctypes.c_double()
    xv, yv = x.values(), y.values()
    rc = lib.sk_propagate_split(sk._ptr(xv), x.length(), sk._ptr(yv), y.length(), x.dim(), int(order),
                                sk._flags(options), int(gpus), int(block), ctypes.byref(value), ctypes.byref(st))
    sk._check(rc, st)
    return value.value


def strip_bands(ly: int, order: int) -> int:
    nb = ctypes.c_size_t()
    if _capi.load().sk_strip_bands(ly, int(order), ctypes.byref(nb)) != 0:
        raise ValueError("bad length/order")
    return nb.value


def propagate_long_pair_devices(x, y, order: int, devices: Sequence[int],
                                options: Optional[sk.PropagateOptions] = None, diag: bool = False,
                                block: Optional[int] = None):
    """K(1,1) of ONE long pair over several GPUs driven from this process (the
    SURVEY.md section 8b device-list option; the multi-process variant is
    propagate_long_pair_distributed): the same block-cyclic layout, one host
    thread per device, exchange areas reached through peer access (NVLink).
    Returns (value, diag-or-None).  The devices must be distinct: GPUs wait on
    each other, so two of them must never share one (one GPU: sk.propagate)."""
    import threading

    devices = [int(dv) for dv in devices]
    if len(set(devices)) != len(devices):
        raise ValueError("propagate_long_pair_devices: devices must be distinct (strips wait on each other)")
    x, y = sk._as_series(x), sk._as_series(y)
    if len(devices) <= 1:
        lib = _capi.load()
        if devices:
            st = _capi.SkStatus()
            sk._check(lib.sk_set_device(devices[0], ctypes.byref(st)), st)
        r = sk.propagate(x, y, order, options, diag=diag)
        return r.value, (r.diag if diag else None)
    if x.dim() != y.dim():
        raise ValueError("propagate: series dimensions differ")
    lib = _capi.load()
    lx, ly, d = x.length(), y.length(), x.dim()
    world = len(devices)
    bands = strip_bands(ly, order)
    block = block or strip_block(bands, world)
    nblocks = -(-bands // block)
    if nblocks < world:
        raise ValueError(f"{nblocks} blocks of {block} bands cannot feed {world} GPUs")
    st = _capi.SkStatus()
    xbuf = [None] * world  # exchange area (abuf, prog) on each receiving device
    try:
        for g in range(world):
            _, _, in_rounds = strip_plan(ly, order, world, g, block)
            if in_rounds == 0:
                continue
            sk._check(lib.sk_set_device(devices[g], ctypes.byref(st)), st)
            a, p = ctypes.c_void_p(), ctypes.c_void_p()
            sk._check(lib.sk_exchange_alloc(lx, int(order), in_rounds, ctypes.byref(a), ctypes.byref(p),
                                            ctypes.byref(st)), st)
            xbuf[g] = (a, p)
        for g in range(world):
            sk._check(lib.sk_set_device(devices[g], ctypes.byref(st)), st)
            sk._check(lib.sk_enable_peer_access(devices[(g + 1) % world], ctypes.byref(st)), st)
        xv, yv = x.values(), y.values()
        out = [None] * world
        dg = np.full(min(lx, ly) - 1, np.nan) if diag else None
        parts = [np.full(min(lx, ly) - 1, np.nan) if diag else None for _ in range(world)]

        def strip(g):
            s = _capi.SkStatus()
            v = ctypes.c_double(float("nan"))
            rc = lib.sk_set_device(devices[g], ctypes.byref(s))
            if rc == 0:
                sends = any(k + 1 < nblocks for k in range(g, nblocks, world))
                inn, nxt = xbuf[g], xbuf[(g + 1) % world] if sends else None
                rc = lib.sk_propagate_strip(sk._ptr(xv), lx, sk._ptr(yv), ly, d, int(order), sk._flags(options),
                                            world, g, block, inn[0] if inn else None, inn[1] if inn else None,
                                            nxt[0] if nxt else None, nxt[1] if nxt else None, ctypes.byref(v),
                                            sk._ptr(parts[g]) if diag else None, ctypes.byref(s))
            out[g] = (rc, s, v.value)

        threads = [threading.Thread(target=strip, args=(g,)) for g in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        for g in range(world):
            if xbuf[g] is not None:
                lib.sk_exchange_free(xbuf[g][0], xbuf[g][1])
    _raise_first([None if rc == 0 else (int(s.code), int(s.tile_k), int(s.tile_l), s.message.decode(errors="replace"))
                  for rc, s, _ in out])
    if diag:
        for g in range(world):
            sel = ~np.isnan(parts[g])
            dg[sel] = parts[g][sel]
    return out[(nblocks - 1) % world][2], dg
