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
    r.pair_max_abs_rho = out[2].ravel()
    n_ok = int(np.sum(~np.isnan(r.values)))
    r.peak_live_series = sk._peak_live(length - 1, length - 1) if n_ok else 0
    if options.compute_bound:
        r.bound = sk.gram_error_bound(sk.ErrorBoundInputs(m, length, r.max_abs_increment_product, r.min_order))
    else:
        r.bound = math.nan
    return r


# ------------------------------------------------------------ long pairs
def strip_ranges(bands: int, world: int):
    """Contiguous, balanced band ranges [b0, b1) of a long pair, one per rank."""
    return [(bands * g // world, bands * (g + 1) // world) for g in range(world)]


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


def propagate_long_pair_distributed(x, y, order: int, options: Optional[sk.PropagateOptions] = None,
                                    group=None, diag: bool = False):
    """K(1,1) of ONE long pair split into row strips across the ranks of
    `group` (one process per GPU): rank g sweeps a
    contiguous band range and streams its top band's alpha series straight
    into rank g+1's exchange buffer over NVLink (CUDA IPC peer mapping,
    system-scope release/acquire).  Every rank returns (value, diag-or-None);
    diag holds this rank's knots K(a, a) (NaN elsewhere)."""
    import torch.distributed as dist

    x, y = sk._as_series(x), sk._as_series(y)
    if x.dim() != y.dim():
        raise ValueError("propagate: series dimensions differ")
    lib = _capi.load()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lx, ly, d = x.length(), y.length(), x.dim()
    nb = ctypes.c_size_t()
    if lib.sk_strip_bands(ly, int(order), ctypes.byref(nb)) != 0:
        raise ValueError("propagate: bad length/order")
    bands = nb.value
    if bands < world:
        raise ValueError(f"{bands} bands cannot feed {world} GPUs")
    b0, b1 = strip_ranges(bands, world)[rank]
    st = _capi.SkStatus()
    in_a, in_p, out_a, out_p = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    handles = None
    if rank > 0:
        sk._check(lib.sk_exchange_alloc(lx, int(order), ctypes.byref(in_a), ctypes.byref(in_p), ctypes.byref(st)), st)
        ha, hp = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
        sk._check(lib.sk_ipc_handle(in_a, ha, ctypes.byref(st)), st)
        sk._check(lib.sk_ipc_handle(in_p, hp, ctypes.byref(st)), st)
        handles = (bytes(ha), bytes(hp))
    all_handles = [None] * world
    dist.all_gather_object(all_handles, handles, group=group)
    try:
        if rank + 1 < world:
            ha, hp = all_handles[rank + 1]
            sk._check(lib.sk_ipc_open(ctypes.create_string_buffer(ha, 64), ctypes.byref(out_a), ctypes.byref(st)), st)
            sk._check(lib.sk_ipc_open(ctypes.create_string_buffer(hp, 64), ctypes.byref(out_p), ctypes.byref(st)), st)
        dist.barrier(group=group)
        value = ctypes.c_double(float("nan"))
        dg = np.full(min(lx, ly) - 1, np.nan) if diag else None
        xv, yv = x.values(), y.values()
        rc = lib.sk_propagate_strip(sk._ptr(xv), lx, sk._ptr(yv), ly, d, int(order), sk._flags(options), b0, b1,
                                    in_a if rank > 0 else None, in_p if rank > 0 else None,
                                    out_a if rank + 1 < world else None, out_p if rank + 1 < world else None,
                                    ctypes.byref(value), sk._ptr(dg) if dg is not None else None, ctypes.byref(st))
        rec = None if rc == 0 else (int(st.code), int(st.tile_k), int(st.tile_l), st.message.decode(errors="replace"))
        recs = [None] * world
        dist.all_gather_object(recs, (rec, value.value if b1 == bands else None), group=group)
    finally:
        dist.barrier(group=group)
        if rank + 1 < world:
            if out_a.value:
                lib.sk_ipc_close(out_a)
            if out_p.value:
                lib.sk_ipc_close(out_p)
        if rank > 0:
            lib.sk_exchange_free(in_a, in_p)
    err = first_error([r for r, _ in recs])
    if err is not None:
        code, k, l, msg = err
        if code == _capi.SK_NUMERIC_OVERFLOW:
            raise sk.NumericOverflowError(msg, k, l)
        if code == _capi.SK_INCONSISTENT_BOUNDARY:
            raise sk.InconsistentBoundaryError(msg)
        raise RuntimeError(msg)
    final = [v for _, v in recs if v is not None][0]
    return final, dg


def propagate_split_emulated(x, y, order: int, split_band: int, options: Optional[sk.PropagateOptions] = None):
    """One-GPU test of the strip protocol: a single launch whose hand-off from
    band split_band-1 to split_band goes through an exchange buffer exactly
    as between two GPUs (sk_propagate_split)."""
    x, y = sk._as_series(x), sk._as_series(y)
    lib = _capi.load()
    st = _capi.SkStatus()
    value = ctypes.c_double()
    xv, yv = x.values(), y.values()
    rc = lib.sk_propagate_split(sk._ptr(xv), x.length(), sk._ptr(yv), y.length(), x.dim(), int(order),
                                sk._flags(options), int(split_band), ctypes.byref(value), ctypes.byref(st))
    sk._check(rc, st)
    return value.value


def strip_bands(ly: int, order: int) -> int:
    nb = ctypes.c_size_t()
    if _capi.load().sk_strip_bands(ly, int(order), ctypes.byref(nb)) != 0:
        raise ValueError("bad length/order")
    return nb.value


def propagate_long_pair_devices(x, y, order: int, devices: Sequence[int],
                                options: Optional[sk.PropagateOptions] = None, diag: bool = False):
    """K(1,1) of ONE long pair split into row strips over several GPUs driven
    from this process (the SURVEY.md section 8b device-list option; the
    multi-process variant is propagate_long_pair_distributed).  Strip g runs
    on devices[g] in its own host thread; its top band writes alpha' straight
    into devices[g+1]'s exchange buffer through peer access (NVLink), with the
    same system-scope release/acquire protocol.  Returns (value, diag-or-None).
    The devices must be distinct: strips wait on each other, so two of them
    must never share a GPU (one GPU: sk.propagate)."""
    import threading

    devices = [int(d) for d in devices]
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
    if bands < world:
        raise ValueError(f"{bands} bands cannot feed {world} GPUs")
    ranges = strip_ranges(bands, world)
    st = _capi.SkStatus()
    xbuf = [None] * world  # exchange buffer (abuf, prog) on each consumer device
    try:
        for g in range(1, world):
            sk._check(lib.sk_set_device(devices[g], ctypes.byref(st)), st)
            a, p = ctypes.c_void_p(), ctypes.c_void_p()
            sk._check(lib.sk_exchange_alloc(lx, int(order), ctypes.byref(a), ctypes.byref(p), ctypes.byref(st)), st)
            xbuf[g] = (a, p)
        for g in range(world - 1):
            sk._check(lib.sk_set_device(devices[g], ctypes.byref(st)), st)
            sk._check(lib.sk_enable_peer_access(devices[g + 1], ctypes.byref(st)), st)
        xv, yv = x.values(), y.values()
        out = [None] * world
        dg = np.full(min(lx, ly) - 1, np.nan) if diag else None
        parts = [np.full(min(lx, ly) - 1, np.nan) if diag else None for _ in range(world)]

        def strip(g):
            s = _capi.SkStatus()
            v = ctypes.c_double(float("nan"))
            rc = lib.sk_set_device(devices[g], ctypes.byref(s))
            if rc == 0:
                b0, b1 = ranges[g]
                rc = lib.sk_propagate_strip(sk._ptr(xv), lx, sk._ptr(yv), ly, d, int(order), sk._flags(options), b0, b1,
                                            xbuf[g][0] if g > 0 else None, xbuf[g][1] if g > 0 else None,
                                            xbuf[g + 1][0] if g + 1 < world else None,
                                            xbuf[g + 1][1] if g + 1 < world else None, ctypes.byref(v),
                                            sk._ptr(parts[g]) if diag else None, ctypes.byref(s))
            out[g] = (rc, s, v.value)

        threads = [threading.Thread(target=strip, args=(g,)) for g in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        for g in range(1, world):
            if xbuf[g] is not None:
                lib.sk_exchange_free(xbuf[g][0], xbuf[g][1])
    recs = [None if rc == 0 else (int(s.code), int(s.tile_k), int(s.tile_l), s.message.decode(errors="replace"))
            for rc, s, _ in out]
    err = first_error(recs)
    if err is not None:
        code, k, l, msg = err
        if code == _capi.SK_NUMERIC_OVERFLOW:
            raise sk.NumericOverflowError(msg, k, l)
        if code == _capi.SK_INCONSISTENT_BOUNDARY:
            raise sk.InconsistentBoundaryError(msg)
        raise RuntimeError(msg)
    if diag:
        for g in range(world):
            sel = ~np.isnan(parts[g])
            dg[sel] = parts[g][sel]
    return out[-1][2], dg
