"""Python mirror of the reference engine's public API (namespace ``sigker``),
backed by the B200 C-ABI (include/sigker_b200.h).

Names, argument meaning and error behaviour follow the reference headers:
  wavefront.hpp:13-60   PropagateOptions, KernelResult, propagate,
                        propagate_grid, propagate_with_policy, step_tile
  truncation.hpp:10-51  TruncationPolicy, OrderEstimate, estimate_order,
                        bessel_i0, ErrorBoundInputs, gram_error_bound
  gram.hpp:14-55        GramOptions, GramEntryError, GramResult, gram_matrix
  time_series.hpp:13-88 TimeSeries, pad_to_length, increments, IncrementTable
  errors.hpp:10-53      NumericOverflowError, InconsistentBoundaryError
Additions the reference lacks: ``pairwise`` (batched
independent pairs), ``PropagateOptions.strict_corner`` (the corner check
switch), ``propagate(..., diag=True)`` (K at the knots (a, a)) and
``gram_matrix(..., shard, nshards)`` (row-block sharding across ranks).

Every kernel evaluation runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi

K_MAX_ORDER = 64  # tile_series.hpp:12


# ------------------------------------------------------------------ errors
class NumericOverflowError(RuntimeError):
    """errors.hpp:29-41 -- carries the 1-based tile (k along x, l along y)."""

    def __init__(self, message: str, tile_k: int, tile_l: int):
        super().__init__(message)
        self.tile_k = tile_k
        self.tile_l = tile_l


class InconsistentBoundaryError(RuntimeError):
    """errors.hpp:24-27."""


class DeviceError(RuntimeError):
    """No CUDA device / launch failure (the B200 path has no CPU fallback)."""


def _raise(st: _capi.SkStatus):
    msg = st.message.decode(errors="replace")
    if st.code == _capi.SK_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if st.code == _capi.SK_NUMERIC_OVERFLOW:
        raise NumericOverflowError(msg, int(st.tile_k), int(st.tile_l))
    if st.code == _capi.SK_INCONSISTENT_BOUNDARY:
        raise InconsistentBoundaryError(msg)
    if st.code == _capi.SK_CUDA_ERROR:
        raise DeviceError(msg)
    raise RuntimeError(msg)


def _check(rc: int, st: _capi.SkStatus):
    if rc != _capi.SK_OK:
        if st.code == 0:
            st.code = rc
        _raise(st)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------- time series
class TimeSeries:
    """time_series.hpp:13-38: length x dim samples, row-major, finite."""

    def __init__(self, values, dim: Optional[int] = None):
        v = np.asarray(values, dtype=np.float64)
        if dim is None:
            if v.ndim != 2:
                raise ValueError("time series needs a (length, dim) array or an explicit dim")
            dim = v.shape[1]
        if dim == 0:
            raise ValueError("time series dimension must be >= 1")
        v = np.ascontiguousarray(v.reshape(-1))
        if v.size == 0:
            raise ValueError("time series must contain at least one point")
        if v.size % dim != 0:
            raise ValueError("value count is not a multiple of the dimension")
        # time_series.cpp:9-19 (sk_all_finite: threaded exponent test on the host)
        if not _capi.load().sk_all_finite(v.ctypes.data, v.size):
            raise ValueError("time series coordinates must be finite")
        self._v = v.reshape(-1, dim)
        self._v.setflags(write=False)

    def length(self) -> int:
        return self._v.shape[0]

    def dim(self) -> int:
        return self._v.shape[1]

    def values(self) -> np.ndarray:
        return self._v

    def point(self, k: int) -> np.ndarray:
        return self._v[k]

    def knot(self, k: int) -> float:
        return k / (self.length() - 1)

    def __eq__(self, other):
        return isinstance(other, TimeSeries) and self._v.shape == other._v.shape and np.array_equal(self._v, other._v)


def _as_series(x) -> TimeSeries:
    return x if isinstance(x, TimeSeries) else TimeSeries(x)


def pad_to_length(ts: TimeSeries, target_length: int) -> TimeSeries:
    """time_series.cpp:21-30: repeat the last point."""
    ts = _as_series(ts)
    if target_length < ts.length():
        raise ValueError("pad_to_length: target shorter than the series")
    v = ts.values()
    extra = np.repeat(v[-1:], target_length - ts.length(), axis=0)
    return TimeSeries(np.concatenate([v, extra], axis=0))


def increments(ts: TimeSeries) -> np.ndarray:
    """time_series.cpp:32-42 (host helper; the GPU path computes its own)."""
    ts = _as_series(ts)
    if ts.length() < 2:
        raise ValueError("increments: a single point has no increments")
    v = ts.values()
    return v[1:] - v[:-1]


class IncrementTable:
    """time_series.hpp:54-88.  max_abs_rho() is the bit-exact GPU scan."""

    def __init__(self, x, y):
        x, y = _as_series(x), _as_series(y)
        self._xi, self._yi = increments(x), increments(y)
        if x.dim() != y.dim():
            raise ValueError("increment table: series dimensions differ")
        self._x, self._y = x, y
        self._max = None

    def x_count(self):
        return self._xi.shape[0]

    def y_count(self):
        return self._yi.shape[0]

    def dim(self):
        return self._xi.shape[1]

    def rho(self, k: int, l: int) -> float:
        if k >= self.x_count() or l >= self.y_count():
            raise ValueError("rho: tile index out of range")
        acc = 0.0
        for a, b in zip(self._xi[k], self._yi[l]):
            acc += float(a) * float(b)
        return acc

    def max_abs_rho(self) -> float:
        if self._max is None:
            lib = _capi.load()
            st = _capi.SkStatus()
            out = ctypes.c_double()
            xv, yv = self._x.values(), self._y.values()
            rc = lib.sk_max_abs_rho(_ptr(xv), xv.shape[0], _ptr(yv), yv.shape[0], xv.shape[1],
                                    ctypes.byref(out), ctypes.byref(st))
            _check(rc, st)
            self._max = out.value
        return self._max

    def materialize_table(self) -> np.ndarray:
        return self._xi @ self._yi.T


# ----------------------------------------------------------------- policy
@dataclass
class TruncationPolicy:
    """truncation.hpp:10-19: fixed order 7 by default; adaptive searches 8..64."""
    mode: str = "fixed"
    order: int = 7
    tol: float = 1e-12

    @staticmethod
    def fixed(order: int) -> "TruncationPolicy":
        if order < 1 or order > K_MAX_ORDER:
            raise ValueError("fixed truncation order must lie in [1, 64]")
        return TruncationPolicy("fixed", order, 1e-12)

    @staticmethod
    def adaptive(tol: float = 1e-12) -> "TruncationPolicy":
        if not tol > 0.0:
            raise ValueError("adaptive tolerance must be positive")
        return TruncationPolicy("adaptive", 7, tol)


@dataclass
class OrderEstimate:
    order: int = 0
    converged: bool = True


def estimate_order(max_abs_rho: float, length: int, tol: float) -> OrderEstimate:
    """truncation.cpp:41-55."""
    lib = _capi.load()
    st = _capi.SkStatus()
    o, c = ctypes.c_int(), ctypes.c_int()
    rc = lib.sk_estimate_order(float(max_abs_rho), int(length), float(tol), ctypes.byref(o), ctypes.byref(c),
                               ctypes.byref(st))
    _check(rc, st)
    return OrderEstimate(o.value, bool(c.value))


def bessel_i0(x: float) -> float:
    """truncation.cpp:28-39 (host metadata helper)."""
    if x < 0.0:
        raise ValueError("bessel_i0: argument must be nonnegative")
    q = 0.25 * x * x
    term = 1.0
    s = 1.0
    for k in range(1, 1000):
        term *= q / (float(k) * float(k))
        s += term
        if term < s * 2.220446049250313e-16:
            break
    return s


@dataclass
class ErrorBoundInputs:
    family_size: int = 1
    length: int = 2
    max_abs_increment_product: float = 0.0
    order: int = 7


def gram_error_bound(inputs: ErrorBoundInputs) -> float:
    """truncation.cpp:57-87 (Prop. A.1 a-priori Frobenius bound; host metadata)."""
    if inputs.family_size < 1:
        raise ValueError("gram_error_bound: family size must be >= 1")
    if inputs.length < 2:
        raise ValueError("gram_error_bound: length must be >= 2")
    if inputs.max_abs_increment_product < 0.0:
        raise ValueError("gram_error_bound: increment product bound must be >= 0")
    if inputs.order < 0:
        raise ValueError("gram_error_bound: order must be >= 0")
    lm1 = float(inputs.length - 1)
    n = inputs.order
    max_x = lm1 * lm1 * inputs.max_abs_increment_product
    gamma = 0.5 * float(inputs.family_size)
    for nu in range(0, 2 * inputs.length - 2 + 1):
        gamma *= bessel_i0(2.0 * math.sqrt(float(nu) * max_x) / lm1)
    zeta = (1.0 + (2.0 * lm1) / (n + 2.0)) * (2.0 / lm1) ** (n + 1)
    if n + 1 < 171:
        fac = 1.0
        for k in range(1, n + 2):
            fac *= float(k)
        try:
            return gamma * max_x ** (n + 1) * zeta / (fac * fac)
        except OverflowError:
            return math.inf
    log_tail = (n + 1) * math.log(max_x) - 2.0 * math.lgamma(n + 2.0) if max_x > 0 else -math.inf
    return gamma * zeta * math.exp(log_tail)


# -------------------------------------------------------------- wavefront
@dataclass
class PropagateOptions:
    """wavefront.hpp:13-18.  threads / reverse_diagonals are advisory on the
    GPU (results are order-independent by construction); strict_corner is the
    reference's InconsistentBoundaryError check (tile_series.cpp:70-75)."""
    threads: int = 1
    reverse_diagonals: bool = False
    strict_corner: bool = True


@dataclass
class KernelResult:
    """wavefront.hpp:20-32."""
    value: float = 1.0
    order: int = 0
    order_converged: bool = True
    tiles_processed: int = 0
    peak_live_series: int = 0
    grid_rows: int = 0
    grid_cols: int = 0
    grid: np.ndarray = field(default_factory=lambda: np.zeros(0))
    diag: Optional[np.ndarray] = None


def _flags(options: Optional[PropagateOptions], fault: bool = False) -> int:
    f = 0
    if options is None or options.strict_corner:
        f |= _capi.SK_STRICT_CORNER
    if fault or _W_FAULT[0]:
        f |= _capi.SK_W_FAULT
    return f


_W_FAULT = [False]


def set_w_fault_for_testing(enabled: bool) -> None:
    """tile_series.hpp:102-106 negative-control hook (flips W[1][1])."""
    _W_FAULT[0] = bool(enabled)


def _run(x, y, order: int, options: Optional[PropagateOptions], with_grid: bool, diag: bool) -> KernelResult:
    x, y = _as_series(x), _as_series(y)
    if x.dim() != y.dim():
        raise ValueError("propagate: series dimensions differ")
    if x.length() < 2 or y.length() < 2:
        raise ValueError("propagate: both series need length >= 2")
    if order < 1 or order > K_MAX_ORDER:
        raise ValueError("propagate: order must lie in [1, 64]")
    lib = _capi.load()
    st = _capi.SkStatus()
    value = ctypes.c_double()
    peak = ctypes.c_uint64()
    lx, ly = x.length(), y.length()
    grid = np.zeros(lx * ly) if with_grid else None
    dg = np.zeros(min(lx, ly) - 1) if diag else None
    xv, yv = x.values(), y.values()
    rc = lib.sk_propagate(_ptr(xv), lx, _ptr(yv), ly, x.dim(), int(order), _flags(options), ctypes.byref(value),
                          ctypes.byref(peak), _ptr(grid) if grid is not None else None,
                          _ptr(dg) if dg is not None else None, ctypes.byref(st))
    _check(rc, st)
    r = KernelResult(value=value.value, order=order, tiles_processed=(lx - 1) * (ly - 1),
                     peak_live_series=int(peak.value))
    if with_grid:
        r.grid_rows, r.grid_cols, r.grid = lx, ly, grid
    r.diag = dg
    return r


def propagate(x, y, order: int, options: Optional[PropagateOptions] = None, diag: bool = False) -> KernelResult:
    """wavefront.hpp:41-42 (wavefront.cpp:196-199)."""
    return _run(x, y, order, options, False, diag)


def propagate_grid(x, y, order: int, options: Optional[PropagateOptions] = None) -> KernelResult:
    """wavefront.hpp:46-47 (wavefront.cpp:201-204): grid[a * ly + b] = K(sigma_a, tau_b)."""
    return _run(x, y, order, options, True, False)


def propagate_with_policy(x, y, policy: TruncationPolicy, options: Optional[PropagateOptions] = None) -> KernelResult:
    """wavefront.hpp:51-53 (wavefront.cpp:206-221)."""
    x, y = _as_series(x), _as_series(y)
    if policy.mode != "adaptive":
        return propagate(x, y, policy.order, options)
    if x.dim() != y.dim():
        raise ValueError("propagate: series dimensions differ")
    # one batched call: the device order pre-pass proves N from a Cauchy-Schwarz
    # bound of max|rho| and only runs the exact O(l^2 d) scan when it must
    lib = _capi.load()
    st = _capi.SkStatus()
    per = _capi.SkStatus()
    value = np.zeros(1)
    order = np.zeros(1, dtype=np.int32)
    conv = np.zeros(1, dtype=np.int32)
    xv, yv = x.values(), y.values()
    rc = lib.sk_pairwise(_ptr(xv), x.length(), _ptr(yv), y.length(), 1, x.dim(), 1, 7, float(policy.tol),
                         _flags(options), _ptr(value), _ptr(order), _ptr(conv), None, ctypes.byref(per),
                         ctypes.byref(st))
    _check(rc, st)
    if per.code != 0:
        _raise(per)
    lx, ly = x.length(), y.length()
    return KernelResult(value=float(value[0]), order=int(order[0]), order_converged=bool(conv[0]),
                        tiles_processed=(lx - 1) * (ly - 1), peak_live_series=_peak_live(ly - 1, lx - 1))


def step_tile(delta: float, alpha, beta, order: int, fast: bool = False):
    """wavefront.hpp:58-60 (wavefront.cpp:223-237) on the device, bit-identical
    to the reference.  fast=True routes through the factorial-scaled register
    solver of the sweep (diagnostic; order 1..16).  Returns (alpha', beta')."""
    if order < 0 or order > K_MAX_ORDER:
        raise ValueError("step_tile: order must lie in [0, 64]")
    n = order + 1
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    if a.size < n or b.size < n:
        raise ValueError("step_tile: boundary series shorter than the order")
    lib = _capi.load()
    st = _capi.SkStatus()
    oa, ob = np.zeros(n), np.zeros(n)
    tot = ctypes.c_double()
    fn = lib.sk_step_tile_fast if fast else lib.sk_step_tile
    rc = fn(float(delta), _ptr(a), _ptr(b), int(order), _ptr(oa), _ptr(ob), ctypes.byref(tot), ctypes.byref(st))
    _check(rc, st)
    return oa, ob


# ------------------------------------------------------------------ batched
@dataclass
class PairwiseResult:
    values: np.ndarray
    orders: np.ndarray
    converged: np.ndarray
    max_abs_rho: Optional[np.ndarray]
    failures: List[tuple]


def pairwise(xs, ys, policy: Optional[TruncationPolicy] = None, options: Optional[PropagateOptions] = None,
             want_max_abs_rho: bool = False) -> PairwiseResult:
    """Batched independent pairs: entry k == propagate_with_policy(xs[k], ys[k])
    (SURVEY.md section 8b addition).  xs: (npairs, lx, d), ys: (npairs, ly, d).
    Entries that raise NumericOverflowError are NaN and listed in failures as
    (k, tile_k, tile_l, message)."""
    policy = policy or TruncationPolicy()
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    ys = np.ascontiguousarray(ys, dtype=np.float64)
    if xs.ndim != 3 or ys.ndim != 3 or xs.shape[0] != ys.shape[0] or xs.shape[2] != ys.shape[2]:
        raise ValueError("pairwise: xs (npairs, lx, d) and ys (npairs, ly, d) must agree")
    npairs, lx, d = xs.shape
    ly = ys.shape[1]
    lib = _capi.load()
    st = _capi.SkStatus()
    values = np.zeros(npairs)
    orders = np.zeros(npairs, dtype=np.int32)
    conv = np.zeros(npairs, dtype=np.int32)
    mr = np.zeros(npairs) if want_max_abs_rho else None
    per = _status_array(max(npairs, 1))
    adaptive = 1 if policy.mode == "adaptive" else 0
    rc = lib.sk_pairwise(_ptr(xs), lx, _ptr(ys), ly, npairs, d, adaptive, int(policy.order), float(policy.tol),
                         _flags(options), _ptr(values), _ptr(orders), _ptr(conv),
                         _ptr(mr) if mr is not None else None, _ptr(per), ctypes.byref(st))
    _check(rc, st)
    failures = []
    for k in np.flatnonzero(per["code"][:npairs] != 0).tolist():
        e = per[k]
        if e["code"] == _capi.SK_INCONSISTENT_BOUNDARY:
            _raise(_capi.SkStatus.from_buffer_copy(e.tobytes()))
        failures.append((k, int(e["tile_k"]), int(e["tile_l"]), e["message"].decode(errors="replace")))
    return PairwiseResult(values, orders, conv.astype(bool), mr, failures)


# --------------------------------------------------------------------- gram
@dataclass
class GramOptions:
    """gram.hpp:14-18."""
    policy: TruncationPolicy = field(default_factory=TruncationPolicy)
    threads: int = 1
    compute_bound: bool = False
    strict_corner: bool = True
    # GPUs to spread this call over, one host thread each (a sub-shard per
    # device); empty: the current device
    devices: List[int] = field(default_factory=list)
    # also return every entry's exact max|rho| (GramResult.pair_max_abs_rho);
    # without it only the family's maximum is formed (cheaper: one running
    # max for the whole launch lets most tiles skip the exact dot)
    pair_max_abs_rho: bool = False


@dataclass
class GramEntryError:
    row: int
    col: int
    message: str


@dataclass
class GramResult:
    """gram.hpp:26-39."""
    size: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))
    orders: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))
    min_order: int = 0
    max_order: int = 0
    adaptive: bool = False
    orders_converged: bool = True
    max_abs_increment_product: float = 0.0
    bound: float = math.nan
    wall_seconds: float = 0.0
    peak_live_series: int = 0
    failures: List[GramEntryError] = field(default_factory=list)
    pair_max_abs_rho: Optional[np.ndarray] = None


def _peak_live(rows: int, cols: int) -> int:
    # wavefront.cpp live counter in closed form (same as the C-ABI's
    # peak_live_closed_form): 2 per diagonal while both edges prefill, one
    # more when the longer edge keeps prefilling past the shorter one
    m, big = min(rows, cols), max(rows, cols)
    return 2 * m + (1 if big > m else 0)


def _status_array(n: int) -> np.ndarray:
    """n zeroed sk_status records as a numpy structured array (calloc'd pages,
    vectorised code scans) with the C layout of include/sigker_b200.h."""
    S = _capi.SkStatus
    dt = np.dtype({"names": ["code", "tile_k", "tile_l", "message"], "formats": ["<i4", "<u8", "<u8", "S256"],
                   "offsets": [S.code.offset, S.tile_k.offset, S.tile_l.offset, S.message.offset],
                   "itemsize": ctypes.sizeof(S)})
    return np.zeros(n, dtype=dt)


def _gram_failures(lib, count: int) -> List[GramEntryError]:
    """The calling thread's last sk_gram failure records (sparse, row-major)."""
    if count == 0:
        return []
    buf = (_capi.SkGramFailure * count)()
    n = lib.sk_gram_failures(buf, count)
    return [GramEntryError(int(f.row), int(f.col), f.status.message.decode(errors="replace")) for f in buf[:n]]


def gram_matrix(family: Sequence, options: Optional[GramOptions] = None, shard: int = 0,
                nshards: int = 1) -> GramResult:
    """gram.hpp:46 (gram.cpp:16-98).  With nshards > 1 only this shard's
    upper-triangle entries are evaluated (others stay NaN) -- the row-block
    partition of the multi-GPU Gram."""
    import time
    options = options or GramOptions()
    if isinstance(family, np.ndarray) and family.ndim == 3:
        # an (m, length, dim) block is a family of equal-length series already
        # padded (no per-series copies; one finiteness scan, time_series.cpp:9-19)
        padded = np.ascontiguousarray(family, dtype=np.float64)
        if padded.shape[0] == 0:
            raise ValueError("gram_matrix: family must be nonempty")
        if padded.shape[1] < 1 or padded.shape[2] < 1:
            raise ValueError("time series must contain at least one point")
        if not _capi.load().sk_all_finite(padded.ctypes.data, padded.size):
            raise ValueError("time series coordinates must be finite")
        m, max_len, dim = padded.shape
        if max_len < 2:
            padded = np.concatenate([padded, padded], axis=1)
            max_len = 2
    else:
        fam = [_as_series(s) for s in family]
        if not fam:
            raise ValueError("gram_matrix: family must be nonempty")
        dim = fam[0].dim()
        max_len = 0
        for s in fam:
            if s.dim() != dim:
                raise ValueError("gram_matrix: mixed dimensions in family")
            max_len = max(max_len, s.length())
        max_len = max(max_len, 2)
        padded = np.stack([pad_to_length(s, max_len).values() for s in fam])
        m = len(fam)
    adaptive = options.policy.mode == "adaptive"
    scan = adaptive or options.compute_bound
    lib = _capi.load()
    st = _capi.SkStatus()
    values = np.zeros(m * m)
    orders = np.zeros(m * m, dtype=np.int32)
    pmax = np.zeros(m * m)
    maxp = ctypes.c_double()
    conv = ctypes.c_int()
    flags = _capi.SK_STRICT_CORNER if options.strict_corner else 0
    if _W_FAULT[0]:
        flags |= _capi.SK_W_FAULT
    t0 = time.perf_counter()

    def run_shard(sub, nsub, vals, ords, pm, mp, cv, status):
        nf = ctypes.c_size_t()
        rc = lib.sk_gram(_ptr(padded), m, max_len, dim, 1 if adaptive else 0, int(options.policy.order),
                         float(options.policy.tol), flags, 1 if scan else 0, int(sub), int(nsub), _ptr(vals),
                         _ptr(ords), _ptr(pm) if options.pair_max_abs_rho else None, ctypes.byref(mp),
                         ctypes.byref(cv), ctypes.byref(nf), ctypes.byref(status))
        return rc, (_gram_failures(lib, nf.value) if rc == 0 else [])

    devices = list(options.devices)
    if len(devices) <= 1:
        if devices:
            _check(lib.sk_set_device(int(devices[0]), ctypes.byref(st)), st)
        rc, failures = run_shard(shard, nshards, values, orders, pmax, maxp, conv, st)
        _check(rc, st)
    else:
        # one host thread per GPU (ctypes releases the GIL during the call);
        # each evaluates the sub-shard shard * nd + k of nshards * nd
        import threading
        nd = len(devices)
        parts = [dict(values=np.zeros(m * m), orders=np.zeros(m * m, dtype=np.int32), pmax=np.zeros(m * m),
                      maxp=ctypes.c_double(), conv=ctypes.c_int(), st=_capi.SkStatus(), rc=0, failures=[])
                 for _ in range(nd)]

        def work(k):
            p = parts[k]
            p["rc"] = lib.sk_set_device(int(devices[k]), ctypes.byref(p["st"]))
            if p["rc"] == 0:
                p["rc"], p["failures"] = run_shard(shard * nd + k, nshards * nd, p["values"], p["orders"], p["pmax"],
                                                   p["maxp"], p["conv"], p["st"])

        threads = [threading.Thread(target=work, args=(k,)) for k in range(nd)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for p in parts:
            _check(p["rc"], p["st"])
        lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
        owner = np.full(m * m, -1)
        iu, ju = np.triu_indices(m)  # the upper triangle in row-major order, as the shards number it
        for k in range(nd):
            lib.sk_gram_shard_range(m, shard * nd + k, nshards * nd, ctypes.byref(lo), ctypes.byref(hi))
            a, b = iu[lo.value:hi.value], ju[lo.value:hi.value]
            owner[a * m + b] = k
            owner[b * m + a] = k
        values[:] = np.nan
        for k, p in enumerate(parts):
            sel = owner == k
            values[sel] = p["values"][sel]
            orders[sel] = p["orders"][sel]
            pmax[sel] = p["pmax"][sel]
        # sub-shards are consecutive row-major ranges: concatenation keeps the order
        failures = [f for p in parts for f in p["failures"]]
        maxp.value = max(p["maxp"].value for p in parts)
        conv.value = int(all(p["conv"].value for p in parts))
    wall = time.perf_counter() - t0
    r = GramResult(size=m, values=values, orders=orders, adaptive=adaptive, orders_converged=bool(conv.value),
                   wall_seconds=wall)
    r.failures = failures
    computed = orders[orders > 0]
    r.min_order = int(computed.min()) if computed.size else 0
    r.max_order = int(computed.max()) if computed.size else 0
    n_ok = int(np.sum(~np.isnan(values)))
    r.peak_live_series = _peak_live(max_len - 1, max_len - 1) if n_ok else 0
    if scan:
        r.max_abs_increment_product = float(maxp.value)
        r.pair_max_abs_rho = pmax if options.pair_max_abs_rho else None
    if options.compute_bound:
        r.bound = gram_error_bound(ErrorBoundInputs(m, max_len, r.max_abs_increment_product, r.min_order))
    return r


# ------------------------------------------------------------ input side
_HOST_LIB = [None]


def _host_lib():
    """libsigker.so (the C++ drop-in library, host code) for datagen."""
    if _HOST_LIB[0] is None:
        import os
        lib = ctypes.CDLL(os.path.join(os.path.dirname(_capi.LIB_PATH), "libsigker.so"))
        lib.sigker_datagen_brownian.argtypes = [ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_void_p]
        lib.sigker_datagen_brownian.restype = ctypes.c_int
        _HOST_LIB[0] = lib
    return _HOST_LIB[0]


def brownian(length: int, dim: int, seed: int) -> np.ndarray:
    """datagen.hpp brownian (datagen.cpp:78-88): the reference's value stream,
    bit for bit (xoshiro256++ / splitmix64, polar Box-Muller)."""
    out = np.empty((length, dim))
    if _host_lib().sigker_datagen_brownian(length, dim, seed, out.ctypes.data) != 0:
        raise ValueError("brownian: length must be >= 2 and dimension >= 1")
    return out


def brownian_family(length: int, dim: int, seeds: Sequence[int], out: Optional[np.ndarray] = None,
                    threads: int = 8) -> np.ndarray:
    """(len(seeds), length, dim) block of brownian(length, dim, seed) series,
    generated by `threads` host threads (ctypes releases the GIL), into `out`
    if given (e.g. a pinned buffer)."""
    import threading
    seeds = [int(s) for s in seeds]
    if out is None:
        out = np.empty((len(seeds), length, dim))
    lib = _host_lib()
    bad = []

    def work(t):
        for k in range(t, len(seeds), threads):
            if lib.sigker_datagen_brownian(length, dim, seeds[k], out[k].ctypes.data) != 0:
                bad.append(k)

    ts = [threading.Thread(target=work, args=(t,)) for t in range(max(1, threads))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if bad:
        raise ValueError("brownian: length must be >= 2 and dimension >= 1")
    return out


# ---------------------------------------------------------------- helpers
def device_count() -> int:
    return _capi.load().sk_device_count()


def set_device(device: int) -> None:
    st = _capi.SkStatus()
    _check(_capi.load().sk_set_device(int(device), ctypes.byref(st)), st)


def stats_enable(on: bool = True):
    _capi.load().sk_stats_enable(1 if on else 0)


def stats_reset():
    _capi.load().sk_stats_reset()


def stats_get() -> dict:
    s = _capi.SkStats()
    _capi.load().sk_stats_get(ctypes.byref(s))
    return {"sweep_launches": s.sweep_launches, "aux_launches": s.aux_launches, "sweep_ms": s.sweep_ms,
            "tiles": s.tiles, "tile_flops": s.tile_flops, "literal_rechecks": s.literal_rechecks}
