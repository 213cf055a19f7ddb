"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU checkers:

* ``Restatement``: oracle/_build/liboracle.so, the plain-C restatement of the
  reference (oracle/sigker_oracle.c), buildable anywhere with gcc;
* ``Reference``: oracle/_ref/libsigker_ref.so, the UNMODIFIED reference
  engine compiled from /root/reference/proj/src by oracle/Makefile (present
  only where it was built; it travels to the GPU box as a built file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use this.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsigker_ref.so")

P = ctypes.c_void_p
SZ = ctypes.c_size_t


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("tile_k", ctypes.c_uint64), ("tile_l", ctypes.c_uint64),
                ("message", ctypes.c_char * 256)]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def build_oracle():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def ref_available():
    return os.path.exists(REF_SO)


class OracleError(RuntimeError):
    def __init__(self, code, tile_k, tile_l, msg):
        super().__init__(msg)
        self.code, self.tile_k, self.tile_l = code, tile_k, tile_l


def _raise(rc, st):
    if rc != 0:
        raise OracleError(rc, int(st.tile_k), int(st.tile_l), st.message.decode(errors="replace"))


class Restatement:
    """Plain-C restatement of the reference (oracle/sigker_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = ctypes.CDLL(ORACLE_SO)
        L.or_rng_new.restype = P
        L.or_rng_new.argtypes = [ctypes.c_uint64]
        L.or_rng_free.argtypes = [P]
        L.or_rng_uniform01.restype = ctypes.c_double
        L.or_rng_uniform01.argtypes = [P]
        L.or_rng_gaussian.restype = ctypes.c_double
        L.or_rng_gaussian.argtypes = [P]
        L.or_random_series.argtypes = [P, SZ, SZ, ctypes.c_double, P]
        L.or_brownian.argtypes = [SZ, SZ, ctypes.c_uint64, P]
        L.or_fbm.argtypes = [SZ, SZ, ctypes.c_double, ctypes.c_uint64, P]
        L.or_max_abs_rho.argtypes = [P, SZ, P, SZ, SZ, P]
        L.or_step_tile.restype = ctypes.c_double
        L.or_step_tile.argtypes = [ctypes.c_double, P, P, ctypes.c_int, P, P]
        L.or_peak_live.restype = ctypes.c_uint64
        L.or_peak_live.argtypes = [SZ, SZ]
        L.or_propagate.argtypes = [P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_int, P, P, P, ctypes.POINTER(Status)]
        L.or_estimate_order.argtypes = [ctypes.c_double, ctypes.c_double, P, P]
        L.or_bessel_i0.restype = ctypes.c_double
        L.or_bessel_i0.argtypes = [ctypes.c_double]
        L.or_gram_error_bound.restype = ctypes.c_double
        L.or_gram_error_bound.argtypes = [SZ, SZ, ctypes.c_double, ctypes.c_int]
        L.or_gram.argtypes = [P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, P, P, P, P]
        L.or_propagate_probe.argtypes = [P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_int, P, SZ, P, P, P, P, P,
                                         ctypes.POINTER(Status)]
        self.L = L

    # datagen
    def brownian(self, length, dim, seed):
        out = np.zeros((length, dim))
        rc = self.L.or_brownian(length, dim, seed, _ptr(out))
        if rc:
            raise ValueError("brownian: bad arguments")
        return out

    def fbm(self, length, dim, hurst, seed):
        out = np.zeros((length, dim))
        rc = self.L.or_fbm(length, dim, hurst, seed, _ptr(out))
        if rc:
            raise ValueError("fbm failed")
        return out

    def rng(self, seed):
        return _Rng(self.L, seed)

    def max_abs_rho(self, x, y):
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        out = ctypes.c_double()
        self.L.or_max_abs_rho(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], ctypes.byref(out))
        return out.value

    def estimate_order(self, rho, tol):
        o, c = ctypes.c_int(), ctypes.c_int()
        rc = self.L.or_estimate_order(float(rho), float(tol), ctypes.byref(o), ctypes.byref(c))
        if rc:
            raise ValueError("estimate_order: bad arguments")
        return o.value, bool(c.value)

    def step_tile(self, delta, alpha, beta, order):
        n = order + 1
        a = np.ascontiguousarray(alpha[:n], float)
        b = np.ascontiguousarray(beta[:n], float)
        oa, ob = np.zeros(n), np.zeros(n)
        tot = self.L.or_step_tile(float(delta), _ptr(a), _ptr(b), order, _ptr(oa), _ptr(ob))
        return oa, ob, tot

    def peak_live(self, rows, cols):
        return int(self.L.or_peak_live(rows, cols))

    def propagate(self, x, y, order, check_corner=True, grid=False):
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        v = ctypes.c_double()
        pk = ctypes.c_uint64()
        g = np.zeros(x.shape[0] * y.shape[0]) if grid else None
        st = Status()
        rc = self.L.or_propagate(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], order, 1 if check_corner else 0,
                                 ctypes.byref(v), ctypes.byref(pk), _ptr(g) if grid else None, ctypes.byref(st))
        _raise(rc, st)
        return (v.value, int(pk.value), g) if grid else (v.value, int(pk.value))

    def propagate_probe(self, x, y, order, knots=(), check_corner=False):
        """The same sweep with instrumentation: K at the knots (a, a), the worst
        relative corner mismatch, and the first tile (k, l) where the
        reference's corner check (tile_series.cpp:70-75) would throw (0, 0 if
        none).  Returns (value, knot_values, max_corner_rel, (k, l))."""
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        kn = np.ascontiguousarray(knots, dtype=np.uint64)
        kv = np.full(len(kn), np.nan)
        v, mc = ctypes.c_double(), ctypes.c_double()
        ck, cl = ctypes.c_uint64(), ctypes.c_uint64()
        st = Status()
        rc = self.L.or_propagate_probe(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], order,
                                       1 if check_corner else 0, _ptr(kn) if len(kn) else None, len(kn),
                                       _ptr(kv) if len(kn) else None, ctypes.byref(mc), ctypes.byref(ck),
                                       ctypes.byref(cl), ctypes.byref(v), ctypes.byref(st))
        _raise(rc, st)
        return v.value, kv, mc.value, (int(ck.value), int(cl.value))

    def propagate_with_policy(self, x, y, tol, check_corner=True):
        n, conv = self.estimate_order(self.max_abs_rho(x, y), tol)
        return self.propagate(x, y, n, check_corner)[0], n, conv

    def bessel_i0(self, x):
        return self.L.or_bessel_i0(float(x))

    def gram_error_bound(self, m, length, maxp, order):
        return self.L.or_gram_error_bound(m, length, float(maxp), order)

    def gram(self, family, adaptive, order=7, tol=1e-12, check_corner=True):
        fam = np.ascontiguousarray(family, float)
        m, length, dim = fam.shape
        vals = np.zeros(m * m)
        ords = np.zeros(m * m, dtype=np.int32)
        mp = ctypes.c_double()
        nf = ctypes.c_uint64()
        rc = self.L.or_gram(_ptr(fam), m, length, dim, 1 if adaptive else 0, order, tol, 1 if check_corner else 0,
                            _ptr(vals), _ptr(ords), ctypes.byref(mp), ctypes.byref(nf))
        if rc:
            raise OracleError(rc, 0, 0, "gram aborted")
        return vals.reshape(m, m), ords.reshape(m, m), mp.value, int(nf.value)


class _Rng:
    def __init__(self, L, seed):
        self.L = L
        self.h = L.or_rng_new(seed)

    def __del__(self):
        try:
            self.L.or_rng_free(self.h)
        except Exception:
            pass

    def uniform01(self):
        return self.L.or_rng_uniform01(self.h)

    def gaussian(self):
        return self.L.or_rng_gaussian(self.h)

    def random_series(self, length, dim, cap):
        out = np.zeros((length, dim))
        self.L.or_random_series(self.h, length, dim, cap, _ptr(out))
        return out


class Reference:
    """The unmodified reference engine (oracle/_ref/libsigker_ref.so)."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO)
        S = ctypes.POINTER(Status)
        L.ref_propagate.argtypes = [P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_uint, ctypes.c_int, P, P, P, S]
        L.ref_propagate_with_policy.argtypes = [P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                ctypes.c_uint, P, P, P, S]
        L.ref_max_abs_rho.argtypes = [P, SZ, P, SZ, SZ, P, S]
        L.ref_estimate_order.argtypes = [ctypes.c_double, SZ, ctypes.c_double, P, P, S]
        L.ref_step_tile.argtypes = [ctypes.c_double, P, P, ctypes.c_int, P, P, S]
        L.ref_gram.argtypes = [P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint,
                               ctypes.c_int, P, P, P, P, P, P, P, P, S]
        L.ref_pairwise.argtypes = [P, P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint,
                                   P, P, S]
        L.ref_brownian.argtypes = [SZ, SZ, ctypes.c_uint64, P, S]
        L.ref_fbm.argtypes = [SZ, SZ, ctypes.c_double, ctypes.c_uint64, P, S]
        L.ref_gram_error_bound.argtypes = [SZ, SZ, ctypes.c_double, ctypes.c_int, P, S]
        L.ref_bessel_i0.restype = ctypes.c_double
        L.ref_bessel_i0.argtypes = [ctypes.c_double]
        L.ref_rng_stream.argtypes = [ctypes.c_uint64, SZ, ctypes.c_int, P]
        self.L = L

    def propagate(self, x, y, order, threads=1, grid=False, reverse=False):
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        v, pk, st = ctypes.c_double(), ctypes.c_uint64(), Status()
        g = np.zeros(x.shape[0] * y.shape[0]) if grid else None
        rc = self.L.ref_propagate(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], order, threads,
                                  1 if reverse else 0, ctypes.byref(v), ctypes.byref(pk),
                                  _ptr(g) if grid else None, ctypes.byref(st))
        _raise(rc, st)
        return (v.value, int(pk.value), g) if grid else (v.value, int(pk.value))

    def propagate_with_policy(self, x, y, adaptive=True, order=7, tol=1e-12, threads=1):
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        v, o, c, st = ctypes.c_double(), ctypes.c_int(), ctypes.c_int(), Status()
        rc = self.L.ref_propagate_with_policy(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1],
                                              1 if adaptive else 0, order, tol, threads, ctypes.byref(v),
                                              ctypes.byref(o), ctypes.byref(c), ctypes.byref(st))
        _raise(rc, st)
        return v.value, o.value, bool(c.value)

    def max_abs_rho(self, x, y):
        x, y = np.ascontiguousarray(x, float), np.ascontiguousarray(y, float)
        out, st = ctypes.c_double(), Status()
        _raise(self.L.ref_max_abs_rho(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], ctypes.byref(out),
                                      ctypes.byref(st)), st)
        return out.value

    def estimate_order(self, rho, length, tol):
        o, c, st = ctypes.c_int(), ctypes.c_int(), Status()
        _raise(self.L.ref_estimate_order(float(rho), length, float(tol), ctypes.byref(o), ctypes.byref(c),
                                         ctypes.byref(st)), st)
        return o.value, bool(c.value)

    def step_tile(self, delta, alpha, beta, order):
        n = order + 1
        a = np.ascontiguousarray(alpha[:n], float)
        b = np.ascontiguousarray(beta[:n], float)
        oa, ob, st = np.zeros(n), np.zeros(n), Status()
        _raise(self.L.ref_step_tile(float(delta), _ptr(a), _ptr(b), order, _ptr(oa), _ptr(ob), ctypes.byref(st)), st)
        return oa, ob

    def gram(self, family, adaptive=True, order=7, tol=1e-12, threads=1, compute_bound=False):
        fam = np.ascontiguousarray(family, float)
        m, length, dim = fam.shape
        vals = np.zeros(m * m)
        ords = np.zeros(m * m, dtype=np.int32)
        mp, bd, wall = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        pk, nf = ctypes.c_uint64(), ctypes.c_uint64()
        conv, st = ctypes.c_int(), Status()
        _raise(self.L.ref_gram(_ptr(fam), m, length, dim, 1 if adaptive else 0, order, tol, threads,
                               1 if compute_bound else 0, _ptr(vals), _ptr(ords), ctypes.byref(mp), ctypes.byref(bd),
                               ctypes.byref(pk), ctypes.byref(conv), ctypes.byref(nf), ctypes.byref(wall),
                               ctypes.byref(st)), st)
        return dict(values=vals.reshape(m, m), orders=ords.reshape(m, m), max_product=mp.value, bound=bd.value,
                    peak_live=int(pk.value), converged=bool(conv.value), n_failures=int(nf.value),
                    wall_seconds=wall.value)

    def pairwise(self, xs, ys, adaptive=True, order=7, tol=1e-12, threads=1):
        xs, ys = np.ascontiguousarray(xs, float), np.ascontiguousarray(ys, float)
        npairs, length, dim = xs.shape
        vals = np.zeros(npairs)
        ords = np.zeros(npairs, dtype=np.int32)
        st = Status()
        _raise(self.L.ref_pairwise(_ptr(xs), _ptr(ys), npairs, length, dim, 1 if adaptive else 0, order, tol,
                                   threads, _ptr(vals), _ptr(ords), ctypes.byref(st)), st)
        return vals, ords

    def brownian(self, length, dim, seed):
        out, st = np.zeros((length, dim)), Status()
        _raise(self.L.ref_brownian(length, dim, seed, _ptr(out), ctypes.byref(st)), st)
        return out

    def fbm(self, length, dim, hurst, seed):
        out, st = np.zeros((length, dim)), Status()
        _raise(self.L.ref_fbm(length, dim, hurst, seed, _ptr(out), ctypes.byref(st)), st)
        return out

    def rng_stream(self, seed, n, gaussian):
        out = np.zeros(n)
        self.L.ref_rng_stream(seed, n, 1 if gaussian else 0, _ptr(out))
        return out

    def gram_error_bound(self, m, length, maxp, order):
        out, st = ctypes.c_double(), Status()
        _raise(self.L.ref_gram_error_bound(m, length, float(maxp), order, ctypes.byref(out), ctypes.byref(st)), st)
        return out.value

    def bessel_i0(self, x):
        return self.L.ref_bessel_i0(float(x))
