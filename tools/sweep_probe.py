"""Diagnostics: sweep-kernel throughput on arbitrary pair shapes (device-resident
inputs, fixed order, CUDA-event time of the sweep launches only)."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import _capi, sigker as sk  # noqa: E402


def run(npairs, lx, ly, dim, order, reps=3, flags=_capi.SK_STRICT_CORNER):
    rng = np.random.default_rng(0)
    xs = np.cumsum(rng.standard_normal((npairs, lx, dim)) / np.sqrt(lx), axis=1)
    ys = np.cumsum(rng.standard_normal((npairs, ly, dim)) / np.sqrt(ly), axis=1)
    xd = torch.from_numpy(xs).cuda()
    yd = torch.from_numpy(ys).cuda()
    vd = torch.empty(npairs, dtype=torch.float64, device="cuda")
    lib = _capi.load()
    st = _capi.SkStatus()
    lib.sk_set_stream(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
    def once():
        rc = lib.sk_pairwise_device(ctypes.c_void_p(xd.data_ptr()), lx, ctypes.c_void_p(yd.data_ptr()), ly, npairs,
                                    dim, 0, order, 1e-12, flags, ctypes.c_void_p(vd.data_ptr()), None, None, None,
                                    ctypes.byref(st))
        assert rc == 0, st.message
    once()
    sk.stats_enable(True)
    sk.stats_reset()
    for _ in range(reps):
        once()
    s = sk.stats_get()
    sk.stats_enable(False)
    ms = s["sweep_ms"] / s["sweep_launches"]
    tiles = npairs * (lx - 1) * (ly - 1)
    print(f"pairs={npairs:6d} lx={lx:7d} ly={ly:7d} d={dim:3d} N={order:2d}: sweep {ms:8.3f} ms  "
          f"{tiles / ms * 1e3:.3e} tiles/s  {s['tile_flops'] / s['sweep_ms'] / 1e9:.2f} TF/s "
          f"({100 * s['tile_flops'] / s['sweep_ms'] / 1e9 / 37.11:.1f}% of 37.11)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("shapes", nargs="*", default=["256,4096,4096,8,8"])
    ap.add_argument("--no-strict", action="store_true", help="skip the per-tile corner check (bench uses it)")
    a = ap.parse_args()
    for sh in a.shapes:
        run(*[int(v) for v in sh.split(",")], flags=0 if a.no_strict else _capi.SK_STRICT_CORNER)
