"""Cost of the Gram's exact max|rho| metadata (scan_products = 1, the EXACT
sweep with the launch-wide running max) against scan_products = 0 on the
same device-resident family (first M north-star members, one launch)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import _capi, sigker as sk  # noqa: E402

m = int(os.environ.get("AB_M", "64"))
fam = sk.brownian_family(4096, 16, range(1000, 1000 + m))
lib = _capi.load()
dev = torch.device("cuda", 0)
fd = torch.from_numpy(fam).to(dev)
mat = torch.empty(m * m, dtype=torch.float64, device=dev)
st = _capi.SkStatus()
mp = ctypes.c_double(0.0)
cv = ctypes.c_int(0)
nf = ctypes.c_size_t(0)
npairs = m * (m + 1) // 2
for scan in (1, 0, 1, 0):
    def call():
        rc = lib.sk_gram_device(ctypes.c_void_p(fd.data_ptr()), m, 4096, 16, 1, 7, 1e-12, _capi.SK_STRICT_CORNER, scan,
                                0, npairs, ctypes.c_void_p(mat.data_ptr()), ctypes.byref(mp), ctypes.byref(cv),
                                ctypes.byref(nf), ctypes.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())
    call()
    sk.stats_enable(True)
    sk.stats_reset()
    call()
    s = sk.stats_get()
    sk.stats_enable(False)
    print(f"scan_products={scan}: sweep {s['sweep_ms']:.1f} ms, max_product={mp.value!r}", flush=True)
