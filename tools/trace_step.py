import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2502_20392_b200 import _capi
lib = _capi.load()
NP, L, D = 256, 4096, 8
rng = np.random.default_rng(0)
xs = np.cumsum(rng.standard_normal((NP, L, D)) / np.sqrt(L), axis=1)
ys = np.cumsum(rng.standard_normal((NP, L, D)) / np.sqrt(L), axis=1)
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
vd = torch.empty(NP, dtype=torch.float64, device="cuda")
st = _capi.SkStatus()
lib.sk_set_stream(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
orders = np.zeros(NP, dtype=np.int32); conv = np.zeros(NP, dtype=np.int32)
def step():
    rc = lib.sk_pairwise_device(ctypes.c_void_p(xd.data_ptr()), L, ctypes.c_void_p(yd.data_ptr()), L, NP, D, 1, 7, 1e-12,
                                _capi.SK_STRICT_CORNER, ctypes.c_void_p(vd.data_ptr()), orders.ctypes.data_as(ctypes.c_void_p),
                                conv.ctypes.data_as(ctypes.c_void_p), None, ctypes.byref(st))
    assert rc == 0, st.message
for _ in range(3): step()
torch.cuda.synchronize()
pass  # run with SK_TRACE=1 for phase timings
for _ in range(2):
    t0 = time.perf_counter(); step(); torch.cuda.synchronize(); print("wall ms", (time.perf_counter()-t0)*1e3, file=sys.stderr)
