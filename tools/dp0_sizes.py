import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2502_20392_b200 import sigker as sk
loose = sk.PropagateOptions(strict_corner=False)
for L, d in [(257, 64), (1025, 64), (2049, 64), (4097, 64), (1025, 512), (4097, 512), (8193, 512)]:
    x, y = sk.brownian(L, d, 1), sk.brownian(L, d, 2)
    t = time.time()
    try:
        v = sk.propagate(x, y, 8, loose).value
        print(L, d, v, f"{time.time()-t:.3f}s", flush=True)
    except Exception as e:
        print(L, d, "ERR", e, flush=True)
