"""cfg 4 host-phase trace: run with SK_TRACE=1; the last block is a warm call."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2502_20392_b200 import sigker as sk
x, y = sk.brownian(16384, 512, 1), sk.brownian(16384, 512, 2)
pol = sk.TruncationPolicy.adaptive(1e-12)
loose = sk.PropagateOptions(strict_corner=False)
for i in range(3):
    sk.propagate_with_policy(x, y, pol, loose)
print("---- traced call", file=sys.stderr)
t = time.perf_counter()
sk.propagate_with_policy(x, y, pol, loose)
print("wall", time.perf_counter() - t, file=sys.stderr)
