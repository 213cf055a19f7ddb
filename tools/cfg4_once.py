"""One cfg-4-shaped large-d sweep (for ncu captures): l=16384, d=512, N=8."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

L = int(os.environ.get("CFG4_LEN", "16384"))
x, y = sk.brownian(L, 512, 1), sk.brownian(L, 512, 2)
print(sk.propagate(x, y, 8, sk.PropagateOptions(strict_corner=False)).value)
