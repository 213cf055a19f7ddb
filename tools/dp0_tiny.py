import os, sys
sys.path.insert(0, os.getcwd())
from paper_2502_20392_b200 import sigker as sk
x, y = sk.brownian(40, 20, 1), sk.brownian(40, 20, 2)
try:
    print(sk.propagate(x, y, 8, sk.PropagateOptions(strict_corner=False)).value)
except Exception as e:
    print("ERR", e)
