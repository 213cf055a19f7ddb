"""ncu target: one config-5-shaped Gram (96 series, l=4096, d=16, adaptive) -- a single sweep launch."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2502_20392_b200 import sigker as sk
rng = np.random.default_rng(5)
fam = list(np.cumsum(rng.standard_normal((96, 4096, 16)) / 64.0, axis=1))
sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)))
