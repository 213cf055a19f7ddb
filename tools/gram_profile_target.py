"""ncu target: one config-5-shaped Gram -- the first M members (default 96;
SK_PROFILE_M) of the north-star family brownian(4096, 16, 1000 + i),
adaptive: a single sweep launch of skb::sweep_kernel<8,16,EXACT>."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

m = int(os.environ.get("SK_PROFILE_M", "96"))
fam = sk.brownian_family(4096, 16, range(1000, 1000 + m))
sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)))
