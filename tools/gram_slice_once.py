"""One bench step's worth of the north-star Gram (for ncu captures): the
1/32 slice 0 of the N = 1024, l = 4096, d = 16 datagen family, adaptive --
one sweep launch of skb::sweep_kernel<8,16,EXACT> over 16,400 pairs."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

fam = sk.brownian_family(4096, 16, range(1000, 2024))
r = sk.gram_matrix(fam, sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12)), shard=int(os.environ.get("SLICE", "0")),
                   nshards=32)
print("pairs done", int((~__import__("numpy").isnan(r.values)).sum()))
