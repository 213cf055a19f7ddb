"""Per-band timeline of one streaming pair (needs a SK_PROFILE_WAITS build,
SIGKER_B200_LIB=.../libsigker_b200_pw.so): x of length L, y of 32 B + 1
points; prints each band's start/end (us from the first start), dependency
wait and its SM/warp slot."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

L = int(os.environ.get("PROBE_LEN", "4096"))
d = int(os.environ.get("PROBE_DIM", "8"))
loose = sk.PropagateOptions(strict_corner=False)
x = sk.brownian(L, d, 1)
for B in [int(v) for v in os.environ.get("PROBE_BANDS", "2,8,32").split(",")]:
    y = sk.brownian(32 * B + 1, d, 2)
    sk.propagate(x, y, 8, loose)
    path = os.path.join(tempfile.gettempdir(), "utrace.bin")
    os.environ["SK_UTRACE"] = path
    sk.propagate(x, y, 8, loose)
    del os.environ["SK_UTRACE"]
    t = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
    t = t[t[:, 1] > 0]
    t0 = t[:, 1].min()
    print(f"-- bands {B}")
    for row in sorted(t.tolist(), key=lambda r: (r[0] >> 20) & 0xFFFFF):
        b = (row[0] >> 20) & 0xFFFFF
        sm = (row[0] >> 40) & 0xFF
        wp = (row[0] >> 48) & 0xFF
        print(f"band {b:4d} sm {sm:3d} warp {wp:2d}: start {(row[1] - t0) / 1e3:9.1f} end {(row[2] - t0) / 1e3:9.1f} "
              f"wait {(row[3] & ((1 << 40) - 1)) / 1e3:9.1f} us")
