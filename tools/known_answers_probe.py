"""Diagnostics: the known-answer golden cases one at a time (timing + value)."""
import faulthandler
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
faulthandler.dump_traceback_later(int(os.environ.get("KA_TIMEOUT", "60")), exit=True)
from oracle.oracle import Restatement  # noqa: E402  (test infrastructure: input generation only)
from paper_2502_20392_b200 import sigker as sk  # noqa: E402

R = Restatement()
cases = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "known_answers.json")))["cases"]
for c in cases:
    rec = c["recipe"]
    if rec[0] == "brownian":
        _, length, dim, s1, s2, sigma = rec
        x, y = sigma * R.brownian(length, dim, s1), sigma * R.brownian(length, dim, s2)
    else:
        _, length, dim, h, s1, s2 = rec
        x, y = R.fbm(length, dim, h, s1), R.fbm(length, dim, h, s2)
    t0 = time.perf_counter()
    r = sk.propagate_with_policy(x, y, sk.TruncationPolicy.adaptive(1e-12))
    print(c["label"], f"{time.perf_counter() - t0:.3f}s", r.order, abs(r.value - c["value"]) / max(1, abs(c["value"])),
          flush=True)
