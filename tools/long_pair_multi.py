"""Multi-GPU long pair (BASELINE cfg 3) through the strip pipeline:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/long_pair_multi.py --length 1000001 --dim 4

Each rank sweeps a contiguous band range of the one pair on its own GPU and
streams its top band's alpha series into the next rank's exchange buffer over
NVLink (paper_2502_20392_b200.distributed.propagate_long_pair_distributed).
Timed with CUDA events as the max over ranks; rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2502_20392_b200 import sigker as sk  # noqa: E402
from paper_2502_20392_b200.distributed import propagate_long_pair_distributed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=1_000_001)
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--order", type=int, default=8)
    ap.add_argument("--sigma", type=float, default=1.0)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    sk.set_device(local)
    rng = np.random.default_rng(1)
    steps = rng.standard_normal((2, a.length - 1, a.dim)) * np.sqrt(1.0 / (a.length - 1)) * a.sigma
    xy = np.zeros((2, a.length, a.dim))
    np.cumsum(steps, axis=1, out=xy[:, 1:, :])
    dist.barrier()
    t0 = time.perf_counter()
    value, _ = propagate_long_pair_distributed(xy[0], xy[1], a.order, sk.PropagateOptions(strict_corner=False))
    wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    tiles = (a.length - 1) ** 2
    if dist.get_rank() == 0:
        print(json.dumps({"metric": "tile_updates_per_sec", "value": tiles / wall.item(), "n_gpus": dist.get_world_size(),
                          "length": a.length, "dim": a.dim, "order": a.order, "K": value, "seconds": wall.item()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
