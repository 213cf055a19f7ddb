"""Host model of ONE long pair swept by G GPUs (BASELINE cfg 3, SURVEY.md
section 8e): which assignment of 32-row bands to GPUs scales.

The model follows the kernel's streaming schedule (csrc/sk_sweep.cuh):
* each GPU runs W band workers (resident warps: 12 per SM x 148 SMs); its
  bands are claimed in increasing order and hold a worker from the claim on,
  waiting included;
* band b advances one column per step but stays >= LAG steps behind band b-1
  (31 lanes of skew + one 16-column publication chunk + 1); a hand-off that
  crosses GPUs adds XLAG steps (the NVLink store + system-scope flag);
* a GPU's step time is the latency floor (552 ns, one warp per sub-partition,
  measured) or, with a running warps, the throughput time a / W x 861 ns (the
  measured 6.6e10 tile-updates/s over 1776 warps x 32 tiles) -- whichever is
  longer.

Assignments: "contiguous" (GPU g owns bands [g B/G, (g+1) B/G), round 1's
design) and "cyclic" (band blocks of size S dealt round-robin: GPU g owns
blocks g, g+G, g+2G, ...; the top band of every block hands to the next
GPU, GPU G-1 to GPU 0).  Prints the makespan and the scaling efficiency
T(1) / (G T(G)) for each G.

    python tools/strip_sim.py --cols 999999 --gpus 1 2 4 8
"""
import argparse

import numpy as np

LAG = 48          # steps between a band and the one above it (31 + 16 + 1)
XLAG = 16         # extra steps when the hand-off crosses GPUs (~9 us)
TAU_LAT = 552.0   # ns per step, latency floor
TAU_FULL = 861.0  # ns per step with all W workers running
W = 1776          # band workers per GPU


def owners(bands, G, mode, block):
    b = np.arange(bands)
    if mode == "contiguous":
        return np.minimum(b * G // bands, G - 1)
    return (b // block) % G


def simulate(cols, bands, G, mode="cyclic", block=None, dt_ns=500000.0, workers=None):
    """Makespan in seconds.  Within a time step the band chain is advanced
    exactly (band b <= band b-1 - lag, a running min along the chain);
    claims and step times are updated per step of dt_ns."""
    Wk = workers or W
    block = block or Wk
    own = owners(bands, G, mode, block)
    total = float(cols + 31)
    prog = np.zeros(bands)
    claimed = np.zeros(bands, bool)
    xlag = np.full(bands, float(LAG))
    xlag[0] = 0.0
    xlag[1:][own[1:] != own[:-1]] += XLAG
    L = np.cumsum(xlag)
    order = [np.flatnonzero(own == g) for g in range(G)]
    nxt = [0] * G
    first = 0  # bands finish in order: [0, first) are done
    t = 0.0
    while first < bands:
        for g in range(G):
            o = order[g]
            busy = int(np.count_nonzero(claimed[o] & (prog[o] < total)))
            take = min(Wk - busy, len(o) - nxt[g])
            if take > 0:
                claimed[o[nxt[g]:nxt[g] + take]] = True
                nxt[g] += take
        sl = slice(first, bands)
        run = claimed[sl]
        # step time per GPU from the workers that can advance now
        lim = np.empty(bands - first)
        lim[0] = total
        lim[1:] = prog[first:-1] - xlag[first + 1:]
        can = run & (prog[sl] < np.minimum(lim, total))
        a = np.bincount(own[sl][can], minlength=G)
        tau = np.maximum(TAU_LAT, TAU_FULL * a / Wk)
        adv = np.where(run, dt_ns / tau[own[sl]], 0.0)
        c = prog[sl] + adv + L[sl]
        y = np.minimum.accumulate(c)
        prog[sl] = np.maximum(prog[sl], np.minimum(y - L[sl], total))
        while first < bands and prog[first] >= total:
            first += 1
        t += dt_ns
    return t * 1e-9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cols", type=int, default=999_999)
    ap.add_argument("--rows", type=int, default=999_999)
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    a = ap.parse_args()
    bands = (a.rows + 31) // 32
    t1 = simulate(a.cols, bands, 1)
    print(f"l = {a.cols + 1}: {bands} bands; 1 GPU {t1:.2f} s (model)")
    for G in a.gpus:
        for mode in ("contiguous", "cyclic"):
            if G == 1 and mode == "contiguous":
                continue
            tg = simulate(a.cols, bands, G, mode)
            print(f"  G={G} {mode:10s}: {tg:6.2f} s, scaling efficiency {t1 / (G * tg):.1%}")


if __name__ == "__main__":
    main()
