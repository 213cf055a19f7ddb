#!/usr/bin/env python3
"""Benchmark of the B200 signature-kernel path on the north-star Gram workload.

Workload (BASELINE.json configs[4], SURVEY.md section 8d cfg 5): the Gram
matrix of N = 1024 series x_i = datagen::brownian(4096, 16, 1000 + i) (the
reference's own generator, bit for bit), adaptive truncation tol 1e-12
(=> N = 8), as gram_matrix (gram.cpp:16-98) evaluates it: 524,800 upper-
triangle kernel-evals of 4095^2 tile-updates each, plus each pair's exact
max|rho| (GramResult.max_abs_increment_product).  One step = one of the
16 equal slices of the upper-triangle pair range (32,800 kernel-evals,
5.5e11 tile-updates; large enough that a launch's tail -- the last pairs'
critical path -- stays a few percent at 8 GPUs); step s evaluates slice
s mod 16, so 16 steps are the whole Gram.  With --gpus N the slice is split
over N ranks (sk_gram_shard_range arithmetic: rank r owns sub-range s*N + r
of 16*N) and assembled by an NCCL all-reduce of the m x m matrix inside the
timed region: strong scaling.

  value : kernel-evals/s of the whole job, family resident in HBM on every
          rank (sk_gram_device into a device matrix + all-reduce)
  e2e   : the same through the public API (distributed.gram_matrix_
          distributed -> sk_gram): every step copies the pinned host family
          to the device and reads the matrix back (min(K, 4) timed steps:
          the same metric over a shorter run)
  roofline : the dominant kernel (skb::sweep_kernel<8,16,EXACT>): algorithmic
          FP64 flops F(N,d) = 4(N+1)^2 + 2d per tile-update over its
          CUDA-event time (library event pair on the launching stream),
          against the measured B200 FP64 peak (profiles/fp64_peak_r01.txt)
  cpu_baseline : the unmodified reference (oracle/_ref, propagate_with_policy
          per pair, pair-parallel over all host cores) on a bounded sample of
          slice 0's pairs; rank 0 at N = 1
  configs : BASELINE configs 1-4 at N = 1 (rank 0), each checked against the
          reference's goldens (tests/golden/*.json)

`--impl reference` times the reference's own CPU implementation on the same
workload (bounded sample of each step's slice, all host cores; rank 0 only).
`--gpus N` outside torchrun re-launches itself under torch.distributed.run
with N ranks; it fails if fewer than N GPUs are visible.  `--cpu-smoke`
runs the same slicing / assembly / timing over gloo on the CPU with the C
restatement standing in for the GPU (a test of the multi-rank plumbing).
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, LEN, DIM, SEED0, TOL = 1024, 4096, 16, 1000, 1e-12
SLICES = 16
ORDER = 8
FP64_PEAK_TFLOPS = 37.11  # measured: tools/fp64_peak.cu DMMA m8n8k4 (DFMA 34.2); profiles/fp64_peak_r01.txt
CPU_SAMPLE_PAIRS = 16
TOTAL_PAIRS = M * (M + 1) // 2
TILES_PER_PAIR = (LEN - 1) ** 2


# ------------------------------------------------------------ workload math
def pair_range(total, shard, nshards):
    """sk_gram_shard_range: [total*shard/nshards, total*(shard+1)/nshards)."""
    return total * shard // nshards, total * (shard + 1) // nshards


def step_range(step, rank, world, total=TOTAL_PAIRS, slices=SLICES):
    """Rank `rank`'s pairs of step `step`: sub-shard s*world + rank of
    slices*world, s = step mod slices (the ranks tile slice s exactly)."""
    s = step % slices
    return pair_range(total, s * world + rank, slices * world)


def pair_of(t, m=M):
    """(i, j), i <= j, of row-major upper-triangle index t."""
    i, start = 0, 0
    while start + (m - i) <= t:
        start += m - i
        i += 1
    return i, i + (t - start)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            if bits & 0x1:  # idle samples are not "under load"
                continue
            sm.append(s)
            mx.append(m)
            for b, name in self.REASONS.items():
                if bits & b and b != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- launching
def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks (one per GPU) and pass its exit code through."""
    if not args.cpu_smoke and not args.share_gpu:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible", file=sys.stderr)
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------ CPU legs
def golden_cfg5():
    with open(os.path.join(ROOT, "tests", "golden", "scale.json")) as f:
        return json.load(f)["cfg5"]["entries"]


def cpu_reference_sample(family, t0, n, threads=None):
    """The reference (oracle/_ref: unmodified sigker, propagate_with_policy
    per pair, ThreadPool pair-parallel like gram.cpp:51-66) on pairs t0..t0+n
    of the upper triangle; falls back to the C restatement (1 thread).
    Returns (cpu_baseline dict, {(i, j): value})."""
    from oracle import oracle as orc
    pairs = [pair_of(t) for t in range(t0, t0 + n)]
    xs = np.ascontiguousarray(np.stack([family[i] for i, _ in pairs]))
    ys = np.ascontiguousarray(np.stack([family[j] for _, j in pairs]))
    threads = threads or os.cpu_count() or 1
    if orc.ref_available():
        ref = orc.Reference()
        t = time.perf_counter()
        vals, _ = ref.pairwise(xs, ys, adaptive=True, tol=TOL, threads=threads)
        dt = time.perf_counter() - t
        kind, cores = "reference", threads
    else:
        R = orc.Restatement()
        t = time.perf_counter()
        vals = np.array([R.propagate_with_policy(xs[k], ys[k], TOL)[0] for k in range(n)])
        dt = time.perf_counter() - t
        kind, cores = "port", 1
    cb = {"value": n / dt, "unit": "kernel-evals/s", "cores": cores, "kind": kind,
          "tile_updates_per_sec": n * TILES_PER_PAIR / dt,
          "sample": f"{n} Gram entries (upper-triangle pairs {t0}..{t0 + n - 1}: x_i = brownian(4096,16,1000+i), "
                    f"adaptive tol {TOL}), pair-parallel over {cores} thread(s), {dt:.2f} s"}
    return cb, {p: float(v) for p, v in zip(pairs, vals)}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2502_20392_b200 import sigker as sk
    family = sk.brownian_family(LEN, DIM, range(SEED0, SEED0 + M))
    vals = []
    base = None
    for step in range(args.steps):
        lo, _ = step_range(step, 0, 1)
        base, _ = cpu_reference_sample(family, lo, CPU_SAMPLE_PAIRS)
        vals.append(base["value"])
    v = statistics.median(vals)
    base["value"] = v
    line = {"impl": "reference", "metric": "gram_kernel_evals_per_sec", "value": v, "unit": "kernel-evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(1) | {"sample_per_step": f"{CPU_SAMPLE_PAIRS} pairs of the step's slice"},
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "kernel-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(ws):
    return {"workload": f"cfg 5 (BASELINE configs[4]): Gram matrix of N={M} series x_i = datagen::brownian"
                        f"({LEN},{DIM},{SEED0}+i), adaptive tol {TOL}; one step = one 1/{SLICES} slice of the "
                        f"{TOTAL_PAIRS} upper-triangle kernel-evals",
            "m": M, "length": LEN, "dim": DIM, "slices": SLICES, "pairs_per_step": TOTAL_PAIRS // SLICES,
            "tiles_per_step": TOTAL_PAIRS // SLICES * TILES_PER_PAIR,
            "parallelism": f"row-major pair range split over {ws} rank(s), NCCL all-reduce assembly" if ws > 1
            else "1 GPU",
            "l2": "each step's working set (537 MB family + increments) exceeds the 126 MB L2"}


# ------------------------------------------------------- gloo CPU smoke
def run_cpu_smoke(args):
    """The multi-rank plumbing on CPU (gloo): the same step_range split, the
    all-reduce assembly and max-over-ranks timing, with the C restatement
    computing each rank's pairs of a tiny family."""
    import torch
    import torch.distributed as dist
    from oracle.oracle import Restatement
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    R = Restatement()
    m, length = 7, 9
    fam = np.stack([R.brownian(length, 2, 50 + i) for i in range(m)])
    total = m * (m + 1) // 2
    slices = 3
    mats = []
    t0 = time.perf_counter()
    for step in range(slices):
        mat = np.zeros((m, m))
        lo, hi = step_range(step, rank, ws, total, slices)
        for t in range(lo, hi):
            i, j = pair_of(t, m)
            mat[i, j] = mat[j, i] = R.propagate(fam[i], fam[j], ORDER)[0]
        buf = torch.from_numpy(mat)
        if ws > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        mats.append(buf.numpy().copy())
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    full = sum(mats)
    ref, _, _, _ = R.gram(fam, adaptive=False, order=ORDER)
    ok = bool(np.array_equal(full, ref))
    if rank == 0:
        print(json.dumps({"cpu_smoke": True, "world_size": ws, "assembled_equals_single_process": ok,
                          "seconds_max_over_ranks": float(dt.item())}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


# ---------------------------------------------------------- extra configs
def extra_configs(sk, lib, st, capi):
    """BASELINE configs 1-4 at N = 1 through the public API (host inputs),
    each with parity against the reference's goldens."""
    import ctypes
    out = {}
    gold = os.path.join(ROOT, "tests", "golden")
    known = {c["label"]: c for c in json.load(open(os.path.join(gold, "known_answers.json")))["cases"]}
    scale = json.load(open(os.path.join(gold, "scale.json")))
    pol = sk.TruncationPolicy.adaptive(TOL)

    def timed_call(fn, reps=1):
        sk.stats_enable(True)
        sk.stats_reset()
        t = time.perf_counter()
        for _ in range(reps):
            r = fn()
        wall = (time.perf_counter() - t) / reps
        s = sk.stats_get()
        sk.stats_enable(False)
        return r, wall, s

    # cfg 1: latency of one small pair.  Single-pair configs time propagate on
    # TimeSeries built once (datagen::brownian returns a TimeSeries in the
    # reference; its finiteness scan is construction, not propagation)
    x, y = sk.TimeSeries(sk.brownian(1000, 2, 1)), sk.TimeSeries(sk.brownian(1000, 2, 2))
    for _ in range(3):
        sk.propagate_with_policy(x, y, pol)
    r, wall, s = timed_call(lambda: sk.propagate_with_policy(x, y, pol), reps=20)
    # a latency: also the median of single calls (host hiccups -- a page
    # fault, a scheduler tick -- move the mean of 20 ~1 ms calls)
    singles = []
    for _ in range(21):
        t1 = time.perf_counter()
        sk.propagate_with_policy(x, y, pol)
        singles.append(time.perf_counter() - t1)
    out["cfg1"] = {"workload": "single pair l=1000, d=2, adaptive (x=brownian(1000,2,1), y=(..,2))",
                   "seconds_e2e": wall, "seconds_e2e_median": float(np.median(singles)),
                   "tile_updates_per_sec_e2e": 999 ** 2 / wall,
                   "sweep_ms": s["sweep_ms"] / 20, "order": r.order,
                   "rel_err_vs_reference": abs(r.value - known["cfg1"]["value"]) / abs(known["cfg1"]["value"])}
    # cfg 2: 256 pairs l=4096, d=8, device-resident inputs
    xs = sk.brownian_family(4096, 8, [2 * p + 1 for p in range(256)])
    ys = sk.brownian_family(4096, 8, [2 * p + 2 for p in range(256)])
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    xd, yd = torch.from_numpy(xs).to(dev), torch.from_numpy(ys).to(dev)
    vd = torch.empty(256, dtype=torch.float64, device=dev)
    ords = np.zeros(256, dtype=np.int32)

    def cfg2():
        rc = lib.sk_pairwise_device(ctypes.c_void_p(xd.data_ptr()), 4096, ctypes.c_void_p(yd.data_ptr()), 4096, 256,
                                    8, 1, 7, TOL, capi.SK_STRICT_CORNER, ctypes.c_void_p(vd.data_ptr()),
                                    ords.ctypes.data_as(ctypes.c_void_p), None, None, ctypes.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())
    cfg2()
    torch.cuda.synchronize()
    _, wall, s = timed_call(cfg2, reps=5)
    v0 = float(vd[0].item())
    out["cfg2"] = {"workload": "256 pairs l=4096, d=8 (x_p=brownian(4096,8,2p+1), y_p=(..,2p+2)), adaptive, "
                               "inputs resident in HBM",
                   "tile_updates_per_sec": 256 * 4095 ** 2 / wall, "kernel_evals_per_sec": 256 / wall,
                   "ms_per_step": wall * 1e3, "roofline_frac": s["tile_flops"] / (s["sweep_ms"] / 1e3) / 1e12
                   / FP64_PEAK_TFLOPS, "order": int(ords[0]),
                   "rel_err_pair0_vs_reference": abs(v0 - known["cfg2_pair0"]["value"]) / abs(known["cfg2_pair0"]["value"])}
    del xd, yd
    # cfg 4: l=16384, d=512 (large-d path); the reference throws here, the
    # check-free restatement is the golden
    g4 = scale["cfg4"]
    x, y = sk.TimeSeries(sk.brownian(16384, 512, 1)), sk.TimeSeries(sk.brownian(16384, 512, 2))
    loose = sk.PropagateOptions(strict_corner=False)
    sk.propagate_with_policy(x, y, pol, loose)
    r, wall, s = timed_call(lambda: sk.propagate_with_policy(x, y, pol, loose), reps=3)
    out["cfg4"] = {"workload": "single pair l=16384, d=512 (brownian seeds 1/2), adaptive, corner check off "
                               "(the reference throws InconsistentBoundaryError here)",
                   "seconds_e2e": wall, "tile_updates_per_sec_e2e": 16383 ** 2 / wall, "order": r.order,
                   "roofline_frac_e2e": 16383 ** 2 * (4 * 81 + 2 * 512) / wall / 1e12 / FP64_PEAK_TFLOPS,
                   "rel_err_vs_restatement": abs(r.value - g4["restatement"]["value"]) / abs(g4["restatement"]["value"])}
    # cfg 3: one pair l=10^6, d=4 with its prefix knots
    g3 = scale["cfg3"]["sigma1"]["restatement"]
    x, y = sk.TimeSeries(sk.brownian(1_000_000, 4, 1)), sk.TimeSeries(sk.brownian(1_000_000, 4, 2))
    r, wall, s = timed_call(lambda: sk.propagate(x, y, ORDER, loose, diag=True))
    errs = [abs(r.diag[a - 1] - v) / abs(v) for a, v in zip(g3["knots"], g3["values"])]
    out["cfg3"] = {"workload": "single pair l=1,000,000, d=4 (brownian seeds 1/2), N=8 (Cauchy-Schwarz proof), "
                               "corner check off; knots K(a,a) checked",
                   "seconds_e2e": wall, "tile_updates_per_sec_e2e": 999_999 ** 2 / wall,
                   "roofline_frac_sweep": s["tile_flops"] / (s["sweep_ms"] / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                   "knots": g3["knots"], "max_rel_err_knots_vs_reference": max(errs), "value": r.value}
    return out


# -------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip BASELINE configs 1-4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-smoke", action="store_true", help="gloo CPU run of the multi-rank plumbing")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: all ranks on cuda:0 over gloo (the multi-rank GPU path on a 1-GPU box; "
                         "the Gram shards are independent, so sharing one GPU cannot deadlock)")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.cpu_smoke:
        return run_cpu_smoke(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    if ws != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr)
        return 1

    import ctypes
    import torch
    dist = None
    if args.share_gpu:
        local = 0
    elif torch.cuda.device_count() < max(1, ws):
        print(f"bench.py: {ws} rank(s) but {torch.cuda.device_count()} GPU(s) visible", file=sys.stderr)
        return 1
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def allreduce_(t, op):
        if args.share_gpu:  # gloo: through host memory
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)

    from paper_2502_20392_b200 import _capi
    from paper_2502_20392_b200 import sigker as sk
    from paper_2502_20392_b200 import distributed as skd
    lib = _capi.load()
    st = _capi.SkStatus()
    if lib.sk_set_device(local, ctypes.byref(st)) != 0:
        raise RuntimeError(st.message)
    stream = torch.cuda.current_stream()
    if lib.sk_set_stream(ctypes.c_void_p(stream.cuda_stream), ctypes.byref(st)) != 0:
        raise RuntimeError(st.message)

    # the family: datagen on the host (pinned), resident copy in HBM
    fam_pin = torch.empty((M, LEN, DIM), dtype=torch.float64).pin_memory()
    fam_h = fam_pin.numpy()
    sk.brownian_family(LEN, DIM, range(SEED0, SEED0 + M), out=fam_h)
    fam_d = fam_pin.to(dev)
    mat = torch.zeros((M, M), dtype=torch.float64, device=dev)
    acc = torch.zeros((M, M), dtype=torch.float64, device=dev)  # every computed slice, for parity
    maxp = ctypes.c_double()
    conv = ctypes.c_int()
    nf = ctypes.c_size_t()

    def device_step(step):
        lo, hi = step_range(step, rank, ws)
        mat.zero_()
        rc = lib.sk_gram_device(ctypes.c_void_p(fam_d.data_ptr()), M, LEN, DIM, 1, 7, TOL, _capi.SK_STRICT_CORNER,
                                1, lo, hi, ctypes.c_void_p(mat.data_ptr()), ctypes.byref(maxp), ctypes.byref(conv),
                                ctypes.byref(nf), ctypes.byref(st))
        if rc != 0:
            raise RuntimeError(st.message.decode())
        if dist is not None:
            allreduce_(mat, dist.ReduceOp.SUM)
        return mat

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, first):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(steps):
            fn(first + k)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            allreduce_(t, dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # warm-up on the last slices, timed steps from slice 0
    for k in range(args.warmup):
        device_step(SLICES - 1 - (k % SLICES))
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(1.5)  # let nvidia-smi/NVML initialise before the timed region

    def step_acc(step):
        m_ = device_step(step)
        if step < SLICES:
            acc.add_(m_)

    sk.stats_enable(True)
    sk.stats_reset()
    ms = timed(step_acc, args.steps, 0)
    stats = sk.stats_get()
    sk.stats_enable(False)
    clocks = sampler.stop()
    ms_step = ms / args.steps
    pairs_per_step = TOTAL_PAIRS // SLICES
    value = pairs_per_step / (ms_step / 1e3)

    # e2e through the public API (host family in, host matrix out, every step)
    ms_e2e = None
    h2d = M * LEN * DIM * 8
    if not args.no_e2e:
        opts = sk.GramOptions(policy=sk.TruncationPolicy.adaptive(TOL))

        def e2e_step(step):
            s = step % SLICES
            if dist is not None:
                skd.gram_matrix_distributed(fam_h, opts, shard=s, nshards=SLICES,
                                            device=torch.device("cpu") if args.share_gpu else None)
            else:
                sk.gram_matrix(fam_h, opts, shard=s, nshards=SLICES)
        e2e_step(SLICES - 1)
        e2e_steps = min(args.steps, 4)
        ms_e2e = timed(e2e_step, e2e_steps, 0)
    e2e_value = pairs_per_step / (ms_e2e / e2e_steps / 1e3) if ms_e2e else None

    # roofline of the dominant kernel (this rank's launches)
    avg_launch_ms = stats["sweep_ms"] / max(1, stats["sweep_launches"])
    flops_per_launch = stats["tile_flops"] / max(1, stats["sweep_launches"])
    achieved = flops_per_launch / (avg_launch_ms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "sweep_traffic_r02.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    line = {
        "metric": "gram_kernel_evals_per_sec", "value": value, "unit": "kernel-evals/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen::brownian, "
        "the reference's generator, bit-identical)",
        "config": workload_config(ws),
        "tile_updates_per_sec": value * TILES_PER_PAIR,
        "e2e": None if e2e_value is None else {
            "value": e2e_value, "unit": "kernel-evals/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": M * M * 8, "path": "distributed.gram_matrix_distributed -> sk_gram (pinned "
            "host family copied to the device every step; matrix back to the host)" if ws > 1 else
            "sigker.gram_matrix -> sk_gram (pinned host family copied to the device every step; matrix back)",
            "bytes_note": "per rank"},
        "roofline": {"bound": "fp64", "kernel": "skb::sweep_kernel<8,16,EXACT>", "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": traffic, "peak_source": "measured FP64 (DMMA m8n8k4) peak, profiles/fp64_peak_r01.txt "
                     "(MEASURED_PEAKS.json has no FP64 entry)",
                     "flops_per_tile": 4 * (ORDER + 1) ** 2 + 2 * DIM, "sweep_ms_per_launch": avg_launch_ms,
                     "sweep_share_of_step": stats["sweep_ms"] / ms if ms > 0 else None},
        "clocks": clocks,
        "gpu_launches": int(stats["sweep_launches"] + stats["aux_launches"]),
        "literal_rechecks": int(stats["literal_rechecks"]),
    }
    # parity of the computed slices against the reference's goldens
    if rank == 0:
        A = acc.cpu().numpy()
        done = set()
        for step in range(min(args.steps, SLICES)):
            done.add(step)
        errs = []
        for e in golden_cfg5():
            if (e["linear"] * SLICES) // TOTAL_PAIRS in done:
                errs.append(abs(A[e["i"], e["j"]] - e["value"]) / abs(e["value"]))
        line["parity"] = {"golden_entries_checked": len(errs), "max_rel_err": max(errs) if errs else None,
                          "tolerance": 1e-10, "reference": "tests/golden/scale.json (reference "
                          "propagate_with_policy per entry)"}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb, ref_vals = cpu_reference_sample(fam_h, 0, CPU_SAMPLE_PAIRS)
        line["cpu_baseline"] = cb
        A = acc.cpu().numpy()
        line["parity"]["in_run_pairs_checked"] = len(ref_vals)
        line["parity"]["in_run_max_rel_err"] = max(abs(A[i, j] - v) / abs(v) for (i, j), v in ref_vals.items())
    if rank == 0 and ws == 1 and not args.no_extras:
        # the configs run on the library's own stream, not torch's default stream
        lib.sk_set_stream(None, ctypes.byref(st))
        line["configs"] = extra_configs(sk, lib, st, _capi)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
