#!/usr/bin/env python3
"""Benchmark of the B200 signature-kernel path (BASELINE.json configs[1]).

Workload (per rank): 256 independent pairs of synthetic Brownian paths,
l = 4096, d = 8, adaptive truncation tol 1e-12 (=> N = 8 for every pair), i.e.
256 x 4095^2 = 4.29e9 tile-updates per step.  Metric: tile-updates/s
(BASELINE.json: "tile-updates/sec and Gram kernel-evals/sec vs roofline");
kernel-evals/s (pairs/s) is reported beside it.

  value : whole-job tile-updates/s with the inputs resident in HBM (device
          entry point sk_pairwise_device: increments + order pre-pass + sweep)
  e2e   : the same through the public host API sk_pairwise (pinned host
          inputs -> H2D -> compute -> D2H values) every step
  roofline : the sweep kernel (dominant) -- algorithmic FP64 flops
          F(N,d) = 4(N+1)^2 + 2d per tile-update over its CUDA-event time,
          against the measured B200 FP64 peak (profiles/fp64_peak_r01.txt)
  cpu_baseline : the reference engine (oracle/_ref, kind "reference") or the
          C restatement (kind "port") on a bounded sample of the same pairs,
          all host cores, rank 0 at N = 1 only

`--impl reference` times the reference's own CPU implementation on the same
config (bounded sample per step; rank 0 only under torchrun).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LEN, DIM, NPAIRS, TOL = 4096, 8, 256, 1e-12
FP64_PEAK_TFLOPS = 37.11  # measured: tools/fp64_peak.cu DMMA m8n8k4 (DFMA 34.2); profiles/fp64_peak_r01.txt
CPU_SAMPLE_PAIRS = 16


def brownian_family(n, length, dim, seed):
    """Synthetic Brownian paths (variance 1/(l-1) per step, datagen.cpp:78-88 shape)."""
    rng = np.random.default_rng(seed)
    steps = rng.standard_normal((n, length - 1, dim)) * np.sqrt(1.0 / (length - 1))
    out = np.zeros((n, length, dim))
    np.cumsum(steps, axis=1, out=out[:, 1:, :])
    return out


def workload(rank):
    xs = brownian_family(NPAIRS, LEN, DIM, 1000 + 2 * rank)
    ys = brownian_family(NPAIRS, LEN, DIM, 1001 + 2 * rank)
    return xs, ys


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


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_sample(xs, ys, kind_pref="reference"):
    """Time the reference CPU path on a bounded sample (all host threads)."""
    from oracle import oracle as orc
    n = min(CPU_SAMPLE_PAIRS, xs.shape[0])
    threads = os.cpu_count() or 1
    xs_s, ys_s = np.ascontiguousarray(xs[:n]), np.ascontiguousarray(ys[:n])
    tiles = n * (xs.shape[1] - 1) * (ys.shape[1] - 1)
    if kind_pref == "reference" and orc.ref_available():
        ref = orc.Reference()
        t0 = time.perf_counter()
        vals, ords = ref.pairwise(xs_s, ys_s, adaptive=True, tol=TOL, threads=threads)
        dt = time.perf_counter() - t0
        kind, cores = "reference", threads
    else:
        R = orc.Restatement()
        t0 = time.perf_counter()
        vals = np.array([R.propagate_with_policy(xs_s[k], ys_s[k], TOL)[0] for k in range(n)])
        dt = time.perf_counter() - t0
        kind, cores = "port", 1
    return {"value": tiles / dt, "unit": "tile-updates/s", "cores": cores, "kind": kind,
            "sample": f"{n} of the {xs.shape[0]} pairs (l={xs.shape[1]}, d={xs.shape[2]}, adaptive tol {TOL}), "
                      f"pair-parallel over {cores} thread(s), {dt:.2f} s"}, vals


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    xs, ys = workload(0)
    for _ in range(args.warmup):
        pass  # the reference CPU path has no warm-up state worth paying for
    vals = []
    times = []
    base = None
    for _ in range(args.steps):
        cb, _v = cpu_reference_sample(xs, ys)
        base = cb
        vals.append(cb["value"])
    v = statistics.median(vals)
    base["value"] = v
    line = {"impl": "reference", "metric": "tile_updates_per_sec", "value": v, "unit": "tile-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"batched pairwise kernels, {NPAIRS} pairs of l={LEN}, d={DIM} Brownian paths, "
                                   f"adaptive tol {TOL} (BASELINE configs[1]); bounded sample of "
                                   f"{CPU_SAMPLE_PAIRS} pairs per step", "pairs": NPAIRS, "length": LEN, "dim": DIM},
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "tile-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_2502_20392_b200 import _capi
    from paper_2502_20392_b200 import sigker as sk
    import ctypes
    lib = _capi.load()
    st = _capi.SkStatus()
    if lib.sk_set_device(torch.cuda.current_device(), ctypes.byref(st)) != 0:
        raise RuntimeError(st.message)
    stream = torch.cuda.current_stream()
    if lib.sk_set_stream(ctypes.c_void_p(stream.cuda_stream), ctypes.byref(st)) != 0:
        raise RuntimeError(st.message)

    xs_h, ys_h = workload(rank)
    xs_pin = torch.from_numpy(xs_h).pin_memory()
    ys_pin = torch.from_numpy(ys_h).pin_memory()
    xs_d = xs_pin.to(dev)
    ys_d = ys_pin.to(dev)
    vals_d = torch.empty(NPAIRS, dtype=torch.float64, device=dev)
    orders = np.zeros(NPAIRS, dtype=np.int32)
    conv = np.zeros(NPAIRS, dtype=np.int32)
    per = (_capi.SkStatus * NPAIRS)()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    tiles_per_step = NPAIRS * (LEN - 1) * (LEN - 1)

    def device_step():
        flush.zero_()
        rc = lib.sk_pairwise_device(ctypes.c_void_p(xs_d.data_ptr()), LEN, ctypes.c_void_p(ys_d.data_ptr()), LEN,
                                    NPAIRS, DIM, 1, 7, TOL, _capi.SK_STRICT_CORNER,
                                    ctypes.c_void_p(vals_d.data_ptr()), orders.ctypes.data_as(ctypes.c_void_p),
                                    conv.ctypes.data_as(ctypes.c_void_p), per, ctypes.byref(st))
        if rc != 0:
            raise RuntimeError(st.message.decode())

    vals_h = np.zeros(NPAIRS)
    mr_h = None

    def e2e_step():
        flush.zero_()
        rc = lib.sk_pairwise(ctypes.c_void_p(xs_pin.data_ptr()), LEN, ctypes.c_void_p(ys_pin.data_ptr()), LEN,
                             NPAIRS, DIM, 1, 7, TOL, _capi.SK_STRICT_CORNER, vals_h.ctypes.data_as(ctypes.c_void_p),
                             orders.ctypes.data_as(ctypes.c_void_p), conv.ctypes.data_as(ctypes.c_void_p), None,
                             per, ctypes.byref(st))
        if rc != 0:
            raise RuntimeError(st.message.decode())

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    time.sleep(1.5)  # let nvidia-smi/NVML finish initialising before the timed region
    sk.stats_enable(True)
    sk.stats_reset()
    ms = timed(device_step, args.steps)
    stats = sk.stats_get()
    # per-step device times (diagnostic, stderr)
    per_step = []
    for _ in range(min(3, args.steps)):
        per_step.append(timed(device_step, 1))
    print(f"[bench] per-step ms: {[round(x, 2) for x in per_step]}", file=sys.stderr)
    sk.stats_enable(False)
    clocks = sampler.stop()
    ms_step = ms / args.steps
    value = ws * tiles_per_step / (ms_step / 1e3)

    # e2e through the host API
    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    ms_e2e = timed(e2e_step, args.steps)
    e2e_value = ws * tiles_per_step / (ms_e2e / args.steps / 1e3)
    vals_dev = vals_d.cpu().numpy()

    avg_launch_ms = stats["sweep_ms"] / max(1, stats["sweep_launches"])
    flops_per_launch = stats["tile_flops"] / max(1, stats["sweep_launches"])
    achieved = flops_per_launch / (avg_launch_ms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "sweep_traffic_r01.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    line = {
        "metric": "tile_updates_per_sec", "value": value, "unit": "tile-updates/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"batched pairwise kernels, {NPAIRS} pairs of l={LEN}, d={DIM} synthetic Brownian "
                               f"paths per GPU, adaptive tol {TOL} (BASELINE configs[1])",
                   "pairs_per_gpu": NPAIRS, "length": LEN, "dim": DIM, "order": int(orders[0]),
                   "tiles_per_step": ws * tiles_per_step, "l2": "flushed (256 MB write) before every step; "
                   "inputs 134 MB > L2", "parallelism": f"pairs sharded, {ws} rank(s), no collective"},
        "kernel_evals_per_sec": ws * NPAIRS / (ms_step / 1e3),
        "e2e": {"value": e2e_value, "unit": "tile-updates/s", "h2d_bytes_per_step": int(xs_h.nbytes + ys_h.nbytes),
                "d2h_bytes_per_step": int(NPAIRS * 8)},
        "roofline": {"bound": "fp64", "kernel": "skb::sweep_kernel<8,8>", "achieved": achieved,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": traffic, "peak_source": "measured FP64 (DMMA) peak, profiles/fp64_peak_r01.txt",
                     "flops_per_tile": 4 * 9 * 9 + 2 * DIM, "sweep_ms_per_launch": avg_launch_ms,
                     "sweep_share_of_step": stats["sweep_ms"] / ms if ms > 0 else None},
        "clocks": clocks,
        "gpu_launches": int(stats["sweep_launches"] + stats["aux_launches"]),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb, ref_vals = cpu_reference_sample(xs_h, ys_h)
        line["cpu_baseline"] = cb
        n = len(ref_vals)
        errs = np.abs(vals_dev[:n] - ref_vals) / np.maximum(1.0, np.abs(ref_vals))
        line["parity"] = {"pairs_checked": int(n), "max_rel_err": float(errs.max()), "tolerance": 1e-10,
                          "e2e_equals_device": bool(np.array_equal(vals_h, vals_dev))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
