"""Multi-process paths through the real GPU code (no injected oracle):

* the row-block sharded Gram (distributed.gram_matrix_distributed, SURVEY.md
  section 8e) with two ranks -- two processes on the one GPU of this box, gloo
  for the host-side collectives -- each rank running its sk_gram shard on the
  device; the assembled matrix, orders and failure records must equal one
  single-process call bit for bit (gram.cpp:74-77 failure semantics included);
* the long-pair strip hand-off's CUDA IPC plumbing (sk_exchange_alloc ->
  sk_ipc_handle in one process, sk_ipc_open in another): handles round-trip
  and both processes see the same device memory.

Ranks whose kernels wait on each other must not share one GPU (the strip
pipeline itself is covered on one GPU by the single-launch emulation,
test_strip_protocol_emulated_on_one_gpu); these tests only share it for
independent work and plain memory traffic."""
import ctypes
import multiprocessing as mp
import os
import random
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _family():
    sys.path.insert(0, ROOT)
    from oracle.oracle import Restatement
    R = Restatement()
    rng = R.rng(905)
    fam = [rng.random_series(40 + 3 * k, 2, 1.0) for k in range(9)]
    big = rng.random_series(45, 2, 1.0) * 3e3  # |delta| > 1.25e5 against the larger series
    fam.append(big)
    return fam


def _gram_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_20392_b200 import sigker as sk
        from paper_2502_20392_b200.distributed import gram_matrix_distributed
        sk.set_device(0)
        opts = sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12), strict_corner=False, compute_bound=True)
        r = gram_matrix_distributed(_family(), opts)
        q.put((rank, np.asarray(r.values).tobytes(), np.asarray(r.orders).tolist(),
               [(f.row, f.col, f.message) for f in r.failures], r.max_abs_increment_product))
    except Exception as e:  # surface the error in the parent
        q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


def test_sharded_gram_over_two_ranks_matches_one_call(sk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randint(0, 3000)
    procs = [ctx.Process(target=_gram_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, vals, *_ in res:
        assert not isinstance(vals, str), (rank, vals)
    opts = sk.GramOptions(policy=sk.TruncationPolicy.adaptive(1e-12), strict_corner=False, compute_bound=True)
    one = sk.gram_matrix(_family(), opts)
    assert one.failures, "the scaled member must overflow against something"
    for rank, vals, orders, failures, maxp in res:
        assert vals == np.asarray(one.values).tobytes(), rank
        assert orders == np.asarray(one.orders).tolist()
        assert failures == [(f.row, f.col, f.message) for f in one.failures]
        assert maxp == one.max_abs_increment_product


def _cudart():
    import torch  # noqa: F401  (loads the CUDA runtime torch ships)
    for name in ("libcudart.so", "libcudart.so.12"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    import glob
    import torch as _t
    cands = glob.glob(os.path.join(os.path.dirname(_t.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    return ctypes.CDLL(cands[0])


def _ipc_reader(handle_a, handle_p, nbytes, q):
    sys.path.insert(0, ROOT)
    try:
        from paper_2502_20392_b200 import _capi
        lib = _capi.load()
        st = _capi.SkStatus()
        a, p = ctypes.c_void_p(), ctypes.c_void_p()
        rc = lib.sk_ipc_open(ctypes.create_string_buffer(handle_a, 64), ctypes.byref(a), ctypes.byref(st))
        rc |= lib.sk_ipc_open(ctypes.create_string_buffer(handle_p, 64), ctypes.byref(p), ctypes.byref(st))
        if rc:
            q.put(("open failed", st.message.decode()))
            return
        rt = _cudart()
        buf = np.zeros(nbytes // 8)
        rt.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), a, ctypes.c_size_t(nbytes), 2)  # device -> host
        pattern = np.arange(nbytes // 8, dtype=np.float64) * 0.5 + 3.0
        rt.cudaMemcpy(a, ctypes.c_void_p(pattern.ctypes.data), ctypes.c_size_t(nbytes), 1)  # host -> device
        ctr = np.array([1234567], dtype=np.uint64)
        rt.cudaMemcpy(p, ctypes.c_void_p(ctr.ctypes.data), ctypes.c_size_t(8), 1)
        rt.cudaDeviceSynchronize()
        lib.sk_ipc_close(a)
        lib.sk_ipc_close(p)
        q.put(("ok", buf.tolist()[:4]))
    except Exception as e:
        q.put(("error", repr(e)))


def test_ipc_exchange_buffers_round_trip(sk):
    """The consumer side of a strip boundary allocates the exchange buffer and
    progress counter and exports both; a second process maps them and writes;
    the first sees the writes (and its own zeroed counter before)."""
    from paper_2502_20392_b200 import _capi
    lib = _capi.load()
    st = _capi.SkStatus()
    lx, order = 4097, 8
    a, p = ctypes.c_void_p(), ctypes.c_void_p()
    assert lib.sk_exchange_alloc(lx, order, 1, ctypes.byref(a), ctypes.byref(p), ctypes.byref(st)) == 0, st.message
    try:
        ha, hp = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
        assert lib.sk_ipc_handle(a, ha, ctypes.byref(st)) == 0, st.message
        assert lib.sk_ipc_handle(p, hp, ctypes.byref(st)) == 0, st.message
        rt = _cudart()
        nbytes = 4096 * 8
        ctr = np.array([99], dtype=np.uint64)
        rt.cudaMemcpy(ctypes.c_void_p(ctr.ctypes.data), p, ctypes.c_size_t(8), 2)
        assert ctr[0] == 0  # sk_exchange_alloc zeroed the progress counter
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        proc = ctx.Process(target=_ipc_reader, args=(bytes(ha), bytes(hp), nbytes, q))
        proc.start()
        status, payload = q.get(timeout=120)
        proc.join(timeout=60)
        assert status == "ok", payload
        back = np.zeros(nbytes // 8)
        rt.cudaMemcpy(ctypes.c_void_p(back.ctypes.data), a, ctypes.c_size_t(nbytes), 2)
        assert np.array_equal(back, np.arange(nbytes // 8, dtype=np.float64) * 0.5 + 3.0)
        rt.cudaMemcpy(ctypes.c_void_p(ctr.ctypes.data), p, ctypes.c_size_t(8), 2)
        assert ctr[0] == 1234567
        assert lib.sk_exchange_reset(p, 1, ctypes.byref(st)) == 0
        rt.cudaMemcpy(ctypes.c_void_p(ctr.ctypes.data), p, ctypes.c_size_t(8), 2)
        assert ctr[0] == 0
    finally:
        lib.sk_exchange_free(a, p)


def test_bench_multi_rank_gpu_path_on_one_gpu():
    """bench.py's N-rank GPU path -- sk_gram_device per rank on its share of
    each slice, all-reduce assembly, max-over-ranks timing, parity of the
    assembled slice against the reference's goldens -- with two ranks sharing
    the box's one GPU over gloo (--share-gpu; the shards never wait on each
    other)."""
    import json
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--share-gpu", "--steps", "1",
                          "--warmup", "1", "--no-extras", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["parity"]["golden_entries_checked"] >= 1
    assert line["parity"]["max_rel_err"] <= 1e-10
