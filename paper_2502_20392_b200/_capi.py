"""ctypes binding of the C-ABI in include/sigker_b200.h (libsigker_b200.so).

This is the binding a maintainer of the reference would add on the Python
side; the C++ mirror of the reference API lives in
include/sigker/*.hpp.  The library is built in-tree by
paper_2502_20392_b200/csrc/Makefile (``__graft_entry__.build()``).  There is
no CPU fallback: importing works without a GPU, every compute call then
fails loudly with SK_CUDA_ERROR.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SIGKER_B200_LIB", os.path.join(_HERE, "libsigker_b200.so"))

SK_OK = 0
SK_INVALID_ARGUMENT = 1
SK_NUMERIC_OVERFLOW = 2
SK_INCONSISTENT_BOUNDARY = 3
SK_INTERNAL = 4
SK_CUDA_ERROR = 5

SK_STRICT_CORNER = 1
SK_W_FAULT = 4

# Every symbol include/sigker_b200.h declares (tests check the export list).
EXPORTED = [
    "sk_abi_version", "sk_device_count", "sk_set_device", "sk_set_stream",
    "sk_propagate", "sk_max_abs_rho", "sk_estimate_order", "sk_step_tile",
    "sk_step_tile_fast", "sk_pairwise", "sk_pairwise_device", "sk_gram", "sk_gram_device", "sk_gram_failures",
    "sk_gram_shard_range", "sk_all_finite",
    "sk_stats_enable", "sk_stats_reset", "sk_stats_get", "sk_release",
    "sk_strip_bands", "sk_strip_plan", "sk_exchange_alloc", "sk_exchange_reset", "sk_exchange_free", "sk_ipc_handle",
    "sk_ipc_open", "sk_ipc_close", "sk_enable_peer_access", "sk_propagate_strip", "sk_propagate_split",
]


class SkStatus(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("tile_k", ctypes.c_uint64),
                ("tile_l", ctypes.c_uint64), ("message", ctypes.c_char * 256)]


class SkGramFailure(ctypes.Structure):
    _fields_ = [("row", ctypes.c_uint32), ("col", ctypes.c_uint32), ("status", SkStatus)]


class SkStats(ctypes.Structure):
    _fields_ = [("sweep_launches", ctypes.c_uint64), ("aux_launches", ctypes.c_uint64),
                ("sweep_ms", ctypes.c_double), ("tiles", ctypes.c_double),
                ("tile_flops", ctypes.c_double), ("literal_rechecks", ctypes.c_uint64)]


_lib = None

P = ctypes.c_void_p
DP = ctypes.POINTER(ctypes.c_double)
IP = ctypes.POINTER(ctypes.c_int)
SZ = ctypes.c_size_t
ST = ctypes.POINTER(SkStatus)


def load():
    """Load libsigker_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            "libsigker_b200.so is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "sk_abi_version": ([], ctypes.c_int),
        "sk_device_count": ([], ctypes.c_int),
        "sk_set_device": ([ctypes.c_int, ST], ctypes.c_int),
        "sk_set_stream": ([P, ST], ctypes.c_int),
        "sk_propagate": ([P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_uint32, P, P, P, P, ST], ctypes.c_int),
        "sk_max_abs_rho": ([P, SZ, P, SZ, SZ, P, ST], ctypes.c_int),
        "sk_estimate_order": ([ctypes.c_double, SZ, ctypes.c_double, P, P, ST], ctypes.c_int),
        "sk_step_tile": ([ctypes.c_double, P, P, ctypes.c_int, P, P, P, ST], ctypes.c_int),
        "sk_step_tile_fast": ([ctypes.c_double, P, P, ctypes.c_int, P, P, P, ST], ctypes.c_int),
        "sk_pairwise": ([P, SZ, P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint32,
                         P, P, P, P, P, ST], ctypes.c_int),
        "sk_pairwise_device": ([P, SZ, P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                ctypes.c_uint32, P, P, P, P, ST], ctypes.c_int),
        "sk_gram": ([P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint32, ctypes.c_int,
                     SZ, SZ, P, P, P, P, P, P, ST], ctypes.c_int),
        "sk_gram_device": ([P, SZ, SZ, SZ, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint32,
                            ctypes.c_int, SZ, SZ, P, P, P, P, ST], ctypes.c_int),
        "sk_gram_failures": ([P, SZ], SZ),
        "sk_gram_shard_range": ([SZ, SZ, SZ, P, P], ctypes.c_int),
        "sk_all_finite": ([P, SZ], ctypes.c_int),
        "sk_stats_enable": ([ctypes.c_int], ctypes.c_int),
        "sk_stats_reset": ([], ctypes.c_int),
        "sk_stats_get": ([ctypes.POINTER(SkStats)], ctypes.c_int),
        "sk_release": ([], ctypes.c_int),
        "sk_strip_bands": ([SZ, ctypes.c_int, P], ctypes.c_int),
        "sk_strip_plan": ([SZ, ctypes.c_int, SZ, SZ, SZ, P, P, P], ctypes.c_int),
        "sk_exchange_alloc": ([SZ, ctypes.c_int, SZ, P, P, ST], ctypes.c_int),
        "sk_exchange_reset": ([P, SZ, ST], ctypes.c_int),
        "sk_exchange_free": ([P, P], ctypes.c_int),
        "sk_ipc_handle": ([P, P, ST], ctypes.c_int),
        "sk_ipc_open": ([P, P, ST], ctypes.c_int),
        "sk_ipc_close": ([P], ctypes.c_int),
        "sk_enable_peer_access": ([ctypes.c_int, ST], ctypes.c_int),
        "sk_propagate_strip": ([P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_uint32, SZ, SZ, SZ, P, P, P, P, P, P, ST],
                               ctypes.c_int),
        "sk_propagate_split": ([P, SZ, P, SZ, SZ, ctypes.c_int, ctypes.c_uint32, SZ, SZ, P, ST], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib
