"""ctypes binding of the C ABI in include/rsot_cuda.h (librsot_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if
the library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_size_t, c_uint8, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSOT_LIB_PATH") or os.path.join(_HERE, "lib", "librsot_b200.so")

RSOT_CUDA_OK = 0
RSOT_CUDA_INVALID_ARGUMENT = -1
RSOT_CUDA_RUNTIME_ERROR = -2
RSOT_CUDA_NO_DEVICE = -3
RSOT_CUDA_UNSUPPORTED = -4


class RsotCudaScalars(ctypes.Structure):
    _fields_ = [
        ("J", c_double),
        ("D", c_double),
        ("atoms_visited", c_uint64),
        ("candidate_pairs", c_uint64),
        ("empty_candidate_atoms", c_uint64),
    ]


# (name, restype, argtypes) for every symbol include/rsot_cuda.h declares.
_SIGNATURES = [
    ("rsot_cuda_abi_version", c_int, []),
    ("rsot_cuda_last_error", c_char_p, []),
    ("rsot_cuda_ctx_create", c_int, [c_int, POINTER(c_void_p)]),
    ("rsot_cuda_ctx_destroy", c_int, [c_void_p]),
    ("rsot_cuda_ctx_stream", c_void_p, [c_void_p]),
    ("rsot_cuda_ctx_synchronize", c_int, [c_void_p]),
    ("rsot_cuda_ctx_num_sms", c_int, [c_void_p]),
    ("rsot_cuda_comm_unique_id", c_int, [POINTER(c_uint8)]),
    ("rsot_cuda_ctx_set_comm", c_int, [c_void_p, c_int, c_int, POINTER(c_uint8)]),
    ("rsot_cuda_shard_range", None, [c_size_t, c_int, c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    ("rsot_cuda_targets_create", c_int, [c_void_p, c_void_p, c_void_p, c_size_t, POINTER(c_void_p)]),
    ("rsot_cuda_targets_destroy", c_int, [c_void_p]),
    ("rsot_cuda_targets_size", c_size_t, [c_void_p]),
    ("rsot_cuda_atoms_create", c_int, [c_void_p, c_void_p, c_void_p, c_size_t, POINTER(c_void_p)]),
    ("rsot_cuda_atoms_create_partitioned", c_int,
     [c_void_p, c_void_p, c_void_p, c_size_t, POINTER(c_void_p)]),
    ("rsot_cuda_ctx_set_virtual_rank", c_int, [c_void_p, c_int, c_int]),
    ("rsot_cuda_atoms_destroy", c_int, [c_void_p]),
    ("rsot_cuda_atoms_size", c_size_t, [c_void_p]),
    ("rsot_cuda_eval", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_void_p, POINTER(RsotCudaScalars)]),
    ("rsot_cuda_eval_device", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p]),
    ("rsot_cuda_check_status", c_int, [c_void_p]),
    ("rsot_cuda_eval_debug", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_void_p, POINTER(RsotCudaScalars),
      c_void_p, c_void_p, c_void_p]),
    ("rsot_cuda_nearest", c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("rsot_cuda_covering_cost", c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_double)]),
    ("rsot_cuda_softmax_refine", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_double, c_double, c_void_p]),
    ("rsot_cuda_ctx_set_timing", c_int, [c_void_p, c_int]),
    ("rsot_cuda_ctx_set_precision", c_int, [c_void_p, c_int]),
    ("rsot_cuda_eval_cost", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_int, c_void_p,
                                    POINTER(RsotCudaScalars)]),
    ("rsot_cuda_plan_candidates", c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p, c_void_p]),
    ("rsot_cuda_plan_moments", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("rsot_cuda_eval_debug_cost", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_int,
                                          c_void_p, POINTER(RsotCudaScalars), c_void_p, c_void_p, c_void_p]),
    ("rsot_cuda_last_kernel_ms", c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_double)]),
    ("rsot_cuda_measure_fp64_peak", c_int, [c_void_p, POINTER(c_double)]),
    ("rsot_cuda_kernel_launches", c_uint64, []),
    ("rsot_cuda_eval_virtual_world", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_int, c_void_p, POINTER(RsotCudaScalars)]),
    ("rsot_cuda_host_rank_sum", None, [c_void_p, c_int, c_size_t, c_void_p]),
    ("rsot_cuda_atoms_create_local", c_int, [c_void_p, c_void_p, c_void_p, c_size_t, POINTER(c_void_p)]),
    ("rsot_cuda_covering_cost_kind", c_int, [c_void_p, c_void_p, c_void_p, c_int, POINTER(c_double)]),
    ("rsot_cuda_measure_fp32_peaks", c_int, [c_void_p, POINTER(c_double), POINTER(c_double)]),
    ("rsot_cuda_host_finalize", None, [c_void_p, c_void_p, c_size_t, c_double, c_void_p, c_void_p]),
]

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads librsot_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the sm_100a extension with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    try:
        # one NCCL per process: with torch loaded first, the library's lazy
        # dlopen("libnccl.so.2") binds torch's bundled NCCL; the other order
        # would bind the system one and break a later `import torch`
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = ctypes.CDLL(path)
    for name, restype, argtypes in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


class RsotCudaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rsot_cuda error {code}: {msg}")
        self.code = code


def check(code: int) -> None:
    if code == RSOT_CUDA_OK:
        return
    msg = load().rsot_cuda_last_error().decode(errors="replace")
    if code == RSOT_CUDA_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    raise RsotCudaError(code, msg)
