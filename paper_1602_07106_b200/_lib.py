"""ctypes binding of ``libparba_b200.so`` (include/parba_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute call raises ``GenerationError``.  Device buffers are torch tensors
(allocation and streams only -- torch is plumbing here, the compute is the
library's CUDA kernels).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import GenerationError, ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
# PARBA_LIB selects another build of the same library (e.g. the
# -DPARBA_DEBUG_CHECKS=1 build of tools/check_build.sh); default: in-tree.
LIB_PATH = os.environ.get("PARBA_LIB") or os.path.join(HERE, "libparba_b200.so")

PARBA_OK, PARBA_EINVAL, PARBA_ECUDA, PARBA_ENOMEM, PARBA_EINFEASIBLE = 0, 1, 2, 3, 4
HASH_CRC, HASH_SIMPLE = 0, 1
FLAG_NO_SELF_LOOPS, FLAG_NO_PARALLEL_EDGES = 1, 2

# Every symbol include/parba_b200.h declares (checked by tests/test_boundary.py).
EXPORTS = (
    "parba_version", "parba_last_error", "parba_device_count", "parba_hash",
    "parba_resolve_chains", "parba_generate", "parba_generate_targets", "parba_edges_at", "parba_degree_window",
    "parba_degree_full", "parba_count_ids", "parba_generate_host", "parba_write_binary", "parba_degree_window_host",
    "parba_degseq_prefix", "parba_degseq_rank", "parba_rank1", "parba_node_of_edges", "parba_count_pairs",
    "parba_multi_run", "parba_multi_run_shards", "parba_crc32c", "parba_mulhi_u64", "parba_degseq_dense",
    "parba_peak_int32", "parba_peak_write", "parba_debug_mod", "parba_debug_mod_check", "parba_debug_rcp_bound",
    "parba_bb_fill", "parba_degree_full_routed_ok", "parba_degree_full_routed", "parba_ipc_alloc", "parba_ipc_open",
    "parba_ipc_close", "parba_ipc_free", "parba_peer_atomics_ok",
)
MOD_FP31, MOD_FP_NARROW, MOD_FP_WIDE, MOD_INT, MOD_FP31_SERIES, MOD_FP_NARROW_SERIES, MOD_FP_WIDE_SERIES, \
    MOD_FP31_SERIES1, MOD_FP_WIDE_SERIES1, MOD_FP32, MOD_FP32_SERIES = range(11)
MULTI_STORE, MULTI_WINDOW, MULTI_FULL, MULTI_DISCARD = 0, 1, 2, 3


class CParams(ctypes.Structure):
    """parba_params_t."""

    _fields_ = [
        ("n", ctypes.c_uint64),
        ("d", ctypes.c_uint64),
        ("n0", ctypes.c_uint64),
        ("m0", ctypes.c_uint64),
        ("m", ctypes.c_uint64),
        ("hash_kind", ctypes.c_uint32),
        ("crc_seed0", ctypes.c_uint32),
        ("crc_seed1", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("simple_mult", ctypes.c_uint64),
        ("seed_edges", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("reserved2", ctypes.c_uint32),
        ("max_attempts", ctypes.c_uint64),
        ("base_seed0", ctypes.c_uint32),
        ("base_seed1", ctypes.c_uint32),
        ("base_mult", ctypes.c_uint64),
        ("degree_prefix", ctypes.c_void_p),
        ("rank", ctypes.c_void_p),
        ("owners", ctypes.c_void_p),
        ("dense_owner", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library; raise loudly when it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise GenerationError(
                f"CUDA library {path} is missing; build it with "
                "`python -m paper_1602_07106_b200.build` (there is no CPU fallback)"
            )
        L = ctypes.CDLL(path)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        P = ctypes.POINTER(CParams)
        sig = {
            "parba_version": ([], i32),
            "parba_last_error": ([], ctypes.c_char_p),
            "parba_device_count": ([], i32),
            "parba_hash": ([P, vp, u64, vp, vp], i32),
            "parba_resolve_chains": ([P, vp, u64, u64, vp, vp, vp], i32),
            "parba_generate": ([P, u64, u64, vp, vp, vp], i32),
            "parba_generate_targets": ([P, u64, u64, vp, vp, vp], i32),
            "parba_edges_at": ([P, vp, u64, vp, vp, vp], i32),
            "parba_degree_window": ([P, u64, u64, u64, vp, vp, vp], i32),
            "parba_degree_full": ([P, u64, u64, vp, vp, vp], i32),
            "parba_count_ids": ([vp, u64, u64, vp, vp], i32),
            "parba_generate_host": ([P, u64, u64, vp, vp, i32], i32),
            "parba_write_binary": ([P, u64, u64, i32, u64, vp, i32], i32),
            "parba_degree_window_host": ([P, u64, u64, u64, vp, vp, i32], i32),
            "parba_degseq_prefix": ([vp, u64, u64, vp, vp], i32),
            "parba_degseq_rank": ([vp, u64, u64, u64, vp, vp, ctypes.POINTER(u64), vp], i32),
            "parba_rank1": ([vp, vp, u64, vp, vp], i32),
            "parba_node_of_edges": ([P, vp, u64, vp, ctypes.c_uint32, vp], i32),
            "parba_count_pairs": ([vp, u64, u64, vp, vp], i32),
            "parba_crc32c": ([ctypes.c_uint32, vp, u64, vp, vp], i32),
            "parba_mulhi_u64": ([vp, vp, u64, vp, vp], i32),
            "parba_degseq_dense": ([vp, u64, u64, u64, vp, vp], i32),
            "parba_multi_run": ([P, i32, vp, i32, u64, vp, ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double)],
                                i32),
            "parba_bb_fill": ([P, vp, vp, vp, ctypes.POINTER(i32), vp], i32),
            "parba_debug_mod": ([i32, vp, vp, vp, u64, vp, vp], i32),
            "parba_debug_mod_check": ([i32, u64, u64, u64, u64, vp, vp, vp], i32),
            "parba_debug_rcp_bound": ([i32, i32, vp, vp], i32),
            "parba_peak_int32": ([vp, ctypes.POINTER(ctypes.c_double), vp], i32),
            "parba_peak_write": ([vp, u64, vp], i32),
            "parba_multi_run_shards": ([P, i32, vp, vp, vp, i32, u64, vp, vp, ctypes.POINTER(ctypes.c_double)], i32),
            "parba_degree_full_routed_ok": ([P, u64, u64], i32),
            "parba_degree_full_routed": ([P, u64, u64, i32, vp, u64, vp, vp], i32),
            "parba_ipc_alloc": ([u64, ctypes.POINTER(vp), vp], i32),
            "parba_ipc_open": ([vp, ctypes.POINTER(vp)], i32),
            "parba_ipc_close": ([vp], i32),
            "parba_ipc_free": ([vp], i32),
            "parba_peer_atomics_ok": ([i32, i32], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name, None)
            if fn is None:  # older builds (tools/ab.py A/B); tests check every export
                continue
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def check(rc: int) -> None:
    if rc == PARBA_OK:
        return
    msg = load().parba_last_error().decode(errors="replace")
    if rc == PARBA_EINVAL:
        raise ParameterError(msg)
    if rc == PARBA_EINFEASIBLE:
        from .errors import InfeasibleTargetsError

        raise InfeasibleTargetsError(msg)
    raise GenerationError(msg)


def torch_cuda():
    """torch with a usable CUDA device, else GenerationError (no CPU path)."""
    import torch

    if not torch.cuda.is_available():
        raise GenerationError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def stream_ptr(torch, device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_device_u64(torch, arr, device) -> "torch.Tensor":
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return torch.from_numpy(a.view(np.int64)).to(device)
