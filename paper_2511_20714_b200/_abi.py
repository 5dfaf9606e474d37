"""ctypes binding of libinferix_b200.so (include/ifx_abi.h).

The library is built in-tree by `paper_2511_20714_b200._build` (or
`__graft_entry__.build()`); there is no fallback: if it is missing, importing the
hot-path modules raises. Status codes are mapped onto the reference exception
classes (errors.py:4-33).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    CapacityError,
    ConfigError,
    CudaError,
    DimensionError,
    InferixError,
    MaskError,
    OutOfRangeError,
)

LIB_PATH = os.environ.get("IFX_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libinferix_b200.so")  # override: A/B builds

OK, EDIM, EMASK, ECAPACITY, ERANGE, ECONFIG, ECUDA, EUNSUPPORTED, ENCCL = 0, 1, 2, 3, 4, 5, 16, 17, 18
SELF_ATTN, CROSS_ATTN = 0, 1
F32, BF16 = 0, 1

_ERRORS = {EDIM: DimensionError, EMASK: MaskError, ECAPACITY: CapacityError,
           ERANGE: OutOfRangeError, ECONFIG: ConfigError, ECUDA: CudaError,
           EUNSUPPORTED: DimensionError, ENCCL: CudaError}

# every symbol include/ifx_abi.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "ifx_last_error", "ifx_version",
    "ifx_pt_create", "ifx_pt_destroy", "ifx_pt_append", "ifx_pt_offload", "ifx_pt_evict_window",
    "ifx_pt_clear_cross", "ifx_pt_touch_range", "ifx_pt_touch_indices", "ifx_pt_range",
    "ifx_pt_stats", "ifx_pt_snapshot", "ifx_pt_drain_moves", "ifx_pt_pool_extent", "ifx_pt_slots",
    "ifx_pt_batch_begin", "ifx_pt_batch_end", "ifx_pt_pending",
    "ifx_kv_append", "ifx_kv_gather", "ifx_kv_append_latent", "ifx_kv_gather_latent", "ifx_kv_move_pages", "ifx_kv_copy_runs", "ifx_host_alloc", "ifx_host_free",
    "ifx_dev_alloc", "ifx_dev_free",
    "ifx_attn_fwd", "ifx_attn_workspace_bytes", "ifx_attn_combine",
    "ifx_rms_bf16", "ifx_rope_qk", "ifx_group_softmax", "ifx_group_softmax_rs", "ifx_ulysses_pack", "ifx_ulysses_unpack",
    "ifx_copy_blocks", "ifx_gemm_bf16", "ifx_gemm_fused", "ifx_gemm_tiles_n",
    "ifx_noise_normal_f32",
    "ifx_ipc_handle", "ifx_ipc_open", "ifx_ipc_close", "ifx_memcpy2d", "ifx_peer_barrier",
    "ifx_comm_unique_id", "ifx_comm_init", "ifx_comm_destroy", "ifx_comm_size",
    "ifx_comm_all_to_all", "ifx_comm_all_gather",
)


class KvPool(ctypes.Structure):
    """Mirror of `ifx_kv_pool` (include/ifx_abi.h)."""

    _fields_ = [
        ("dev_k", ctypes.c_void_p), ("dev_v", ctypes.c_void_p),
        ("host_k", ctypes.c_void_p), ("host_v", ctypes.c_void_p),
        ("width", ctypes.c_int64), ("page_len", ctypes.c_int64), ("type", ctypes.c_int),
    ]


class AttnParams(ctypes.Structure):
    """Mirror of `ifx_attn_params` (include/ifx_abi.h)."""

    _fields_ = [
        ("q", ctypes.c_void_p), ("q_ld", ctypes.c_int64), ("n_q", ctypes.c_int64),
        ("k_ctx", ctypes.c_void_p), ("v_ctx", ctypes.c_void_p), ("ctx_ld", ctypes.c_int64),
        ("ctx_rows", ctypes.c_int64), ("ctx_row0", ctypes.c_int64), ("n_ctx", ctypes.c_int64),
        ("k_cur", ctypes.c_void_p), ("v_cur", ctypes.c_void_p), ("cur_ld", ctypes.c_int64),
        ("n_cur", ctypes.c_int64),
        ("o", ctypes.c_void_p), ("o_ld", ctypes.c_int64),
        ("heads", ctypes.c_int64), ("head_dim", ctypes.c_int64), ("scale", ctypes.c_float),
        ("mask", ctypes.c_void_p), ("mask_ld", ctypes.c_int64),
        ("row_max", ctypes.c_void_p), ("row_sum", ctypes.c_void_p),
        ("ctx_slots", ctypes.c_void_p), ("ctx_page_len", ctypes.c_int64),
        ("ctx_first_token", ctypes.c_int64),
        ("k_stage", ctypes.c_void_p), ("v_stage", ctypes.c_void_p), ("stage_rows", ctypes.c_int64),
        ("ctx_tile_runs", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_int64),
        ("o_peer", ctypes.c_void_p * 8), ("o_peer_rows", ctypes.c_int64), ("o_row0", ctypes.c_int64),
    ]


class GemmParams(ctypes.Structure):
    """Mirror of `ifx_gemm_params` (include/ifx_abi.h)."""

    _fields_ = [
        ("a", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("b", ctypes.c_void_p), ("ldb", ctypes.c_int64),
        ("c", ctypes.c_void_p), ("ldc", ctypes.c_int64), ("c_type", ctypes.c_int),
        ("relu", ctypes.c_int),
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
        ("beta", ctypes.c_float), ("rs_eps", ctypes.c_float),
        ("rs_part", ctypes.c_void_p), ("rs_ld", ctypes.c_int64), ("rs_parts", ctypes.c_int64),
        ("rs_dim", ctypes.c_int64),
        ("emit_b", ctypes.c_void_p), ("emit_ld", ctypes.c_int64),
        ("emit_ss", ctypes.c_void_p), ("emit_ss_ld", ctypes.c_int64),
        ("rope_cos", ctypes.c_void_p), ("rope_sin", ctypes.c_void_p),
        ("rope_row0", ctypes.c_int64), ("rope_q0", ctypes.c_int64), ("rope_k0", ctypes.c_int64),
        ("rope_pairs", ctypes.c_int64), ("rope_hs", ctypes.c_int64), ("rope_heads", ctypes.c_int64),
        ("page_pool", ctypes.c_void_p), ("page_slots", ctypes.c_void_p),
        ("page_first_token", ctypes.c_int64), ("page_token0", ctypes.c_int64),
        ("page_k_col0", ctypes.c_int64), ("page_v_col0", ctypes.c_int64),
        ("scatter", ctypes.c_void_p), ("scatter_w", ctypes.c_int64), ("scatter_blocks", ctypes.c_int64),
    ]


_lib = None
_lock = threading.Lock()
I64 = ctypes.c_int64
P = ctypes.c_void_p
PI64 = ctypes.POINTER(ctypes.c_int64)


def lib() -> ctypes.CDLL:
    """Load the native library once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            import torch  # noqa: F401  (torch's CUDA libraries first: one cuBLASLt per process)
            L = ctypes.CDLL(LIB_PATH)
            L.ifx_last_error.restype = ctypes.c_char_p
            L.ifx_pt_create.argtypes = [I64, I64, I64, I64, I64, ctypes.POINTER(P)]
            L.ifx_pt_destroy.argtypes = [P]
            L.ifx_pt_destroy.restype = None
            L.ifx_pt_append.argtypes = [P, I64, ctypes.c_int, I64, I64, PI64, PI64, PI64, PI64, I64, PI64]
            L.ifx_pt_offload.argtypes = [P, PI64, I64, PI64]
            L.ifx_pt_evict_window.argtypes = [P, I64, PI64]
            L.ifx_pt_clear_cross.argtypes = [P, PI64]
            L.ifx_pt_touch_range.argtypes = [P, I64, ctypes.c_int, I64, I64]
            L.ifx_pt_touch_indices.argtypes = [P, I64, ctypes.c_int, PI64, I64]
            L.ifx_pt_range.argtypes = [P, I64, ctypes.c_int, PI64, PI64]
            L.ifx_pt_stats.argtypes = [P, PI64, I64]
            L.ifx_pt_snapshot.argtypes = [P, PI64, I64, PI64]
            L.ifx_pt_drain_moves.argtypes = [P, PI64, I64, PI64]
            L.ifx_pt_batch_begin.argtypes = [P]
            L.ifx_pt_batch_end.argtypes = [P]
            L.ifx_pt_pending.argtypes = [P, I64, PI64]
            L.ifx_pt_pool_extent.argtypes = [P, PI64]
            L.ifx_pt_slots.argtypes = [P, I64, ctypes.c_int, I64, I64, P, I64, PI64, PI64]
            PPOOL = ctypes.POINTER(KvPool)
            L.ifx_kv_append.argtypes = [P, P, I64, ctypes.c_int, PPOOL, P, I64, I64, I64, P]
            L.ifx_kv_gather.argtypes = [PPOOL, P, I64, P, I64, I64, P, P, P]
            L.ifx_kv_append_latent.argtypes = [P, P, I64, ctypes.c_int, I64, P, I64, PPOOL, P, I64,
                                               I64, I64, P]
            L.ifx_kv_gather_latent.argtypes = [PPOOL, P, I64, P, I64, I64, I64, P, I64, P, P, I64,
                                               ctypes.c_int, P]
            L.ifx_kv_move_pages.argtypes = [PPOOL, P, I64, ctypes.c_int, P]
            L.ifx_kv_copy_runs.argtypes = [PPOOL, PI64, I64, ctypes.c_int, P]
            L.ifx_host_alloc.argtypes = [I64, ctypes.POINTER(P)]
            L.ifx_host_free.argtypes = [P]
            L.ifx_dev_alloc.argtypes = [I64, ctypes.POINTER(P)]
            L.ifx_dev_free.argtypes = [P]
            L.ifx_attn_fwd.argtypes = [ctypes.POINTER(AttnParams), P]
            L.ifx_attn_workspace_bytes.argtypes = [ctypes.POINTER(AttnParams), PI64]
            L.ifx_rms_bf16.argtypes = [P, I64, I64, P, ctypes.c_float, P, P, P]
            L.ifx_copy_blocks.argtypes = [P, P, P, I64, I64, P]
            L.ifx_gemm_bf16.argtypes = [P, I64, P, I64, P, I64, ctypes.c_int, I64, I64, I64,
                                        ctypes.c_float, ctypes.c_int, P]
            L.ifx_gemm_fused.argtypes = [ctypes.POINTER(GemmParams), PI64, P]
            L.ifx_gemm_tiles_n.argtypes = [I64, I64, I64, PI64]
            L.ifx_group_softmax.argtypes = [P, I64, I64, I64, I64, ctypes.c_float, P, I64, P]
            L.ifx_group_softmax_rs.argtypes = [P, I64, I64, I64, I64, ctypes.c_float, P, I64, P,
                                               I64, I64, I64, P]
            L.ifx_rope_qk.argtypes = [P, I64, I64, I64, I64, I64, I64, I64, P, P, I64, P]
            L.ifx_ulysses_pack.argtypes = [P, I64, I64, I64, I64, I64, ctypes.c_int, P, P]
            L.ifx_ulysses_unpack.argtypes = [P, I64, I64, I64, I64, ctypes.c_int, P, I64, P]
            L.ifx_ipc_handle.argtypes = [P, P]
            L.ifx_ipc_open.argtypes = [P, ctypes.POINTER(P)]
            L.ifx_ipc_close.argtypes = [P]
            L.ifx_memcpy2d.argtypes = [P, I64, P, I64, I64, I64, P]
            L.ifx_attn_combine.argtypes = [P, I64, P, P, I64, I64, I64, I64, P, I64, P, P, P]
            L.ifx_peer_barrier.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, P,
                                           ctypes.c_int, P]
            L.ifx_comm_unique_id.argtypes = [P]
            L.ifx_comm_init.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
            L.ifx_comm_destroy.argtypes = [P]
            L.ifx_comm_size.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
            L.ifx_comm_all_to_all.argtypes = [P, P, PI64, PI64, P, PI64, PI64, P]
            L.ifx_comm_all_gather.argtypes = [P, P, I64, P, P]
            L.ifx_noise_normal_f32.argtypes = [ctypes.POINTER(ctypes.c_uint64), I64, P, ctypes.c_int]
            _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = lib().ifx_last_error().decode(errors="replace")
    cls = _ERRORS.get(rc, InferixError)
    raise cls(f"{what}: {msg}" if what else msg)
