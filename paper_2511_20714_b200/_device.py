"""Device-side helpers shared by the façades: stream handle, tensor coercion, launchers.

PyTorch is plumbing here (device memory, streams, cuBLAS GEMMs); every hot-path
kernel is ours and is reached through `_abi` (include/ifx_abi.h).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _abi
from .errors import DimensionError

# Count of OUR kernels enqueued (K1/K2/K7/RMS/Ulysses); bench.py reports the delta over
# its timed region as `gpu_launches`.
LAUNCHES = [0]


def count_launch(n: int = 1) -> None:
    LAUNCHES[0] += n


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_20714_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = torch._C._cuda_getCurrentRawStream  # one C call (torch.cuda.current_stream()
# resolves the device index through Python on every call: ~10 us per launch measured)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    return _raw_stream(torch._C._cuda_getDevice())


def to_device(x, dtype=torch.float32) -> torch.Tensor:
    """numpy / list / tensor -> CUDA tensor of `dtype` (copy only if needed)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype)
    a = np.asarray(x, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def row_ld(t: torch.Tensor) -> int:
    """Row stride (elements) of a 2-D tensor whose rows are contiguous."""
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise DimensionError("expected a 2-D tensor with contiguous rows")
    return t.stride(0)


_WS: dict = {}


def _workspace(dev: torch.device, nbytes: int) -> torch.Tensor:
    """Grow-only per-device scratch for K1's split-KV partials (stream-ordered reuse)."""
    w = _WS.get(dev)
    if w is None or w.numel() < nbytes:
        w = _WS[dev] = torch.empty(max(nbytes, 1 << 20), device=dev, dtype=torch.uint8)
    return w


def attn_fwd(q: torch.Tensor, heads: int, head_dim: int, out: torch.Tensor,
             ctx_k: torch.Tensor | None = None, ctx_v: torch.Tensor | None = None,
             ctx_row0: int = 0, n_ctx: int = 0,
             cur_k: torch.Tensor | None = None, cur_v: torch.Tensor | None = None,
             scale: float | None = None, mask: torch.Tensor | None = None,
             row_max: torch.Tensor | None = None, row_sum: torch.Tensor | None = None,
             split_kv: bool = True, stream=None, ctx_slots: torch.Tensor | None = None,
             page_len: int = 0, first_token: int = 0, stage_k: torch.Tensor | None = None,
             stage_v: torch.Tensor | None = None, tile_runs: torch.Tensor | None = None,
             o_peers=None, o_rows: int = 0, o_row0: int = 0) -> torch.Tensor:
    """Enqueue K1 (attn_fwd_sm100.cu): out = softmax(q [ctx∥cur]^T * scale) [ctx∥cur].

    q/out: [n_q, heads*head_dim] bf16 (row-strided views allowed). cur_*: [n_cur,
    heads*head_dim] views. Context, contiguous: rows [ctx_row0, ctx_row0+n_ctx) of ctx_k/v.
    Paged (ctx_slots given): ctx_k/v are the KV pool, the context is tokens [ctx_row0,
    ctx_row0+n_ctx) whose pages from first_token on sit in slot codes ctx_slots (int32
    device tensor; codes < 0 address stage_k/v); tile_runs = tile_run_codes(codes, page_len).
    o_peers: O scatter over peer memory (the Ulysses head->sequence re-shard in K1's
    epilogue): output row r is sequence row g = o_row0 + r, written to row g % o_rows of
    the buffer at address o_peers[g // o_rows] (row stride = out's); `out` only supplies
    the row stride then.
    """
    p = _abi.AttnParams()
    p.q, p.q_ld, p.n_q = q.data_ptr(), row_ld(q), q.shape[0]
    if n_ctx > 0:
        p.k_ctx, p.v_ctx = ctx_k.data_ptr(), ctx_v.data_ptr()
        p.ctx_ld, p.ctx_rows = row_ld(ctx_k), ctx_k.shape[0]
        p.ctx_row0, p.n_ctx = ctx_row0, n_ctx
        if ctx_slots is not None:
            p.ctx_slots, p.ctx_page_len, p.ctx_first_token = ctx_slots.data_ptr(), page_len, first_token
            if tile_runs is not None:
                p.ctx_tile_runs = tile_runs.data_ptr()
            if stage_k is not None:
                p.k_stage, p.v_stage, p.stage_rows = stage_k.data_ptr(), stage_v.data_ptr(), stage_k.shape[0]
    if cur_k is not None and cur_k.shape[0] > 0:
        p.k_cur, p.v_cur = cur_k.data_ptr(), cur_v.data_ptr()
        p.cur_ld, p.n_cur = row_ld(cur_k), cur_k.shape[0]
    p.o, p.o_ld = out.data_ptr(), row_ld(out)
    if o_peers is not None:
        for i, a in enumerate(o_peers):
            p.o_peer[i] = a
        p.o_peer_rows, p.o_row0 = o_rows, o_row0
    p.heads, p.head_dim = heads, head_dim
    p.scale = (1.0 / math.sqrt(head_dim)) if scale is None else scale
    if mask is not None:
        p.mask, p.mask_ld = mask.data_ptr(), mask.stride(0)
    if row_max is not None:
        p.row_max, p.row_sum = row_max.data_ptr(), row_sum.data_ptr()
    L = _abi.lib()
    if split_kv and row_max is None:  # let the library split under-filled launches
        # = ifx_attn_workspace_bytes (8 splits), without the extra ctypes round trip
        need = 8 * p.n_q * heads * head_dim * 2 + 2 * 8 * heads * p.n_q * 4 + 256
        ws = _workspace(q.device, need)
        p.workspace, p.workspace_bytes = ws.data_ptr(), ws.numel()
    rc = L.ifx_attn_fwd(ctypes.byref(p), stream_ptr(stream))
    _abi.check(rc, "attn_fwd")
    LAUNCHES[0] += 1
    return out


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, beta: float = 0.0,
         relu: bool = False, stream=None) -> torch.Tensor:
    """out = relu?(a @ b + beta * out) on cuBLASLt through ifx_gemm_bf16: bf16 a [M, K] and
    b [K, N] (rows contiguous), fp32 accumulate, out fp32 or bf16 [M, N]."""
    M, K = a.shape
    N = b.shape[1]
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or b.shape[0] != K or \
            tuple(out.shape) != (M, N):
        raise DimensionError("gemm expects bf16 a [M, K], b [K, N] and out [M, N]")
    _abi.check(_abi.lib().ifx_gemm_bf16(a.data_ptr(), row_ld(a), b.data_ptr(), row_ld(b),
                                        out.data_ptr(), row_ld(out), dtype_code(out.dtype), M, N,
                                        K, float(beta), int(relu), stream_ptr(stream)), "gemm")
    return out


RMS_EPS = 1e-6  # engine.py:26


class RowNorm:
    """RMS statistics a G1 producer leaves for its consumer: the bf16 copy of the fp32 rows
    (the consumer's A) and per-column-tile sums of squares [rows, parts] (its row scale)."""

    __slots__ = ("rows_bf16", "ss", "parts", "dim")

    def __init__(self, rows_bf16: torch.Tensor, ss: torch.Tensor, parts: int, dim: int):
        self.rows_bf16, self.ss, self.parts, self.dim = rows_bf16, ss, parts, dim


def gemm_tiles_n(m: int, n: int, k: int) -> int:
    """Sum-of-squares parts per row G1 emits for an [m, k] x [k, n] product."""
    out = ctypes.c_int64()
    _abi.check(_abi.lib().ifx_gemm_tiles_n(m, n, k, ctypes.byref(out)), "gemm_tiles_n")
    return out.value


_G1_ARGS: dict = {}  # gemm_fused argument blocks by call signature (pointers, shapes)


def gemm_fused(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None, beta: float = 0.0,
               relu: bool = False, norm_in: RowNorm | None = None, norm_out: RowNorm | None = None,
               rope=None, page=None, scatter=None, stream=None) -> int:
    """G1 (gemm_sm100.cu): out = f(a @ b) on tcgen05, bf16 a [M, K] / b [K, N], fp32
    accumulate; out bf16, or fp32 with out = beta * out + f(.).

    norm_in:  a holds bf16 copies of fp32 rows whose RMS statistics are norm_in.ss: the
              product is scaled by rsqrt(mean(row^2) + 1e-6) (engine.py:171-173).
    norm_out: (fp32 out) also write the new rows as bf16 to norm_out.rows_bf16 and their
              per-tile sums of squares to norm_out.ss (norm_out.parts is set).
    rope:     (cos, sin, row0, pairs, head_stride, heads, q_col0, k_col0) 3D RoPE tables.
    page:     (pool abi, slots tensor, first_token, token0, k_col0, v_col0) page write.
    scatter:  (table, block_width): bf16 output column blocks stored into peers' buffers
              (device int64 table [blocks, 2, 4], ifx_gemm_params.scatter); out may be None.
    Returns the column tile count (norm_out.parts).

    The argument block of a call without a page write is cached on its pointers and shapes:
    the engine repeats the same calls on the same buffers every pass, and re-filling the
    ctypes struct was most of the host cost of a launch."""
    key = None
    if page is None:
        key = (a.data_ptr(), a.shape, a.stride(0), b.data_ptr(), b.shape, b.stride(0),
               None if out is None else (out.data_ptr(), out.shape, out.stride(0), out.dtype),
               beta, relu,
               None if norm_in is None else (norm_in.ss.data_ptr(), norm_in.parts, norm_in.dim),
               None if norm_out is None else (norm_out.rows_bf16.data_ptr(), norm_out.ss.data_ptr()),
               None if rope is None else (rope[0].data_ptr(), rope[1].data_ptr(), *rope[2:]),
               None if scatter is None else (scatter[0].data_ptr(), scatter[1]))
        hit = _G1_ARGS.get(key)
        if hit is not None:
            pref, tn, tref = hit
            _abi.check(_abi.lib().ifx_gemm_fused(pref, tref, stream_ptr(stream)), "gemm_fused")
            LAUNCHES[0] += 1
            if norm_out is not None:
                norm_out.parts, norm_out.dim = tn.value, b.shape[1]
            return tn.value
    M, K = a.shape
    N = b.shape[1]
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or b.shape[0] != K or \
            (out is not None and tuple(out.shape) != (M, N)) or (out is None and scatter is None):
        raise DimensionError("gemm expects bf16 a [M, K], b [K, N] and out [M, N]")
    p = _abi.GemmParams()
    p.a, p.lda, p.b, p.ldb = a.data_ptr(), row_ld(a), b.data_ptr(), row_ld(b)
    if out is not None:
        p.c, p.ldc, p.c_type = out.data_ptr(), row_ld(out), dtype_code(out.dtype)
    else:
        p.c, p.ldc, p.c_type = None, N, dtype_code(torch.bfloat16)
    if scatter is not None:
        table, width = scatter
        p.scatter, p.scatter_w, p.scatter_blocks = table.data_ptr(), width, table.shape[0]
    p.m, p.n, p.k, p.beta, p.relu = M, N, K, float(beta), int(relu)
    if norm_in is not None:
        p.rs_part, p.rs_ld, p.rs_parts = norm_in.ss.data_ptr(), norm_in.ss.stride(0), norm_in.parts
        p.rs_dim, p.rs_eps = norm_in.dim, RMS_EPS
    if norm_out is not None:
        p.emit_b, p.emit_ld = norm_out.rows_bf16.data_ptr(), row_ld(norm_out.rows_bf16)
        p.emit_ss, p.emit_ss_ld = norm_out.ss.data_ptr(), norm_out.ss.stride(0)
    if rope is not None:
        cos, sin, row0, pairs, hs, heads, q0, k0 = rope
        p.rope_cos, p.rope_sin, p.rope_row0 = cos.data_ptr(), sin.data_ptr(), row0
        p.rope_pairs, p.rope_hs, p.rope_heads, p.rope_q0, p.rope_k0 = pairs, hs, heads, q0, k0
    keep = None
    if page is not None:
        pool, slots, first, token0, kc0, vc0 = page
        keep = pool
        p.page_pool = ctypes.addressof(pool)
        p.page_slots, p.page_first_token, p.page_token0 = slots.data_ptr(), first, token0
        p.page_k_col0, p.page_v_col0 = kc0, vc0
    tn = ctypes.c_int64()
    _abi.check(_abi.lib().ifx_gemm_fused(ctypes.byref(p), ctypes.byref(tn), stream_ptr(stream)),
               "gemm_fused")
    del keep
    LAUNCHES[0] += 1
    if key is not None:
        if len(_G1_ARGS) > 4096:
            _G1_ARGS.clear()
        _G1_ARGS[key] = (ctypes.byref(p), tn, ctypes.byref(tn))  # byref keeps p alive
    if norm_out is not None:
        norm_out.parts, norm_out.dim = tn.value, N
    return tn.value


def tile_run_codes(codes: np.ndarray, page_len: int) -> np.ndarray:
    """Per 128-key tile of a paged context (K1's ctx_tile_runs): the first page's slot code
    when the tile's pages are one consecutive run of one pool, else INT32_MIN. The last
    tile counts as a run only if it has all its pages (K1 then reads finite rows past the
    context end and masks them)."""
    ppt = 128 // page_len
    n = len(codes)
    n_tiles = -(-n // ppt)
    pad = np.full(n_tiles * ppt, np.iinfo(np.int32).min, dtype=np.int64)
    pad[:n] = codes
    t = pad.reshape(n_tiles, ppt)
    step = np.where(t[:, :1] >= 0, 1, -1)
    run = (t == t[:, :1] + step * np.arange(ppt)[None, :]).all(axis=1) & (t[:, -1] != np.iinfo(np.int32).min)
    return np.where(run, t[:, 0], np.iinfo(np.int32).min).astype(np.int32)


def rms_bf16(x: torch.Tensor, out: torch.Tensor, tvec: torch.Tensor | None = None,
             t: float = 0.0, x_out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Enqueue the fused RMS-norm (engine.py:171-173): out = bf16(rms(x + t*tvec))."""
    rows, width = x.shape
    _abi.check(_abi.lib().ifx_rms_bf16(x.data_ptr(), rows, width, ptr(tvec), float(t),
                                       ptr(x_out), out.data_ptr(), stream_ptr(stream)), "rms")
    LAUNCHES[0] += 1
    return out


def rope_qk(qkv: torch.Tensor, heads: int, head_stride: int, pairs: int, q_col0: int, k_col0: int,
            cos: torch.Tensor, sin: torch.Tensor, tab_row0: int = 0, stream=None) -> torch.Tensor:
    """Enqueue the in-place 3D RoPE of the Q and K column blocks of a bf16 QKV buffer."""
    _abi.check(_abi.lib().ifx_rope_qk(qkv.data_ptr(), qkv.shape[0], row_ld(qkv), heads,
                                      head_stride, pairs, q_col0, k_col0, cos.data_ptr(),
                                      sin.data_ptr(), tab_row0, stream_ptr(stream)), "rope")
    LAUNCHES[0] += 1
    return qkv


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _abi.F32
    if dt == torch.bfloat16:
        return _abi.BF16
    raise DimensionError(f"unsupported dtype {dt}")
