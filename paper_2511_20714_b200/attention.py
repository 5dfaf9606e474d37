"""Attention primitives — drop-in for `inferix.attention` on B200.

Reference: /root/reference/pkg/src/inferix/attention.py. Same names and error behaviour
(DimensionError for bad shapes / non-finite input, MaskError for a fully masked row or a
zero denominator), but the math runs in the K1 tcgen05 kernel (bf16 operands, fp32
softmax and accumulation) on CUDA tensors. Tolerance vs the fp32 reference is stated in
DESIGN.md §Parity (max-abs 2e-2 on unit-scale inputs).

Head widths that are not 64/128 are zero-padded to the next supported width (zeros do
not change q.k, and padded V columns are sliced off); the scale stays 1/sqrt(d).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ._device import attn_fwd, require_cuda, to_device
from .errors import DimensionError, MaskError

NEG_INF = float("-inf")


def block_causal_mask(num_blocks: int, block_len: int) -> torch.Tensor:
    """attention.py:27-35 — token i (block b_i) may attend j iff b_j <= b_i."""
    if num_blocks < 1 or block_len < 1:
        raise DimensionError("num_blocks and block_len must be >= 1")
    blk = torch.arange(num_blocks * block_len, device=require_cuda()) // block_len
    return blk[None, :] <= blk[:, None]


def windowed_block_causal_mask(num_blocks: int, block_len: int, window_tokens) -> torch.Tensor:
    """attention.py:38-58 — additionally j >= b_i*block_len - window_tokens."""
    mask = block_causal_mask(num_blocks, block_len)
    if window_tokens is None:
        return mask
    if window_tokens < 0:
        raise DimensionError("window_tokens must be >= 0")
    n = num_blocks * block_len
    idx = torch.arange(n, device=mask.device)
    lo = (idx // block_len) * block_len - window_tokens
    return mask & (idx[None, :] >= lo[:, None])


def _finite(x, name: str) -> torch.Tensor:
    t = to_device(x, torch.float32)
    if not bool(torch.isfinite(t).all()):
        raise DimensionError(f"{name} contains non-finite values")
    return t


def _check(q, k, v, mask):
    """attention.py:61-71."""
    if q.dim() != 2 or k.dim() != 2 or v.dim() != 2:
        raise DimensionError("q, k, v must be rank-2 [tokens, dim]")
    if q.shape[1] != k.shape[1]:
        raise DimensionError(f"q dim {q.shape[1]} != k dim {k.shape[1]}")
    if k.shape[0] != v.shape[0]:
        raise DimensionError(f"k rows {k.shape[0]} != v rows {v.shape[0]}")
    if tuple(mask.shape) != (q.shape[0], k.shape[0]):
        raise DimensionError(f"mask shape {tuple(mask.shape)} != ({q.shape[0]}, {k.shape[0]})")


def _padded(x: torch.Tensor, width: int) -> torch.Tensor:
    out = torch.zeros(x.shape[0], width, device=x.device, dtype=torch.bfloat16)
    out[:, :x.shape[1]] = x
    return out


def _run(q, k, v, mask, want_stats: bool):
    """One K1 launch, single head, any d <= 128 (padded), optional dense mask."""
    n, d = q.shape
    dv = v.shape[1]
    width = 64 if max(d, dv) <= 64 else 128
    if max(d, dv) > 128:
        raise DimensionError("head width > 128 is not supported by the B200 kernel")
    qp, kp, vp = _padded(q, width), _padded(k, width), _padded(v, width)
    out = torch.empty(n, width, device=q.device, dtype=torch.bfloat16)
    m8 = None
    if mask is not None and not bool(mask.all()):
        m8 = mask.to(torch.uint8).contiguous()
    rm = rs = None
    if want_stats:
        rm = torch.empty(n, device=q.device, dtype=torch.float32)
        rs = torch.empty(n, device=q.device, dtype=torch.float32)
    attn_fwd(qp, 1, width, out, kp, vp, 0, k.shape[0], scale=1.0 / math.sqrt(d), mask=m8,
             row_max=rm, row_sum=rs)
    return out[:, :dv].float(), rm, rs


def scaled_dot_attention(q, k, v, mask) -> torch.Tensor:
    """attention.py:74-94 — softmax(q k^T / sqrt(d)) v over the allowed entries of mask."""
    q, k, v = _finite(q, "q"), _finite(k, "k"), _finite(v, "v")
    mask = torch.as_tensor(np.asarray(mask, dtype=bool) if not isinstance(mask, torch.Tensor)
                           else mask, device=q.device).bool()
    _check(q, k, v, mask)
    if not bool(mask.any(dim=1).all()):
        raise MaskError("query row with no allowed key")
    return _run(q, k, v, mask, False)[0]


@dataclass
class AttentionPartial:
    """attention.py:97-116 — acc = sum exp(logit - row_max) v, row_max, denom."""
    acc: torch.Tensor
    row_max: torch.Tensor
    denom: torch.Tensor

    @property
    def num_queries(self) -> int:
        return self.acc.shape[0]

    @property
    def head_dim(self) -> int:
        return self.acc.shape[1]


def empty_partial(num_queries: int, head_dim: int) -> AttentionPartial:
    """attention.py:119-125."""
    dev = require_cuda()
    return AttentionPartial(torch.zeros(num_queries, head_dim, device=dev),
                            torch.full((num_queries,), NEG_INF, device=dev),
                            torch.zeros(num_queries, device=dev))


def attention_partial(q, k_shard, v_shard, mask_shard) -> AttentionPartial:
    """attention.py:127-154 — partial over one key shard; dead rows keep (-inf, 0, 0).

    K1 returns the normalised output plus (max, denominator) in the log2 domain; the
    reference convention (natural-log max, acc = out * denom) is rebuilt here."""
    q, k, v = _finite(q, "q"), _finite(k_shard, "k"), _finite(v_shard, "v")
    mask = torch.as_tensor(mask_shard, device=q.device).bool()
    _check(q, k, v, mask)
    if k.shape[0] == 0:
        return empty_partial(q.shape[0], v.shape[1])
    out, m2, l = _run(q, k, v, mask, True)
    dead = l <= 0
    row_max = torch.where(dead, torch.full_like(m2, NEG_INF), m2 * math.log(2.0))
    denom = torch.where(dead, torch.zeros_like(l), l)
    acc = torch.where(dead[:, None], torch.zeros_like(out), out * denom[:, None])
    return AttentionPartial(acc, row_max, denom)


def merge_partials(a: AttentionPartial, b: AttentionPartial) -> AttentionPartial:
    """attention.py:157-173 — associative, commutative online-softmax merge."""
    if tuple(a.acc.shape) != tuple(b.acc.shape):
        raise DimensionError(f"partial shapes differ: {tuple(a.acc.shape)} vs {tuple(b.acc.shape)}")
    new_max = torch.maximum(a.row_max, b.row_max)
    safe = torch.where(torch.isfinite(new_max), new_max, torch.zeros_like(new_max))

    def factor(p):
        f = torch.exp(p.row_max - safe)
        return torch.where(torch.isfinite(p.row_max), f, torch.zeros_like(f))

    fa, fb = factor(a), factor(b)
    return AttentionPartial(a.acc * fa[:, None] + b.acc * fb[:, None], new_max,
                            a.denom * fa + b.denom * fb)


def finalize_partial(p: AttentionPartial) -> torch.Tensor:
    """attention.py:176-180."""
    if not bool((p.denom > 0).all()):
        raise MaskError("finalize with zero denominator (query saw no keys)")
    return p.acc / p.denom[:, None]


def multi_head_attention(q: torch.Tensor, heads: int, out: torch.Tensor | None = None,
                         ctx_k=None, ctx_v=None, ctx_row0: int = 0, n_ctx: int = 0,
                         cur_k=None, cur_v=None) -> torch.Tensor:
    """The `_mha` hook (engine.py:176-182) on device: all heads, keys = [ctx rows ∥ cur].

    q / cur_k / cur_v: [n, heads*dh] bf16 row-strided views (e.g. slices of a fused QKV
    projection); ctx_*: KV-cache slabs read in place from row ctx_row0."""
    d = q.shape[1]
    dh = d // heads
    if out is None:
        out = torch.empty(q.shape[0], d, device=q.device, dtype=torch.bfloat16)
    return attn_fwd(q, heads, dh, out, ctx_k, ctx_v, ctx_row0, n_ctx, cur_k, cur_v)
