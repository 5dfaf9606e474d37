"""Oracle: single-head fp32 softmax attention and online-softmax partials.

Test infrastructure only (see oracle/__init__.py). Restates
`/root/reference/pkg/src/inferix/attention.py`.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from .errors import DimensionError, MaskError

_F32 = np.float32
_NEG_INF = _F32(-np.inf)


def _finite_f32(a) -> np.ndarray:
    """attention.py:20-24 — cast to fp32, reject NaN/Inf."""
    out = np.asarray(a, dtype=_F32)
    if not np.isfinite(out).all():
        raise DimensionError("non-finite input")
    return out


def _shape_check(q, k, v, mask):
    """attention.py:61-71 — rank-2 operands, matching widths/rows, mask [n, m]."""
    if min(q.ndim, k.ndim, v.ndim) != 2 or max(q.ndim, k.ndim, v.ndim) != 2:
        raise DimensionError("operands must be [tokens, dim]")
    if k.shape[1] != q.shape[1]:
        raise DimensionError("q/k width mismatch")
    if v.shape[0] != k.shape[0]:
        raise DimensionError("k/v row mismatch")
    if mask.shape != (q.shape[0], k.shape[0]):
        raise DimensionError("mask shape mismatch")


def block_causal_mask(num_blocks: int, block_len: int) -> np.ndarray:
    """attention.py:27-35 — token i sees token j iff block(j) <= block(i)."""
    if num_blocks < 1 or block_len < 1:
        raise DimensionError("num_blocks and block_len must be >= 1")
    b = np.repeat(np.arange(num_blocks), block_len)
    return b[:, None] >= b[None, :]


def windowed_block_causal_mask(num_blocks: int, block_len: int, window_tokens):
    """attention.py:38-58 — additionally j >= block(i)*block_len - window."""
    vis = block_causal_mask(num_blocks, block_len)
    if window_tokens is None:
        return vis
    if window_tokens < 0:
        raise DimensionError("window_tokens must be >= 0")
    n = num_blocks * block_len
    first_visible = (np.arange(n) // block_len) * block_len - window_tokens
    return vis & (np.arange(n)[None, :] >= first_visible[:, None])


def _scale(d: int):
    # attention.py:87 — 1/sqrt(d) computed in fp32
    return _F32(1.0) / _F32(np.sqrt(_F32(d)))


def scaled_dot_attention(q, k, v, mask) -> np.ndarray:
    """attention.py:74-94 — max-subtracted masked softmax(q k^T / sqrt(d)) v."""
    q, k, v = _finite_f32(q), _finite_f32(k), _finite_f32(v)
    mask = np.asarray(mask, dtype=bool)
    _shape_check(q, k, v, mask)
    if not mask.any(axis=1).all():
        raise MaskError("a query row has no visible key")
    s = (q @ k.T) * _scale(q.shape[1])
    s = np.where(mask, s, _NEG_INF).astype(_F32)
    e = np.exp((s - s.max(axis=1, keepdims=True)).astype(_F32), dtype=_F32)
    e = np.where(mask, e, _F32(0.0))
    z = e.sum(axis=1, keepdims=True, dtype=_F32)
    return ((e / z) @ v).astype(_F32)


class AttentionPartial(NamedTuple):
    """attention.py:97-116 — (acc = sum exp(l - m) v, row max m, denominator)."""

    acc: np.ndarray
    row_max: np.ndarray
    denom: np.ndarray


def empty_partial(n: int, d: int) -> AttentionPartial:
    """attention.py:119-125 — merge identity."""
    return AttentionPartial(np.zeros((n, d), _F32), np.full(n, _NEG_INF, _F32),
                            np.zeros(n, _F32))


def attention_partial(q, k, v, mask) -> AttentionPartial:
    """attention.py:127-154 — partial over one key shard; dead rows keep -inf/0."""
    q, k, v = _finite_f32(q), _finite_f32(k), _finite_f32(v)
    mask = np.asarray(mask, dtype=bool)
    _shape_check(q, k, v, mask)
    if k.shape[0] == 0:
        return empty_partial(q.shape[0], v.shape[1])
    s = (q @ k.T) * _scale(q.shape[1])
    s = np.where(mask, s, _NEG_INF).astype(_F32)
    m = s.max(axis=1)
    live = np.isfinite(m)
    shift = np.where(live, m, _F32(0.0))
    e = np.exp((s - shift[:, None]).astype(_F32), dtype=_F32)
    e = np.where(mask, e, _F32(0.0))
    z = e.sum(axis=1, dtype=_F32)
    acc = (e @ v).astype(_F32)
    acc[~live] = 0.0
    z[~live] = 0.0
    return AttentionPartial(acc, m.astype(_F32), z)


def merge_partials(a: AttentionPartial, b: AttentionPartial) -> AttentionPartial:
    """attention.py:157-173 — associative/commutative log-sum-exp merge."""
    if a.acc.shape != b.acc.shape:
        raise DimensionError("partial shapes differ")
    m = np.maximum(a.row_max, b.row_max)
    ref = np.where(np.isfinite(m), m, _F32(0.0))

    def factor(p):
        f = np.exp((p.row_max - ref).astype(_F32), dtype=_F32)
        return np.where(np.isfinite(p.row_max), f, _F32(0.0)).astype(_F32)

    fa, fb = factor(a), factor(b)
    return AttentionPartial(
        (a.acc * fa[:, None] + b.acc * fb[:, None]).astype(_F32),
        m.astype(_F32),
        (a.denom * fa + b.denom * fb).astype(_F32),
    )


def finalize_partial(p: AttentionPartial) -> np.ndarray:
    """attention.py:176-180 — acc / denom; zero denominator is a MaskError."""
    if not (p.denom > 0).all():
        raise MaskError("zero denominator")
    return (p.acc / p.denom[:, None]).astype(_F32)


def multi_head(q, k, v, heads: int, mask) -> np.ndarray:
    """engine.py:176-182 (`_mha`) — per-head column slices, concatenated."""
    dh = q.shape[1] // heads
    cols = [slice(h * dh, (h + 1) * dh) for h in range(heads)]
    return np.concatenate([scaled_dot_attention(q[:, c], k[:, c], v[:, c], mask)
                           for c in cols], axis=1)
