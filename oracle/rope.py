"""Oracle: 3D (frame, row, column) rotary position embedding — TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED: the reference has no positional encoding ("positions enter only through
the mask", /root/reference/pkg/src/inferix/attention.py:6). BASELINE.json's
north star asks the B200 path to fuse 3D RoPE on Q/K; this restatement defines the
semantics the CUDA kernel (`ifx_rope_qk`) is checked against, following the Wan2.1
convention: head_dim d is split into d - 4*(d//6) frame dims and 2*(d//6) dims each for the
latent row and column; each part rotates interleaved pairs (2k, 2k+1) by
pos * theta^(-2k/part).

Token i of block b (frames_per_block F, latent grid gh x gw) sits at frame b*F + i//(gh*gw),
row (i % (gh*gw)) // gw, column i % gw. Cached K is stored post-RoPE, so context tokens keep
the positions they were generated at.
"""

from __future__ import annotations

import numpy as np


def rope_parts(head_dim: int):
    s = head_dim // 6
    return head_dim - 4 * s, 2 * s, 2 * s


def rope_tables(grid, first_frame: int, head_dim: int, theta: float = 10000.0):
    """cos, sin [F*gh*gw, head_dim//2] float32 for one block starting at `first_frame`."""
    frames, gh, gw = grid
    i = np.arange(frames * gh * gw)
    pos = (first_frame + i // (gh * gw), (i % (gh * gw)) // gw, i % gw)
    angs = []
    for p, n in zip(pos, rope_parts(head_dim)):
        inv = theta ** (-np.arange(0, n, 2, dtype=np.float64) / n)
        angs.append(p[:, None].astype(np.float64) * inv[None, :])
    ang = np.concatenate(angs, axis=1)
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x, cos, sin, heads: int):
    """Rotate interleaved pairs of every head of x [n, heads*head_dim] (fp32)."""
    n, width = x.shape
    d = width // heads
    xr = x.reshape(n, heads, d // 2, 2).astype(np.float32)
    a, b = xr[..., 0], xr[..., 1]
    c, s = cos[:, None, :], sin[:, None, :]
    out = np.stack([a * c - b * s, a * s + b * c], axis=-1)
    return out.reshape(n, width).astype(np.float32)
