"""Oracle: Ulysses head<->sequence re-shard and its communication model.

Test infrastructure only (see oracle/__init__.py). Restates
`/root/reference/pkg/src/inferix/parallel.py:38-298,312-364` without the
simulated queue fabric: the all-to-all is a transpose of the send matrix and the
trace is the list of (sender, receiver, bytes) it implies.
"""

from __future__ import annotations

import numpy as np

from .attention import attention_partial, empty_partial, finalize_partial, merge_partials, multi_head
from .errors import DimensionError

FLOAT_BYTES = 4  # parallel.py:38


def equal_shards(seq_len: int, world: int) -> list:
    """parallel.py:312-314 — first `rem` shards get one extra token."""
    q, r = divmod(seq_len, world)
    return [q + int(i < r) for i in range(world)]


def all_to_all(send):
    """parallel.py:101-111 — recv[j][i] = send[i][j]; returns (recv, trace)."""
    w = len(send)
    if any(len(row) != w for row in send):
        raise DimensionError("send matrix must be world_size x world_size")
    trace = [(i, j, _nbytes(send[i][j])) for i in range(w) for j in range(w)]
    return [[send[i][j] for i in range(w)] for j in range(w)], trace


def _nbytes(payload) -> int:
    if isinstance(payload, np.ndarray):
        return payload.size * FLOAT_BYTES
    return sum(_nbytes(p) for p in payload)


def dense_reference(q_shards, k_shards, v_shards, heads, mask):
    """parallel.py:130-137."""
    out = multi_head(np.concatenate(q_shards), np.concatenate(k_shards),
                     np.concatenate(v_shards), heads, mask)
    cuts = np.cumsum([0] + [s.shape[0] for s in q_shards])
    return [out[cuts[i]:cuts[i + 1]] for i in range(len(q_shards))]


def ulysses_attention(q_shards, k_shards, v_shards, heads, mask):
    """parallel.py:140-169 — seq->head a2a, local MHA on heads/W, head->seq a2a.

    Returns (per-rank outputs, trace of both all-to-alls)."""
    w = len(q_shards)
    if heads % w:
        raise DimensionError(f"heads {heads} not divisible by world_size {w}")
    hpw = heads // w
    width = q_shards[0].shape[1] // heads * hpw
    cols = [slice(j * width, (j + 1) * width) for j in range(w)]
    fwd = [[(q_shards[i][:, cols[j]], k_shards[i][:, cols[j]], v_shards[i][:, cols[j]])
            for j in range(w)] for i in range(w)]
    recv, tr1 = all_to_all(fwd)
    local = [multi_head(*(np.concatenate([recv[j][i][n] for i in range(w)]) for n in range(3)),
                        hpw, mask) for j in range(w)]
    cuts = np.cumsum([0] + [s.shape[0] for s in q_shards])
    back = [[local[j][cuts[i]:cuts[i + 1]] for i in range(w)] for j in range(w)]
    recv2, tr2 = all_to_all(back)
    return [np.concatenate(recv2[i], axis=1) for i in range(w)], tr1 + tr2


def predict_communication(strategy, shard_lens, heads, head_dim, world):
    """parallel.py:317-343 — (messages, bytes) excluding self-sends."""
    w, d = world, heads * head_dim
    if w == 1:
        return 0, 0
    n = sum(shard_lens)
    if strategy == "ulysses":
        return 2 * w * (w - 1), (w - 1) * 4 * n * (d // w) * FLOAT_BYTES
    if strategy == "ring_pass_kv":
        return w * (w - 1), (w - 1) * 2 * n * d * FLOAT_BYTES
    if strategy == "ring_pass_q":
        rot = n * d + n * (d + 2 * heads)
        return w * (w - 1) + w, ((w - 1) * rot + n * (d + 2 * heads)) * FLOAT_BYTES
    raise DimensionError(f"unknown strategy {strategy!r}")


STRATEGIES = ("ulysses", "ring_pass_kv", "ring_pass_q")


def choose_strategy(seq_len, heads, world, cost_per_message=1e-6, cost_per_byte=1e-9,
                    head_dim=8):
    """parallel.py:349-364 — argmin cost; ulysses skipped if heads % W."""
    lens = equal_shards(seq_len, world)
    best = None
    for s in STRATEGIES:
        if s == "ulysses" and heads % world:
            continue
        m, b = predict_communication(s, lens, heads, head_dim, world)
        c = cost_per_message * m + cost_per_byte * b
        if best is None or c < best[1]:
            best = (s, c, m, b)
    return {"strategy": best[0], "cost": best[1], "messages": best[2], "bytes": best[3]}


def _offsets(shards) -> list:
    """parallel.py:114-118."""
    return [0] + list(np.cumsum([s.shape[0] for s in shards]))


def _pbytes(p) -> int:
    """parallel.py:41-49 for an AttentionPartial: acc + row_max + denom elements."""
    return (p.acc.size + p.row_max.size + p.denom.size) * FLOAT_BYTES


def ring_attention_pass_kv(q_shards, k_shards, v_shards, mask, heads=1):
    """parallel.py:172-244 (lockstep schedule) — K/V rotate W-1 steps; each rank merges a
    partial per head over every visiting shard. Returns (outputs, trace)."""
    w = len(q_shards)
    dh = q_shards[0].shape[1] // heads
    qo, ko = _offsets(q_shards), _offsets(k_shards)
    parts = [[empty_partial(q_shards[i].shape[0], dh) for _ in range(heads)] for i in range(w)]
    cur = [(k_shards[i], v_shards[i], i) for i in range(w)]
    trace = []
    for step in range(w):
        for i in range(w):
            k, v, o = cur[i]
            m = mask[qo[i]:qo[i + 1], ko[o]:ko[o + 1]]
            for h in range(heads):
                sl = slice(h * dh, (h + 1) * dh)
                parts[i][h] = merge_partials(parts[i][h], attention_partial(q_shards[i][:, sl], k[:, sl], v[:, sl], m))
        if step < w - 1:
            trace += [(i, (i + 1) % w, _nbytes((cur[i][0], cur[i][1]))) for i in range(w)]
            cur = [(cur[(i - 1) % w][0], cur[(i - 1) % w][1], cur[(i - 1) % w][2]) for i in range(w)]
    return [np.concatenate([finalize_partial(p) for p in parts[i]], axis=1) for i in range(w)], trace


def ring_attention_pass_q(q_shards, k_shards, v_shards, mask, heads=1):
    """parallel.py:247-298 — Q and its partials rotate, K/V stay, then a gather to the
    owners. Returns (outputs, trace)."""
    w = len(q_shards)
    dh = q_shards[0].shape[1] // heads
    qo, ko = _offsets(q_shards), _offsets(k_shards)
    trav = [(q_shards[i], [empty_partial(q_shards[i].shape[0], dh) for _ in range(heads)], i)
            for i in range(w)]
    trace = []
    for step in range(w):
        for i in range(w):
            q, parts, o = trav[i]
            m = mask[qo[o]:qo[o + 1], ko[i]:ko[i + 1]]
            for h in range(heads):
                sl = slice(h * dh, (h + 1) * dh)
                parts[h] = merge_partials(parts[h], attention_partial(q[:, sl], k_shards[i][:, sl], v_shards[i][:, sl], m))
        if step < w - 1:
            trace += [(i, (i + 1) % w, trav[i][0].size * FLOAT_BYTES + sum(_pbytes(p) for p in trav[i][1]))
                      for i in range(w)]
            trav = [trav[(i - 1) % w] for i in range(w)]
    out = [None] * w
    for i in range(w):
        q, parts, o = trav[i]
        out[o] = np.concatenate([finalize_partial(p) for p in parts], axis=1)
        trace.append((i, o, sum(_pbytes(p) for p in parts)))
    return out, trace
