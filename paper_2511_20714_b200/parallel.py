"""Ulysses sequence/head parallelism on B200 — drop-in for `inferix.parallel`'s Ulysses path.

Reference: /root/reference/pkg/src/inferix/parallel.py. Two layers:

1. The reference's in-process API (WorkerGroup / all_to_all / ulysses_attention /
   dense_reference / predict_communication / choose_strategy, parallel.py:38-169,304-364)
   with the same trace and byte accounting (FLOAT_BYTES = 4) so the cost model stays
   checkable; local attention runs in K1.

2. The real thing, one process per GPU (`torch.distributed`, NCCL over NVLink/NVSwitch):
   `UlyssesComm` re-shards a rank's sequence slice of the fused Q|K|V projection into the
   full sequence of its head group with ONE all-to-all (pack kernel -> a2a), and the
   attention output back with one all-to-all (a2a -> unpack kernel). `UlyssesEngine`
   runs the generate-and-cache loop with activations sequence-sharded, attention
   head-sharded, the KV cache head-sharded and rank-local (never communicated), the page
   table replicated and identical on every rank, and cross-attention sequence-sharded
   against replicated prompt K/V (no communication).

3. The same exchange over NVLink peer memory instead of NCCL (`P2PExchange`, the default
   when every rank can map every other rank's arena): `PeerMesh` opens each rank's arena
   in every other rank through CUDA IPC; G1's scatter epilogue writes each Q/K/V column
   block straight into the owner's head-group buffer, K1 scatters its output rows back
   into the sequence owners' buffers, and a graph-capturable barrier kernel
   (ifx_peer_barrier) orders the two passes — no pack/unpack kernels and no all-to-all
   launches. Head counts that do not divide the world use the grouped plan
   (`grouped_split`: G head groups x R <= 2 query-row slices, one K1 launch per rank).

The reference's per-strategy entry points also exist over real ranks
(`ulysses_attention_dist`, `ring_attention_pass_kv_dist`, `ring_attention_pass_q_dist`,
`sequence_parallel_attention`), with the same SpTrace byte accounting as layer 1.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .attention import (AttentionPartial, attention_partial, empty_partial, finalize_partial, merge_partials,
                        scaled_dot_attention)
from .errors import ConfigError, DimensionError

FLOAT_BYTES = 4  # parallel.py:38 — the reference's cost model counts fp32 elements


# ===================================================================== reference API
def _payload_bytes(payload) -> int:
    """parallel.py:41-49."""
    if isinstance(payload, (np.ndarray, torch.Tensor)):
        return int(np.prod(tuple(payload.shape))) * FLOAT_BYTES
    if isinstance(payload, AttentionPartial):
        return sum(_payload_bytes(t) for t in (payload.acc, payload.row_max, payload.denom))
    if isinstance(payload, (tuple, list)):
        return sum(_payload_bytes(p) for p in payload)
    raise DimensionError(f"untraceable payload type {type(payload)!r}")


@dataclass
class TraceRecord:
    """parallel.py:52-60."""
    step: int
    sender: int
    receiver: int
    bytes: int
    tag: str

    def to_line(self) -> str:
        return f"{self.step}\t{self.sender}\t{self.receiver}\t{self.bytes}\t{self.tag}"


class WorkerGroup:
    """parallel.py:63-98 — world_size simulated ranks with FIFO channels and a send trace."""

    def __init__(self, world_size: int):
        if world_size < 1:
            raise DimensionError("world_size must be >= 1")
        self.world_size = world_size
        self.channels = {(i, j): [] for i in range(world_size) for j in range(world_size)}
        self.trace: list = []
        self._lock = threading.Lock()
        self._step = 0

    def send(self, sender: int, receiver: int, payload, tag: str = ""):
        with self._lock:
            self.trace.append(TraceRecord(self._step, sender, receiver, _payload_bytes(payload), tag))
            self.channels[(sender, receiver)].append(payload)

    def recv(self, sender: int, receiver: int, timeout: float = 10.0):
        with self._lock:
            return self.channels[(sender, receiver)].pop(0)

    def advance_step(self):
        with self._lock:
            self._step += 1

    def total_bytes(self, tag=None) -> int:
        return sum(r.bytes for r in self.trace if tag is None or r.tag == tag)

    def message_count(self, tag=None) -> int:
        return sum(1 for r in self.trace if tag is None or r.tag == tag)

    def export_trace(self) -> str:
        return "\n".join(r.to_line() for r in self.trace)


def all_to_all(group: WorkerGroup, per_worker_send):
    """parallel.py:101-111 — recv[j][i] == send[i][j]; every pair is one message."""
    w = group.world_size
    if len(per_worker_send) != w or any(len(row) != w for row in per_worker_send):
        raise DimensionError("send matrix must be world_size x world_size")
    for i in range(w):
        for j in range(w):
            group.send(i, j, per_worker_send[i][j], tag="a2a")
    recv = [[group.recv(i, j) for i in range(w)] for j in range(w)]
    group.advance_step()
    return recv


def equal_shards(seq_len: int, world_size: int) -> list:
    """parallel.py:312-314."""
    base, rem = divmod(seq_len, world_size)
    return [base + (1 if i < rem else 0) for i in range(world_size)]


def _dev(x) -> torch.Tensor:
    return x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float32)).cuda()


def _mha_dense(q, k, v, heads, mask):
    """parallel.py:121-127 — per-head K1 launches."""
    dh = q.shape[1] // heads
    return torch.cat([scaled_dot_attention(q[:, h * dh:(h + 1) * dh], k[:, h * dh:(h + 1) * dh],
                                           v[:, h * dh:(h + 1) * dh], mask)
                      for h in range(heads)], dim=1)


def dense_reference(q_shards, k_shards, v_shards, heads, mask):
    """parallel.py:130-137."""
    q = torch.cat([_dev(s) for s in q_shards])
    k = torch.cat([_dev(s) for s in k_shards])
    v = torch.cat([_dev(s) for s in v_shards])
    out = _mha_dense(q, k, v, heads, _dev_mask(mask))
    cuts = np.cumsum([0] + [s.shape[0] for s in q_shards])
    return [out[cuts[i]:cuts[i + 1]] for i in range(len(q_shards))]


def _dev_mask(mask) -> torch.Tensor:
    return mask.bool() if isinstance(mask, torch.Tensor) else torch.as_tensor(np.asarray(mask, bool)).cuda()


def ulysses_attention(group: WorkerGroup, q_shards, k_shards, v_shards, heads, mask):
    """parallel.py:140-169 — sequence-sharded in/out via head repartitioning (simulated
    ranks, device tensors, K1 local attention)."""
    w = group.world_size
    if heads % w != 0:
        raise DimensionError(f"heads {heads} not divisible by world_size {w}")
    qs, ks, vs = ([_dev(s) for s in x] for x in (q_shards, k_shards, v_shards))
    d = qs[0].shape[1]
    hpw = heads // w
    cw = hpw * (d // heads)
    col = lambda j: slice(j * cw, (j + 1) * cw)  # noqa: E731
    send = [[(qs[i][:, col(j)], ks[i][:, col(j)], vs[i][:, col(j)]) for j in range(w)] for i in range(w)]
    recv = all_to_all(group, send)
    m = _dev_mask(mask)
    outs = []
    for j in range(w):
        q = torch.cat([recv[j][i][0] for i in range(w)])
        k = torch.cat([recv[j][i][1] for i in range(w)])
        v = torch.cat([recv[j][i][2] for i in range(w)])
        outs.append(_mha_dense(q, k, v, hpw, m))
    cuts = np.cumsum([0] + [s.shape[0] for s in qs])
    back = [[outs[j][cuts[i]:cuts[i + 1]] for i in range(w)] for j in range(w)]
    recv_back = all_to_all(group, back)
    return [torch.cat(recv_back[i], dim=1) for i in range(w)]


def _shard_offsets(shards) -> list:
    """parallel.py:114-118 — cumulative row offsets of a shard list."""
    return [0] + list(np.cumsum([s.shape[0] for s in shards]))


def _heads_partial(q, k, v, heads: int, m, parts):
    """Merge one key shard into every head's running partial (attention.py:127-173): one
    K1 launch per head with partial statistics, merged on device."""
    dh = q.shape[1] // heads
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        parts[h] = merge_partials(parts[h], attention_partial(q[:, sl], k[:, sl], v[:, sl], m))
    return parts


def ring_attention_pass_kv(group: WorkerGroup, q_shards, k_shards, v_shards, mask, heads: int = 1,
                           threads: bool = False):
    """parallel.py:172-244 — K/V shards rotate around the ring (W-1 steps, one 'kv' message
    per rank per step), every rank merges partials over each visiting shard. The
    lockstep schedule is used for either `threads` value: the result and the trace are
    the same as the reference's (deterministic rotation), only the scheduling differs."""
    w = group.world_size
    qs, ks, vs = ([_dev(s) for s in x] for x in (q_shards, k_shards, v_shards))
    m = _dev_mask(mask)
    dh = qs[0].shape[1] // heads
    q_off, kv_off = _shard_offsets(qs), _shard_offsets(ks)
    parts = [[empty_partial(qs[i].shape[0], dh) for _ in range(heads)] for i in range(w)]
    cur = [(ks[i], vs[i], i) for i in range(w)]
    for step in range(w):
        for i in range(w):
            k, v, owner = cur[i]
            _heads_partial(qs[i], k, v, heads,
                           m[q_off[i]:q_off[i + 1], kv_off[owner]:kv_off[owner + 1]], parts[i])
        if step < w - 1:
            owners = [c[2] for c in cur]
            for i in range(w):
                group.send(i, (i + 1) % w, (cur[i][0], cur[i][1]), tag="kv")
            cur = [(*group.recv((i - 1) % w, i), owners[(i - 1) % w]) for i in range(w)]
            group.advance_step()
    return [torch.cat([finalize_partial(p) for p in parts[i]], dim=1) for i in range(w)]


def ring_attention_pass_q(group: WorkerGroup, q_shards, k_shards, v_shards, mask, heads: int = 1):
    """parallel.py:247-298 — Q and its per-head partials rotate while K/V stay; after W
    steps the finished partials are sent to their owners ('gather')."""
    w = group.world_size
    qs, ks, vs = ([_dev(s) for s in x] for x in (q_shards, k_shards, v_shards))
    m = _dev_mask(mask)
    dh = qs[0].shape[1] // heads
    q_off, kv_off = _shard_offsets(qs), _shard_offsets(ks)
    trav = [(qs[i], [empty_partial(qs[i].shape[0], dh) for _ in range(heads)], i) for i in range(w)]
    for step in range(w):
        for i in range(w):
            q, parts, owner = trav[i]
            _heads_partial(q, ks[i], vs[i], heads,
                           m[q_off[owner]:q_off[owner + 1], kv_off[i]:kv_off[i + 1]], parts)
        if step < w - 1:
            for i in range(w):
                q, parts, _ = trav[i]
                group.send(i, (i + 1) % w, (q, *parts), tag="q")
            nxt = []
            for i in range(w):
                payload = group.recv((i - 1) % w, i)
                nxt.append((payload[0], list(payload[1:]), trav[(i - 1) % w][2]))
            trav = nxt
            group.advance_step()
    out = [None] * w
    for i in range(w):
        q, parts, owner = trav[i]
        if owner == i:
            out[i] = torch.cat([finalize_partial(p) for p in parts], dim=1)
        else:
            group.send(i, owner, tuple(parts), tag="gather")
    for i in range(w):
        if out[i] is None:
            holder = next(j for j in range(w) if trav[j][2] == i)
            out[i] = torch.cat([finalize_partial(p) for p in group.recv(holder, i)], dim=1)
    return out


@dataclass
class LinkCostModel:
    """parallel.py:305-309 — cost = cost_per_message * messages + cost_per_byte * bytes."""
    cost_per_message: float = 1e-6
    cost_per_byte: float = 1e-9


def predict_communication(strategy, shard_lens, heads, head_dim, world_size, elem_bytes=FLOAT_BYTES):
    """parallel.py:317-343 — (messages, bytes) on the wire, self-sends excluded.
    `elem_bytes` (B200 extension) = 2 for the bf16 activations UlyssesComm moves."""
    w, d = world_size, heads * head_dim
    if w == 1:
        return 0, 0
    n = sum(shard_lens)
    if strategy == "ulysses":
        return 2 * w * (w - 1), (w - 1) * 4 * n * (d // w) * elem_bytes
    if strategy == "ring_pass_kv":
        return w * (w - 1), (w - 1) * 2 * n * d * elem_bytes
    if strategy == "ring_pass_q":
        rot = n * d + n * (d + 2 * heads)
        return w * (w - 1) + w, ((w - 1) * rot + n * (d + 2 * heads)) * elem_bytes
    raise DimensionError(f"unknown strategy {strategy!r}")


STRATEGIES = ("ulysses", "ring_pass_kv", "ring_pass_q")


def choose_strategy(seq_len, heads, world_size, link_cost_model: LinkCostModel, head_dim: int = 8):
    """parallel.py:349-364 — argmin predicted cost; ties break in listed order."""
    shard_lens = equal_shards(seq_len, world_size)
    best = None
    for name in STRATEGIES:
        if name == "ulysses" and heads % world_size != 0:
            continue
        msgs, nbytes = predict_communication(name, shard_lens, heads, head_dim, world_size)
        cost = link_cost_model.cost_per_message * msgs + link_cost_model.cost_per_byte * nbytes
        if best is None or cost < best[1]:
            best = (name, cost, msgs, nbytes)
    name, cost, msgs, nbytes = best
    return {"strategy": name, "cost": cost, "messages": msgs, "bytes": nbytes}


# ===================================================================== real multi-GPU path
def _pack_cuda(src: torch.Tensor, groups: int, world: int, chunk: int) -> torch.Tensor:
    from ._device import count_launch, dtype_code, row_ld, stream_ptr
    n = src.shape[0]
    dst = torch.empty(world, n, groups, chunk, device=src.device, dtype=src.dtype)
    _abi.check(_abi.lib().ifx_ulysses_pack(src.data_ptr(), n, groups, world, chunk, row_ld(src),
                                           dtype_code(src.dtype), dst.data_ptr(), stream_ptr()),
               "ulysses_pack")
    count_launch()
    return dst


def _unpack_cuda(src: torch.Tensor, out: torch.Tensor, groups: int, world: int, chunk: int):
    from ._device import count_launch, dtype_code, row_ld, stream_ptr
    n = out.shape[0]
    _abi.check(_abi.lib().ifx_ulysses_unpack(src.data_ptr(), n, groups, world, chunk,
                                             dtype_code(out.dtype), out.data_ptr(), row_ld(out),
                                             stream_ptr()), "ulysses_unpack")
    count_launch()
    return out


class UlyssesComm:
    """Head<->sequence re-shard over a torch.distributed group (NCCL on NVLink/NVSwitch).

    seq_to_head: rank r's [n, G*W*c] (G groups, e.g. Q|K|V, each W per-peer head chunks of
    c columns) -> [W*n, G*c], the FULL sequence (ranks hold contiguous sequence slices in
    rank order) for rank r's heads. head_to_seq is the inverse for one group.
    One all-to-all per direction; `trace` accumulates (messages, bytes) excluding self."""

    def __init__(self, group=None, pack=None, unpack=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._pack = pack or _pack_cuda
        self._unpack = unpack or _unpack_cuda
        self.messages = 0
        self.bytes = 0  # counted at enqueue: a pass captured in a CUDA graph counts once
        if dist.get_backend(group) == "nccl":  # communicator up before any graph capture
            t = torch.zeros(self.world, device="cuda")
            dist.all_to_all_single(torch.empty_like(t), t, group=group)

    def _a2a(self, send: torch.Tensor) -> torch.Tensor:
        recv = torch.empty_like(send)
        if send.is_cuda and self.dist.get_backend(self.group) != "nccl":
            # non-NCCL group (e.g. gloo tests of several ranks sharing one GPU): stage on host
            r = torch.empty(send.shape, dtype=send.dtype)
            self.dist.all_to_all_single(r, send.cpu(), group=self.group)
            recv.copy_(r)
        else:
            self.dist.all_to_all_single(recv, send, group=self.group)
        w = self.world
        self.messages += w - 1
        self.bytes += send.numel() * send.element_size() * (w - 1) // w
        return recv

    def a2a_var(self, send: torch.Tensor, send_sizes, recv: torch.Tensor, recv_sizes) -> torch.Tensor:
        """All-to-all with per-peer sizes (elements), for the balanced re-shard."""
        if send.is_cuda and self.dist.get_backend(self.group) != "nccl":
            r = torch.empty(recv.shape, dtype=recv.dtype)
            self.dist.all_to_all_single(r, send.cpu(), recv_sizes, send_sizes, group=self.group)
            recv.copy_(r)
        else:
            self.dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=self.group)
        self.messages += sum(1 for k, sz in enumerate(send_sizes) if sz and k != self.rank)
        self.bytes += sum(sz for k, sz in enumerate(send_sizes) if k != self.rank) * send.element_size()
        return recv

    def seq_to_head(self, x: torch.Tensor, groups: int) -> torch.Tensor:
        n = x.shape[0]
        chunk = x.shape[1] // (groups * self.world)
        packed = self._pack(x, groups, self.world, chunk)  # [W, n, G, c]
        recv = self._a2a(packed)                            # [W(src), n, G, c]
        return recv.view(self.world * n, groups * chunk)

    def head_to_seq(self, y: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        chunk = y.shape[1]
        n = y.shape[0] // self.world
        recv = self._a2a(y.contiguous().view(self.world, n, 1, chunk))  # [W(src heads), n, 1, c]
        return self._unpack(recv, out, 1, self.world, chunk)


class NativeComm:
    """The C-ABI's NCCL communicator (include/ifx_abi.h ifx_comm_*) — what a host without
    torch.distributed binds (SURVEY §8(b) `ifx_comm_init`): the reference's WorkerGroup +
    all_to_all (parallel.py:63-111) as a real collective on the current CUDA device.
    `NativeComm.unique_id()` on rank 0, shipped to every rank out of band, then
    `NativeComm(uid, world, rank)` on each. `all_to_all` has UlyssesComm.a2a_var's meaning
    (per-peer element counts, contiguous per-peer chunks); `all_gather` concatenates every
    rank's buffer in rank order."""

    def __init__(self, uid: bytes, world: int, rank: int):
        import ctypes
        if len(uid) != 128:
            raise DimensionError("an NCCL unique id is 128 bytes")
        self._h = ctypes.c_void_p()
        _abi.check(_abi.lib().ifx_comm_init(uid, world, rank, ctypes.byref(self._h)), "comm_init")
        self.world, self.rank = world, rank

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        buf = ctypes.create_string_buffer(128)
        _abi.check(_abi.lib().ifx_comm_unique_id(buf), "comm_unique_id")
        return buf.raw

    def all_to_all(self, send: torch.Tensor, send_sizes, recv: torch.Tensor, recv_sizes,
                   stream=None) -> torch.Tensor:
        import ctypes
        from ._device import stream_ptr
        if len(send_sizes) != self.world or len(recv_sizes) != self.world:
            raise DimensionError("one send and one receive size per rank")
        if sum(send_sizes) > send.numel() or sum(recv_sizes) > recv.numel() or \
                send.dtype != recv.dtype or not send.is_contiguous() or not recv.is_contiguous():
            raise DimensionError("all_to_all sizes exceed the contiguous buffers")
        es = send.element_size()
        arr = lambda v: (ctypes.c_int64 * self.world)(*v)  # noqa: E731
        so = np.concatenate([[0], np.cumsum(send_sizes)[:-1]]) * es
        ro = np.concatenate([[0], np.cumsum(recv_sizes)[:-1]]) * es
        _abi.check(_abi.lib().ifx_comm_all_to_all(
            self._h, send.data_ptr(), arr(so.tolist()), arr([n * es for n in send_sizes]),
            recv.data_ptr(), arr(ro.tolist()), arr([n * es for n in recv_sizes]),
            stream_ptr(stream)), "comm_all_to_all")
        return recv

    def all_gather(self, send: torch.Tensor, recv: torch.Tensor, stream=None) -> torch.Tensor:
        from ._device import stream_ptr
        nb = send.numel() * send.element_size()
        if recv.numel() * recv.element_size() < nb * self.world or not send.is_contiguous() or \
                not recv.is_contiguous():
            raise DimensionError("all_gather needs world x the send bytes, contiguous")
        _abi.check(_abi.lib().ifx_comm_all_gather(self._h, send.data_ptr(), nb, recv.data_ptr(),
                                                  stream_ptr(stream)), "comm_all_gather")
        return recv

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _abi.check(_abi.lib().ifx_comm_destroy(self._h), "comm_destroy")
            self._h = None

    def __del__(self):
        import sys
        if sys.is_finalizing():  # CUDA / NCCL may already be torn down at interpreter exit
            return
        try:
            self.close()
        except Exception:
            pass


class BalancedPlan:
    """Ulysses re-shard for heads that do not divide the ranks, without dummy heads.

    The (head, query row) grid of a block, head-major, is cut into W equal ranges: rank k
    attends segments (h, r0, r1) covering H*T/W query rows in total (e.g. 12 heads on 8
    ranks: 1.5 heads each instead of 2 padded ones), holds K/V of the <= ceil(H/W)+1 heads
    its segments touch (its KV-cache shard; a head split across two ranks is cached on
    both), and activations stay sequence-sharded (rank i owns rows [i*n, (i+1)*n)).
    Static per runner: the byte-block descriptors of the four copies around the two
    all-to-alls (K5b `ifx_copy_blocks`) and the all-to-all split sizes."""

    def __init__(self, heads: int, T: int, world: int, rank: int, dhp: int, dev):
        if T % world or (heads * T) % world:
            raise DimensionError("block_len must split evenly over the ranks")
        n, per = T // world, heads * T // world
        segs = []
        for k in range(world):
            g, g1, sk = k * per, (k + 1) * per, []
            while g < g1:
                h, r = divmod(g, T)
                e = min(g1, (h + 1) * T)
                sk.append((h, r, r + e - g))
                g = e
            segs.append(sk)
        heads_of = [sorted({h for h, _, _ in sk}) for sk in segs]
        self.n, self.T, self.world, self.rank, self.dhp = n, T, world, rank, dhp
        self.segs, self.heads_of = segs[rank], heads_of[rank]
        self.hl = len(self.heads_of)
        Dp, eb = heads * dhp, 2  # bf16
        rb = dhp * eb            # bytes of one head row

        def qrows(seg, i):
            _, r0, r1 = seg
            a, b = max(r0, i * n), min(r1, (i + 1) * n)
            return a, max(0, b - a)

        # --- seq -> head: what this rank sends to k, and what it receives from i
        pack, self.send_sizes, off = [], [], 0
        for k in range(world):
            start = off
            for (h, r0, r1) in segs[k]:
                a, m = qrows((h, r0, r1), rank)
                if m:
                    pack.append(((a - rank * n) * 3 * Dp * eb + h * rb, 3 * Dp * eb, off, rb, m, rb))
                    off += m * rb
            for which in (1, 2):  # K then V of k's heads, my n rows
                for h in heads_of[k]:
                    pack.append((which * Dp * eb + h * rb, 3 * Dp * eb, off, rb, n, rb))
                    off += n * rb
            self.send_sizes.append((off - start) // eb)
        self.send_elems = off // eb
        # receive layout: Q region [QR, dhp] (segments stacked), K / V regions [T, hl*dhp]
        self.seg_base, qr = [], 0
        for (h, r0, r1) in self.segs:
            self.seg_base.append(qr)
            qr += r1 - r0
        self.qr = qr
        kv_w = self.hl * rb
        k_off, v_off = qr * rb, qr * rb + T * kv_w
        self.region_bytes = v_off + T * kv_w
        unpack, self.recv_sizes, off = [], [], 0
        for i in range(world):
            start = off
            for si, seg in enumerate(self.segs):
                a, m = qrows(seg, i)
                if m:
                    unpack.append((off, rb, (self.seg_base[si] + a - seg[1]) * rb, rb, m, rb))
                    off += m * rb
            for reg in (k_off, v_off):
                for hi_, h in enumerate(self.heads_of):
                    unpack.append((off, rb, reg + i * n * kv_w + hi_ * rb, kv_w, n, rb))
                    off += n * rb
            self.recv_sizes.append((off - start) // eb)
        self.recv_elems = off // eb
        self.k_off, self.v_off, self.kv_w = k_off, v_off, kv_w
        # --- head -> seq: O rows of my segments back to their sequence owners
        opack, self.o_send_sizes, off = [], [], 0
        for i in range(world):
            start = off
            for si, seg in enumerate(self.segs):
                a, m = qrows(seg, i)
                if m:
                    opack.append(((self.seg_base[si] + a - seg[1]) * rb, rb, off, rb, m, rb))
                    off += m * rb
            self.o_send_sizes.append((off - start) // eb)
        self.o_send_elems = off // eb
        ounpack, self.o_recv_sizes, off = [], [], 0
        for k in range(world):
            start = off
            for (h, r0, r1) in segs[k]:
                a, m = qrows((h, r0, r1), rank)
                if m:
                    ounpack.append((off, rb, (a - rank * n) * Dp * eb + h * rb, Dp * eb, m, rb))
                    off += m * rb
            self.o_recv_sizes.append((off - start) // eb)
        self.o_recv_elems = off // eb

        def dev_desc(d):
            t = torch.tensor(d if d else [[0] * 6], dtype=torch.int64).to(dev)
            return t, len(d), max((x[4] for x in d), default=0)

        self.pack, self.unpack = dev_desc(pack), dev_desc(unpack)
        self.opack, self.ounpack = dev_desc(opack), dev_desc(ounpack)


def _copy_blocks(src: torch.Tensor, dst: torch.Tensor, desc) -> None:
    from ._device import count_launch, stream_ptr
    t, nb, max_rows = desc
    if nb:
        _abi.check(_abi.lib().ifx_copy_blocks(src.data_ptr(), dst.data_ptr(), t.data_ptr(), nb,
                                              max_rows, stream_ptr()), "copy_blocks")
        count_launch()


class PeerMesh:
    """Symmetric device arenas over NVLink / NVSwitch peer memory, one per rank.

    Each rank allocates one arena (cudaMalloc via ifx_dev_alloc, outside torch's caching
    allocator), exports its CUDA IPC handle, and maps every peer's arena (handles exchanged
    with all_gather_object over the group: host plumbing, no data). Kernels then store
    straight into a peer's arena (`addr(peer, offset)`) and `barrier()` (ifx_peer_barrier,
    graph-capturable) orders the phases. Arena = [signal pad 32 B | epoch counter | data]."""

    HEAD = 256  # pad (uint32[8]) at 0, this rank's epoch counter at 64, data from 256

    def __init__(self, comm, nbytes: int, timeout_ms: int | None = None):
        if getattr(comm, "loopback", False):
            self._init_loopback(comm, nbytes, timeout_ms)
            return
        import ctypes
        import os

        from .engine import _DevBuf
        self.comm = comm
        W, r = comm.world, comm.rank
        if W > 8:
            raise ConfigError("peer meshes span at most the 8 GPUs of one box")
        self.nbytes = int(nbytes)
        self.buf = _DevBuf(self.HEAD + self.nbytes)
        raw = torch.as_tensor(self.buf, device=torch.device("cuda", torch.cuda.current_device()))
        raw[:self.HEAD].zero_()
        torch.cuda.synchronize()
        L = _abi.lib()
        self._opened = []
        bases = []
        if W == 1:
            bases = [self.buf.ptr]
        else:
            h = (ctypes.c_char * 64)()
            _abi.check(L.ifx_ipc_handle(ctypes.c_void_p(self.buf.ptr), h), "ipc_handle")
            hs = [None] * W
            comm.dist.all_gather_object(hs, bytes(h), group=comm.group)
            err = None
            for i in range(W):
                if i == r:
                    bases.append(self.buf.ptr)
                    continue
                pp = ctypes.c_void_p()
                rc = L.ifx_ipc_open(ctypes.c_char_p(hs[i]), ctypes.byref(pp))
                if rc != _abi.OK:
                    err = f"rank {r} cannot map rank {i}: {L.ifx_last_error().decode()}"
                    break
                self._opened.append(pp.value)
                bases.append(pp.value)
            errs = [None] * W  # every rank learns whether the mesh is complete
            comm.dist.all_gather_object(errs, err, group=comm.group)
            if any(errs):
                self.close()
                raise ConfigError("peer mesh: " + "; ".join(e for e in errs if e))
        comm.dist.barrier(group=comm.group)  # every pad zeroed before any barrier kernel
        self.bases = bases
        self._pads = (ctypes.c_void_p * W)(*bases)
        self._counter = ctypes.c_void_p(self.buf.ptr + 64)
        self.timeout_ms = int(timeout_ms or os.environ.get("IFX_PEER_TIMEOUT_MS", 60000))
        self.barriers = 0

    def _init_loopback(self, comm, nbytes, timeout_ms):
        """One process standing in for rank comm.rank of comm.world (tools/rank_probe.py):
        every 'peer' arena is a slice of one local allocation, barriers pass at once. The
        kernels run exactly one rank's launches (the scatter stores land in local HBM
        instead of crossing NVLink; peers' rows stay stale): a compute-only timing probe."""
        import ctypes
        import os

        from .engine import _DevBuf
        self.comm, W = comm, comm.world
        self.nbytes = int(nbytes)
        self.stride = (self.HEAD + self.nbytes + 255) // 256 * 256
        self.buf = _DevBuf(self.stride * W)
        raw = torch.as_tensor(self.buf, device=torch.device("cuda", torch.cuda.current_device()))
        raw.zero_()
        self._opened = []
        self.bases = [self.buf.ptr + p * self.stride for p in range(W)]
        self._own = self.bases[comm.rank]
        self._pads = (ctypes.c_void_p * 1)(self._own)
        self._counter = ctypes.c_void_p(self._own + 64)
        self.timeout_ms = int(timeout_ms or os.environ.get("IFX_PEER_TIMEOUT_MS", 60000))
        self.barriers = 0
        self.loopback = True

    def addr(self, peer: int, offset: int = 0) -> int:
        """Address (in this process) of byte `offset` of `peer`'s data region."""
        return self.bases[peer] + self.HEAD + int(offset)

    def local(self, offset: int, rows: int, width: int, dtype=torch.bfloat16) -> torch.Tensor:
        """[rows, width] view of this rank's own data region at byte `offset`."""
        t = torch.as_tensor(self.buf, device=torch.device("cuda", torch.cuda.current_device()))
        es = torch.empty((), dtype=dtype).element_size()
        n = rows * width * es
        o = self.HEAD + offset + (self._own - self.buf.ptr if getattr(self, "loopback", False) else 0)
        return t[o:o + n].view(dtype).view(rows, width)

    def barrier(self) -> None:
        from ._device import count_launch, stream_ptr
        lb = getattr(self, "loopback", False)
        _abi.check(_abi.lib().ifx_peer_barrier(self._pads, 1 if lb else self.comm.world,
                                               0 if lb else self.comm.rank,
                                               self._counter, self.timeout_ms, stream_ptr()),
                   "peer_barrier")
        count_launch()
        self.barriers += 1

    def close(self) -> None:
        import ctypes
        for pp in self._opened:
            _abi.lib().ifx_ipc_close(ctypes.c_void_p(pp))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


class LoopbackComm:
    """Stand-in for UlyssesComm in a single process that runs ONE rank's share of a W-rank
    Ulysses job (tools/rank_probe.py): the world-1 process group does the plumbing, the peer
    mesh loops back (PeerMesh._init_loopback). Timing only — other ranks' data never arrive."""

    loopback = True

    def __init__(self, world: int, rank: int = 0):
        import torch.distributed as dist
        self.dist, self.group = dist, None
        self.world, self.rank = world, rank
        self.messages = self.bytes = 0


def grouped_split(heads: int, world: int):
    """(G, R) for heads that do not divide the ranks: G head groups x R row slices with
    G * R = W, heads % G == 0, R <= 2 (largest G); None if there is none (balanced plan)."""
    if heads % world == 0:
        return None
    for g in range(world, 0, -1):
        if world % g == 0 and heads % g == 0 and world // g <= 2 and g < world:
            return g, world // g
    return None


class GroupedPlan:
    """Ulysses x sequence split for heads that do not divide the ranks (peer exchange only):
    rank k = g*R + r attends head group g (H/G whole heads) for query rows [r*T/R,
    (r+1)*T/R) against the full sequence's K/V of its heads (the whole block's K/V reaches
    the R ranks of its group). Same query-row work as the balanced plan, but ONE K1 launch
    over whole heads per layer-pass (e.g. 12 heads on 8 ranks: 3 heads x half the rows)."""

    def __init__(self, heads: int, T: int, world: int, rank: int, G: int, R: int):
        self.G, self.R, self.T = G, R, T
        self.g, self.r = divmod(rank, R)
        self.hl = heads // G
        self.rows = T // R
        self.row0 = self.r * self.rows


class P2PExchange:
    """The Ulysses re-shard (parallel.py:150-169) without an all-to-all: G1's QKV epilogue
    stores each head's Q/K/V column block of this rank's n sequence rows straight into the
    rank that attends that head (region R of its arena), K1's epilogue stores each output
    row into the rank that owns that sequence row (region S, [n, Dp]). Two peer barriers
    per layer-pass (after the QKV GEMM; after attention) order the phases; they also cover
    the write-after-read hazards (a rank's next QKV GEMM starts only after every rank's
    attention read R, its next attention only after every rank's wo GEMM read S — so the
    clean pass's page write, which reads this rank's K/V from R, runs before the second).

    Layouts (`layout`): whole heads (heads % W == 0: R = [T, 3*wl]); grouped (GroupedPlan:
    Q [T/R, wl] of the rank's row slice, K and V [T, wl]); balanced (BalancedPlan: Q
    segments stacked, K and V [T, hl*dhp]) when a head's rows and K/V reach at most two
    ranks (two scatter entries per column block; `layout` raises ConfigError otherwise)."""

    def __init__(self, runner, comm):
        m = runner.model
        W, r, n, T = comm.world, comm.rank, runner.n, m.config.block_len
        H, dhp, Dp = m.heads_pad, m.dh_pad, m.attn_width
        balanced = runner.plan is not None
        grouped = (runner.grouped.G, runner.grouped.R) if runner.grouped is not None else None
        r_bytes = self.region_bytes(H, T, W, dhp, balanced, grouped)
        self.s_off = max(r_bytes) // 256 * 256 + 256
        self.mesh = PeerMesh(comm, self.s_off + n * Dp * 2)
        table, self.o_peers = self.layout(H, T, W, r, dhp, balanced, self.mesh.addr, self.s_off,
                                          grouped)
        self.table = torch.from_numpy(table.reshape(3 * H, 8)).to(runner.x.device)
        if balanced:
            self.r_view = self.mesh.local(0, r_bytes[r] // 2, 1).view(-1)
        elif grouped is not None:
            gp = runner.grouped
            wl = gp.hl * dhp
            self.q_view = self.mesh.local(0, gp.rows, wl)
            self.k_view = self.mesh.local(gp.rows * wl * 2, T, wl)
            self.v_view = self.mesh.local((gp.rows + T) * wl * 2, T, wl)
        else:
            self.r_view = self.mesh.local(0, T, 3 * (H // W) * dhp)
        self.s_view = self.mesh.local(self.s_off, n, Dp)
        self.n = n

    @classmethod
    def region_bytes(cls, H, T, W, dhp, balanced, grouped=None):
        """Bytes of each rank's receive region R (whole-head: [T, 3*wl]; balanced: the Q
        segments stacked, then K and V [T, hl*dhp]; grouped: Q [T/R, wl], K, V [T, wl])."""
        if grouped is not None:
            G, R = grouped
            return [(T // R + 2 * T) * (H // G) * dhp * 2] * W
        if not balanced:
            return [T * 3 * (H // W) * dhp * 2] * W
        segs, heads = cls._segments(H, T, W)
        return [sum(r1 - r0 for _, r0, r1 in segs[k]) * dhp * 2 + 2 * T * len(heads[k]) * dhp * 2
                for k in range(W)]

    @classmethod
    def layout(cls, H, T, W, r, dhp, balanced, addr, s_off, grouped=None):
        """Rank r's G1 scatter table [3H blocks, 2 entries, (address, row stride, row_lo,
        row_hi)] over the Q|K|V column blocks of its n rows, and K1's per-peer O addresses.
        addr(peer, byte offset) -> address of that byte of the peer's data region."""
        n, rb = T // W, dhp * 2
        table = np.zeros((3 * H, 2, 4), dtype=np.int64)
        fill = np.zeros(3 * H, dtype=np.int64)

        def put(blk, a, ld, lo, hi):
            e = fill[blk]
            if e >= 2:
                raise ConfigError("a head reaches more than two ranks")
            table[blk, e] = (a, ld, lo, hi)
            fill[blk] += 1
        if grouped is not None:
            G, R = grouped
            hl, rows = H // G, T // R
            wl = hl * dhp
            rs = (r * n) // rows  # the row slice this rank's sequence rows fall in
            for h in range(H):
                g, j = divmod(h, hl)
                # Q rows -> the group's rank for this row slice, at row r*n - rs*rows + rr
                put(h, addr(g * R + rs, ((r * n - rs * rows) * wl + j * dhp) * 2), wl * 2, 0, n)
                for r2 in range(R):  # K / V rows -> every row slice of the group
                    put(H + h, addr(g * R + r2, ((rows + r * n) * wl + j * dhp) * 2), wl * 2, 0, n)
                    put(2 * H + h, addr(g * R + r2, ((rows + T + r * n) * wl + j * dhp) * 2),
                        wl * 2, 0, n)
            g = r // R
            return table, [addr(p, s_off + g * hl * dhp * 2) for p in range(W)]
        if not balanced:
            hl = H // W
            wl = hl * dhp
            for g in range(3):
                for h in range(H):
                    p, j = divmod(h, hl)
                    put(g * H + h, addr(p, (r * n) * 3 * wl * 2 + (g * wl + j * dhp) * 2),
                        3 * wl * 2, 0, n)
            # K1 over this rank's hl heads, all T rows: row g -> row owner g // n, at the
            # columns of this rank's heads
            return table, [addr(p, s_off + r * hl * dhp * 2) for p in range(W)]
        segs, heads = cls._segments(H, T, W)
        for k in range(W):
            kv_w = len(heads[k]) * rb
            qr_k = sum(r1 - r0 for (_, r0, r1) in segs[k])
            k_off, v_off = qr_k * rb, qr_k * rb + T * kv_w
            base = 0
            for (h, r0, r1) in segs[k]:
                a, b = max(r0, r * n), min(r1, (r + 1) * n)
                if b > a:  # local row rr -> Q row base + (r*n + rr - r0) of rank k
                    put(h, addr(k, (base + r * n - r0) * rb), rb, a - r * n, b - r * n)
                base += r1 - r0
            for hi_, h in enumerate(heads[k]):
                put(H + h, addr(k, k_off + (r * n) * kv_w + hi_ * rb), kv_w, 0, n)
                put(2 * H + h, addr(k, v_off + (r * n) * kv_w + hi_ * rb), kv_w, 0, n)
        # K1 per segment (one head): O row i is sequence row r0 + i -> its owner, at the
        # head's columns (attn(col_off=h*dhp*2, row0=r0))
        return table, [addr(p, s_off) for p in range(W)]

    @staticmethod
    def _segments(H, T, W):
        per = H * T // W
        segs = []
        for k in range(W):
            g, g1, sk = k * per, (k + 1) * per, []
            while g < g1:
                h, rr = divmod(g, T)
                e = min(g1, (h + 1) * T)
                sk.append((h, rr, rr + e - g))
                g = e
            segs.append(sk)
        return segs, [sorted({h for h, _, _ in sk}) for sk in segs]

    def attn(self, col_off: int = 0, row0: int = 0):
        """K1 with its O scattered to the row owners' S regions (+ col_off bytes)."""
        import functools

        from ._device import attn_fwd
        return functools.partial(attn_fwd, o_peers=[a + col_off for a in self.o_peers],
                                 o_rows=self.n, o_row0=row0)


class UlyssesRunner:
    """BlockRunner (engine.py) for one Ulysses rank: sequence-sharded activations,
    head-sharded attention over the rank-local KV shard (engine.py:185-221 semantics)."""

    def __init__(self, model, comm: UlyssesComm, attn=None, p2p: bool = False):
        from ._device import attn_fwd
        self.model, self.comm = model, comm
        c = model.config
        W = comm.world
        if c.block_len % W:
            raise DimensionError(f"block_len {c.block_len} not divisible by world_size {W}")
        self.n = c.block_len // W
        dev = model.time_vec.device
        # heads divisible by the ranks: classic Ulysses (whole heads per rank, K5 pack);
        # otherwise the balanced plan (query rows of a head split across ranks)
        self.plan = None
        self.grouped = None
        gs = grouped_split(model.heads_pad, W) if (model.heads_pad % W and p2p) else None
        if gs is not None:  # peer exchange: whole head groups x row slices, one K1 launch
            self.grouped = GroupedPlan(model.heads_pad, c.block_len, W, comm.rank, *gs)
            self.hl = self.grouped.hl
        elif model.heads_pad % W:
            self.plan = BalancedPlan(model.heads_pad, c.block_len, W, comm.rank, model.dh_pad, dev)
            self.hl = self.plan.hl
        else:
            self.hl = model.heads_pad // W
        self.wl = self.hl * model.dh_pad
        self._attn = attn or attn_fwd
        D, Dp, n, T = c.model_dim, model.attn_width, self.n, c.block_len
        if self.plan is not None:
            pl = self.plan
            self.b_send = torch.empty(pl.send_elems, device=dev, dtype=torch.bfloat16)
            self.b_recv = torch.empty(pl.recv_elems, device=dev, dtype=torch.bfloat16)
            self.b_region = torch.empty(pl.region_bytes // 2, device=dev, dtype=torch.bfloat16)
            self.b_o = torch.empty(pl.qr, model.dh_pad, device=dev, dtype=torch.bfloat16)
            self.b_osend = torch.empty(max(1, pl.o_send_elems), device=dev, dtype=torch.bfloat16)
            self.b_orecv = torch.empty(max(1, pl.o_recv_elems), device=dev, dtype=torch.bfloat16)
        self.x = torch.empty(n, D, device=dev)
        self.h = torch.empty(n, D, device=dev, dtype=torch.bfloat16)
        self.qkv = torch.empty(n, 3 * Dp, device=dev, dtype=torch.bfloat16)
        self.attn_h = torch.empty(T, self.wl, device=dev, dtype=torch.bfloat16)
        self.attn_s = torch.empty(n, Dp, device=dev, dtype=torch.bfloat16)
        self.ffn = torch.empty(n, 2 * D, device=dev, dtype=torch.bfloat16)
        self.eps = torch.empty(n, D, device=dev)
        self.cross_bufs = {}
        self.attn_events = None
        from .engine import _Stager
        self.stager = _Stager(dev)
        self._tv = self._gpool = self._cap = self._graph = None  # CUDA-graph state (_euler_steps)
        self._warm = False
        self._tail = None  # event after the last block's clean pass (_euler_steps: GPU idle?)
        # the re-shard over peer memory (G1 scatter epilogue + K1 O scatter) instead of
        # pack -> all-to-all -> unpack
        self.xch = None
        if p2p:
            if attn is not None:
                raise ConfigError("the peer-scatter exchange runs K1 itself (no attention hook)")
            self.xch = P2PExchange(self, comm)
        # G1 with the norms fused into the projections' epilogues (engine _forward_g1) when
        # it beats cuBLASLt + the RMS kernel on this rank's shapes (small row counts: wave
        # and launch bound), chosen by timing both once (IFX_G1=all / off forces it)
        from ._device import RowNorm
        self.norm = RowNorm(self.h, torch.empty(n, 2 * -(-D // 64), device=dev), 0, D)
        self.g1_all = self.xch is not None and self._choose_g1_all()

    def _balanced_attention(self, li, ctx, sc, ev):
        """BalancedPlan: re-shard (one all-to-all), one K1 per segment (a head's query rows,
        that head's cached columns and own K/V), re-shard back. Returns this rank's K / V
        [T, hl*dhp] (the page write of the clean pass)."""
        pl, dhp = self.plan, self.model.dh_pad
        _copy_blocks(self.qkv, self.b_send, pl.pack)
        self.comm.a2a_var(self.b_send, pl.send_sizes, self.b_recv, pl.recv_sizes)
        _copy_blocks(self.b_recv, self.b_region, pl.unpack)
        T = pl.T
        kv = self.b_region[pl.k_off // 2:].view(-1)[:2 * T * self.wl].view(2, T, self.wl)
        kc, vc = kv[0], kv[1]
        qreg = self.b_region[:pl.qr * dhp].view(pl.qr, dhp)
        if ev is not None:
            from .engine import timing_event
            e0 = timing_event()
            e0.record()
        last = len(pl.segs) - 1
        for si, (h, r0, r1) in enumerate(pl.segs):
            hi_ = pl.heads_of.index(h)
            b, m = pl.seg_base[si], r1 - r0
            c0, c1 = hi_ * dhp, (hi_ + 1) * dhp
            ctx.attend(li, qreg[b:b + m], 1, dhp, self.b_o[b:b + m], kc[:, c0:c1], vc[:, c0:c1], sc,
                       attn=self._attn, cols=(c0, c1), first=si == 0, last=si == last)
        if ev is not None:
            e1 = timing_event()
            e1.record()
            ev.append((e0, e1))
        _copy_blocks(self.b_o, self.b_osend, pl.opack)
        self.comm.a2a_var(self.b_osend, pl.o_send_sizes, self.b_orecv, pl.o_recv_sizes)
        _copy_blocks(self.b_orecv, self.attn_s, pl.ounpack)
        return kc, vc

    def _p2p_attention(self, li, ctx, sc, ev, lw, rope, append=None, norm_in=None):
        """QKV projection scattered into the attending ranks (G1 epilogue, RoPE fused), a
        peer barrier, K1 with O scattered to the row owners, the clean pass's page write of
        this rank's K / V (`append(kc, vc)`: before the barrier, because once every rank
        passed it the peers' next QKV epilogue overwrites region R), a peer barrier."""
        from ._device import gemm_fused
        from .engine import timing_event
        m, x = self.model, self.xch
        c, dhp, wl = m.config, m.dh_pad, self.wl
        rspec = None if rope is None else (rope[0], rope[1], self.comm.rank * self.n,
                                           c.head_dim // 2, dhp, m.heads_pad, 0, m.attn_width)
        gemm_fused(self.h, lw.wqkv, None, norm_in=norm_in, rope=rspec, scatter=(x.table, dhp))
        x.mesh.barrier()
        if ev is not None:
            e0 = timing_event()
            e0.record()
        if self.grouped is not None:  # whole heads, this rank's row slice of the queries
            kc, vc = x.k_view, x.v_view
            ctx.attend(li, x.q_view, self.hl, dhp, x.s_view, kc, vc, sc,
                       attn=x.attn(row0=self.grouped.row0))
        elif self.plan is None:
            R = x.r_view
            q, kc, vc = R[:, :wl], R[:, wl:2 * wl], R[:, 2 * wl:]
            ctx.attend(li, q, self.hl, dhp, x.s_view, kc, vc, sc, attn=x.attn())
        else:
            pl, T = self.plan, self.plan.T
            kv = x.r_view[pl.k_off // 2:][:2 * T * wl].view(2, T, wl)
            kc, vc = kv[0], kv[1]
            qreg = x.r_view[:pl.qr * dhp].view(pl.qr, dhp)
            last = len(pl.segs) - 1
            for si, (h, r0, r1) in enumerate(pl.segs):
                hi_ = pl.heads_of.index(h)
                b, mm = pl.seg_base[si], r1 - r0
                c0, c1 = hi_ * dhp, (hi_ + 1) * dhp
                ctx.attend(li, qreg[b:b + mm], 1, dhp, x.s_view, kc[:, c0:c1], vc[:, c0:c1], sc,
                           attn=x.attn(col_off=h * dhp * 2, row0=r0), cols=(c0, c1),
                           first=si == 0, last=si == last)
        if ev is not None:
            e1 = timing_event()
            e1.record()
            ev.append((e0, e1))
        if append is not None:
            append(kc, vc)
        x.mesh.barrier()

    def _rms(self, x, out, tvec=None, t=0.0, x_out=None):
        from ._device import rms_bf16
        return rms_bf16(x, out, tvec, t, x_out)

    def _choose_g1_all(self) -> bool:
        """Time this rank's wo / w1 / w2 on G1 (fused residual + norm statistics, norm as a
        row scale) against cuBLASLt plus the RMS kernels they replace; QKV is on G1 either
        way (scatter epilogue)."""
        from . import engine as E
        from ._device import gemm, gemm_fused
        if E.G1 in ("all", "off", "qkv"):
            return E.G1 == "all"
        lw, norm = self.model.layers[0], self.norm
        self.x.normal_()
        self.h.copy_(self.x)
        self.ffn.normal_()

        def timed(fn, n=6):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n

        def lt():
            gemm(self.attn_s, lw.wo, self.x, beta=1.0)
            for _ in range(2):
                self._rms(self.x, self.h)
            gemm(self.h, lw.w1, self.ffn, relu=True)
            gemm(self.ffn, lw.w2, self.x, beta=1.0)
            self._rms(self.x, self.h)

        def g1():
            gemm_fused(self.attn_s, lw.wo, self.x, beta=1.0, norm_out=norm)
            gemm_fused(self.h, lw.w1, self.ffn, relu=True, norm_in=norm)
            gemm_fused(self.ffn, lw.w2, self.x, beta=1.0, norm_out=norm)

        t_lt, t_g1 = min(timed(lt) for _ in range(2)), min(timed(g1) for _ in range(2))
        self.g1_choice = {"cublaslt_rms_ms": t_lt, "g1_fused_ms": t_g1}
        use = t_g1 < 0.95 * t_lt
        comm = self.comm
        if comm.world > 1 and not getattr(comm, "loopback", False):
            votes = [None] * comm.world  # one decision for all ranks (rank 0's timing)
            comm.dist.all_gather_object(votes, use, group=comm.group)
            use = votes[0]
        return use

    def forward(self, latent, t, ctx, cross, cache, collect_kv=False, chunk_index=0, eps_out=None,
                rope=None):
        from ._device import gemm
        from .engine import _cross_attend, _ffn_up, _residual
        from .kvcache import SELF_ATTN
        m = self.model
        c = m.config
        sc = 1.0 / math.sqrt(c.head_dim)
        if self.g1_all:
            return self._forward_g1(latent, t, ctx, cross, cache, collect_kv, chunk_index,
                                    eps_out, rope, sc)
        for li, lw in enumerate(m.layers):
            if li == 0:
                if isinstance(t, torch.Tensor):  # t*time_vec on device (graph replays)
                    self._rms(latent, self.h, t, 1.0, self.x)
                else:
                    self._rms(latent, self.h, m.time_vec, t, self.x)
            else:
                self._rms(self.x, self.h)
            ev = self.attn_events
            if self.xch is not None:
                app = None
                if collect_kv:  # rank-local page write of this rank's heads
                    def app(kc, vc, li=li):
                        cache.append_block(li, kc, vc, kind=SELF_ATTN, chunk_index=chunk_index)
                self._p2p_attention(li, ctx, sc, ev, lw, rope, app)
                attn_s = self.xch.s_view
            else:
                kc, vc = self._a2a_attention(li, ctx, sc, ev, lw, rope)
                attn_s = self.attn_s
            _residual(self.x, attn_s, lw.wo)
            if cross is not None:  # sequence-sharded vs replicated prompt K/V: no comm
                self._rms(self.x, self.h)
                _cross_attend(self, cross[li], self.x, self.h, sc)
            self._rms(self.x, self.h)
            _ffn_up(self.h, lw.w1, self.ffn)
            _residual(self.x, self.ffn, lw.w2)
            if collect_kv and self.xch is None:  # rank-local page write of this rank's heads
                cache.append_block(li, kc, vc, kind=SELF_ATTN, chunk_index=chunk_index)
        if eps_out is not None:
            self._rms(self.x, self.h)
            gemm(self.h, m.w_out, eps_out)

    def _forward_g1(self, latent, t, ctx, cross, cache, collect_kv, chunk_index, eps_out, rope, sc):
        """forward() with every projection on G1 and the RMS norms in the epilogues (engine
        BlockRunner._forward_g1): the residual GEMMs emit the bf16 rows and their sums of
        squares, the next projection applies the norm as a row scale."""
        from ._device import gemm_fused
        from .engine import _cross_attend_g1
        from .kvcache import SELF_ATTN
        m, norm = self.model, self.norm
        for li, lw in enumerate(m.layers):
            if li == 0:  # x = latent + t*time_vec fused into the first norm (engine.py:199)
                if isinstance(t, torch.Tensor):
                    self._rms(latent, self.h, t, 1.0, self.x)
                else:
                    self._rms(latent, self.h, m.time_vec, t, self.x)
                nin = None
            else:
                nin = norm
            app = None
            if collect_kv:
                def app(kc, vc, li=li):
                    cache.append_block(li, kc, vc, kind=SELF_ATTN, chunk_index=chunk_index)
            self._p2p_attention(li, ctx, sc, self.attn_events, lw, rope, app, norm_in=nin)
            gemm_fused(self.xch.s_view, lw.wo, self.x, beta=1.0, norm_out=norm)
            if cross is not None:
                _cross_attend_g1(self, cross[li], norm, sc)
            gemm_fused(self.h, lw.w1, self.ffn, relu=True, norm_in=norm)
            gemm_fused(self.ffn, lw.w2, self.x, beta=1.0, norm_out=norm)
        if eps_out is not None:
            gemm_fused(self.h, m.w_out, eps_out, norm_in=norm)

    def _a2a_attention(self, li, ctx, sc, ev, lw, rope):
        """QKV projection, pack -> all-to-all -> K1 -> all-to-all -> unpack (NCCL)."""
        from ._device import gemm
        from .engine import timing_event
        m, c, dhp, wl = self.model, self.model.config, self.model.dh_pad, self.wl
        gemm(self.h, lw.wqkv, self.qkv)
        if rope is not None:  # this rank's rows of the block: table rows rank*n ..
            from ._device import rope_qk
            rope_qk(self.qkv, m.heads_pad, dhp, c.head_dim // 2, 0, m.attn_width, rope[0],
                    rope[1], tab_row0=self.comm.rank * self.n)
        if self.plan is None:
            qkv_h = self.comm.seq_to_head(self.qkv, 3)          # [T, 3*wl] local heads
            q, kc, vc = qkv_h[:, :wl], qkv_h[:, wl:2 * wl], qkv_h[:, 2 * wl:]
            if ev is not None:
                e0 = timing_event()
                e0.record()
            ctx.attend(li, q, self.hl, dhp, self.attn_h, kc, vc, sc, attn=self._attn)
            if ev is not None:
                e1 = timing_event()
                e1.record()
                ev.append((e0, e1))
            self.comm.head_to_seq(self.attn_h, self.attn_s)      # [n, Dp]
        else:
            kc, vc = self._balanced_attention(li, ctx, sc, ev)
        return kc, vc

    def denoise(self, latent, schedule, ctx, cross, cache, chunk_index):
        from .engine import _euler_steps, rope_tables
        rope = rope_tables(self.model.config, chunk_index, latent.device)
        # graph capture needs the all-to-alls on the GPU stream: NCCL only (a gloo group
        # stages them through the host)
        nccl = self.comm.dist.get_backend(self.comm.group) == "nccl" or self.xch is not None
        _euler_steps(self, latent, schedule, ctx, cross, cache, self.eps, rope, graphs_ok=nccl,
                     first_block=chunk_index == 0)
        self.forward(latent, 0.0, ctx, cross, cache, collect_kv=cache is not None,
                     chunk_index=chunk_index, rope=rope)
        self._tail = torch.cuda.Event()
        self._tail.record()
        return latent

    def release_graphs(self) -> None:
        """Free the captured pass graph (before destroying the NCCL process group)."""
        self._graph = None


class UlyssesEngine:
    """Engine.generate (engine.py:368-411) across the ranks of `comm`. Every rank runs the
    same page-table calls in the same order, so bookkeeping stays identical everywhere."""

    def __init__(self, model, comm: UlyssesComm, kv_config=None, attn=None, p2p: bool | None = None):
        """p2p: re-shard through peer memory (P2PExchange) instead of NCCL all-to-alls.
        Default (None): IFX_ULYSSES=p2p|nccl, else p2p when no attention hook is given and
        the plan allows it (heads >= ranks)."""
        import os

        from .engine import default_kv_config
        self.model, self.comm = model, comm
        self.kv_config = kv_config or default_kv_config(model.config)
        if self.kv_config.latent is not None:  # the up-projection mixes every head's columns
            raise ConfigError("latent KV mode is not supported with head-sharded (Ulysses) caches")
        self.runner = None
        if p2p is None:
            mode = os.environ.get("IFX_ULYSSES", "auto")
            p2p = mode == "p2p"
            if mode == "auto" and attn is None and model.heads_pad >= comm.world:
                try:  # peer mesh failures are agreed across ranks: all fall back together
                    self.runner = UlyssesRunner(model, comm, attn, p2p=True)
                except ConfigError as e:
                    import warnings
                    warnings.warn(f"Ulysses: peer-memory exchange unavailable ({e}); "
                                  "using NCCL all-to-alls", RuntimeWarning)
        if self.runner is None:
            self.runner = UlyssesRunner(model, comm, attn, p2p=bool(p2p))
        self.cache = None

    def generate(self, request, noise_provider=None, gather: bool = True, to_host: bool = False):
        """Returns per-block full latents (gathered) if `gather`, else local shards; with
        `to_host` as pinned host tensors, each block's copy running on a side stream while
        the next block computes."""
        from .engine import (_block_context, _cross_kv, _init_noise_pinned,
                             _prompt_for_chunk, embed_prompt)
        from .kvcache import CROSS_ATTN, KvCache
        request.validate()
        m, c, r = self.model, self.model.config, self.runner
        T, n, rank = c.block_len, r.n, self.comm.rank
        retired = self.cache._pt if self.cache is not None else None  # freed after block 0
        self.cache = KvCache(self.kv_config, dtype=torch.bfloat16,
                             reserve_tokens=T * request.num_blocks, row_width=r.wl,
                             cross_row_width=m.attn_width)
        # the reference's seeded host noise (engine.py:280-282), generated bit-exactly by the
        # native parallel PCG64 parser; each rank copies only its sequence slice to the GPU
        make_noise = noise_provider or (lambda ch: _init_noise_pinned(c, request.seed, ch))
        # the next block's noise is drawn (and pinned) on a host thread while this block's
        # passes are enqueued: a rank at 8 GPUs is close to enqueue-bound
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(1)
        nxt = pool.submit(make_noise, 0)
        cur = None
        out = []
        for chunk in range(request.num_blocks):
            prompt = _prompt_for_chunk(request.prompt_schedule, chunk)
            if prompt != cur:
                if cur is not None:
                    self.cache.clear_cross_attention()
                for li, (kc, vc) in enumerate(_cross_kv(m, embed_prompt(m, prompt))):
                    self.cache.append_block(li, kc, vc, kind=CROSS_ATTN, chunk_index=chunk)
                cur = prompt
            noise = nxt.result()
            if chunk + 1 < request.num_blocks:
                nxt = pool.submit(make_noise, chunk + 1)
            full = noise if isinstance(noise, torch.Tensor) else torch.from_numpy(noise)
            lat = full[rank * n:(rank + 1) * n].to(m.time_vec.device, torch.float32,
                                                   non_blocking=True).clone()
            ctx, cross = _block_context(m, self.cache, None, r.stager, len(request.schedule.steps) + 1)
            r.denoise(lat, request.schedule, ctx, cross, self.cache, chunk)
            retired = None
            if request.kv_window is not None:
                self.cache.evict_window(request.kv_window)
            if gather:
                parts = [torch.empty_like(lat) for _ in range(self.comm.world)]
                self.comm.dist.all_gather(parts, lat, group=self.comm.group)
                lat = torch.cat(parts)
            if to_host:
                from .engine import _copy_stream
                main = torch.cuda.current_stream()
                cs = _copy_stream(lat.device, 1)
                cs.wait_stream(main)
                host = torch.empty(lat.shape, dtype=lat.dtype, pin_memory=True)
                with torch.cuda.stream(cs):
                    host.copy_(lat, non_blocking=True)
                lat.record_stream(cs)
                lat = host
            out.append(lat)
        pool.shutdown(wait=False)
        if to_host:
            from .engine import _copy_stream
            _copy_stream(torch.device("cuda", torch.cuda.current_device()), 1).synchronize()
        return out


# ============================================ sequence-parallel attention across real ranks
# The reference's three strategies (parallel.py:140-298) run on an in-process WorkerGroup;
# these are their multi-GPU counterparts: each rank passes ITS shards and gets ITS output
# rows. Transport is peer memory (a PeerMesh per comm, grown on demand): shards are staged
# into each rank's arena, peers PULL what they need with the DMA copy engines over NVLink
# (ifx_memcpy2d, overlapped with the previous step's K1 on a copy stream) or K1 / the copy
# engines PUSH results into the owner's arena, and ifx_peer_barrier orders the phases. The
# per-shard partials are K1's (normalised output, row max, denominator) and are merged by
# K4 (`ifx_attn_combine`) — the reference's merge_partials / finalize_partial
# (attention.py:157-180) on device.
class SpTrace:
    """Inter-rank traffic of the calls on this rank (sender != receiver): messages and
    logical bytes (unpadded bf16 elements), like WorkerGroup.total_bytes."""

    def __init__(self):
        self.messages = 0
        self.bytes = 0

    def add(self, nbytes: int, messages: int = 1) -> None:
        self.messages += messages
        self.bytes += int(nbytes)


def _sp_mesh(comm, nbytes: int) -> PeerMesh:
    """The comm's sequence-parallel mesh, re-created (collectively: every rank asks for the
    same size, which depends only on the global shard lengths) when too small."""
    mesh = getattr(comm, "_sp_mesh", None)
    if mesh is None or mesh.nbytes < nbytes:
        if mesh is not None:
            torch.cuda.synchronize()
            mesh.close()
        mesh = PeerMesh(comm, max(int(nbytes), 1 << 20))
        comm._sp_mesh = mesh
    return mesh


class _SpCall:
    """Arena layout of one sequence-parallel call (byte offsets identical on every rank)."""

    def __init__(self, comm, q, k, v, heads, mask):
        from .errors import MaskError
        W, r = comm.world, comm.rank
        q, k, v = (_dev(x) for x in (q, k, v))
        if q.dim() != 2 or k.dim() != 2 or v.shape != k.shape or q.shape[1] != k.shape[1]:
            raise DimensionError("q [n, d], k / v [m, d] shards expected")
        d = q.shape[1]
        if heads < 1 or d % heads:
            raise DimensionError(f"model dim {d} not divisible by heads {heads}")
        dh = d // heads
        if dh > 128:
            raise DimensionError("head_dim above 128 is not supported")
        lens = [None] * W
        comm.dist.all_gather_object(lens, (q.shape[0], k.shape[0]), group=comm.group)
        self.q_lens, self.kv_lens = [a for a, _ in lens], [b for _, b in lens]
        self.q_off = [0] + list(np.cumsum(self.q_lens))
        self.kv_off = [0] + list(np.cumsum(self.kv_lens))
        N, M = int(self.q_off[-1]), int(self.kv_off[-1])
        if mask is None:
            mask = np.ones((N, M), dtype=bool)
        mk = torch.as_tensor(np.asarray(mask) if not isinstance(mask, torch.Tensor) else mask)
        if tuple(mk.shape) != (N, M):
            raise DimensionError(f"mask {tuple(mk.shape)} does not match [{N}, {M}]")
        if not bool(mk.bool().any(dim=1).all()):  # scaled_dot_attention / finalize raise
            raise MaskError("query row with no allowed key")
        self.mask = mk.to(q.device, torch.uint8).contiguous()
        self.W, self.r, self.heads, self.dh, self.d = W, r, heads, dh, d
        self.dhp = 64 if dh <= 64 else 128
        self.wp = heads * self.dhp  # padded row width (elements)
        self.n_max, self.m_max = max(max(self.q_lens), 1), max(max(self.kv_lens), 1)
        self.N, self.M = N, M
        off = 0

        def region(nbytes):
            nonlocal off
            o = off
            off += (int(nbytes) + 255) // 256 * 256
            return o
        rb = self.wp * 2
        self.o_qp, self.o_kp, self.o_vp = (region(self.n_max * rb), region(self.m_max * rb),
                                           region(self.m_max * rb))
        self.o_po = region(W * self.n_max * rb)
        self.o_pm = region(W * heads * self.n_max * 4)
        self.o_pl = region(W * heads * self.n_max * 4)
        self.o_out = region(self.n_max * rb)
        self.o_buf = region(2 * max(self.n_max, self.m_max) * rb * 2)  # pull double buffers
        self.total = off
        self.mesh = _sp_mesh(comm, self.total)
        self.q, self.k, self.v = q, k, v
        self.trace = getattr(comm, "sp_trace", None)
        if self.trace is None:
            self.trace = comm.sp_trace = SpTrace()

    def local(self, off, rows, width, dtype=torch.bfloat16):
        return self.mesh.local(off, rows, width, dtype)

    def stage(self):
        """Own shards -> the arena, each head zero-padded to dhp columns; partial slots
        reset (max -inf, denominator 0: a shard without keys contributes nothing)."""
        hp, dh = self.dhp, self.dh
        for x, o in ((self.q, self.o_qp), (self.k, self.o_kp), (self.v, self.o_vp)):
            n = x.shape[0]
            dst = self.local(o, max(n, 1), self.wp)
            dst.zero_()
            if n:
                src = x.to(torch.bfloat16).contiguous().view(n, self.heads, dh)
                dst[:n].view(n, self.heads, hp)[:, :, :dh].copy_(src)
        # partial slot s of this rank's rows: O [n, wp] at o_po + s*n*rb, max / denominator
        # [heads, n] at o_pm / o_pl + s*heads*n*4 (K1's statistics layout, K4's input)
        self.local(self.o_po, self.W * self.n_max, self.wp).zero_()  # 0-weight slots stay finite
        self.local(self.o_pm, self.W * self.heads, self.n_max, torch.float32).fill_(float("-inf"))
        self.local(self.o_pl, self.W * self.heads, self.n_max, torch.float32).zero_()

    def slot(self, owner: int, s: int):
        """Addresses (in owner's arena) of partial slot s of owner's rows."""
        n, rb = self.q_lens[owner], self.wp * 2
        a = self.mesh.addr
        return (a(owner, self.o_po + s * n * rb), a(owner, self.o_pm + s * self.heads * n * 4),
                a(owner, self.o_pl + s * self.heads * n * 4))

    def pull(self, dst, src, width_b, rows, dpitch, spitch, stream):
        from ._device import stream_ptr
        if rows:
            _abi.check(_abi.lib().ifx_memcpy2d(dst, dpitch, src, spitch, width_b, rows,
                                               stream_ptr(stream)), "memcpy2d")

    def partial(self, q_t, k_t, v_t, n_k, mask_view, po, pm, pl):
        """K1 over one key shard with partial statistics, written to (po, pm, pl) (raw
        addresses, possibly in a peer's arena)."""
        from ._device import attn_fwd
        if q_t.shape[0] == 0 or n_k == 0:
            return
        p_out = _RawRows(po, q_t.shape[0], self.wp)
        attn_fwd(q_t, self.heads, self.dhp, p_out, k_t, v_t, 0, n_k, scale=1.0 / math.sqrt(self.dh),
                 mask=mask_view, row_max=_RawRows(pm, 1, 1, torch.float32),
                 row_sum=_RawRows(pl, 1, 1, torch.float32), split_kv=False)

    def combine(self):
        from ._device import count_launch, stream_ptr
        n = self.q_lens[self.r]
        out = self.local(self.o_out, self.n_max, self.wp)
        if n:
            mesh = self.mesh
            _abi.check(_abi.lib().ifx_attn_combine(
                mesh.addr(self.r, self.o_po), self.wp, mesh.addr(self.r, self.o_pm),
                mesh.addr(self.r, self.o_pl), self.W, n, self.heads, self.dhp,
                out.data_ptr(), self.wp, None, None, stream_ptr()), "attn_combine")
            count_launch()
        return out

    def result(self, out):
        n = self.q_lens[self.r]
        y = out[:n].view(n, self.heads, self.dhp)[:, :, :self.dh].reshape(n, self.d)
        return y.float()


class _RawRows:
    """A [rows, width] stand-in for attn_fwd's output / statistics arguments at a raw device
    address (e.g. inside a peer's arena): attn_fwd only reads data_ptr() and the row stride."""

    def __init__(self, addr: int, rows: int, width: int, dtype=torch.bfloat16):
        self._addr, self.shape, self.dtype = int(addr), (rows, width), dtype

    def data_ptr(self) -> int:
        return self._addr

    def stride(self, dim=None):
        s = (self.shape[1], 1)
        return s if dim is None else s[dim]

    def dim(self) -> int:
        return 2


def ulysses_attention_dist(comm, q, k, v, heads: int, mask=None):
    """parallel.py:140-169 across real ranks. Each rank pulls its heads' columns of every
    rank's Q/K/V shard (copy engines, NVLink), attends them over the whole sequence with
    one K1, and pushes each owner's output rows into its arena; two peer barriers."""
    W, r = comm.world, comm.rank
    if heads % W:
        raise DimensionError(f"heads {heads} not divisible by world_size {W}")
    c = _SpCall(comm, q, k, v, heads, mask)
    mesh, hl = c.mesh, heads // W
    hw, rb = hl * c.dhp * 2, c.wp * 2
    c.stage()
    # pull region (reused): Q [N, hl*dhp] | K [M, hl*dhp] | V [M, hl*dhp] | O [N, hl*dhp]
    need = (2 * c.N + 2 * c.M) * hw
    buf = torch.empty(need // 2, device=c.q.device, dtype=torch.bfloat16)
    uq = buf[:c.N * hw // 2].view(c.N, hl * c.dhp)
    uk = buf[c.N * hw // 2:(c.N + c.M) * hw // 2].view(c.M, hl * c.dhp)
    uv = buf[(c.N + c.M) * hw // 2:(c.N + 2 * c.M) * hw // 2].view(c.M, hl * c.dhp)
    uo = buf[(c.N + 2 * c.M) * hw // 2:].view(c.N, hl * c.dhp)
    mesh.barrier()
    st = torch.cuda.current_stream()
    for i in range(W):
        col = r * hw
        c.pull(uq[c.q_off[i]:].data_ptr(), mesh.addr(i, c.o_qp) + col, hw, c.q_lens[i], hw, rb, st)
        c.pull(uk[c.kv_off[i]:].data_ptr(), mesh.addr(i, c.o_kp) + col, hw, c.kv_lens[i], hw, rb, st)
        c.pull(uv[c.kv_off[i]:].data_ptr(), mesh.addr(i, c.o_vp) + col, hw, c.kv_lens[i], hw, rb, st)
        if i != r:
            c.trace.add(hl * c.dh * 2 * (c.q_lens[i] + 2 * c.kv_lens[i]))
    from ._device import attn_fwd
    attn_fwd(uq, hl, c.dhp, uo, uk, uv, 0, c.M, scale=1.0 / math.sqrt(c.dh), mask=c.mask)
    for i in range(W):  # each owner's rows of this rank's heads -> the owner's arena
        c.pull(mesh.addr(i, c.o_out) + r * hw, uo[c.q_off[i]:].data_ptr(), hw, c.q_lens[i], rb, hw, st)
        if i != r:
            c.trace.add(hl * c.dh * 2 * c.q_lens[i])
    mesh.barrier()
    out = c.result(c.local(c.o_out, c.n_max, c.wp))
    mesh.barrier()  # nobody re-stages this arena while a peer still reads it
    return out


def ring_attention_pass_kv_dist(comm, q, k, v, mask=None, heads: int = 1):
    """parallel.py:172-244 across real ranks: the K/V shards visit every rank in ring order
    (owner r-s at step s); the next shard is pulled from its owner's arena on a copy stream
    while K1 attends the current one; one partial per step, merged by K4."""
    W, r = comm.world, comm.rank
    c = _SpCall(comm, q, k, v, heads, mask)
    mesh, rb = c.mesh, c.wp * 2
    c.stage()
    mesh.barrier()
    main = torch.cuda.current_stream()
    cp = torch.cuda.Stream()
    n = c.q_lens[r]
    qv = c.local(c.o_qp, c.n_max, c.wp)[:n]
    bufs = [(c.o_buf + j * 2 * c.m_max * rb, c.o_buf + (j * 2 + 1) * c.m_max * rb) for j in range(2)]
    ready = [torch.cuda.Event() for _ in range(W)]
    free = [torch.cuda.Event() for _ in range(2)]

    def fetch(s):
        o = (r - s) % W
        kb, vb = bufs[s % 2]
        if s >= 2:
            cp.wait_event(free[s % 2])
        c.pull(mesh.addr(r, kb), mesh.addr(o, c.o_kp), rb, c.kv_lens[o], rb, rb, cp)
        c.pull(mesh.addr(r, vb), mesh.addr(o, c.o_vp), rb, c.kv_lens[o], rb, rb, cp)
        ready[s].record(cp)
        c.trace.add(2 * c.kv_lens[o] * c.d * 2)
    cp.wait_stream(main)
    if W > 1:
        fetch(1)
    for s in range(W):
        o = (r - s) % W
        if s == 0:
            kt, vt = c.local(c.o_kp, c.m_max, c.wp), c.local(c.o_vp, c.m_max, c.wp)
        else:
            main.wait_event(ready[s])
            kb, vb = bufs[s % 2]
            kt, vt = c.local(kb, c.m_max, c.wp), c.local(vb, c.m_max, c.wp)
        if s + 1 < W and s + 1 >= 2:  # buffer (s+1)%2 was read by step s-1's K1
            free[(s + 1) % 2].record(main)
            fetch(s + 1)
        po, pm, pl = c.slot(r, s)
        mv = c.mask[c.q_off[r]:c.q_off[r] + n, c.kv_off[o]:c.kv_off[o] + c.kv_lens[o]]
        c.partial(qv, kt, vt, c.kv_lens[o], mv, po, pm, pl)
    out = c.result(c.combine())
    mesh.barrier()  # every peer finished pulling this rank's shards
    return out


def ring_attention_pass_q_dist(comm, q, k, v, mask=None, heads: int = 1):
    """parallel.py:247-298 across real ranks: K/V stay; every rank's Q visits this rank
    (pulled from its owner's arena on a copy stream, overlapping the previous step), K1
    writes the partial of that Q against the local K/V straight into the OWNER's partial
    slot (its arena, over NVLink), and after one peer barrier each owner merges its W
    partials with K4 (the reference's traveling partial + final gather, reassociated)."""
    W, r = comm.world, comm.rank
    c = _SpCall(comm, q, k, v, heads, mask)
    mesh, rb = c.mesh, c.wp * 2
    c.stage()
    mesh.barrier()
    main = torch.cuda.current_stream()
    cp = torch.cuda.Stream()
    m = c.kv_lens[r]
    kt, vt = c.local(c.o_kp, c.m_max, c.wp), c.local(c.o_vp, c.m_max, c.wp)
    bufs = [c.o_buf + j * c.n_max * rb for j in range(2)]
    ready = [torch.cuda.Event() for _ in range(W)]
    free = [torch.cuda.Event() for _ in range(2)]

    def fetch(s):
        o = (r - s) % W
        if s >= 2:
            cp.wait_event(free[s % 2])
        c.pull(mesh.addr(r, bufs[s % 2]), mesh.addr(o, c.o_qp), rb, c.q_lens[o], rb, rb, cp)
        ready[s].record(cp)
        c.trace.add(c.q_lens[o] * c.d * 2)
    cp.wait_stream(main)
    if W > 1:
        fetch(1)
    for s in range(W):
        o = (r - s) % W
        if s == 0:
            qt = c.local(c.o_qp, c.n_max, c.wp)[:c.q_lens[o]]
        else:
            main.wait_event(ready[s])
            qt = c.local(bufs[s % 2], c.n_max, c.wp)[:c.q_lens[o]]
        if s + 1 < W and s + 1 >= 2:
            free[(s + 1) % 2].record(main)
            fetch(s + 1)
        # the partial lands in owner o's slot r: partials (normalised O, max, denominator)
        po, pm, pl = c.slot(o, r)
        mv = c.mask[c.q_off[o]:c.q_off[o] + c.q_lens[o], c.kv_off[r]:c.kv_off[r] + m]
        c.partial(qt, kt, vt, m, mv, po, pm, pl)
        if o != r and m and c.q_lens[o]:
            c.trace.add(c.q_lens[o] * (c.d + 2 * c.heads) * 2)
    mesh.barrier()
    out = c.result(c.combine())
    mesh.barrier()
    return out


STRATEGY_FNS = {"ulysses": ulysses_attention_dist, "ring_pass_kv": ring_attention_pass_kv_dist,
                "ring_pass_q": ring_attention_pass_q_dist}


def sequence_parallel_attention(comm, q, k, v, heads: int, mask=None, strategy: str | None = None,
                                link: LinkCostModel | None = None):
    """The strategy menu of parallel.py:300-364 dispatched on real ranks: `strategy` None
    picks choose_strategy(seq_len, heads, world, link, head_dim) on the global length (the
    default link model is NVLink-like: 5 us per message, 1/700 GB/s per byte). Returns
    (this rank's output rows [n, d] fp32, the strategy used)."""
    if strategy is None:
        lens = [None] * comm.world
        comm.dist.all_gather_object(lens, int(_dev(q).shape[0]), group=comm.group)
        d = _dev(q).shape[1]
        link = link or LinkCostModel(cost_per_message=5e-6, cost_per_byte=1.0 / 700e9)
        strategy = choose_strategy(sum(lens), heads, comm.world, link, head_dim=d // heads)["strategy"]
    if strategy not in STRATEGY_FNS:
        raise DimensionError(f"unknown strategy {strategy!r}")
    fn = STRATEGY_FNS[strategy]
    out = fn(comm, q, k, v, heads, mask) if strategy == "ulysses" else fn(comm, q, k, v, mask, heads)
    return out, strategy
