"""CPU check of the balanced Ulysses re-shard plan (parallel.BalancedPlan): heads that do
not divide the ranks are split by query rows instead of padded with dummy heads.

The four block-copy descriptor sets (K5b `ifx_copy_blocks`) and the all-to-all split sizes
are executed here with numpy on byte buffers for every rank; the test checks that each rank
receives exactly its segments' Q rows and its heads' full K/V, and that the attention
outputs land back in every rank's sequence slice at the right columns."""

import numpy as np
import pytest
import torch

from paper_2511_20714_b200.parallel import BalancedPlan


def _exec(desc, src: np.ndarray, dst: np.ndarray):
    t, nb, _ = desc
    for s_off, s_ld, d_off, d_ld, rows, rb in t.numpy()[:nb]:
        for r in range(rows):
            dst[d_off + r * d_ld:d_off + r * d_ld + rb] = src[s_off + r * s_ld:s_off + r * s_ld + rb]


def _a2a(sends, send_sizes, recv_sizes, eb=2):
    """sends[i] bytes of rank i, split by send_sizes[i] (elements) -> recv buffers."""
    W = len(sends)
    outs = []
    for k in range(W):
        parts = []
        for i in range(W):
            off = sum(send_sizes[i][:k]) * eb
            parts.append(sends[i][off:off + send_sizes[i][k] * eb])
            assert len(parts[-1]) == recv_sizes[k][i] * eb
        outs.append(np.concatenate(parts))
    return outs


@pytest.mark.parametrize("heads,world,T,dhp", [(12, 8, 64, 8), (3, 2, 16, 8), (5, 4, 8, 16), (7, 3, 12, 8)])
def test_balanced_plan_round_trip(heads, world, T, dhp):
    rng = np.random.default_rng(heads * 100 + world)
    Dp, n = heads * dhp, T // world
    qkv = rng.integers(0, 2**15, size=(T, 3 * Dp), dtype=np.uint16)  # bf16 bit patterns
    plans = [BalancedPlan(heads, T, world, r, dhp, torch.device("cpu")) for r in range(world)]
    work = [sum(r1 - r0 for _, r0, r1 in p.segs) for p in plans]
    assert work == [heads * T // world] * world  # balanced query rows
    sends = []
    for r, p in enumerate(plans):
        src = np.ascontiguousarray(qkv[r * n:(r + 1) * n]).view(np.uint8).ravel()
        buf = np.zeros(p.send_elems * 2, np.uint8)
        _exec(p.pack, src, buf)
        sends.append(buf)
    recvs = _a2a(sends, [p.send_sizes for p in plans], [p.recv_sizes for p in plans])
    outs_h = []
    for r, p in enumerate(plans):
        region = np.zeros(p.region_bytes, np.uint8)
        _exec(p.unpack, recvs[r], region)
        reg = region.view(np.uint16)
        q = reg[:p.qr * dhp].reshape(p.qr, dhp)
        kv = reg[p.k_off // 2:p.k_off // 2 + 2 * T * p.hl * dhp].reshape(2, T, p.hl * dhp)
        for si, (h, r0, r1) in enumerate(p.segs):
            b = p.seg_base[si]
            assert np.array_equal(q[b:b + r1 - r0], qkv[r0:r1, h * dhp:(h + 1) * dhp])
        for hi, h in enumerate(p.heads_of):
            assert np.array_equal(kv[0][:, hi * dhp:(hi + 1) * dhp], qkv[:, Dp + h * dhp:Dp + (h + 1) * dhp])
            assert np.array_equal(kv[1][:, hi * dhp:(hi + 1) * dhp], qkv[:, 2 * Dp + h * dhp:2 * Dp + (h + 1) * dhp])
        # "attention output" = the Q rows themselves, sent back to their sequence owners
        o = np.ascontiguousarray(q).view(np.uint8).ravel()
        buf = np.zeros(max(1, p.o_send_elems) * 2, np.uint8)
        _exec(p.opack, o, buf)
        outs_h.append(buf)
    back = _a2a(outs_h, [p.o_send_sizes for p in plans], [p.o_recv_sizes for p in plans])
    for r, p in enumerate(plans):
        attn_s = np.zeros(n * Dp * 2, np.uint8)
        _exec(p.ounpack, back[r], attn_s)
        assert np.array_equal(attn_s.view(np.uint16).reshape(n, Dp), qkv[r * n:(r + 1) * n, :Dp])
