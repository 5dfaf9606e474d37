"""CPU check of the peer-memory Ulysses exchange layout (parallel.P2PExchange.layout).

The exchange has no all-to-all: G1's epilogue stores each Q/K/V column block of a rank's n
sequence rows into the arena of the rank that attends that head, following a scatter table
of (address, row stride, row_lo, row_hi) entries (ifx_gemm_params.scatter), and K1 stores
each output row into the arena of the rank that owns the sequence row (ifx_attn_params
o_peer). Here every rank's table is executed with numpy on byte arenas (addresses =
peer * 2^40 + offset), the same way the kernels address them, and the result must equal
the receive layout of the NCCL path (parallel.py:150-169 of the reference: each rank sees
the full sequence of its heads' Q/K/V) and, after the O scatter, each rank's [n, Dp] slice
of the attention output."""

import numpy as np
import pytest
import torch

from paper_2511_20714_b200.parallel import BalancedPlan, P2PExchange

BIG = 1 << 40


def _addr(p, off):
    return p * BIG + off


def _scatter_rows(arenas, table, src, blk_w):
    """G1's scatter epilogue: src [n, 3H*blk_w] uint16 rows of one rank."""
    for blk in range(table.shape[0]):
        for a, ld, lo, hi in table[blk]:
            if hi <= 0:
                continue
            p, off = divmod(int(a), BIG)
            for rr in range(lo, hi):
                o = off + rr * ld
                arenas[p][o:o + blk_w * 2] = src[rr, blk * blk_w:(blk + 1) * blk_w].view(np.uint8)


def _o_scatter(arenas, o_peers, rows, out, n, o_ld, row0=0, col_off=0):
    """K1's epilogue: output row r (all its head columns) -> sequence row row0 + r."""
    for r in range(rows):
        g = row0 + r
        p, off = divmod(o_peers[g // n] + col_off, BIG)
        o = off + (g % n) * o_ld * 2
        arenas[p][o:o + out.shape[1] * 2] = out[r].view(np.uint8)


@pytest.mark.parametrize("heads,world,T,dhp,balanced", [
    (4, 2, 16, 8, False), (8, 4, 32, 16, False), (40, 8, 64, 8, False),
    (12, 8, 64, 8, True), (3, 2, 16, 8, True), (5, 4, 8, 16, True), (7, 3, 12, 8, True)])
def test_p2p_layout_equals_all_to_all(heads, world, T, dhp, balanced):
    rng = np.random.default_rng(heads * 100 + world)
    Dp, n = heads * dhp, T // world
    qkv = rng.integers(0, 2**15, size=(T, 3 * Dp), dtype=np.uint16)  # bf16 bit patterns
    rb = P2PExchange.region_bytes(heads, T, world, dhp, balanced)
    s_off = max(rb) // 256 * 256 + 256
    arenas = [np.zeros(s_off + n * Dp * 2, np.uint8) for _ in range(world)]
    layouts = [P2PExchange.layout(heads, T, world, r, dhp, balanced, _addr, s_off)
               for r in range(world)]
    for r in range(world):  # every rank's QKV GEMM epilogue
        _scatter_rows(arenas, layouts[r][0], np.ascontiguousarray(qkv[r * n:(r + 1) * n]), dhp)
    for r in range(world):
        reg = arenas[r][:rb[r]].view(np.uint16)
        o_peers = layouts[r][1]
        if not balanced:
            hl = heads // world
            wl = hl * dhp
            R = reg.reshape(T, 3 * wl)
            for g in range(3):
                for j in range(hl):
                    h = r * hl + j
                    assert np.array_equal(R[:, g * wl + j * dhp:g * wl + (j + 1) * dhp],
                                          qkv[:, g * Dp + h * dhp:g * Dp + (h + 1) * dhp])
            # "attention output" of the rank's heads = their Q columns, all T rows
            _o_scatter(arenas, o_peers, T, np.ascontiguousarray(R[:, :wl]), n, Dp)
        else:
            p = BalancedPlan(heads, T, world, r, dhp, torch.device("cpu"))
            assert rb[r] == p.region_bytes
            q = reg[:p.qr * dhp].reshape(p.qr, dhp)
            kv = reg[p.k_off // 2:p.k_off // 2 + 2 * T * p.hl * dhp].reshape(2, T, p.hl * dhp)
            for si, (h, r0, r1) in enumerate(p.segs):
                b = p.seg_base[si]
                assert np.array_equal(q[b:b + r1 - r0], qkv[r0:r1, h * dhp:(h + 1) * dhp])
            for hi, h in enumerate(p.heads_of):
                assert np.array_equal(kv[0][:, hi * dhp:(hi + 1) * dhp], qkv[:, Dp + h * dhp:Dp + (h + 1) * dhp])
                assert np.array_equal(kv[1][:, hi * dhp:(hi + 1) * dhp], qkv[:, 2 * Dp + h * dhp:2 * Dp + (h + 1) * dhp])
            for si, (h, r0, r1) in enumerate(p.segs):  # one K1 per segment
                b = p.seg_base[si]
                _o_scatter(arenas, o_peers, r1 - r0, np.ascontiguousarray(q[b:b + r1 - r0]), n, Dp,
                           row0=r0, col_off=h * dhp * 2)
    for r in range(world):  # every rank's S region = its rows of every head's output
        S = arenas[r][s_off:].view(np.uint16).reshape(n, Dp)
        assert np.array_equal(S, qkv[r * n:(r + 1) * n, :Dp])


@pytest.mark.parametrize("heads,world,T,dhp", [(12, 8, 64, 8), (6, 4, 32, 16), (3, 2, 16, 8),
                                                (10, 4, 16, 8)])
def test_p2p_grouped_layout(heads, world, T, dhp):
    """Grouped plan (G head groups x R row slices): rank g*R + r receives Q rows of slice r
    for its H/G heads and the whole sequence's K/V of those heads; one K1 over the slice's
    rows writes each output row to its sequence owner."""
    from paper_2511_20714_b200.parallel import GroupedPlan, grouped_split
    gs = grouped_split(heads, world)
    assert gs is not None
    G, R = gs
    rng = np.random.default_rng(heads + world)
    Dp, n = heads * dhp, T // world
    qkv = rng.integers(0, 2**15, size=(T, 3 * Dp), dtype=np.uint16)
    rb = P2PExchange.region_bytes(heads, T, world, dhp, False, gs)
    s_off = max(rb) // 256 * 256 + 256
    arenas = [np.zeros(s_off + n * Dp * 2, np.uint8) for _ in range(world)]
    layouts = [P2PExchange.layout(heads, T, world, r, dhp, False, _addr, s_off, gs)
               for r in range(world)]
    for r in range(world):
        _scatter_rows(arenas, layouts[r][0], np.ascontiguousarray(qkv[r * n:(r + 1) * n]), dhp)
    for k in range(world):
        gp = GroupedPlan(heads, T, world, k, G, R)
        wl = gp.hl * dhp
        reg = arenas[k][:rb[k]].view(np.uint16)
        q = reg[:gp.rows * wl].reshape(gp.rows, wl)
        kk = reg[gp.rows * wl:(gp.rows + T) * wl].reshape(T, wl)
        vv = reg[(gp.rows + T) * wl:(gp.rows + 2 * T) * wl].reshape(T, wl)
        cols = slice(gp.g * wl, (gp.g + 1) * wl)
        assert np.array_equal(q, qkv[gp.row0:gp.row0 + gp.rows, cols])
        assert np.array_equal(kk, qkv[:, Dp:2 * Dp][:, cols])
        assert np.array_equal(vv, qkv[:, 2 * Dp:][:, cols])
        _o_scatter(arenas, layouts[k][1], gp.rows, np.ascontiguousarray(q), n, Dp, row0=gp.row0)
    for r in range(world):
        S = arenas[r][s_off:].view(np.uint16).reshape(n, Dp)
        assert np.array_equal(S, qkv[r * n:(r + 1) * n, :Dp])


def test_p2p_layout_rejects_three_way_heads():
    # 1 head on 4 ranks: its K/V would reach all 4 (two scatter entries per block)
    from paper_2511_20714_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        P2PExchange.layout(1, 16, 4, 0, 8, True, _addr, 1 << 20)
