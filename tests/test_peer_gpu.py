"""Peer-memory building blocks of the Ulysses exchange, on one GPU: G1's scatter epilogue
(ifx_gemm_params.scatter) and K1's O scatter (ifx_attn_params.o_peer) against the plain
outputs, and the cross-rank barrier (ifx_peer_barrier) eagerly and inside a CUDA graph.
The multi-process versions (CUDA IPC mappings between ranks) are in test_ulysses_gpu.py."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _bf(x):
    return x.to(torch.bfloat16)


def test_gemm_scatter_matches_plain_output():
    from paper_2511_20714_b200._device import gemm_fused

    torch.manual_seed(0)
    M, K, blk = 300, 256, 128
    nblk = 6
    N = nblk * blk
    a = _bf(torch.randn(M, K, device="cuda"))
    b = _bf(torch.randn(K, N, device="cuda") / 16)
    plain = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gemm_fused(a, b, plain)
    # two destinations with different row strides; block i rows [lo, hi) go to dst0, the
    # rest to dst1 (like a head's query rows split between two ranks)
    dst0 = torch.zeros(M + 7, nblk * blk + 64, device="cuda", dtype=torch.bfloat16)
    dst1 = torch.zeros(nblk, M, blk, device="cuda", dtype=torch.bfloat16)
    table = np.zeros((nblk, 2, 4), dtype=np.int64)
    cuts = [0, 40, 128, 150, 299, 300]
    for i in range(nblk):
        c = cuts[i]
        table[i, 0] = (dst0.data_ptr() + (7 * dst0.shape[1] + i * blk) * 2, dst0.shape[1] * 2, 0, c)
        table[i, 1] = (dst1[i].data_ptr(), blk * 2, c, M)
    t = torch.from_numpy(table.reshape(nblk, 8)).cuda()
    gemm_fused(a, b, None, scatter=(t, blk))
    torch.cuda.synchronize()
    for i in range(nblk):
        c = cuts[i]
        want = plain[:, i * blk:(i + 1) * blk]
        assert torch.equal(dst0[7:7 + c, i * blk:(i + 1) * blk], want[:c])
        assert torch.equal(dst1[i, c:], want[c:])
        assert not dst1[i, :c].any() and not dst0[7 + c:7 + M, i * blk:(i + 1) * blk].any()


@pytest.mark.parametrize("n_q,n_ctx,heads,row0", [(600, 0, 2, 0), (600, 900, 2, 0),
                                                   (200, 1000, 1, 170)])
def test_attn_o_scatter_matches_plain_output(n_q, n_ctx, heads, row0):
    """Output rows spread over three 'ranks' of n rows each (n_q=200 with a few heads
    takes the split-KV + K4 combine path, which scatters instead)."""
    from paper_2511_20714_b200._device import attn_fwd

    torch.manual_seed(1)
    D = heads * 128
    q = _bf(torch.randn(n_q, D, device="cuda"))
    kc = _bf(torch.randn(max(n_ctx, 1), D, device="cuda"))
    vc = _bf(torch.randn(max(n_ctx, 1), D, device="cuda"))
    kn = _bf(torch.randn(n_q, D, device="cuda"))
    vn = _bf(torch.randn(n_q, D, device="cuda"))
    plain = torch.empty(n_q, D, device="cuda", dtype=torch.bfloat16)
    attn_fwd(q, heads, 128, plain, kc, vc, 0, n_ctx, kn, vn)
    n = (row0 + n_q + 2) // 3
    ld = D + 128  # the owners' buffers are wider (all heads), this call's heads at col 64
    bufs = [torch.zeros(n, ld, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    attn_fwd(q, heads, 128, bufs[0], kc, vc, 0, n_ctx, kn, vn,
             o_peers=[b.data_ptr() + 64 * 2 for b in bufs], o_rows=n, o_row0=row0)
    torch.cuda.synchronize()
    got = torch.cat(bufs)[row0:row0 + n_q, 64:64 + D]
    assert torch.equal(got, plain)
    assert not torch.cat(bufs)[:row0].any()


def _barrier_fn():
    from paper_2511_20714_b200 import _abi
    from paper_2511_20714_b200._device import stream_ptr

    arena = torch.zeros(64, device="cuda", dtype=torch.int32)
    pads = (ctypes.c_void_p * 1)(arena.data_ptr())
    counter = ctypes.c_void_p(arena.data_ptr() + 128)

    def barrier():
        _abi.check(_abi.lib().ifx_peer_barrier(pads, 1, 0, counter, 10000, stream_ptr()), "barrier")
    return arena, barrier


def test_peer_barrier_world1_eager_and_graph():
    arena, barrier = _barrier_fn()
    for _ in range(5):
        barrier()
    torch.cuda.synchronize()
    assert int(arena[32]) == 5 and int(arena[0]) == 5  # epoch counter, own flag
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g.capture_begin()
        barrier()
        barrier()
        g.capture_end()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(arena[32]) == 11 and int(arena[0]) == 11  # replays advance the epoch


def test_peer_barrier_rejects_bad_meshes():
    from paper_2511_20714_b200 import _abi
    from paper_2511_20714_b200.errors import DimensionError

    arena = torch.zeros(64, device="cuda", dtype=torch.int32)
    pads = (ctypes.c_void_p * 2)(arena.data_ptr(), arena.data_ptr() + 4)  # misaligned pad
    with pytest.raises(DimensionError):
        _abi.check(_abi.lib().ifx_peer_barrier(pads, 2, 0, ctypes.c_void_p(arena.data_ptr() + 128),
                                               100, None), "barrier")
    with pytest.raises(DimensionError):
        _abi.check(_abi.lib().ifx_peer_barrier(pads, 9, 0, ctypes.c_void_p(arena.data_ptr() + 128),
                                               100, None), "barrier")


@pytest.mark.parametrize("splits,hd", [(1, 128), (3, 128), (8, 64), (32, 128)])
def test_attn_combine_matches_torch(splits, hd):
    """K4 alone (ifx_attn_combine): merge `splits` normalised partials with their (max,
    denominator) statistics, some splits dead (max -inf), vs the merge in torch fp64
    (attention.py:157-180)."""
    from paper_2511_20714_b200 import _abi
    from paper_2511_20714_b200._device import stream_ptr

    torch.manual_seed(splits)
    n, H = 300, 3
    D = H * hd
    po = torch.randn(splits, n, D, device="cuda").bfloat16()
    pm = torch.randn(splits, H, n, device="cuda") * 3
    pl = torch.rand(splits, H, n, device="cuda") * 5 + 0.1
    if splits > 1:  # a dead split for every row of head 1, a row dead in all but one split
        pm[0, 1] = float("-inf")
        pm[1:, 0, 7] = float("-inf")
    out = torch.empty(n, D, device="cuda", dtype=torch.bfloat16)
    rmax = torch.empty(H, n, device="cuda")
    rsum = torch.empty(H, n, device="cuda")
    _abi.check(_abi.lib().ifx_attn_combine(po.data_ptr(), D, pm.data_ptr(), pl.data_ptr(), splits, n,
                                           H, hd, out.data_ptr(), D, rmax.data_ptr(), rsum.data_ptr(),
                                           stream_ptr()), "combine")
    torch.cuda.synchronize()
    M = pm.double().amax(0)                                   # [H, n]
    w = torch.where(pm.isinf(), torch.zeros_like(pl.double()), pl.double() * torch.exp2(pm.double() - M))
    den = w.sum(0)                                            # [H, n]
    o = po.double().view(splits, n, H, hd)
    want = (o * w.permute(0, 2, 1)[..., None]).sum(0) / den.t()[..., None]
    assert torch.allclose(out.double().view(n, H, hd), want, atol=2e-2, rtol=1e-2)
    assert torch.allclose(rsum.double(), den, rtol=1e-4) and torch.allclose(rmax.double(), M)


def test_native_comm_world1_all_to_all_and_all_gather():
    """ifx_comm_* on one GPU (NCCL allows one rank per device, so world 1 here; the
    multi-rank exchange is the same NCCL group call UlyssesComm.a2a_var makes): the
    variable-size byte all-to-all and the all-gather, also inside a CUDA graph."""
    from paper_2511_20714_b200.parallel import NativeComm

    comm = NativeComm(NativeComm.unique_id(), 1, 0)
    try:
        send = torch.arange(1000, device="cuda", dtype=torch.float32)
        recv = torch.zeros(1200, device="cuda")
        comm.all_to_all(send, [1000], recv, [1000])
        torch.cuda.synchronize()
        assert torch.equal(recv[:1000], send) and not recv[1000:].any()
        g = torch.zeros(64, device="cuda", dtype=torch.uint8)
        h = torch.randint(0, 255, (64,), device="cuda", dtype=torch.uint8)  # e.g. an IPC handle
        comm.all_gather(h, g)
        torch.cuda.synchronize()
        assert torch.equal(g, h)
        s = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            graph.capture_begin()
            comm.all_to_all(send, [1000], recv, [1000], stream=s)
            graph.capture_end()
        send.mul_(3)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(recv[:1000], send)
        del graph
    finally:
        comm.close()
