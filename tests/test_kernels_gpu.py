"""GPU numerics of the individual kernels vs plain PyTorch fp32 references.

K1 attention, K2 append, K7 gather, fused RMS, Ulysses pack/unpack.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_attn(q, k, v, heads, scale=None, mask=None):
    n, d = q.shape
    dh = d // heads
    scale = scale or 1.0 / math.sqrt(dh)
    qf, kf, vf = q.float(), k.float(), v.float()
    outs = []
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        s = (qf[:, sl] @ kf[:, sl].T) * scale
        if mask is not None:
            s = s.masked_fill(~mask, float("-inf"))
        outs.append(torch.softmax(s, dim=1) @ vf[:, sl])
    return torch.cat(outs, dim=1)


CASES = [
    # heads, head_dim, n_q, n_ctx, ctx_row0, n_cur
    (12, 128, 4680, 9360, 0, 4680),   # c2 shape, 2 cached blocks (split-KV path)
    (2, 128, 700, 5000, 3, 300),
    (3, 64, 300, 2600, 0, 257),
    (2, 64, 128, 0, 0, 128),
    (1, 128, 128, 0, 0, 128),
    (4, 64, 768, 768, 0, 768),
    (3, 128, 200, 300, 5, 77),
    (2, 128, 130, 1000, 17, 0),
    (12, 128, 520, 384, 0, 520),
    (1, 128, 64, 3, 0, 0),
    (2, 64, 33, 0, 0, 2),
    # K1s (few keys: cross-attention to a prompt), dispatched inside ifx_attn_fwd
    (12, 128, 4680, 3, 0, 0),
    (12, 128, 1000, 3, 5, 2),
    (4, 64, 600, 0, 0, 17),
    (40, 128, 300, 8, 1, 0),
    (40, 128, 300, 32, 1, 0),
    (3, 128, 400, 33, 0, 0),   # 33 keys: K1 (K1s takes <= 32)
]


@pytest.mark.parametrize("case", CASES)
def test_attention_matches_torch(case):
    from paper_2511_20714_b200._device import attn_fwd

    heads, hd, n_q, n_ctx, row0, n_cur = case
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 2**31)
    dev = "cuda"
    q = torch.randn(n_q, d, device=dev, generator=g).bfloat16()
    slab_rows = row0 + n_ctx + 40
    ks = torch.randn(slab_rows, d, device=dev, generator=g).bfloat16()
    vs = torch.randn(slab_rows, d, device=dev, generator=g).bfloat16()
    qkv = torch.randn(max(n_cur, 1), 3 * d, device=dev, generator=g).bfloat16()[:n_cur]
    kc, vc = qkv[:, d:2 * d], qkv[:, 2 * d:]
    out = torch.empty(n_q, d, device=dev, dtype=torch.bfloat16)
    attn_fwd(q, heads, hd, out, ks, vs, row0, n_ctx, kc if n_cur else None, vc if n_cur else None)
    torch.cuda.synchronize()
    k = torch.cat([ks[row0:row0 + n_ctx], kc])
    v = torch.cat([vs[row0:row0 + n_ctx], vc])
    ref = _ref_attn(q, k, v, heads)
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2, err


def test_attention_large_scores_and_masks():
    """Large logits exercise the lazy-rescale path; a dense mask exercises masking."""
    from paper_2511_20714_b200._device import attn_fwd

    heads, hd, n_q, n = 2, 128, 256, 700
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(5)
    q = (torch.randn(n_q, d, device="cuda", generator=g) * 3).bfloat16()
    k = (torch.randn(n, d, device="cuda", generator=g) * 3).bfloat16()
    # increasing key scale so the running max keeps growing across tiles
    k = (k.float() * torch.linspace(0.2, 2.0, n, device="cuda")[:, None]).bfloat16()
    v = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    mask = torch.rand(n_q, n, device="cuda", generator=g) < 0.6
    mask[:, 0] = True
    out = torch.empty(n_q, d, device="cuda", dtype=torch.bfloat16)
    attn_fwd(q, heads, hd, out, k, v, 0, n)
    torch.cuda.synchronize()
    ref = _ref_attn(q, k, v, heads)
    assert (out.float() - ref).abs().max().item() < 3e-2
    m8 = mask.to(torch.uint8).contiguous()
    attn_fwd(q, heads, hd, out, k, v, 0, n, mask=m8)
    torch.cuda.synchronize()
    ref = _ref_attn(q, k, v, heads, mask=mask)
    assert (out.float() - ref).abs().max().item() < 3e-2


@pytest.mark.parametrize("heads,n_q,n", [(5, 4680, 3000), (12, 2000, 1500)])
def test_attention_persistent_items_rescale_and_mask(heads, n_q, n):
    """More items than SMs (185 / 192 items on 148 persistent CTAs, uneven items per CTA):
    every item restarts its online softmax and reuses the TMEM accumulators and S buffers
    of the previous one; growing logits force O rescales inside each item."""
    from paper_2511_20714_b200._device import attn_fwd

    hd = 128
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(heads * 7 + n)
    q = (torch.randn(n_q, d, device="cuda", generator=g) * 2).bfloat16()
    k = torch.randn(n, d, device="cuda", generator=g)
    k = (k * torch.linspace(0.1, 2.5, n, device="cuda")[:, None]).bfloat16()
    v = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    out = torch.empty(n_q, d, device="cuda", dtype=torch.bfloat16)
    attn_fwd(q, heads, hd, out, k, v, 0, n)
    torch.cuda.synchronize()
    ref = _ref_attn(q, k, v, heads)
    assert (out.float() - ref).abs().max().item() < 3e-2
    mask = torch.rand(n_q, n, device="cuda", generator=g) < 0.5
    mask[:, n // 2] = True
    attn_fwd(q, heads, hd, out, k, v, 0, n, mask=mask.to(torch.uint8).contiguous())
    torch.cuda.synchronize()
    ref = _ref_attn(q, k, v, heads, mask=mask)
    assert (out.float() - ref).abs().max().item() < 3e-2


def test_attention_persistent_split_kv():
    """5 heads x 37 query tiles under-fill 148 SMs, so the key range is split (4 ways here):
    740 items, 5 per persistent CTA, each writing a partial merged by K4."""
    from paper_2511_20714_b200._device import attn_fwd

    heads, hd, n_q, n_ctx = 5, 128, 4680, 9000
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn(n_q, d, device="cuda", generator=g).bfloat16()
    ks = (torch.randn(n_ctx, d, device="cuda", generator=g)
          * torch.linspace(0.3, 1.8, n_ctx, device="cuda")[:, None]).bfloat16()
    vs = torch.randn(n_ctx, d, device="cuda", generator=g).bfloat16()
    qkv = torch.randn(n_q, 3 * d, device="cuda", generator=g).bfloat16()
    out = torch.empty(n_q, d, device="cuda", dtype=torch.bfloat16)
    attn_fwd(q, heads, hd, out, ks, vs, 0, n_ctx, qkv[:, d:2 * d], qkv[:, 2 * d:])
    torch.cuda.synchronize()
    ref = _ref_attn(q, torch.cat([ks, qkv[:, d:2 * d]]), torch.cat([vs, qkv[:, 2 * d:]]), heads)
    assert (out.float() - ref).abs().max().item() < 2e-2


def _pool(kd, vd, hk, hv, w, page_len, dt):
    from paper_2511_20714_b200 import _abi
    p = _abi.KvPool()
    p.dev_k, p.dev_v = kd.data_ptr(), vd.data_ptr()
    p.host_k, p.host_v = hk, hv
    p.width, p.page_len = w, page_len
    p.type = _abi.BF16 if dt == torch.bfloat16 else _abi.F32
    return p


def test_kv_append_gather_move_bit_exact():
    """K2 / K7 / K6 over a device pool + a mapped pinned host pool, scattered slots."""
    import ctypes

    from paper_2511_20714_b200 import _abi
    from paper_2511_20714_b200._device import stream_ptr
    from paper_2511_20714_b200.kvcache import _HostBuf

    L = _abi.lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    code = lambda dt: _abi.BF16 if dt == torch.bfloat16 else _abi.F32  # noqa: E731
    for src_dt, dst_dt in [(torch.float32, torch.float32), (torch.float32, torch.bfloat16),
                           (torch.bfloat16, torch.bfloat16)]:
        t, w, P = 37, 256, 8
        esz = 2 if dst_dt == torch.bfloat16 else 4
        src = torch.randn(t, 3 * w, device="cuda", generator=g).to(src_dt)
        ks, vs = src[:, w:2 * w], src[:, 2 * w:]
        kd = torch.zeros(10 * P, w, device="cuda", dtype=dst_dt)
        vd = torch.zeros_like(kd)
        hk, hv = _HostBuf(6 * P * w * esz), _HostBuf(6 * P * w * esz)
        pool = _pool(kd, vd, hk.ptr, hv.ptr, w, P, dst_dt)
        # stream tokens [first, ...): token0 = first + 3 sits mid-page; pages on both tiers
        slots_np = [7, -1 - 4, 2, -1 - 0, 9, 5]
        slots = torch.tensor(slots_np, device="cuda", dtype=torch.int32)
        first, token0 = 32, 35
        _abi.check(L.ifx_kv_append(ks.data_ptr(), vs.data_ptr(), 3 * w, code(src_dt), ctypes.byref(pool),
                                   slots.data_ptr(), first, token0, t, stream_ptr()))
        torch.cuda.synchronize()
        hk_t = hk.bytes_view().view(dst_dt).view(-1, w)
        for r in range(t):
            rel = token0 + r - first
            c = slots_np[rel // P]
            row = (c if c >= 0 else -1 - c) * P + rel % P
            got = kd[row].cpu() if c >= 0 else hk_t[row]
            assert torch.equal(got, ks[r].to(dst_dt).cpu()), (r, c)
        toks = torch.tensor([36, 35, 70, 36, 60], device="cuda", dtype=torch.int64)
        ko = torch.empty(5, w, device="cuda", dtype=dst_dt)
        vo = torch.empty_like(ko)
        _abi.check(L.ifx_kv_gather(ctypes.byref(pool), slots.data_ptr(), first, toks.data_ptr(), 0, 5,
                                   ko.data_ptr(), vo.data_ptr(), stream_ptr()))
        torch.cuda.synchronize()
        idx = (toks - token0).long()
        assert torch.equal(ko, ks.to(dst_dt)[idx]) and torch.equal(vo, vs.to(dst_dt)[idx])
        ko2 = torch.empty(t, w, device="cuda", dtype=dst_dt)
        vo2 = torch.empty_like(ko2)
        _abi.check(L.ifx_kv_gather(ctypes.byref(pool), slots.data_ptr(), first, None, token0, t,
                                   ko2.data_ptr(), vo2.data_ptr(), stream_ptr()))
        torch.cuda.synchronize()
        assert torch.equal(ko2, ks.to(dst_dt)) and torch.equal(vo2, vs.to(dst_dt))
        # K6: device slot 7 -> host slot 5, host slot 4 -> device slot 0 (whole pages)
        before_d7, before_h4 = kd[7 * P:8 * P].cpu().clone(), hk_t[4 * P:5 * P].clone()
        for d, pairs in ((0, [[7, 5]]), (1, [[0, 4]])):
            mv = torch.tensor(pairs, device="cuda", dtype=torch.int64)
            _abi.check(L.ifx_kv_move_pages(ctypes.byref(pool), mv.data_ptr(), 1, d, stream_ptr()))
        torch.cuda.synchronize()
        assert torch.equal(hk_t[5 * P:6 * P], before_d7)
        assert torch.equal(kd[0:P].cpu(), before_h4)


PAGED = [
    # heads, head_dim, page_len, n_ctx, lo (window start inside the first page), n_cur, staged
    (12, 128, 16, 9360, 0, 4680, False),
    (2, 128, 16, 5000, 5, 300, True),
    (3, 64, 8, 2600, 3, 257, True),
    (2, 128, 32, 1000, 31, 0, False),
    (1, 128, 128, 700, 100, 64, True),
    (4, 64, 64, 37, 0, 128, True),
]


@pytest.mark.parametrize("case", PAGED)
def test_paged_attention_matches_torch(case):
    """K1 paged mode: context pages scattered over the pool (and the staging pool for
    negative codes), window start inside the first page."""
    import numpy as np

    from paper_2511_20714_b200._device import attn_fwd, tile_run_codes

    heads, hd, P, n_ctx, lo, n_cur, staged = case
    d = heads * hd
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 2**31)
    n_q = 300
    rows = lo + n_ctx
    n_pages = -(-rows // P)
    k_log = torch.randn(n_pages * P, d, device="cuda", generator=g).bfloat16()
    v_log = torch.randn(n_pages * P, d, device="cuda", generator=g).bfloat16()
    perm = torch.randperm(n_pages + 5, generator=torch.Generator().manual_seed(3))[:n_pages]
    pool_k = torch.zeros((n_pages + 5) * P, d, device="cuda", dtype=torch.bfloat16)
    pool_v = torch.zeros_like(pool_k)
    stage_k = torch.zeros(n_pages * P, d, device="cuda", dtype=torch.bfloat16)
    stage_v = torch.zeros_like(stage_k)
    codes = []
    for i in range(n_pages):
        src = slice(i * P, (i + 1) * P)
        if staged and i % 3 == 1:
            stage_k[i * P:(i + 1) * P], stage_v[i * P:(i + 1) * P] = k_log[src], v_log[src]
            codes.append(-1 - i)
        else:
            s = int(perm[i])
            pool_k[s * P:(s + 1) * P], pool_v[s * P:(s + 1) * P] = k_log[src], v_log[src]
            codes.append(s)
    slots = torch.tensor(codes, device="cuda", dtype=torch.int32)
    q = torch.randn(n_q, d, device="cuda", generator=g).bfloat16()
    qkv = torch.randn(max(n_cur, 1), 3 * d, device="cuda", generator=g).bfloat16()[:n_cur]
    kc, vc = qkv[:, d:2 * d], qkv[:, 2 * d:]
    out = torch.empty(n_q, d, device="cuda", dtype=torch.bfloat16)
    first = 1000 * P
    k = torch.cat([k_log[lo:lo + n_ctx], kc])
    v = torch.cat([v_log[lo:lo + n_ctx], vc])
    ref = _ref_attn(q, k, v, heads)
    # with and without the per-tile run table; a run table over consecutive slots too
    runs = torch.from_numpy(tile_run_codes(np.array(codes, np.int32), P)).cuda()
    for tr in (None, runs):
        out.zero_()
        attn_fwd(q, heads, hd, out, pool_k, pool_v, first + lo, n_ctx, kc if n_cur else None,
                 vc if n_cur else None, ctx_slots=slots, page_len=P, first_token=first,
                 stage_k=stage_k if staged else None, stage_v=stage_v if staged else None,
                 tile_runs=tr)
        torch.cuda.synchronize()
        err = (out.float() - ref).abs().max().item()
        assert err < 2e-2, err
    # the same context laid out in consecutive slots: every full tile is a run
    seq = torch.arange(n_pages, device="cuda", dtype=torch.int32)
    runs = torch.from_numpy(tile_run_codes(np.arange(n_pages, dtype=np.int32), P)).cuda()
    attn_fwd(q, heads, hd, out, k_log, v_log, first + lo, n_ctx, kc if n_cur else None,
             vc if n_cur else None, ctx_slots=seq, page_len=P, first_token=first, tile_runs=runs)
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("width", [1536, 200, 5120])
def test_rms_matches_torch(width):
    """Rows up to 1,536 wide stay in registers (one read of x); wider rows take two passes."""
    from paper_2511_20714_b200._device import rms_bf16

    x = torch.randn(777, width, device="cuda")
    tv = torch.randn(width, device="cuda")
    y = torch.empty(777, width, device="cuda", dtype=torch.bfloat16)
    xo = torch.empty_like(x)
    rms_bf16(x, y, tv, 0.75, xo)
    torch.cuda.synchronize()
    xc = x + 0.75 * tv
    ref = xc / torch.sqrt((xc * xc).mean(-1, keepdim=True) + 1e-6)
    assert torch.allclose(xo, xc, atol=1e-5)
    assert (y.float() - ref).abs().max().item() < 2e-2
    rms_bf16(x, y)  # no time conditioning
    torch.cuda.synchronize()
    ref = x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6)
    assert (y.float() - ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("groups", [1, 3])
def test_ulysses_pack_unpack_roundtrip(groups):
    from paper_2511_20714_b200 import _abi
    from paper_2511_20714_b200._device import stream_ptr

    L = _abi.lib()
    n, world, chunk = 93, 4, 384
    width = groups * world * chunk
    x = torch.randn(n, width + 64, device="cuda").bfloat16()  # row stride > width
    packed = torch.empty(world, n, groups, chunk, device="cuda", dtype=torch.bfloat16)
    _abi.check(L.ifx_ulysses_pack(x.data_ptr(), n, groups, world, chunk, width + 64, _abi.BF16,
                                  packed.data_ptr(), stream_ptr()))
    back = torch.zeros(n, width, device="cuda", dtype=torch.bfloat16)
    _abi.check(L.ifx_ulysses_unpack(packed.data_ptr(), n, groups, world, chunk, _abi.BF16,
                                    back.data_ptr(), width, stream_ptr()))
    torch.cuda.synchronize()
    ref = x[:, :width].reshape(n, groups, world, chunk).permute(2, 0, 1, 3)
    assert torch.equal(packed, ref)
    assert torch.equal(back, x[:, :width])


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(4680, 4608, 1536), (4680, 1536, 3072), (77, 96, 64)])
def test_gemm_lt_matches_torch(M, N, K):
    """ifx_gemm_bf16 (cuBLASLt, per-shape algorithm) against fp32 torch: bf16 out, fp32 out,
    fp32 residual with beta = 1 and the ReLU epilogue."""
    from paper_2511_20714_b200._device import gemm
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(K, N, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ref = a.float() @ b.float()
    o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gemm(a, b, o16)
    torch.testing.assert_close(o16.float(), ref, atol=2e-2, rtol=1e-2)
    o32 = torch.randn(M, N, device="cuda", generator=g)
    x0 = o32.clone()
    gemm(a, b, o32, beta=1.0)
    torch.testing.assert_close(o32, x0 + ref, atol=2e-3, rtol=1e-3)
    gemm(a, b, o16, relu=True)
    torch.testing.assert_close(o16.float(), ref.clamp_min(0), atol=2e-2, rtol=1e-2)
    # a strided A (a column block of a wider buffer), as the engine passes it
    wide = torch.randn(M, K + 64, device="cuda", generator=g).bfloat16()
    gemm(wide[:, 32:32 + K], b, o32)
    torch.testing.assert_close(o32, wide[:, 32:32 + K].float() @ b.float(), atol=2e-3, rtol=1e-3)
