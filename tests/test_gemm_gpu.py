"""G1 (csrc/gemm_sm100.cu), the hand-written tcgen05 GEMM behind the engine's projections,
against a plain PyTorch fp32 reference of the same op (the bf16 operands upcast).

Tolerances: bf16 output = one bf16 rounding of an fp32 accumulation (rel 2^-8 of the
largest |value| in the row block, plus fp32 summation-order noise); fp32 output 1e-3 rel.
The fused page write is bit-exact against the bf16 output columns it copies.
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev():
    from paper_2511_20714_b200 import _device as D
    return D


def _ref(a, b):
    return a.float() @ b.float()


def _close(got, want, rel=1.0 / 128):
    scale = want.abs().amax(dim=1, keepdim=True).clamp_min(1e-6)
    err = ((got.float() - want).abs() / scale).max().item()
    assert err <= rel, err
    return err


@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (100, 40, 40), (300, 192, 1536), (4680, 1536, 1536),
                                   (4680, 4608, 1536), (4680, 1536, 3072), (777, 3072, 200),
                                   (4680, 5120, 5120)])
def test_gemm_bf16_out_vs_torch(M, N, K):
    D = _dev()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(K, N, device="cuda", generator=g) / K ** 0.5).bfloat16()
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    D.gemm_fused(a, b, out)
    _close(out, _ref(a, b))


def test_gemm_strided_operands_and_relu():
    """A and C as column slices of wider buffers (the QKV / attention layouts), ReLU."""
    D = _dev()
    g = torch.Generator(device="cuda").manual_seed(1)
    abuf = torch.randn(500, 3 * 256, device="cuda", generator=g).bfloat16()
    a = abuf[:, 256:512]
    b = (torch.randn(256, 320, device="cuda", generator=g) / 16).bfloat16()
    cbuf = torch.zeros(500, 640, device="cuda", dtype=torch.bfloat16)
    c = cbuf[:, 64:384]
    D.gemm_fused(a, b, c, relu=True)
    _close(c, torch.relu(_ref(a, b)))
    assert (cbuf[:, :64] == 0).all() and (cbuf[:, 384:] == 0).all()


def test_gemm_residual_emit_and_row_scale():
    """fp32 residual C = C + A B with the next norm's statistics emitted, then a consumer
    GEMM that applies the RMS row scale (engine.py:171-173) after its product."""
    D = _dev()
    M, Dm = 4680, 1536
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(M, Dm, device="cuda", generator=g)
    x0 = x.clone()
    a = torch.randn(M, 1536, device="cuda", generator=g).bfloat16()
    w = (torch.randn(1536, Dm, device="cuda", generator=g) / 40).bfloat16()
    tiles = D.gemm_tiles_n(M, Dm, 1536)
    norm = D.RowNorm(torch.empty(M, Dm, device="cuda", dtype=torch.bfloat16),
                     torch.full((M, tiles), float("nan"), device="cuda"), 0, Dm)
    parts = D.gemm_fused(a, w, x, beta=1.0, norm_out=norm)
    assert parts == tiles == norm.parts  # sum-of-squares parts per row
    want = x0 + _ref(a, w)
    assert ((x - want).abs().max() / want.abs().max()).item() < 1e-5
    assert torch.equal(norm.rows_bf16, x.bfloat16())
    ss = norm.ss.double().sum(1)
    assert torch.allclose(ss, (x.double() ** 2).sum(1), rtol=1e-5)
    # consumer: h = rms(x) (fp32), out = h @ w2, here as bf16(x) @ w2 * rsqrt(mean + eps)
    w2 = (torch.randn(Dm, 4608, device="cuda", generator=g) / 40).bfloat16()
    out = torch.empty(M, 4608, device="cuda", dtype=torch.bfloat16)
    D.gemm_fused(norm.rows_bf16, w2, out, norm_in=norm)
    h = x / torch.sqrt((x * x).mean(1, keepdim=True) + 1e-6)
    _close(out, _ref(h.bfloat16(), w2), rel=1.0 / 64)  # bf16(x) vs bf16(h) operand rounding


def test_gemm_fp32_out_beta0_and_bad_args():
    from paper_2511_20714_b200.errors import DimensionError

    D = _dev()
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(129, 96, device="cuda", generator=g).bfloat16()
    b = torch.randn(96, 40, device="cuda", generator=g).bfloat16()
    out = torch.full((129, 40), 7.0, device="cuda")
    D.gemm_fused(a, b, out)
    assert ((out - _ref(a, b)).abs().max() / _ref(a, b).abs().max()).item() < 1e-5
    with pytest.raises(DimensionError):
        D.gemm_fused(a, b[:, :36], out[:, :36])  # N % 8
    with pytest.raises(DimensionError):
        D.gemm_fused(a, b, out.bfloat16(), beta=1.0)  # beta needs fp32 C


def test_gemm_rope_epilogue_vs_separate_pass():
    """3D RoPE fused into the QKV epilogue == QKV GEMM then the rope_qk kernel (up to the
    extra bf16 rounding of the unfused path)."""
    from paper_2511_20714_b200 import engine as E

    D = _dev()
    H, dh, T = 4, 128, 3 * 64
    Dp = H * dh
    cfg = E.ModelConfig(layers=1, heads=H, head_dim=dh, block_len=T, frame_shape=(4, 4),
                        prompt_dim=8, rope_grid=(3, 8, 8))
    cos, sin = E.rope_tables(cfg, 2, torch.device("cuda"))
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.randn(T, Dp, device="cuda", generator=g).bfloat16()
    w = (torch.randn(Dp, 3 * Dp, device="cuda", generator=g) / 20).bfloat16()
    pairs = dh // 2
    fused = torch.empty(T, 3 * Dp, device="cuda", dtype=torch.bfloat16)
    D.gemm_fused(a, w, fused, rope=(cos, sin, 0, pairs, dh, H, 0, Dp))
    ref = _ref(a, w)
    sep = ref.bfloat16().clone()
    D.rope_qk(sep, H, dh, pairs, 0, Dp, cos, sin)
    _close(fused, sep.float(), rel=1.0 / 64)
    _close(fused[:, 2 * Dp:], ref[:, 2 * Dp:])  # V is not rotated
    # exact check of the math on fp32: rotate the fp32 product by the tables
    r = ref[:, :2 * Dp].reshape(T, 2, H, pairs, 2)
    c, s = cos[:T].reshape(T, 1, 1, pairs), sin[:T].reshape(T, 1, 1, pairs)
    rot = torch.stack([r[..., 0] * c - r[..., 1] * s, r[..., 0] * s + r[..., 1] * c], -1)
    _close(fused[:, :2 * Dp], rot.reshape(T, 2 * Dp))


@pytest.mark.parametrize("page_len,token0", [(16, 0), (16, 4680 * 2), (8, 3)])
def test_gemm_page_write_epilogue(page_len, token0):
    """The clean pass's page write fused into the QKV epilogue: K / V columns land in the
    slots of their pages (device and mapped-host pool), bit-identical to the QKV output."""
    from paper_2511_20714_b200 import _abi

    D = _dev()
    T, Dp = 4680, 1536
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(T, Dp, device="cuda", generator=g).bfloat16()
    w = (torch.randn(Dp, 3 * Dp, device="cuda", generator=g) / 40).bfloat16()
    first = token0 - (token0 % page_len)
    n_pages = -(-(token0 + T - first) // page_len)
    rng = np.random.default_rng(page_len)
    dev_slots = rng.permutation(n_pages + 5)[:n_pages]
    codes = np.where(rng.random(n_pages) < 0.2, -1 - np.arange(n_pages), dev_slots).astype(np.int32)
    slots = torch.from_numpy(codes).cuda()
    dev_k = torch.zeros((n_pages + 5) * page_len, Dp, device="cuda", dtype=torch.bfloat16)
    dev_v = torch.zeros_like(dev_k)
    hb = n_pages * page_len * Dp * 2
    hk, hv = ctypes.c_void_p(), ctypes.c_void_p()
    _abi.check(_abi.lib().ifx_host_alloc(hb, ctypes.byref(hk)))
    _abi.check(_abi.lib().ifx_host_alloc(hb, ctypes.byref(hv)))
    try:
        pool = _abi.KvPool()
        pool.dev_k, pool.dev_v, pool.host_k, pool.host_v = dev_k.data_ptr(), dev_v.data_ptr(), hk, hv
        pool.width, pool.page_len, pool.type = Dp, page_len, _abi.BF16
        qkv = torch.empty(T, 3 * Dp, device="cuda", dtype=torch.bfloat16)
        D.gemm_fused(a, w, qkv, page=(pool, slots, first, token0, Dp, 2 * Dp))
        torch.cuda.synchronize()
        host_k = np.ctypeslib.as_array(ctypes.cast(hk, ctypes.POINTER(ctypes.c_uint16)), (hb // 2,))
        host_v = np.ctypeslib.as_array(ctypes.cast(hv, ctypes.POINTER(ctypes.c_uint16)), (hb // 2,))
        dk = dev_k.view(torch.int16).cpu().numpy().view(np.uint16)
        dv = dev_v.view(torch.int16).cpu().numpy().view(np.uint16)
        want = qkv.view(torch.int16).cpu().numpy().view(np.uint16)
        for r in range(T):
            rel = token0 + r - first
            code = int(codes[rel // page_len])
            row = (code if code >= 0 else -1 - code) * page_len + rel % page_len
            if code >= 0:
                gk, gv = dk[row], dv[row]
            else:
                gk, gv = host_k[row * Dp:(row + 1) * Dp], host_v[row * Dp:(row + 1) * Dp]
            assert np.array_equal(gk, want[r, Dp:2 * Dp]), r
            assert np.array_equal(gv, want[r, 2 * Dp:]), r
        _close(qkv, _ref(a, w))
    finally:
        torch.cuda.synchronize()
        _abi.lib().ifx_host_free(hk)
        _abi.lib().ifx_host_free(hv)


def test_gemm_inside_cuda_graph():
    """G1 launches are capturable (the engine replays its denoise passes as graphs)."""
    D = _dev()
    g = torch.Generator(device="cuda").manual_seed(6)
    a = torch.randn(4680, 1536, device="cuda", generator=g).bfloat16()
    b = (torch.randn(1536, 1536, device="cuda", generator=g) / 40).bfloat16()
    out = torch.empty(4680, 1536, device="cuda", dtype=torch.bfloat16)
    D.gemm_fused(a, b, out)
    eager = out.clone()
    out.zero_()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        graph.capture_begin()
        D.gemm_fused(a, b, out, stream=s)
        graph.capture_end()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


@pytest.mark.parametrize("mode", ["all", "qkv"])
@pytest.mark.parametrize("case", [
    dict(rope_grid=None, cap=10**6),
    dict(rope_grid=(2, 8, 8), cap=10**6),
    dict(rope_grid=(2, 8, 8), cap=24),   # device tier full: fused page writes to host pages
])
def test_engine_g1_paths_vs_oracle(monkeypatch, mode, case):
    """The engine with G1 on every projection ("all": RMS norms fused into the epilogues,
    engine.py:171-173) or on the QKV projection only ("qkv": RoPE + clean-pass page write
    in its epilogue) vs the numpy oracle: latents within the stated tolerance, page table
    bit-exact (also when the fused page write lands on pinned-host pages)."""
    from oracle import engine as OE
    from paper_2511_20714_b200 import engine as E

    monkeypatch.setattr(E, "G1", mode)
    kw = dict(layers=2, heads=4, head_dim=64, block_len=128, frame_shape=(4, 4), prompt_dim=8,
              rope_grid=case["rope_grid"])
    req = dict(num_blocks=3, seed=4, prompt_schedule=[(0, "a b c"), (2, "d")])
    sched = [1.0, 0.5]
    mc = E.ModelConfig(**kw)
    model = E.build_model(mc)
    eng = E.Engine(model, E.default_kv_config(mc, capacity_pages_device=case["cap"],
                                              capacity_pages_host=4096))
    got = np.stack([b.latent for b in eng.generate(E.GenerationRequest(
        schedule=E.DenoiseSchedule(sched), **req))])
    r = E._runner(model)
    assert (r.g1, r.g1_qkv) == ((True, False) if mode == "all" else (False, True))
    omc = OE.ModelConfig(**kw)
    want, ocache = OE.generate_sequence(OE.ToyModel(omc), OE.GenerationRequest(
        schedule=OE.DenoiseSchedule(sched), **req),
        kv_config=OE.default_kv_config(omc, capacity_pages_device=case["cap"], capacity_pages_host=4096))
    want = np.stack(want)
    a, b = got.ravel().astype(np.float64), want.ravel().astype(np.float64)
    cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
    assert np.abs(got - want).max() <= 2e-2 and cos > 0.999
    assert eng.cache.state() == ocache.state()
