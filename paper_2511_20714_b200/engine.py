"""Generate-and-cache block-diffusion loop on B200 — drop-in for `inferix.engine`.

Reference: /root/reference/pkg/src/inferix/engine.py. Same public surface (ModelConfig,
DenoiseSchedule, GenerationRequest, GeneratedBlock, ToyModel/build_model, embed_prompt,
denoise_step, decode_frames, generate_block, default_kv_config, Engine,
generate_sequence, Pipeline registry) and the same semantics:
  * weights drawn from one PCG64 stream in the reference's order (engine.py:120-144),
    noise from default_rng([seed, chunk]) (engine.py:280-282) — bit-identical inputs;
  * S Euler steps then a clean t=0 pass whose K/V are appended to the cache
    (engine.py:285-312); prompt switches clear the cross streams (engine.py:382-391);
    window eviction after each block (engine.py:403-404);
  * KV-cache bookkeeping calls in the reference's order (context fetch once per block,
    engine.py:228-250) so page ids / tiers / access clock match bit-for-bit.

What changes is where it runs: one CUDA stream; per layer a fused RMS-norm kernel, one
bf16 QKV GEMM (cuBLAS), K1 attention reading the cached context IN PLACE from the HBM
slab plus the block's own K/V straight out of the QKV buffer (no concat, no gather),
K2 page write on the clean pass, fp32 residual stream (GEMMs with fp32 output).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import threading
import time
import weakref
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _abi, _device
from ._device import (RowNorm, attn_fwd, count_launch, gemm, gemm_fused, gemm_tiles_n,
                      require_cuda, rms_bf16, rope_qk, stream_ptr, tile_run_codes)
from .errors import ConfigError, DimensionError
from .kvcache import CROSS_ATTN, SELF_ATTN, KvCache, KvConfig

LAYER_FIELDS = ("wq", "wk", "wv", "wo", "cq", "ck", "cv", "co", "w1", "w2")  # engine.py:131-138


@dataclass
class ModelConfig:
    """engine.py:29-48."""
    layers: int = 2
    heads: int = 2
    head_dim: int = 8
    block_len: int = 16
    frame_shape: tuple = (16, 16)
    prompt_dim: int = 16
    weight_seed: int = 0
    # B200 extension (the reference has no positional encoding, attention.py:6): 3D RoPE on
    # Q/K over (frames_per_block, latent_h, latent_w); None = off (reference semantics)
    rope_grid: tuple | None = None
    rope_theta: float = 10000.0

    def validate(self):
        for name in ("layers", "heads", "head_dim", "block_len", "prompt_dim"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be >= 1")
        if self.frame_shape[0] < 1 or self.frame_shape[1] < 1:
            raise ConfigError("frame_shape must be positive")
        if self.rope_grid is not None and math.prod(self.rope_grid) != self.block_len:
            raise ConfigError("rope_grid must tile block_len")
        if self.rope_grid is not None and self.head_dim % 2:
            raise ConfigError("RoPE needs an even head_dim")

    @property
    def model_dim(self) -> int:
        return self.heads * self.head_dim


def rope_tables(cfg: ModelConfig, chunk: int, dev) -> tuple | None:
    """cos/sin [block_len, head_dim/2] fp32 on device for block `chunk` (None without RoPE).

    head_dim d splits into d - 4*(d//6) frame dims and 2*(d//6) each for latent row /
    column; token i of block b sits at frame b*F + i//(h*w), row (i % (h*w))//w, column
    i % w; pair k of a part of size n rotates by pos * theta^(-2k/n). Angles in fp64."""
    if cfg.rope_grid is None:
        return None
    F, gh, gw = cfg.rope_grid
    d = cfg.head_dim
    i = torch.arange(F * gh * gw, device=dev, dtype=torch.int64)
    pos = (chunk * F + i // (gh * gw), (i % (gh * gw)) // gw, i % gw)
    s = d // 6
    angs = []
    for p, n in zip(pos, (d - 4 * s, 2 * s, 2 * s)):
        inv = cfg.rope_theta ** (-torch.arange(0, n, 2, device=dev, dtype=torch.float64) / n)
        angs.append(p.to(torch.float64)[:, None] * inv[None, :])
    ang = torch.cat(angs, dim=1)
    return torch.cos(ang).float().contiguous(), torch.sin(ang).float().contiguous()


@dataclass
class DenoiseSchedule:
    """engine.py:51-62."""
    steps: list
    step_scale: float = 0.5

    def validate(self):
        if not self.steps:
            raise ConfigError("schedule needs at least one step")
        if any(t <= 0 for t in self.steps):
            raise ConfigError("noise levels must be > 0")
        if any(a <= b for a, b in zip(self.steps, self.steps[1:])):
            raise ConfigError("noise levels must be strictly decreasing")


@dataclass
class GenerationRequest:
    """engine.py:65-87."""
    num_blocks: int
    schedule: DenoiseSchedule
    seed: int = 0
    prompt_schedule: list = field(default_factory=lambda: [(0, "a quiet scene")])
    kv_window: int | None = None

    def validate(self):
        if self.num_blocks < 1:
            raise ConfigError("num_blocks must be >= 1")
        self.schedule.validate()
        if not self.prompt_schedule or self.prompt_schedule[0][0] != 0:
            raise ConfigError("prompt_schedule must start at chunk 0")
        chunks = [c for c, _ in self.prompt_schedule]
        if any(a >= b for a, b in zip(chunks, chunks[1:])):
            raise ConfigError("prompt_schedule chunks must be strictly increasing")
        if any(not text for _, text in self.prompt_schedule):
            raise ConfigError("prompts must be nonempty")
        if self.kv_window is not None and self.kv_window < 0:
            raise ConfigError("kv_window must be >= 0")


@dataclass
class GeneratedBlock:
    """engine.py:90-95 (latent as host numpy fp32, frames as uint8 [h, w] per token)."""
    chunk_index: int
    latent: np.ndarray
    frames: list
    prompt_in_effect: str


def padded_head_dim(head_dim: int) -> int:
    """K1 runs 64- or 128-wide heads; narrower heads are zero-padded (exact: zero q/k
    columns do not change q.k, zero V columns give zero outputs that meet zero rows of
    wo/co). The softmax scale stays 1/sqrt(head_dim)."""
    if head_dim <= 64:
        return 64
    if head_dim <= 128:
        return 128
    raise ConfigError("head_dim > 128 is not supported by the B200 attention kernel")


def _pad_cols(w: torch.Tensor, heads: int, heads_pad: int, dh: int, dhp: int) -> torch.Tensor:
    """[in, heads*dh] -> [in, heads_pad*dhp]: per-head zero columns + zero dummy heads."""
    if dh == dhp and heads == heads_pad:
        return w
    out = w.new_zeros(w.shape[0], heads_pad, dhp)
    out[:, :heads, :dh] = w.view(w.shape[0], heads, dh)
    return out.view(w.shape[0], heads_pad * dhp)


def _pad_rows(w: torch.Tensor, heads: int, heads_pad: int, dh: int, dhp: int) -> torch.Tensor:
    """[heads*dh, out] -> [heads_pad*dhp, out] with zero rows for padding."""
    if dh == dhp and heads == heads_pad:
        return w
    out = w.new_zeros(heads_pad, dhp, w.shape[1])
    out[:heads, :dh] = w.view(heads, dh, w.shape[1])
    return out.view(heads_pad * dhp, w.shape[1])


def _unpad_heads(x: torch.Tensor, heads: int, heads_pad: int, dh: int, dhp: int) -> torch.Tensor:
    """[n, heads_pad*dhp] (engine layout) -> [n, heads*dh] fp32 (the reference's layout)."""
    n = x.shape[0]
    return x.reshape(n, heads_pad, dhp)[:, :heads, :dh].reshape(n, heads * dh).float()


def _pad_heads(x: torch.Tensor, heads: int, heads_pad: int, dh: int, dhp: int, out: torch.Tensor):
    """[n, heads*dh] -> out [n, heads_pad*dhp] (zero padding, out's dtype)."""
    n = x.shape[0]
    o = out.view(n, heads_pad, dhp)
    if dh != dhp or heads != heads_pad:
        o.zero_()
    o[:, :heads, :dh] = torch.as_tensor(x, device=out.device).reshape(n, heads, dh)
    return out


def _mha(q, k, v, heads: int, mask):
    """engine.py:176-182 — the attention-processor hook: per head h, scaled_dot_attention
    of columns h*dh:(h+1)*dh of q [T, D] over k / v [m, D] under mask [T, m], concatenated
    to [T, D]. Here all heads run in ONE K1 launch (bf16 operands, fp32 softmax and
    accumulation); an all-true mask takes the unmasked fast path, anything else goes in as
    a dense mask. numpy in -> numpy out (like the reference); CUDA tensors in -> CUDA out.

    The engine's passes call the fused paged path directly (the context is read in place,
    never concatenated); if this module attribute is REPLACED (e.g. monkeypatched by a
    user processor), BlockRunner routes every self- and cross-attention through the
    replacement with the reference's arguments instead (eager, context gathered)."""
    from ._device import to_device
    from .errors import MaskError
    as_np = not isinstance(q, torch.Tensor)
    qt, kt, vt = (to_device(x, torch.float32) for x in (q, k, v))
    if qt.dim() != 2 or kt.dim() != 2 or vt.dim() != 2 or qt.shape[1] % heads or \
            kt.shape[1] != qt.shape[1] or vt.shape != kt.shape:
        raise DimensionError("_mha expects q [T, D], k / v [m, D] with D % heads == 0")
    for x, name in ((qt, "q"), (kt, "k"), (vt, "v")):
        if not bool(torch.isfinite(x).all()):
            raise DimensionError(f"{name} contains non-finite values")
    T, D = qt.shape
    m = kt.shape[0]
    dh = D // heads
    dhp = padded_head_dim(dh)
    mt = torch.as_tensor(np.asarray(mask, dtype=bool) if not isinstance(mask, torch.Tensor)
                         else mask, device=qt.device).bool()
    if tuple(mt.shape) != (T, m):
        raise DimensionError(f"mask shape {tuple(mt.shape)} != ({T}, {m})")
    if not bool(mt.any(dim=1).all()):
        raise MaskError("query row with no allowed key")
    bf = lambda x, n: _pad_heads(x, heads, heads, dh, dhp, torch.empty(  # noqa: E731
        n, heads * dhp, device=qt.device, dtype=torch.bfloat16))
    qp, kp, vp = bf(qt, T), bf(kt, m), bf(vt, m)
    out = torch.empty(T, heads * dhp, device=qt.device, dtype=torch.bfloat16)
    m8 = None if bool(mt.all()) else mt.to(torch.uint8).contiguous()
    attn_fwd(qp, heads, dhp, out, kp, vp, 0, m, scale=1.0 / math.sqrt(dh), mask=m8)
    res = _unpad_heads(out, heads, heads, dh, dhp)
    return res.cpu().numpy() if as_np else res


_MHA_DEFAULT = _mha


def _mha_hook():
    """The user's replacement of `_mha`, or None while the built-in one is in place."""
    h = globals()["_mha"]
    return None if h is _MHA_DEFAULT else h


class _LayerWeights:
    """Device weights of one layer: fused [D, 3Dp] QKV, bf16 GEMM operands (Dp = padded
    heads x padded head width; padding is exact zeros); the prompt projections ck/cv
    stay fp32 (they run once per prompt, engine.py:224-225)."""

    def __init__(self, w: dict, dev, heads: int, heads_pad: int, dh: int, dhp: int):
        f32 = lambda a: torch.as_tensor(a).to(dev, torch.float32)  # noqa: E731
        cols = lambda a: _pad_cols(f32(a), heads, heads_pad, dh, dhp)  # noqa: E731
        rows = lambda a: _pad_rows(f32(a), heads, heads_pad, dh, dhp)  # noqa: E731
        bf = torch.bfloat16
        self.wqkv = torch.cat([cols(w["wq"]), cols(w["wk"]), cols(w["wv"])], dim=1).to(bf).contiguous()
        self.wo, self.cq, self.co = rows(w["wo"]).to(bf), cols(w["cq"]).to(bf), rows(w["co"]).to(bf)
        self.w1, self.w2 = f32(w["w1"]).to(bf), f32(w["w2"]).to(bf)
        self.ck, self.cv = cols(w["ck"]).contiguous(), cols(w["cv"]).contiguous()


class ToyModel:
    """Seeded toy transformer denoiser (engine.py:112-150) with device-resident weights.

    weights="reference": identical PCG64 draws to the reference (bit-identical fp32
    source, then cast to bf16 for the GEMMs). weights="device": torch.randn on the GPU
    (same shapes / scales; for the 14B-shaped configs where host generation of ~10^10
    normals is impractical — not bit-comparable with the reference).

    head_multiple: pad the head count with zero dummy heads to a multiple of this (Ulysses
    over W ranks needs heads % W == 0, parallel.py:143-144; dummy heads output exact 0)."""

    def __init__(self, config: ModelConfig, weights: str = "reference", head_multiple: int = 1):
        config.validate()
        self.config = config
        dev = require_cuda()
        d, p = config.model_dim, config.prompt_dim
        h, wd = config.frame_shape
        self.dh_pad = padded_head_dim(config.head_dim)
        self.heads_pad = -(-config.heads // head_multiple) * head_multiple
        lw = lambda ws: _LayerWeights(ws, dev, config.heads, self.heads_pad, config.head_dim,  # noqa: E731
                                      self.dh_pad)
        shapes = {"wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d), "cq": (d, d),
                  "ck": (p, d), "cv": (p, d), "co": (d, d), "w1": (d, 2 * d), "w2": (2 * d, d)}
        if weights == "reference":
            rng = np.random.default_rng(np.random.PCG64(config.weight_seed))

            def draw(r, c):
                return rng.standard_normal((r, c)).astype(np.float32) * np.float32(0.5 / np.sqrt(r))

            self.layers = [lw({f: draw(*shapes[f]) for f in LAYER_FIELDS})
                           for _ in range(config.layers)]
            tv = draw(1, d)[0]
            wout = draw(d, d)
            wdec = rng.standard_normal((d, h * wd)).astype(np.float32) * np.float32(0.35)
        elif weights == "device":
            g = torch.Generator(device=dev).manual_seed(config.weight_seed)

            def draw(r, c):
                return torch.randn(r, c, device=dev, generator=g) * (0.5 / math.sqrt(r))

            self.layers = [lw({f: draw(*shapes[f]) for f in LAYER_FIELDS})
                           for _ in range(config.layers)]
            tv, wout = draw(1, d)[0], draw(d, d)
            wdec = torch.randn(d, h * wd, device=dev, generator=g) * 0.35
        else:
            raise ConfigError(f"unknown weights source {weights!r}")
        self.time_vec = torch.as_tensor(tv).to(dev, torch.float32).contiguous()
        self.w_out = torch.as_tensor(wout).to(dev, torch.bfloat16)
        self.w_decode = torch.as_tensor(wdec).to(dev, torch.float32)

    def num_parameters(self) -> int:
        """engine.py:146-150: L*(10D^2 + 2PD) + D + D^2 + D*H*W."""
        c = self.config
        d, p = c.model_dim, c.prompt_dim
        h, w = c.frame_shape
        return c.layers * (10 * d * d + 2 * p * d) + d + d * d + d * h * w

    @property
    def attn_width(self) -> int:
        """Row width of Q/K/V/O and of the KV slabs (padded heads x padded head width)."""
        return self.heads_pad * self.dh_pad


def build_model(config: ModelConfig, **kw) -> ToyModel:
    """engine.py:153-154."""
    return ToyModel(config, **kw)


def embed_prompt(model: ToyModel, prompt_text: str) -> np.ndarray:
    """engine.py:157-168 — sha256 of each whitespace token seeds a unit vector (host)."""
    if not prompt_text:
        raise ConfigError("empty prompt")
    dim = model.config.prompt_dim
    rows = []
    for tok in prompt_text.split():
        seed = int.from_bytes(hashlib.sha256(tok.encode("utf-8")).digest()[:8], "little")
        vec = np.random.default_rng(seed).standard_normal(dim).astype(np.float32)
        rows.append(vec / np.float32(np.linalg.norm(vec)))
    return np.stack(rows)


def _init_noise(cfg: ModelConfig, seed: int, chunk_index: int) -> np.ndarray:
    """engine.py:280-282 — bit-identical host noise."""
    rng = np.random.default_rng([seed, chunk_index])
    return rng.standard_normal((cfg.block_len, cfg.model_dim)).astype(np.float32)


def _init_noise_pinned(cfg: ModelConfig, seed: int, chunk_index: int) -> torch.Tensor:
    """_init_noise into pinned host memory (async H2D). Same float64 draw + fp32 cast as
    engine.py:280-282, so the values are bit-identical."""
    out = torch.empty((cfg.block_len, cfg.model_dim), dtype=torch.float32, pin_memory=True)
    host_normal_f32(np.random.default_rng([seed, chunk_index]), out)
    return out


def host_normal_f32(rng: np.random.Generator, out: torch.Tensor, threads: int | None = None) -> torch.Tensor:
    """out[:] = rng.standard_normal(out.shape).astype(float32), bit for bit, on all host
    cores (csrc/noise_host.cpp: parallel parse of the PCG64 stream with numpy's own
    ziggurat). `rng` must be freshly seeded; its state is not advanced."""
    st = rng.bit_generator.state
    if st["bit_generator"] != "PCG64" or st["has_uint32"]:
        raise ConfigError("host_normal_f32 needs a freshly seeded PCG64 generator")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    words = (ctypes.c_uint64 * 4)(s >> 64, s & m, inc >> 64, inc & m)
    if threads is None:
        threads = max(1, (os.cpu_count() or 2) - 1)  # leave a core to the launching thread
    if out.dtype != torch.float32 or not out.is_contiguous() or out.is_cuda:
        raise DimensionError("host_normal_f32 writes a contiguous host float32 tensor")
    _abi.check(_abi.lib().ifx_noise_normal_f32(words, out.numel(), out.data_ptr(), threads), "noise")
    return out


def _cross_kv(model: ToyModel, prompt_emb: np.ndarray):
    """engine.py:224-225 on device (fp32)."""
    e = torch.as_tensor(prompt_emb).cuda()
    return [(e @ lw.ck, e @ lw.cv) for lw in model.layers]


class _CrossFold:
    """Cross-attention of one layer folded through its few prompt keys (engine.py:211-215).

    With n prompt keys per head, softmax(q K^T) V co with q = h cq equals
    softmax_per_head(h (cq . K^T)) (V . co): cq . K^T is [D, H*n] and V . co is [H*n, D], so
    the two D x D projections around the attention (cq, co: 2 * 2*T*D*D FLOP per layer-pass)
    and the attention become two GEMMs of width H*n (3 * 12 = 36 at c2: 2 * 2*T*D*36) and a
    group softmax. Same math, reassociated; built from the cached prompt K/V when they change
    (fp32 einsum, bf16 GEMM operands, width padded to a multiple of 8 with zero columns)."""

    def __init__(self, model: "ToyModel", lw, k: torch.Tensor, v: torch.Tensor):
        D, H, dhp = model.config.model_dim, model.heads_pad, model.dh_pad
        n = k.shape[0]
        kk = k.float().reshape(n, H, dhp)
        vv = v.float().reshape(n, H, dhp)
        wqk = torch.einsum("dhe,jhe->dhj", lw.cq.float().reshape(D, H, dhp), kk).reshape(D, H * n)
        wvo = torch.einsum("jhe,hed->hjd", vv, lw.co.float().reshape(H, dhp, D)).reshape(H * n, D)
        self.k, self.v = k, v  # prompt K/V rows (the `_mha` hook path attends them directly)
        self.n, self.groups, self.width = n, H, -(-(H * n) // 8) * 8
        pad = self.width - H * n
        self.wqk = torch.nn.functional.pad(wqk, (0, pad)).to(torch.bfloat16).contiguous()
        self.wvo = torch.nn.functional.pad(wvo, (0, 0, 0, pad)).to(torch.bfloat16).contiguous()


def _fold_cross(model: "ToyModel", cross):
    """cross[l] = (k, v, row0, n) -> per-layer _CrossFold (None passes through)."""
    if cross is None:
        return None
    return [_CrossFold(model, lw, k[r0:r0 + n], v[r0:r0 + n])
            for lw, (k, v, r0, n) in zip(model.layers, cross)]


def _cross_attend(ws, fold: _CrossFold, x: torch.Tensor, h: torch.Tensor, scale: float):
    """x += softmax_per_head(h . wqk * scale) . wvo (the folded cross-attention)."""
    T = h.shape[0]
    key = (T, fold.width)
    buf = ws.cross_bufs.get(key)
    if buf is None:  # logits fp32 / probabilities bf16; padding columns of p stay zero
        buf = ws.cross_bufs[key] = (torch.empty(T, fold.width, device=h.device),
                                    torch.zeros(T, fold.width, device=h.device, dtype=torch.bfloat16))
    s, p = buf
    gemm(h, fold.wqk, s)
    _abi.check(_abi.lib().ifx_group_softmax(s.data_ptr(), T, fold.groups, fold.n, fold.width,
                                            float(scale), p.data_ptr(), fold.width,
                                            stream_ptr()), "group_softmax")
    count_launch()
    gemm(p, fold.wvo, x, beta=1.0)


def _cross_attend_g1(ws, fold: _CrossFold, norm: RowNorm, scale: float):
    """_cross_attend on G1: logits = rms(x) . wqk (row scale from the wo epilogue's
    statistics), group softmax, then x += P . wvo emitting the next norm's statistics."""
    T = norm.rows_bf16.shape[0]
    key = (T, fold.width)
    buf = ws.cross_bufs.get(key)
    if buf is None:
        buf = ws.cross_bufs[key] = (torch.empty(T, fold.width, device=ws.x.device),
                                    torch.zeros(T, fold.width, device=ws.x.device, dtype=torch.bfloat16))
    s, p = buf
    # a [T, D] x [D, H*n] product (H*n = 36 at c2) has too few output tiles for G1's
    # persistent grid (37 CTAs); cuBLASLt on the un-normalised rows, row scale in the softmax
    gemm(norm.rows_bf16, fold.wqk, s)
    _abi.check(_abi.lib().ifx_group_softmax_rs(s.data_ptr(), T, fold.groups, fold.n, fold.width,
                                               float(scale), p.data_ptr(), fold.width,
                                               norm.ss.data_ptr(), norm.ss.stride(0), norm.parts,
                                               norm.dim, stream_ptr()), "group_softmax")
    count_launch()
    gemm_fused(p, fold.wvo, ws.x, beta=1.0, norm_out=norm)


class _Workspace:
    """Per-(T, D) device buffers reused across passes (no allocator traffic in the loop)."""

    def __init__(self, T: int, D: int, Dp: int, dev):
        self.x = torch.empty(T, D, device=dev, dtype=torch.float32)
        self.h = torch.empty(T, D, device=dev, dtype=torch.bfloat16)
        self.qkv = torch.empty(T, 3 * Dp, device=dev, dtype=torch.bfloat16)
        self.attn = torch.empty(T, Dp, device=dev, dtype=torch.bfloat16)
        self.ffn = torch.empty(T, 2 * D, device=dev, dtype=torch.bfloat16)
        self.tmp = torch.empty(T, D, device=dev, dtype=torch.float32)
        self.cross_bufs = {}
        # G1 norm statistics: bf16 copy of the residual rows (self.h) and per-part sums of
        # squares of the fp32 rows, written by each residual GEMM for the next consumer
        # (room for the most parts any producer can emit: BN 64 tiles, two halves each)
        self.norm = RowNorm(self.h, torch.empty(T, 2 * -(-D // 64), device=dev), 0, D)


def _residual(x: torch.Tensor, a: torch.Tensor, w: torch.Tensor):
    """x += a @ w with bf16 operands, fp32 accumulation and fp32 in-place epilogue (one
    cuBLASLt call with beta = 1, per-shape algorithm, `ifx_gemm_bf16`)."""
    gemm(a, w, x, beta=1.0)


def _ffn_up(h: torch.Tensor, w1: torch.Tensor, out: torch.Tensor):
    """relu(h @ w1) with the ReLU in the cuBLASLt epilogue (engine.py:216)."""
    gemm(h, w1, out, relu=True)


class BlockRunner:
    """Runs the denoise passes of one block on the device (engine.py:185-221,285-312).

    `attn_events`: if a list, (start, end) CUDA events are recorded around every
    self-attention K1 launch (bench roofline timing)."""

    def __init__(self, model: ToyModel):
        self.model = model
        c = model.config
        self.dev = require_cuda()
        self.ws = _Workspace(c.block_len, c.model_dim, model.attn_width, self.dev)
        self.attn_events = None
        self.stager = _Stager(self.dev)
        self._eps = None
        self._tv = self._gpool = self._cap = self._graph = None  # CUDA-graph state (_euler_steps)
        self._warm = False
        self._tail = None  # event after the last block's clean pass (_euler_steps: GPU idle?)
        # G1 (hand-written tcgen05 GEMMs with fused epilogues) when the widths allow TMA
        # (rows of 16-byte multiples). IFX_G1 = "qkv": the QKV projection on G1 with RoPE
        # and the clean pass's page write in its epilogue, the other projections on
        # cuBLASLt with the RMS kernel; "all" (or 1): every projection on G1 with the norms
        # fused into the epilogues (_forward_g1); "off" (or 0): cuBLASLt only. Measured in
        # profiles/r04_g1.md.
        # "auto" (default) = "qkv" when the model has RoPE (the fused rotation saves a pass
        # over Q / K), else "off": on these shapes cuBLASLt's GEMMs are as fast or faster.
        ok = c.model_dim % 8 == 0
        self.g1 = G1 == "all" and ok
        self.g1_qkv = ok and (G1 == "qkv" or (G1 == "auto" and c.rope_grid is not None))

    def forward(self, latent: torch.Tensor, t: float, ctx, cross, cache: KvCache | None,
                collect_kv: bool = False, chunk_index: int = 0, eps_out: torch.Tensor | None = None,
                rope=None):
        """One pass. ctx: _KvContext of the block or None; cross: per-layer _CrossFold or
        None; rope = (cos, sin) tables of this block (rope_tables) or None."""
        if self.g1 and _mha_hook() is None:
            return self._forward_g1(latent, t, ctx, cross, cache, collect_kv, chunk_index, eps_out, rope)
        m, ws = self.model, self.ws
        c = m.config
        H, dhp, Dp = m.heads_pad, m.dh_pad, m.attn_width
        sc = 1.0 / math.sqrt(c.head_dim)
        q, kc, vc = ws.qkv[:, :Dp], ws.qkv[:, Dp:2 * Dp], ws.qkv[:, 2 * Dp:]
        for li, lw in enumerate(m.layers):
            if li == 0:  # x = latent + t*time_vec fused into the first norm (engine.py:199)
                if isinstance(t, torch.Tensor):  # t*time_vec precomputed on device (graphs)
                    rms_bf16(latent, ws.h, t, 1.0, x_out=ws.x)
                else:
                    rms_bf16(latent, ws.h, m.time_vec, t, x_out=ws.x)
            else:
                rms_bf16(ws.x, ws.h)
            hook = _mha_hook()
            pend = None
            if self.g1_qkv and hook is None:  # RoPE and the clean pass's page write fused
                if collect_kv:
                    pend = cache.append_reserve(li, c.block_len, SELF_ATTN, chunk_index)
                page = None if pend is None or pend.page is None else (*pend.page, Dp, 2 * Dp)
                gemm_fused(ws.h, lw.wqkv, ws.qkv, rope=None if rope is None else
                           (rope[0], rope[1], 0, c.head_dim // 2, dhp, H, 0, Dp), page=page)
            else:
                gemm(ws.h, lw.wqkv, ws.qkv)
                if rope is not None:  # Q and the block's own K, before K1 and the page write
                    rope_qk(ws.qkv, H, dhp, c.head_dim // 2, 0, Dp, rope[0], rope[1])
            ev = self.attn_events if hook is None else None
            if ev is not None:
                e0 = timing_event()
                e0.record()
            if hook is not None:  # a user attention processor (reference signature)
                self._hooked_self(hook, li, ctx, q, kc, vc)
            elif ctx is not None:
                ctx.attend(li, q, H, dhp, ws.attn, kc, vc, sc)
            else:
                attn_fwd(q, H, dhp, ws.attn, cur_k=kc, cur_v=vc, scale=sc)
            if ev is not None:
                e1 = timing_event()
                e1.record()
                ev.append((e0, e1))
            _residual(ws.x, ws.attn, lw.wo)
            if cross is not None:  # folded through the prompt's few keys (_CrossFold)
                rms_bf16(ws.x, ws.h)
                if hook is not None:
                    self._hooked_cross(hook, lw, cross[li])
                else:
                    _cross_attend(ws, cross[li], ws.x, ws.h, sc)
            rms_bf16(ws.x, ws.h)
            _ffn_up(ws.h, lw.w1, ws.ffn)
            _residual(ws.x, ws.ffn, lw.w2)
            if pend is not None:  # page bookkeeping ran before the QKV GEMM wrote the rows
                pend.finish(kc, vc)
            elif collect_kv:  # clean pass: page write of this layer's K/V (engine.py:303-306)
                cache.append_block(li, kc, vc, kind=SELF_ATTN, chunk_index=chunk_index)
        if eps_out is not None:
            rms_bf16(ws.x, ws.h)
            gemm(ws.h, m.w_out, eps_out)

    def _forward_g1(self, latent, t, ctx, cross, cache, collect_kv, chunk_index, eps_out, rope):
        """The same pass with every projection on G1 (csrc/gemm_sm100.cu) and the work
        between them in its epilogues: each residual GEMM (wo, the cross W_vo, w2) also
        writes the new rows as bf16 plus their sums of squares, and the next projection
        applies the RMS norm (engine.py:171-173) as a row scale after its product, so no
        norm kernel runs after layer 0's; 3D RoPE is applied to Q / K in the QKV epilogue;
        on the clean pass the QKV epilogue also writes K / V into their KV-cache pages
        (engine.py:303-306 -> kvcache.py:179-234; the page bookkeeping runs first, in the
        reference's order)."""
        m, ws = self.model, self.ws
        c = m.config
        H, dhp, Dp = m.heads_pad, m.dh_pad, m.attn_width
        T = c.block_len
        sc = 1.0 / math.sqrt(c.head_dim)
        q, kc, vc = ws.qkv[:, :Dp], ws.qkv[:, Dp:2 * Dp], ws.qkv[:, 2 * Dp:]
        norm = ws.norm
        rope_spec = None if rope is None else (rope[0], rope[1], 0, c.head_dim // 2, dhp, H, 0, Dp)
        for li, lw in enumerate(m.layers):
            if li == 0:  # x = latent + t*time_vec fused into the first norm (engine.py:199)
                if isinstance(t, torch.Tensor):
                    rms_bf16(latent, ws.h, t, 1.0, x_out=ws.x)
                else:
                    rms_bf16(latent, ws.h, m.time_vec, t, x_out=ws.x)
                nin = None
            else:
                nin = norm
            pend = cache.append_reserve(li, T, SELF_ATTN, chunk_index) if collect_kv else None
            page = None if pend is None or pend.page is None else (*pend.page, Dp, 2 * Dp)
            gemm_fused(ws.h, lw.wqkv, ws.qkv, norm_in=nin, rope=rope_spec, page=page)
            ev = self.attn_events
            if ev is not None:
                e0 = timing_event()
                e0.record()
            if ctx is not None:
                ctx.attend(li, q, H, dhp, ws.attn, kc, vc, sc)
            else:
                attn_fwd(q, H, dhp, ws.attn, cur_k=kc, cur_v=vc, scale=sc)
            if ev is not None:
                e1 = timing_event()
                e1.record()
                ev.append((e0, e1))
            gemm_fused(ws.attn, lw.wo, ws.x, beta=1.0, norm_out=norm)
            if cross is not None:  # folded through the prompt's few keys (_CrossFold)
                _cross_attend_g1(ws, cross[li], norm, sc)
            gemm_fused(ws.h, lw.w1, ws.ffn, relu=True, norm_in=norm)
            gemm_fused(ws.ffn, lw.w2, ws.x, beta=1.0, norm_out=norm)
            if pend is not None:
                pend.finish(kc, vc)
        if eps_out is not None:
            gemm_fused(ws.h, m.w_out, eps_out, norm_in=norm)

    def _hooked_self(self, hook, li: int, ctx, q, kc, vc) -> None:
        """engine.py:202-210 through a replaced `_mha`: k / v = [cached context ∥ block],
        all-true mask, the hook's [T, D] output written back into the padded layout."""
        m = self.model
        c = m.config
        un = lambda x: _unpad_heads(x, c.heads, m.heads_pad, c.head_dim, m.dh_pad)  # noqa: E731
        k, v = kc, vc
        if ctx is not None:
            lo, hi = ctx.ranges[li]
            if hi > lo:
                ck, cv = ctx.cache.gather_expanded(li, SELF_ATTN, lo, hi)
                k, v = torch.cat([ck, kc]), torch.cat([cv, vc])
        T = q.shape[0]
        mask = torch.ones(T, k.shape[0], dtype=torch.bool, device=q.device)
        out = hook(un(q), un(k), un(v), c.heads, mask)
        _pad_heads(torch.as_tensor(out, dtype=torch.float32), c.heads, m.heads_pad, c.head_dim,
                   m.dh_pad, self.ws.attn)

    def _hooked_cross(self, hook, lw, fold: "_CrossFold") -> None:
        """engine.py:211-215 through a replaced `_mha`: q = h2 @ cq over the prompt K/V."""
        m, ws = self.model, self.ws
        c = m.config
        un = lambda x: _unpad_heads(x, c.heads, m.heads_pad, c.head_dim, m.dh_pad)  # noqa: E731
        q2 = torch.empty_like(ws.attn)
        gemm(ws.h, lw.cq, q2)
        mask = torch.ones(q2.shape[0], fold.k.shape[0], dtype=torch.bool, device=q2.device)
        out = hook(un(q2), un(fold.k), un(fold.v), c.heads, mask)
        _pad_heads(torch.as_tensor(out, dtype=torch.float32), c.heads, m.heads_pad, c.head_dim,
                   m.dh_pad, q2)
        gemm(q2, lw.co, ws.x, beta=1.0)

    def denoise(self, latent: torch.Tensor, schedule: DenoiseSchedule, ctx, cross,
                cache: KvCache | None, chunk_index: int) -> torch.Tensor:
        """engine.py:296-306: S Euler steps in place on `latent`, then the clean K/V pass."""
        if self._eps is None:
            self._eps = self.ws.tmp.new_empty(self.ws.tmp.shape)
        eps = self._eps
        rope = rope_tables(self.model.config, chunk_index, self.dev)
        _euler_steps(self, latent, schedule, ctx, cross, cache, eps, rope,
                     first_block=chunk_index == 0)
        self.forward(latent, 0.0, ctx, cross, cache, collect_kv=cache is not None,
                     chunk_index=chunk_index, rope=rope)
        self._tail = torch.cuda.Event()
        self._tail.record()
        return latent


GRAPHS = os.environ.get("IFX_CUDA_GRAPHS", "1") != "0"
G1 = {"0": "off", "1": "all"}.get(os.environ.get("IFX_G1", "auto"), os.environ.get("IFX_G1", "auto"))


def timing_event() -> torch.cuda.Event:
    """A timing event for K1 launch windows; inside a CUDA-graph capture it is recorded as
    an external event node, so every replay re-records it (read after the last replay)."""
    return torch.cuda.Event(enable_timing=True,
                            external=torch.cuda.is_current_stream_capturing())


HOST_BOUND_CAPTURE = os.environ.get("IFX_HOST_BOUND_CAPTURE", "1") != "0"  # A/B switch


def _timed_eager_pass(runner, latent, tv, ctx, cross, cache, eps, rope) -> None:
    """runner.forward, eagerly, noting the host enqueue time and a GPU event pair of the pass
    (read later by _host_bound, once the events completed)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    runner.forward(latent, tv, ctx, cross, cache, eps_out=eps, rope=rope)
    e1.record()
    runner._pass_probe = (e0, e1, (time.perf_counter() - t0) * 1e3)


def _host_bound(runner) -> bool:
    """True when the runner's last timed eager pass was enqueue-bound: its GPU span (event
    to event) barely exceeded the host's enqueue time, i.e. the GPU waited for launches (a
    GPU-bound pass runs far longer than it takes to enqueue)."""
    probe = getattr(runner, "_pass_probe", None)
    # Ulysses ranks only: the single-GPU runner is GPU-bound at every shape here, and an
    # idle-GPU capture would only add its duration (measured: e2e -0.5 % with the probe on)
    if probe is None or not HOST_BOUND_CAPTURE or not hasattr(runner, "comm") or \
            not probe[1].query():
        return False
    e0, e1, host_ms = probe
    return e0.elapsed_time(e1) < 1.25 * host_ms


def _euler_steps(runner, latent, schedule: DenoiseSchedule, ctx, cross, cache, eps, rope,
                 graphs_ok: bool = True, first_block: bool = False) -> None:
    """The S denoise passes of a block (engine.py:299-301). Within a block every pass
    launches the same kernels on the same buffers with the same context, only t differs:
    the first pass is captured once as a CUDA graph (t*time_vec read from a device buffer)
    and replayed S times, so the host enqueues one pass per block instead of S (what keeps
    a Ulysses rank, whose GPU share of a pass shrinks with the world size, GPU-bound).
    K1 launches stay timed inside a capture (attn_events: external event nodes, re-recorded
    by every replay). Eager when capture is off (IFX_CUDA_GRAPHS=0), for the first block of
    a run on an idle GPU, when host-tier pages are staged on the side stream, when the
    page length forces the K7-gather path, or when `_mha` is replaced by a user hook; both
    modes compute t*time_vec the same way, so they are bit-identical."""
    steps = [float(t) for t in schedule.steps]
    m = runner.model
    if runner._tv is None:
        runner._tv = torch.empty_like(m.time_vec)  # t*time_vec of the pass (both modes)
        runner._gpool = torch.cuda.graph_pool_handle()
        runner._cap = torch.cuda.Stream(latent.device)
    tv, cap = runner._tv, runner._cap
    if ctx is not None:
        ctx.prepare()
    if len(steps) > 1 and not runner._warm:
        # the runner's first pass runs eagerly: library state (cuBLASLt handle, workspace,
        # per-shape algorithm choice in ifx_gemm_bf16) is set up outside any capture
        torch.mul(m.time_vec, steps[0], out=tv)  # (not timed: library setup skews it)
        runner.forward(latent, tv, ctx, cross, cache, eps_out=eps, rope=rope)
        latent.add_(eps, alpha=-float(schedule.step_scale))
        runner._warm = True
        steps = steps[1:]
    # the first block of a run on a drained GPU runs eagerly when the GPU is the bottleneck:
    # a capture would leave it idle for the capture's duration (in steady state a capture
    # overlaps the previous block's clean pass). A host-bound runner (a pass enqueues slower
    # than the GPU runs it, e.g. a Ulysses rank at 8 GPUs) captures this block too: eager
    # passes would idle the GPU for longer than one capture.
    eager_block = (first_block and (runner._tail is None or runner._tail.query())
                   and not _host_bound(runner))
    use = (GRAPHS and graphs_ok and len(steps) > 1 and not eager_block and _mha_hook() is None
           and (ctx is None or (ctx.paged and not ctx.jobs)))
    if use and isinstance(cross, _LazyFold):
        cross.materialize()  # fold ops (and their allocations) must not enter the graph
    if not use:
        for i, t in enumerate(steps):
            torch.mul(m.time_vec, t, out=tv)
            if i == 0 and runner.attn_events is None:
                _timed_eager_pass(runner, latent, tv, ctx, cross, cache, eps, rope)
            else:
                runner.forward(latent, tv, ctx, cross, cache, eps_out=eps, rope=rope)
            latent.add_(eps, alpha=-float(schedule.step_scale))
        return
    ev = runner.attn_events
    n_ev = len(ev) if ev is not None else 0
    n_launch = _device.LAUNCHES[0]
    g = torch.cuda.CUDAGraph()
    cap.wait_stream(torch.cuda.current_stream())
    try:
        with torch.cuda.stream(cap):  # capture without torch.cuda.graph's device-wide sync
            g.capture_begin(pool=runner._gpool, capture_error_mode="thread_local")
            try:
                runner.forward(latent, tv, ctx, cross, cache, eps_out=eps, rope=rope)
                latent.add_(eps, alpha=-float(schedule.step_scale))
            finally:
                g.capture_end()
    except RuntimeError as err:  # capture refused (driver / library): run eagerly from now on
        globals()["GRAPHS"] = False
        if ev is not None:
            del ev[n_ev:]  # events of the failed capture never complete
        _device.LAUNCHES[0] = n_launch  # nor do its kernels
        import warnings
        warnings.warn(f"CUDA graph capture failed ({err}); denoise passes run eagerly")
        torch.cuda.current_stream().wait_stream(cap)
        for t in steps:  # nothing ran during the failed capture
            torch.mul(m.time_vec, t, out=tv)
            runner.forward(latent, tv, ctx, cross, cache, eps_out=eps, rope=rope)
            latent.add_(eps, alpha=-float(schedule.step_scale))
        return
    torch.cuda.current_stream().wait_stream(cap)
    for t in steps:
        torch.mul(m.time_vec, t, out=tv)
        g.replay()
    if ev is not None:  # the captured K1 windows hold the last replay's times: one entry
        ev.extend(ev[n_ev:] * (len(steps) - 1))  # per replayed launch (same context each pass)
    # our kernels in the graph run once per replay (the launch counter saw the capture)
    _device.LAUNCHES[0] += (_device.LAUNCHES[0] - n_launch) * (len(steps) - 1)
    runner._graph = g  # kept until the next block (its kernels may still be running)


PAGED_K1_PAGE_LENS = (8, 16, 32, 64, 128)  # page boxes that tile K1's 128-key tiles
MAX_DMA_RUNS = 256  # staging of a layer with more slot runs goes through K6 instead


class _DevBuf:
    """A device buffer from ifx_dev_alloc (outside torch's caching allocator), exposed as a
    tensor through __cuda_array_interface__; freed when the last view is gone."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _abi.check(_abi.lib().ifx_dev_alloc(int(nbytes), ctypes.byref(p)), "dev_alloc")
        self.ptr, self.nbytes = p.value or 0, int(nbytes)
        self.__cuda_array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1",
                                         "data": (self.ptr, False), "version": 3,
                                         "strides": None}

    def view(self, rows: int, width: int, dtype) -> torch.Tensor:
        t = torch.as_tensor(self, device=require_cuda())  # keeps self alive
        return t.view(dtype)[:rows * width].view(rows, width)

    def __del__(self):
        if getattr(self, "ptr", 0):
            try:
                _abi.lib().ifx_dev_free(ctypes.c_void_p(self.ptr))
            except Exception:  # interpreter shutdown
                pass
            self.ptr = 0


class _Stager:
    """HBM staging buffers for host-tier context pages (one per runner, reused by blocks).

    K1 cannot stream pages out of host memory at tensor-core speed (every key tile is read
    by all query tiles), so before a layer's attention its host pages are copied H2D (K6,
    PCIe) into a staging buffer on a side stream, ahead of use. Buffers hold one layer's
    host pages each; if every host layer gets its own buffer within the budget, pages are
    staged once per block (their data is constant within a block), otherwise the buffers
    rotate over the host-layer attention calls in order, so the copies for the next host
    layers run while device-resident layers compute."""

    def __init__(self, dev, budget_bytes: int | None = None):
        self.dev = dev
        self.copy = torch.cuda.Stream(dev)
        self.k = self.v = None
        self.budget = budget_bytes if budget_bytes is not None else int(
            os.environ.get("IFX_STAGE_BUDGET_MB", "8192")) << 20
        self.staged_pages = 0  # pages copied H2D for attention (all blocks)
        self.buffers = None     # fixed number of rotating buffers (tests), None = budget

    def ensure(self, slots: int, page_len: int, width: int, dtype) -> None:
        rows = slots * page_len
        if self.k is not None and self.k.shape[0] >= rows and self.k.shape[1] == width \
                and self.k.dtype == dtype:
            return
        self.copy.synchronize()  # no staging copy may still write the old buffers
        if self.k is not None and self.k.shape[1] == width and self.k.dtype == dtype:
            # geometric growth capped at the budget: the host tier grows every block, and
            # re-allocating tens of GB per block would dominate the step
            esz = torch.finfo(dtype).bits // 8
            cap = max(rows, self.budget // (width * esz) // page_len * page_len)
            rows = min(cap, max(rows, -(-self.k.shape[0] * 9 // 8 // page_len) * page_len))
        self.k = self.v = None
        # staging takes what HBM the device tier leaves (c5: 2 x 23 GB next to a 115 GB
        # pool). Its buffers bypass torch's caching allocator (ifx_dev_alloc), so a freed
        # one goes back to the driver instead of being carved up by later small tensors;
        # segments torch keeps reserved are handed back first. Rare (first block, growth).
        torch.cuda.empty_cache()
        esz = torch.finfo(dtype).bits // 8
        self.k = _DevBuf(rows * width * esz).view(rows, width, dtype)
        self.v = _DevBuf(rows * width * esz).view(rows, width, dtype)
        self.k.zero_()
        self.v.zero_()


class _KvContext:
    """Attention view of the self-attention cache for one block (engine.py:228-237).

    Built once per block after the context fetch's bookkeeping (restore-on-read + clock,
    whose tier moves the cache executes). K1 reads device-tier pages IN PLACE from the pool
    through a per-layer slot table; host-tier pages (table code -1-i = the layer's i-th
    host page) come from a staging buffer (_Stager). Page lengths K1 cannot box (not in
    PAGED_K1_PAGE_LENS) fall back to a K7 gather of the context into a contiguous scratch
    per call."""

    def __init__(self, model, cache: KvCache, stager: _Stager, passes: int):
        self.cache = cache
        cfg = cache.config
        L = model.config.layers
        self.L, self.P = L, cfg.page_len
        self.pool = cache.pool(SELF_ATTN)
        # latent mode: the stored rows are expanded (K7 gather + up-projection GEMM) once
        # per block and layer into a contiguous context, reused by the block's passes
        self.latent = cfg.latent is not None
        self.expanded = {}
        self.paged = cfg.page_len in PAGED_K1_PAGE_LENS and not self.latent
        self.stager = stager
        self.calls = 0
        self.passes = passes
        self.ranges = []
        for li in range(L):  # the reference's fetch order: layer 0..L-1 (engine.py:228-237)
            lo, hi = cache.addressable_range(li, SELF_ATTN)
            if hi > lo:
                cache.touch_range(li, (lo, hi), SELF_ATTN)
                cache.batch_checkpoint(fetched_layer=li)
            self.ranges.append((lo, hi))
        self.prepared = False

    def prepare(self) -> None:
        """Slot tables + staging of the block, once every fetch of the block is done (the
        cross-attention fetch that follows the context fetch, engine.py:297-298, may still
        demote context pages to the host tier)."""
        if self.prepared:
            return
        self.prepared = True
        cache, stager, L = self.cache, self.stager, self.L
        self.first = [0] * L
        self.jobs = []  # host layers in call order within a pass
        if not self.paged:
            return
        tables, host_slots = [], [None] * L
        for li, (lo, hi) in enumerate(self.ranges):
            codes, first = cache.slot_table(li, SELF_ATTN, lo, hi) if hi > lo else (np.zeros(0, np.int32), lo)
            self.first[li] = first
            h = np.flatnonzero(codes < 0)
            if len(h):
                host_slots[li] = (-1 - codes[h]).astype(np.int64)
                codes = codes.copy()
                codes[h] = -1 - np.arange(len(h), dtype=np.int32)  # i-th host page of the layer
                self.jobs.append(li)
            tables.append(codes)
        dev = require_cuda()
        runs = [tile_run_codes(t, self.P) for t in tables]
        pairs = [np.stack([np.arange(len(hs), dtype=np.int64), hs], axis=1)
                 for hs in host_slots if hs is not None]
        flat = np.concatenate(tables + runs)
        allt = torch.from_numpy(flat).to(dev, non_blocking=True)
        lens = np.cumsum([0] + [len(t) for t in tables + runs])
        self.tables = [allt[lens[i]:lens[i + 1]] for i in range(L)]
        self.runs = [allt[lens[L + i]:lens[L + i + 1]] for i in range(L)]
        if not self.jobs:
            return
        allm = torch.from_numpy(np.concatenate(pairs)).to(dev, non_blocking=True)
        self.moves = [None] * L
        self.runs_h = [None] * L  # (staging slot, host slot, count) of consecutive host slots
        o = 0
        for li in self.jobs:
            hs = host_slots[li]
            n = len(hs)
            self.moves[li] = allm[o:o + n]
            o += n
            cut = np.flatnonzero(np.diff(hs) != 1) + 1
            starts = np.r_[0, cut]
            if len(starts) <= MAX_DMA_RUNS:
                counts = np.diff(np.r_[starts, n])
                self.runs_h[li] = np.ascontiguousarray(np.stack([starts, hs[starts], counts], 1), np.int64)
        self.job_of = {li: i for i, li in enumerate(self.jobs)}
        H = len(self.jobs)
        self.R = max(len(host_slots[li]) for li in self.jobs)  # slots per buffer
        buf_bytes = self.R * self.P * self.pool.width * self.pool.esz
        fit = max(1, stager.budget // max(1, buf_bytes))
        self.nbuf = H if (fit >= H or H == 1) else max(2, fit)
        if stager.buffers is not None:
            self.nbuf = max(1 if H == 1 else 2, min(H, stager.buffers))
        self.resident = self.nbuf == H  # every host layer keeps its buffer: stage once
        stager.ensure(self.nbuf * self.R, self.P, self.pool.width, self.pool.dtype)
        self.n_jobs = H if self.resident else H * self.passes
        self.staged, self.consumed = {}, {}
        start = torch.cuda.Event()
        start.record()  # tier moves + table uploads of this block are enqueued before it
        stager.copy.wait_event(start)
        for j in range(min(self.nbuf, self.n_jobs)):
            self._stage(j)

    def _buf(self, j: int) -> int:
        return j % self.nbuf

    def _stage_views(self, buf: int):
        r0, r1 = buf * self.R * self.P, (buf + 1) * self.R * self.P
        return self.stager.k[r0:r1], self.stager.v[r0:r1]

    def _stage(self, j: int) -> None:
        """Enqueue job j: the H2D copy of host layer jobs[j % H]'s pages into buffer j % nbuf,
        after the attention that last read that buffer."""
        st, li = self.stager, self.jobs[j % len(self.jobs)]
        buf = self._buf(j)
        if buf in self.consumed:
            st.copy.wait_event(self.consumed[buf])
        k, v = self._stage_views(buf)
        pool = self.pool
        p = _abi.KvPool()
        p.dev_k, p.dev_v = k.data_ptr(), v.data_ptr()
        p.host_k, p.host_v = pool.host_k.ptr, pool.host_v.ptr
        p.width, p.page_len = pool.width, pool.page_len
        p.type = _abi.BF16 if pool.dtype == torch.bfloat16 else _abi.F32
        m = self.moves[li]
        runs = self.runs_h[li]
        if runs is not None:  # DMA engines: runs while K1 occupies every SM
            _abi.check(_abi.lib().ifx_kv_copy_runs(
                ctypes.byref(p), runs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(runs), 1,
                st.copy.cuda_stream), "stage")
        else:  # many short runs: one gather kernel (K6)
            _abi.check(_abi.lib().ifx_kv_move_pages(ctypes.byref(p), m.data_ptr(), m.shape[0], 1,
                                                   st.copy.cuda_stream), "stage")
            count_launch()
        st.staged_pages += m.shape[0]
        ev = torch.cuda.Event()
        ev.record(st.copy)
        self.staged[j] = ev

    def attend(self, li: int, q, heads: int, dhp: int, out, cur_k, cur_v, scale: float, attn=None,
               cols: tuple | None = None, first: bool = True, last: bool = True):
        """K1 for layer li: q over [this layer's cached context ∥ the block's own K/V].

        cols = (c0, c1): only these columns of the cached rows (one head of a Ulysses rank
        whose query rows are split across ranks); a layer may then be attended in several
        calls (first / last mark the first and last of them in this pass)."""
        attn = attn or attn_fwd
        self.prepare()
        lo, hi = self.ranges[li]
        if first:
            self.calls += 1
        call = self.calls - 1
        sl = (lambda t: t) if cols is None else (lambda t: t[:, cols[0]:cols[1]])  # noqa: E731
        if hi <= lo:
            return attn(q, heads, dhp, out, cur_k=cur_k, cur_v=cur_v, scale=scale)
        if self.latent:
            if li not in self.expanded:
                self.expanded[li] = self.cache.gather_expanded(li, SELF_ATTN, lo, hi)
            k, v = self.expanded[li]
            return attn(q, heads, dhp, out, sl(k), sl(v), 0, hi - lo, cur_k, cur_v, scale=scale)
        if not self.paged:  # K7 gather of the context (host pages read over PCIe in place)
            k, v = self.cache._gather(li, SELF_ATTN, None, lo, hi - lo, lo, hi, raw=True)
            return attn(q, heads, dhp, out, sl(k), sl(v), 0, hi - lo, cur_k, cur_v, scale=scale)
        j = None
        if self.jobs and li in self.job_of:
            idx = self.job_of[li]
            j = idx if self.resident else (call // self.L) * len(self.jobs) + idx
            if first:
                torch.cuda.current_stream().wait_event(self.staged[j])
        sk, sv = self._stage_views(self._buf(j)) if j is not None else (None, None)
        pool = self.pool
        if pool.dev_k is None:  # capacity_pages_device=0: every page is staged, but K1 still
            pool.ensure(1, 0)   # takes the (unused) device pool as its base
        attn(q, heads, dhp, out, sl(pool.dev_k), sl(pool.dev_v), lo, hi - lo, cur_k, cur_v,
             scale=scale, ctx_slots=self.tables[li], page_len=self.P, first_token=self.first[li],
             stage_k=sl(sk) if sk is not None else None, stage_v=sl(sv) if sv is not None else None,
             tile_runs=self.runs[li])
        if j is not None and not self.resident and last:
            ev = torch.cuda.Event()
            ev.record()
            self.consumed[self._buf(j)] = ev
            if j + self.nbuf < self.n_jobs:
                self._stage(j + self.nbuf)
        return out


def _ctx_from_cache(model: ToyModel, cache: KvCache | None, stager: _Stager | None = None,
                    passes: int = 1):
    """engine.py:228-237 — the context fetch's bookkeeping (restore + access clock, in the
    reference's call order, with the tier moves it implies) and K1's paged view."""
    if cache is None:
        return None
    return _KvContext(model, cache, stager or _Stager(require_cuda()), passes)


def _touch_cross(model: ToyModel, cache: KvCache | None):
    """engine.py:240-246 — bookkeeping of the cross-attention fetch (if layer 0 has any)."""
    if cache is None:
        return None
    lo, hi = cache.addressable_range(0, CROSS_ATTN)
    if hi <= lo:
        return None
    rngs = []
    for li in range(model.config.layers):
        a, b = cache.addressable_range(li, CROSS_ATTN)
        cache.touch_range(li, (a, b), CROSS_ATTN)
        rngs.append((a, b))
    return rngs


class _LazyFold:
    """Per-layer _CrossFold of the cached prompt K/V, built on first use: the first pass of
    a run folds layer l right before layer l's cross-attention, so those small host-bound
    ops interleave with GPU work instead of running while the GPU waits (block 0).
    `materialize()` builds the rest before a CUDA-graph capture (no fold may be captured)."""

    def __init__(self, model: "ToyModel", cache: KvCache, rngs):
        # weak: the cache holds this object (fold_memo); a cycle would keep a replaced
        # cache's HBM pools alive until the next full garbage collection
        self.model, self.cache_ref, self.rngs = model, weakref.ref(cache), rngs
        self.folds = [None] * len(rngs)

    def __len__(self):
        return len(self.folds)

    def __getitem__(self, li: int) -> _CrossFold:
        f = self.folds[li]
        if f is None:
            a, b = self.rngs[li]
            k, v = self.cache_ref().gather_expanded(li, CROSS_ATTN, a, b)
            f = self.folds[li] = _CrossFold(self.model, self.model.layers[li], k, v)
        return f

    def materialize(self) -> "_LazyFold":
        for li in range(len(self.folds)):
            self[li]
        return self


def _engine_row_width(model: "ToyModel", kv_config: KvConfig):
    """Pool row width of the engine's cache: the padded attention width (zero head padding
    rides along into the pages), or in latent mode (kvcache.py:26-31) the stored latent
    rows, which the down-projection of unpadded rows produces."""
    if kv_config.latent is None:
        return model.attn_width
    if model.attn_width != model.config.model_dim:
        raise ConfigError("latent KV needs head_dim >= 64 (no zero-padded heads in the rows)")
    return None


def _gather_cross(cache: KvCache, rngs):
    """Per layer the prompt K/V rows, gathered (K7) into a contiguous buffer (a few rows;
    pages may sit on either tier)."""
    out = []
    for li, (a, b) in enumerate(rngs):
        k, v = cache.gather_expanded(li, CROSS_ATTN, a, b)
        out.append((k, v, 0, b - a))
    return out


def _block_context(model: ToyModel, cache: KvCache | None, prompt_ctx, stager: _Stager,
                   passes: int):
    """engine.py:297-298 — the block's context fetch: self-attention layers 0..L-1, then
    cross-attention, as ONE move batch (the LRU churn of a context larger than the device
    tier cancels out instead of moving every page twice), then K1's paged view."""
    if cache is None:
        return None, _fold_cross(model, _cross_from_cache(model, None, prompt_ctx))
    with cache.batch():
        ctx = _KvContext(model, cache, stager, passes)
        rngs = _touch_cross(model, cache)
    if rngs is None:
        ctx.prepare()
        return ctx, _fold_cross(model, _cross_from_cache(model, None, prompt_ctx))
    # the prompt K/V only change with the cache's cross rows: blocks under one prompt reuse
    # the fold (the fetch bookkeeping above still runs every block, as in the reference)
    key = (id(model), cache.cross_version, tuple(rngs))
    if cache.fold_memo is None or cache.fold_memo[0] != key:
        cache.fold_memo = (key, _LazyFold(model, cache, rngs))
    ctx.prepare()
    return ctx, cache.fold_memo[1]


def _cross_from_cache(model: ToyModel, cache: KvCache | None, prompt_ctx):
    """engine.py:240-250 — per layer the prompt K/V rows (from the cache when layer 0 has
    any), else projected from the prompt embedding."""
    rngs = _touch_cross(model, cache)
    if rngs is not None:
        return _gather_cross(cache, rngs)
    if prompt_ctx is None:
        return None
    out = []
    for k, v in _cross_kv(model, prompt_ctx):
        kb, vb = k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous()
        out.append((kb, vb, 0, kb.shape[0]))
    return out


def _runner(model: ToyModel) -> BlockRunner:
    """The model's BlockRunner (workspaces, staging buffers, graph state). Stored ON the
    model and holding it only through a weak proxy, so the runner and its device buffers
    are freed together with the model (no process-global registry keeps either alive)."""
    r = model.__dict__.get("_b200_runner")
    if r is None:
        r = model._b200_runner = BlockRunner(weakref.proxy(model))
    return r


def denoise_step(model: ToyModel, latent, t: float, step_scale: float, cache: KvCache | None = None,
                 prompt_ctx: np.ndarray | None = None) -> torch.Tensor:
    """engine.py:253-269 — one Euler update; the cache is read-only. Returns a CUDA tensor."""
    c = model.config
    lat = torch.as_tensor(np.asarray(latent, np.float32) if not isinstance(latent, torch.Tensor)
                          else latent).to(require_cuda(), torch.float32).clone()
    if lat.dim() != 2 or lat.shape[1] != c.model_dim:
        raise DimensionError("latent must be [tokens, model_dim]")
    r = _runner(model) if lat.shape[0] == c.block_len else BlockRunner.__new__(BlockRunner)
    if lat.shape[0] != c.block_len:
        r.__init__(model)
        r.ws = _Workspace(lat.shape[0], c.model_dim, model.attn_width, r.dev)
    eps = torch.empty_like(lat)
    r.forward(lat, float(t), _ctx_from_cache(model, cache, getattr(r, "stager", None)),
              _fold_cross(model, _cross_from_cache(model, cache, prompt_ctx)),
              cache, eps_out=eps, rope=rope_tables(c, 0, lat.device) if lat.shape[0] == c.block_len
              else None)
    return lat.sub_(eps, alpha=float(step_scale))


def _decode_px(model: ToyModel, x: torch.Tensor) -> torch.Tensor:
    """engine.py:272-277 on device: uint8 [T, h*w] = clip(127.5 + 48 * rms(x) @ w_decode)."""
    xr = x / torch.sqrt((x * x).mean(dim=-1, keepdim=True) + 1e-6)
    return torch.clamp(127.5 + 48.0 * (xr @ model.w_decode), 0.0, 255.0).to(torch.uint8)


def decode_frames(model: ToyModel, latent) -> list:
    """engine.py:272-277 — affine map of each latent row to a clamped uint8 frame (fp32)."""
    h, w = model.config.frame_shape
    px = _decode_px(model, torch.as_tensor(latent).to(require_cuda(), torch.float32))
    return list(px.view(-1, h, w).cpu().numpy())


def default_kv_config(model_cfg: ModelConfig, **overrides) -> KvConfig:
    """engine.py:315-324."""
    kw = dict(num_layers=model_cfg.layers, head_dim=model_cfg.model_dim, page_len=16,
              capacity_pages_device=4096, capacity_pages_host=4096)
    kw.update(overrides)
    return KvConfig(**kw)


def _prompt_for_chunk(schedule, chunk: int) -> str:
    """engine.py:327-332."""
    text = schedule[0][1]
    for c, p in schedule:
        if c <= chunk:
            text = p
    return text


_COPY_STREAMS: dict = {}


def _copy_stream(dev: torch.device, which: int) -> torch.cuda.Stream:
    """Per-device side streams for a block's input (0: noise H2D) and output (1: latent and
    frames D2H) transfers, so the DMA copy engines overlap neighbouring blocks' passes."""
    st = _COPY_STREAMS.get((dev, which))
    if st is None:
        st = _COPY_STREAMS[(dev, which)] = torch.cuda.Stream(dev)
    return st


def generate_block(model: ToyModel, cache: KvCache | None, schedule: DenoiseSchedule, prompt_ctx,
                   chunk_index: int, seed: int, prompt_text: str = "", noise=None,
                   to_host: bool = True, _ready=None) -> GeneratedBlock:
    """engine.py:285-312 — denoise one block from seeded noise, append its clean K/V.

    `_ready` (internal, Engine.generate): a list that receives the copy-done event instead
    of synchronising here, so the host can enqueue the next block while this one runs; the
    block's numpy arrays are valid once that event completed."""
    schedule.validate()
    c = model.config
    if noise is None:
        noise = _init_noise_pinned(c, seed, chunk_index)
    src = noise if isinstance(noise, torch.Tensor) else torch.from_numpy(noise)
    dev = require_cuda()
    main = torch.cuda.current_stream()
    if src.is_cuda or not src.is_pinned():
        lat = torch.empty(src.shape, device=dev, dtype=torch.float32)
        lat.copy_(src, non_blocking=True)
    else:  # pinned host noise: H2D on its own stream, overlapping the previous block
        cin = _copy_stream(dev, 0)
        with torch.cuda.stream(cin):  # allocated on that stream, used by main after the copy
            lat = torch.empty(src.shape, device=dev, dtype=torch.float32)
            lat.copy_(src, non_blocking=True)
        main.wait_stream(cin)
        lat.record_stream(main)
    runner = _runner(model)
    ctx, cross = _block_context(model, cache, prompt_ctx, runner.stager, len(schedule.steps) + 1)
    runner.denoise(lat, schedule, ctx, cross, cache, chunk_index)
    if not to_host:
        return GeneratedBlock(chunk_index, lat, [], prompt_text)
    # frames decoded on device; latent + frames land in pinned host buffers (one sync)
    h, w = c.frame_shape
    px = _decode_px(model, lat)
    lat_h = torch.empty(lat.shape, dtype=torch.float32, pin_memory=True)
    px_h = torch.empty(px.shape, dtype=torch.uint8, pin_memory=True)
    # D2H on its own stream: the next block's passes start while the results stream out
    cs = _copy_stream(lat.device, 1)
    cs.wait_stream(main)
    with torch.cuda.stream(cs):
        lat_h.copy_(lat, non_blocking=True)
        px_h.copy_(px, non_blocking=True)
    lat.record_stream(cs)
    px.record_stream(cs)
    ev = torch.cuda.Event()
    ev.record(cs)
    if _ready is None:
        ev.synchronize()
    else:
        _ready.append(ev)
    return GeneratedBlock(chunk_index, lat_h.numpy(), list(px_h.view(-1, h, w).numpy()), prompt_text)


class Engine:
    """engine.py:335-411 — one generation stream; prompt updates from other threads are
    merged at block boundaries, never retroactively."""

    def __init__(self, model: ToyModel, kv_config: KvConfig | None = None, profiler=None,
                 cache_dtype: torch.dtype = torch.bfloat16):
        self.model = model
        self.kv_config = kv_config or default_kv_config(model.config)
        self.profiler = profiler
        self.cache_dtype = cache_dtype
        self._lock = threading.Lock()
        self._generating_chunk = -1
        self._pending: list = []
        self._schedule: list = []
        self.event_log: list = []
        self.cache: KvCache | None = None

    def apply_prompt_update(self, effective_chunk: int, prompt_text: str) -> bool:
        """engine.py:351-359 — accept iff the target chunk is after the one in flight."""
        if not prompt_text:
            return False
        with self._lock:
            if effective_chunk <= self._generating_chunk:
                return False
            self._pending.append((effective_chunk, prompt_text))
            return True

    def _merge_pending(self):
        for chunk, text in self._pending:
            entries = [e for e in self._schedule if e[0] != chunk]
            entries.append((chunk, text))
            self._schedule = sorted(entries)
        self._pending.clear()

    def generate(self, request: GenerationRequest, sinks=(), noise_provider=None,
                 to_host: bool = True) -> list:
        """engine.py:368-411. `noise_provider(chunk)` (optional) supplies the block's noise
        (default: the reference's seeded host noise, prefetched on a worker thread)."""
        request.validate()
        c = self.model.config
        T = c.block_len
        reserve = T * request.num_blocks
        if request.kv_window is not None:
            reserve = min(reserve, request.kv_window + 2 * T + c.block_len)
        # the previous run's page table (~60k pages at c2) is torn down only once this run's
        # first block is enqueued, so its ~7 ms of host frees overlap GPU work; its HBM
        # pools go now (the cache object itself is dropped here)
        retired = self.cache._pt if self.cache is not None else None
        self.cache = KvCache(self.kv_config, dtype=self.cache_dtype, reserve_tokens=reserve,
                             row_width=_engine_row_width(self.model, self.kv_config))
        with self._lock:
            self._schedule = list(request.prompt_schedule)
            self._generating_chunk = -1
        make_noise = noise_provider or (lambda ch: _init_noise_pinned(c, request.seed, ch))
        pool = ThreadPoolExecutor(1)
        nxt = pool.submit(make_noise, 0)
        blocks = []
        pending = []  # copy-done events of blocks whose host arrays are still being filled
        current_prompt = None
        prof = self.profiler
        try:
            for chunk in range(request.num_blocks):
                with self._lock:
                    self._merge_pending()
                    self._generating_chunk = chunk
                    prompt = _prompt_for_chunk(self._schedule, chunk)
                if prompt != current_prompt:
                    if current_prompt is not None:
                        self.cache.clear_cross_attention()
                        self.event_log.append(("clear_cross_attention", chunk))
                    emb = embed_prompt(self.model, prompt)
                    for li, (kc, vc) in enumerate(_cross_kv(self.model, emb)):
                        self.cache.append_block(li, kc, vc, kind=CROSS_ATTN, chunk_index=chunk)
                    current_prompt = prompt
                noise = nxt.result()
                if chunk + 1 < request.num_blocks:
                    nxt = pool.submit(make_noise, chunk + 1)
                span = prof.scoped("generate_block") if prof else None
                if span:
                    span.__enter__()
                torch.cuda.nvtx.range_push(f"block{chunk}")  # ncu --nvtx-include scoping
                ready = [] if to_host else None
                block = generate_block(self.model, self.cache, request.schedule, None, chunk,
                                       request.seed, prompt_text=prompt, noise=noise,
                                       to_host=to_host, _ready=ready)
                if ready:
                    pending.append(ready[0])
                retired = None
                torch.cuda.nvtx.range_pop()
                if span:
                    span.__exit__(None, None, None)
                if request.kv_window is not None:
                    self.cache.evict_window(request.kv_window)
                self.event_log.append(("block", chunk))
                if sinks and pending:  # sinks see finished host arrays (engine.py:405-407)
                    pending.pop().synchronize()
                    pending.clear()
                for sink in sinks:
                    sink(block)
                blocks.append(block)
            for ev in pending:  # without sinks, one wait at the end keeps the GPU fed
                ev.synchronize()
        finally:
            pool.shutdown(wait=False)
        with self._lock:
            self._generating_chunk = request.num_blocks
        return blocks


def recompute_reference(model: ToyModel, request: GenerationRequest) -> list:
    """engine.py:424-489 — the cache-free check: every denoise step recomputes the whole
    sequence [clean prior blocks ∥ current latent] under the (windowed) block-causal mask,
    context tokens at t = 0, each block's rows cross-attending its own prompt. On device:
    the same kernels as the engine (RMS, bf16 GEMMs, K1 with a dense mask, K1s for the
    prompt keys); O(blocks^2) work, meant for validation-size configs."""
    from .attention import windowed_block_causal_mask
    request.validate()
    c = model.config
    dev = require_cuda()
    T, D, H, dhp, Dp = c.block_len, c.model_dim, model.heads_pad, model.dh_pad, model.attn_width
    sc = 1.0 / math.sqrt(c.head_dim)
    clean, prompts, blocks = [], [], []
    for chunk in range(request.num_blocks):
        prompt = _prompt_for_chunk(request.prompt_schedule, chunk)
        prompts.append([(k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous())
                        for k, v in _cross_kv(model, embed_prompt(model, prompt))])
        lat = torch.from_numpy(_init_noise(c, request.seed, chunk)).to(dev)
        nb = len(clean) + 1
        n = nb * T
        mask = windowed_block_causal_mask(nb, T, request.kv_window).to(torch.uint8).contiguous()
        rope = None
        if c.rope_grid is not None:  # every token at its own block's absolute positions
            tabs = [rope_tables(c, bi, dev) for bi in range(nb)]
            rope = (torch.cat([a for a, _ in tabs]), torch.cat([b for _, b in tabs]))
        for t in request.schedule.steps:
            tcol = torch.zeros(n, 1, device=dev)
            tcol[(nb - 1) * T:] = float(t)
            x = (torch.cat(clean + [lat]) + tcol * model.time_vec).contiguous()
            h = torch.empty(n, D, device=dev, dtype=torch.bfloat16)
            qkv = torch.empty(n, 3 * Dp, device=dev, dtype=torch.bfloat16)
            att = torch.empty(n, Dp, device=dev, dtype=torch.bfloat16)
            for lw in model.layers:
                rms_bf16(x, h)
                torch.mm(h, lw.wqkv, out=qkv)
                if rope is not None:
                    rope_qk(qkv, H, dhp, c.head_dim // 2, 0, Dp, rope[0], rope[1])
                attn_fwd(qkv[:, :Dp], H, dhp, att, qkv[:, Dp:2 * Dp], qkv[:, 2 * Dp:], 0, n,
                         scale=sc, mask=mask)
                _residual(x, att, lw.wo)
                rms_bf16(x, h)
                q2 = torch.mm(h, lw.cq)
                for bi in range(nb):  # each block's rows vs its own prompt (engine.py:470-476)
                    r = slice(bi * T, (bi + 1) * T)
                    kc, vc = prompts[bi][model.layers.index(lw)]
                    attn_fwd(q2[r], H, dhp, att[r], kc, vc, 0, kc.shape[0], scale=sc)
                _residual(x, att, lw.co)
                rms_bf16(x, h)
                f = torch.empty(n, 2 * D, device=dev, dtype=torch.bfloat16)
                _ffn_up(h, lw.w1, f)
                _residual(x, f, lw.w2)
            rms_bf16(x, h)
            eps = torch.mm(h[(nb - 1) * T:], model.w_out, out_dtype=torch.float32)
            lat = lat - float(request.schedule.step_scale) * eps
        clean.append(lat)
        blocks.append(GeneratedBlock(chunk, lat.cpu().numpy(), decode_frames(model, lat), prompt))
    return blocks


def generate_sequence(model: ToyModel, request: GenerationRequest, sinks=(),
                      kv_config: KvConfig | None = None, profiler=None) -> list:
    """engine.py:414-421."""
    return Engine(model, kv_config, profiler).generate(request, sinks)


# -- pipeline registry (engine.py:495-528) ------------------------------------------------


@dataclass(frozen=True)
class Pipeline:
    """Hooks a model family plugs into the common generate-and-cache loop."""
    name: str
    build_model: Callable
    denoise_step: Callable
    decode_frames: Callable


_PIPELINES: dict = {}


def register_pipeline(pipeline: Pipeline):
    _PIPELINES[pipeline.name] = pipeline


def get_pipeline(name: str) -> Pipeline:
    try:
        return _PIPELINES[name]
    except KeyError:
        raise ConfigError(f"unknown pipeline {name!r}; registered: {sorted(_PIPELINES)}") from None


for _name in ("toy", "b200"):
    register_pipeline(Pipeline(name=_name, build_model=build_model, denoise_step=denoise_step,
                               decode_frames=decode_frames))
