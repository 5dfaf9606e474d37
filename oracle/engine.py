"""Oracle: seeded toy block-diffusion DiT and its generate-and-cache loop.

Test infrastructure only (see oracle/__init__.py). Restates
`/root/reference/pkg/src/inferix/engine.py`: weights drawn from one PCG64
stream in the reference's order (engine.py:120-144), Euler denoising with a
clean K/V pass per block (engine.py:285-312), the block loop with prompt
switches / cross clears / window eviction (engine.py:368-411) and the cache-free
recompute oracle (engine.py:424-489).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from .attention import multi_head, windowed_block_causal_mask
from .rope import apply_rope, rope_tables
from .errors import ConfigError, DimensionError
from .kvcache import CROSS_ATTN, SELF_ATTN, KvConfig, create_cache

_F32 = np.float32
_EPS = _F32(1e-6)  # engine.py:26
LAYER_FIELDS = ("wq", "wk", "wv", "wo", "cq", "ck", "cv", "co", "w1", "w2")


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
    # B200 extension (not in the reference): 3D RoPE over (frames_per_block, grid_h, grid_w)
    rope_grid: tuple | None = None
    rope_theta: float = 10000.0

    def validate(self):
        for n in ("layers", "heads", "head_dim", "block_len", "prompt_dim"):
            if getattr(self, n) < 1:
                raise ConfigError(f"{n} must be >= 1")
        if min(self.frame_shape) < 1:
            raise ConfigError("frame_shape must be positive")
        if self.rope_grid is not None and int(np.prod(self.rope_grid)) != self.block_len:
            raise ConfigError("rope_grid must tile block_len")

    def rope(self, chunk: int):
        """(cos, sin) of block `chunk`, or None without RoPE (oracle/rope.py)."""
        if self.rope_grid is None:
            return None
        return rope_tables(self.rope_grid, chunk * self.rope_grid[0], self.head_dim, self.rope_theta)

    @property
    def model_dim(self) -> int:
        return self.heads * self.head_dim


@dataclass
class DenoiseSchedule:
    """engine.py:51-62."""
    steps: list
    step_scale: float = 0.5

    def validate(self):
        if not self.steps:
            raise ConfigError("schedule needs at least one step")
        if min(self.steps) <= 0:
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
        ps = self.prompt_schedule
        if not ps or ps[0][0] != 0:
            raise ConfigError("prompt_schedule must start at chunk 0")
        if any(a[0] >= b[0] for a, b in zip(ps, ps[1:])):
            raise ConfigError("prompt_schedule chunks must be strictly increasing")
        if not all(text for _, text in ps):
            raise ConfigError("prompts must be nonempty")
        if self.kv_window is not None and self.kv_window < 0:
            raise ConfigError("kv_window must be >= 0")


class ToyModel:
    """engine.py:112-150 — draw order: per layer wq wk wv wo cq ck cv co w1 w2,
    then time_vec, w_out, w_decode (scale 0.35, not 0.5/sqrt(rows))."""

    def __init__(self, cfg: ModelConfig, with_decoder: bool = True):
        cfg.validate()
        self.config = cfg
        d, p = cfg.model_dim, cfg.prompt_dim
        gen = np.random.default_rng(np.random.PCG64(cfg.weight_seed))

        def draw(r, c):
            return gen.standard_normal((r, c)).astype(_F32) * _F32(0.5 / np.sqrt(r))

        shapes = {"wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d), "cq": (d, d),
                  "ck": (p, d), "cv": (p, d), "co": (d, d), "w1": (d, 2 * d), "w2": (2 * d, d)}
        self.layers = [{f: draw(*shapes[f]) for f in LAYER_FIELDS} for _ in range(cfg.layers)]
        self.time_vec = draw(1, d)[0]
        self.w_out = draw(d, d)
        h, w = cfg.frame_shape
        self.w_decode = (gen.standard_normal((d, h * w)).astype(_F32) * _F32(0.35)
                         if with_decoder else None)

    def num_parameters(self) -> int:
        n = self.time_vec.size + self.w_out.size + self.w_decode.size
        return n + sum(a.size for lw in self.layers for a in lw.values())


def embed_prompt(cfg: ModelConfig, text: str) -> np.ndarray:
    """engine.py:157-168 — sha256(token)[:8] seeds a unit vector per token."""
    if not text:
        raise ConfigError("empty prompt")
    out = []
    for tok in text.split():
        seed = int.from_bytes(hashlib.sha256(tok.encode("utf-8")).digest()[:8], "little")
        vec = np.random.default_rng(seed).standard_normal(cfg.prompt_dim).astype(_F32)
        out.append(vec / _F32(np.linalg.norm(vec)))
    return np.stack(out)


def rms(x):
    """engine.py:171-173."""
    return (x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True, dtype=_F32) + _EPS)).astype(_F32)


def forward_block(model: ToyModel, latent, t, ctx, cross, collect_kv=False, chunk=0):
    """engine.py:185-221 — one pass over a block; ctx[l] = (K, V) [C, D]. With
    `rope_grid` set (B200 extension) q and the block's own k are rotated at the block's
    positions; cached context K is already rotated."""
    heads = model.config.heads
    rope = model.config.rope(chunk)
    x = (latent + _F32(t) * model.time_vec).astype(_F32)
    kv = []
    for li, w in enumerate(model.layers):
        h = rms(x)
        q, kc, vc = h @ w["wq"], h @ w["wk"], h @ w["wv"]
        if rope is not None:
            q, kc = apply_rope(q, *rope, heads), apply_rope(kc, *rope, heads)
        ck, cvv = ctx[li]
        kk = np.concatenate([ck, kc]) if ck.size else kc
        vv = np.concatenate([cvv, vc]) if cvv.size else vc
        x = x + multi_head(q, kk, vv, heads, np.ones((x.shape[0], kk.shape[0]), bool)) @ w["wo"]
        if cross is not None:
            xk, xv = cross[li]
            hq = rms(x) @ w["cq"]
            x = x + multi_head(hq, xk, xv, heads, np.ones((x.shape[0], xk.shape[0]), bool)) @ w["co"]
        x = x + np.maximum(rms(x) @ w["w1"], _F32(0.0)) @ w["w2"]
        if collect_kv:
            kv.append((kc, vc))
    return (rms(x) @ model.w_out).astype(_F32), (kv if collect_kv else None)


def layer_pass(w, heads, x, ctx_k, ctx_v, xk, xv):
    """One layer of forward_block (engine.py:202-217) — the CPU-baseline work unit."""
    h = rms(x)
    q, kc, vc = h @ w["wq"], h @ w["wk"], h @ w["wv"]
    kk = np.concatenate([ctx_k, kc]) if ctx_k.size else kc
    vv = np.concatenate([ctx_v, vc]) if ctx_v.size else vc
    x = x + multi_head(q, kk, vv, heads, np.ones((x.shape[0], kk.shape[0]), bool)) @ w["wo"]
    hq = rms(x) @ w["cq"]
    x = x + multi_head(hq, xk, xv, heads, np.ones((x.shape[0], xk.shape[0]), bool)) @ w["co"]
    return x + np.maximum(rms(x) @ w["w1"], _F32(0.0)) @ w["w2"]


def cross_kv(model: ToyModel, emb):
    """engine.py:224-225."""
    return [(emb @ w["ck"], emb @ w["cv"]) for w in model.layers]


def context_from_cache(model: ToyModel, cache):
    """engine.py:228-237 — full addressable self-attn range per layer."""
    d = model.config.model_dim
    empty = np.empty((0, d), _F32)
    if cache is None:
        return [(empty, empty)] * model.config.layers
    out = []
    for li in range(model.config.layers):
        lo, hi = cache.addressable_range(li, SELF_ATTN)
        out.append(cache.fetch_range(li, (lo, hi)) if hi > lo else (empty, empty))
    return out


def cross_from_cache(model: ToyModel, cache, prompt_emb):
    """engine.py:240-250 — cross K/V from the cache if layer 0 has any."""
    if cache is not None:
        lo, hi = cache.addressable_range(0, CROSS_ATTN)
        if hi > lo:
            return [cache.fetch_range(li, cache.addressable_range(li, CROSS_ATTN), CROSS_ATTN)
                    for li in range(model.config.layers)]
    return None if prompt_emb is None else cross_kv(model, prompt_emb)


def denoise_step(model, latent, t, step_scale, cache=None, prompt_ctx=None):
    """engine.py:253-269."""
    if latent.ndim != 2 or latent.shape[1] != model.config.model_dim:
        raise DimensionError("latent must be [tokens, model_dim]")
    eps, _ = forward_block(model, latent, t, context_from_cache(model, cache),
                           cross_from_cache(model, cache, prompt_ctx))
    return (latent - _F32(step_scale) * eps).astype(_F32)


def decode_frames(model: ToyModel, latent):
    """engine.py:272-277."""
    h, w = model.config.frame_shape
    px = np.clip(_F32(127.5) + _F32(48.0) * (rms(latent) @ model.w_decode), 0.0, 255.0)
    return [r.reshape(h, w).astype(np.uint8) for r in px]


def init_noise(cfg: ModelConfig, seed: int, chunk: int):
    """engine.py:280-282."""
    return np.random.default_rng([seed, chunk]).standard_normal(
        (cfg.block_len, cfg.model_dim)).astype(_F32)


def generate_block(model, cache, schedule, prompt_ctx, chunk_index, seed):
    """engine.py:285-312 — S Euler steps, clean pass at t=0, append K/V."""
    schedule.validate()
    lat = init_noise(model.config, seed, chunk_index)
    ctx = context_from_cache(model, cache)
    cross = cross_from_cache(model, cache, prompt_ctx)
    for t in schedule.steps:
        eps, _ = forward_block(model, lat, t, ctx, cross, chunk=chunk_index)
        lat = (lat - _F32(schedule.step_scale) * eps).astype(_F32)
    _, kv = forward_block(model, lat, 0.0, ctx, cross, collect_kv=True, chunk=chunk_index)
    if cache is not None:
        for li, (k, v) in enumerate(kv):
            cache.append_block(li, k, v, kind=SELF_ATTN, chunk_index=chunk_index)
    return lat


def default_kv_config(cfg: ModelConfig, **kw) -> KvConfig:
    """engine.py:315-324."""
    args = dict(num_layers=cfg.layers, head_dim=cfg.model_dim, page_len=16,
                capacity_pages_device=4096, capacity_pages_host=4096)
    args.update(kw)
    return KvConfig(**args)


def prompt_for_chunk(schedule, chunk):
    """engine.py:327-332."""
    text = schedule[0][1]
    for c, p in schedule:
        if c <= chunk:
            text = p
    return text


def generate_sequence(model, request: GenerationRequest, kv_config=None):
    """engine.py:368-421 (no prompt mailbox: schedule fixed up front).

    Returns (latents per block, final cache)."""
    request.validate()
    cache = create_cache(kv_config or default_kv_config(model.config))
    cur = None
    lats = []
    for chunk in range(request.num_blocks):
        prompt = prompt_for_chunk(request.prompt_schedule, chunk)
        if prompt != cur:
            if cur is not None:
                cache.clear_cross_attention()
            for li, (kc, vc) in enumerate(cross_kv(model, embed_prompt(model.config, prompt))):
                cache.append_block(li, kc, vc, kind=CROSS_ATTN, chunk_index=chunk)
            cur = prompt
        lats.append(generate_block(model, cache, request.schedule, None, chunk, request.seed))
        if request.kv_window is not None:
            cache.evict_window(request.kv_window)
    return lats, cache


def recompute_reference(model, request: GenerationRequest):
    """engine.py:424-489 — cache-free full recompute (windowed block-causal)."""
    request.validate()
    cfg = model.config
    L, heads = cfg.block_len, cfg.heads
    clean, prompts, out = [], [], []
    for chunk in range(request.num_blocks):
        prompts.append(embed_prompt(cfg, prompt_for_chunk(request.prompt_schedule, chunk)))
        lat = init_noise(cfg, request.seed, chunk)
        nb = len(clean) + 1
        mask = windowed_block_causal_mask(nb, L, request.kv_window)
        rope = None
        if cfg.rope_grid is not None:  # every token at its own block's absolute positions
            tabs = [cfg.rope(bi) for bi in range(nb)]
            rope = (np.concatenate([c for c, _ in tabs]), np.concatenate([s for _, s in tabs]))
        for t in request.schedule.steps:
            tcol = np.zeros((nb * L, 1), _F32)
            tcol[(nb - 1) * L:] = _F32(t)
            x = (np.concatenate(clean + [lat]).astype(_F32) + tcol * model.time_vec).astype(_F32)
            for w in model.layers:
                h = rms(x)
                q, k = h @ w["wq"], h @ w["wk"]
                if rope is not None:
                    q, k = apply_rope(q, *rope, heads), apply_rope(k, *rope, heads)
                x = x + multi_head(q, k, h @ w["wv"], heads, mask) @ w["wo"]
                h2 = rms(x)
                y = np.empty_like(x)
                for bi in range(nb):
                    r = slice(bi * L, (bi + 1) * L)
                    kc, vc = prompts[bi] @ w["ck"], prompts[bi] @ w["cv"]
                    y[r] = multi_head(h2[r] @ w["cq"], kc, vc, heads, np.ones((L, kc.shape[0]), bool))
                x = x + y @ w["co"]
                x = x + np.maximum(rms(x) @ w["w1"], _F32(0.0)) @ w["w2"]
            eps = (rms(x) @ model.w_out)[(nb - 1) * L:].astype(_F32)
            lat = (lat - _F32(request.schedule.step_scale) * eps).astype(_F32)
        clean.append(lat)
        out.append(lat)
    return out
