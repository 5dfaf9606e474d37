#!/usr/bin/env python
"""bench.py — block-diffusion decode hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One "step" is one full generate-and-cache rollout of the configured workload: every
block runs 4 Euler denoise passes + the clean K/V pass over all layers, attending the
paged KV cache of prior blocks, then appends its K/V (engine.py:285-312, 368-411).
Default workload (N=1) is BASELINE.json configs[1]: Wan2.1-1.3B-shaped (30 layers, 12
heads x 128, 4680 tokens = 3 latent frames per block), 7 blocks = 21 latent frames.

value    latent frames/s over the K timed rollouts, inputs (noise) resident in HBM,
         CUDA events on the engine stream, barrier + synchronize on both sides.
e2e      the same metric through the public API `Engine.generate()` with host noise
         (numpy default_rng, exactly the reference's inputs) copied H2D and every block's
         latent + decoded frames copied D2H inside the timed region.
roofline the dominant kernel, K1 attention: algorithmic FLOPs 4*T*(C+T)*D per launch
         summed over the timed region / summed CUDA-event durations of those launches,
         against MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long
         step).
cpu_baseline  the numpy oracle port (oracle/engine.py:layer_pass) on the host cores:
         two layer-passes at the exact shape (b = 0 and 1 cached blocks), extrapolated
         linearly in b to the same rollout.

N > 1 (torchrun, one rank per GPU): the same c2 rollout strong-scaled with Ulysses; the
head <-> sequence re-shard runs through NVLink peer memory (G1's QKV epilogue and K1's O
epilogue store into the consuming rank; peer barriers; `--exchange nccl` for all-to-alls);
12 heads on 8 GPUs use the grouped plan (4 head groups x 2 query-row slices). value = all
ranks' frames / max-over-ranks device time; e2e through UlyssesEngine.generate with host
noise and gathered latents copied to host; roofline = rank 0's K1 launches; stdout carries
only rank 0's JSON line. `--ulysses` runs that engine at N = 1.

--impl reference: the reference's CPU algorithm (the oracle port; the Python reference
cannot travel to the GPU box) on all host cores, same metric/config; each step is one
bounded sample (a pair of layer-passes), extrapolated to the rollout.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "latent frames/sec & attention TFLOP/s (% bf16 peak) at 1/2/4/8 B200 vs CPU ref"
UNIT = "latent frames/s"
FRAMES_PER_BLOCK = 3  # 3 latent frames x 1560 tokens (480p) per block
STEPS = [1.0, 0.75, 0.5, 0.25]

CONFIGS = {
    "c1": dict(layers=2, heads=4, head_dim=64, block_len=768, blocks=3, frame_shape=(16, 16),
               weights="reference",
               desc="c1: tiny random-init DiT (2L, 4 heads x 64, dim 256), 768 tok/block, 3 blocks x 3 frames, 4 steps"),
    "c2": dict(layers=30, heads=12, head_dim=128, block_len=4680, blocks=7, frame_shape=(16, 16),
               weights="reference",
               desc="c2: Wan2.1-1.3B-shaped (30L, 12 heads x 128, dim 1536), 1560 tok/frame x 3-frame blocks, 7 blocks (21 latent frames), 4 steps"),
    "c3": dict(layers=30, heads=12, head_dim=128, block_len=4680, blocks=21, frame_shape=(16, 16),
               weights="reference",
               desc="c3: 1.3B shape long context, 21 blocks (20 cached)"),
    "c4": dict(layers=40, heads=40, head_dim=128, block_len=4680, blocks=3, frame_shape=(16, 16),
               weights="device",
               desc="c4: Wan2.1-14B-shaped (40L, 40 heads x 128, dim 5120), 3 blocks, 4 steps"),
    # c5 on ONE GPU: the cache of a minute-long rollout does not fit HBM, so the pinned host
    # tier is live. Blocks [0, prefill) are appended from synthetic K/V (no denoising), then
    # `blocks` more are generated through generate_block and timed.
    "c5": dict(layers=40, heads=40, head_dim=128, block_len=4680, blocks=2, prefill=58,
               device_blocks=30, stage_budget_gb=24, frame_shape=(16, 16), weights="device",
               desc="c5: Wan2.1-14B-shaped LV rollout on 1 GPU: 60+ cached blocks (30 blocks of "
                    "pages = 115 GB in HBM, the rest on the pinned host tier; cache state of a "
                    "58-block rollout: per-block fetch + append bookkeeping), blocks 60-61 timed"),
}


def attn_flops_per_rollout(c) -> float:
    """4*T*(C+T)*D per (layer, pass); P = steps + 1 passes per block."""
    T, D = c["block_len"], c["heads"] * c["head_dim"]
    P = len(STEPS) + 1
    return sum(4.0 * T * (b * T + T) * D * c["layers"] * P for b in range(c["blocks"]))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("bf16_tflops_sustained") or p["bf16_tflops"], "measured (sustained)"
    except Exception:
        return 1400.0, "fallback (B200_PROFILING.md sustained)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self) -> dict:
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[1]) for r in rows),
                "sm_max_mhz": max(float(r[2]) for r in rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_layer_pass_times(c, n_layers_b0=1, bs=(0, 1), threads=None):
    """Time oracle layer-passes (oracle/engine.py:layer_pass) at the exact (T, D, H)."""
    import numpy as np

    from oracle import engine as OE

    T, H, dh = c["block_len"], c["heads"], c["head_dim"]
    D = H * dh
    g = np.random.default_rng(0)
    s = lambda r, k: (g.standard_normal((r, k)).astype(np.float32) * np.float32(0.5 / np.sqrt(r)))  # noqa: E731
    w = {"wq": s(D, D), "wk": s(D, D), "wv": s(D, D), "wo": s(D, D), "cq": s(D, D), "co": s(D, D),
         "w1": s(D, 2 * D), "w2": s(2 * D, D)}
    x = g.standard_normal((T, D)).astype(np.float32)
    xk = g.standard_normal((3, D)).astype(np.float32)
    out = {}
    for b in bs:
        ck = g.standard_normal((b * T, D)).astype(np.float32)
        t0 = time.perf_counter()
        OE.layer_pass(w, H, x, ck, ck, xk, xk)
        out[b] = time.perf_counter() - t0
    return out


def extrapolate_rollout_seconds(c, t_by_b: dict) -> float:
    """Linear-in-b fit of one layer-pass time, summed over the rollout's blocks."""
    b0, b1 = min(t_by_b), max(t_by_b)
    t0, t1 = t_by_b[b0], t_by_b[b1]
    slope = (t1 - t0) / (b1 - b0) if b1 > b0 else 0.0
    P = len(STEPS) + 1
    return sum((t0 + slope * (b - b0)) * c["layers"] * P for b in range(c["blocks"]))


def cpu_baseline(c, cfgname):
    t = cpu_layer_pass_times(c)
    secs = extrapolate_rollout_seconds(c, t)
    return {"value": c["blocks"] * FRAMES_PER_BLOCK / secs, "unit": UNIT,
            "cores": os.cpu_count(), "kind": "port",
            "sample": (f"oracle numpy layer-pass at {cfgname} shape for b=0,1 cached blocks "
                       f"({t[0]:.2f}s, {t[1]:.2f}s), linear in b, x{c['layers']} layers x5 passes "
                       f"x{c['blocks']} blocks = {secs:.0f}s/rollout (extrapolated)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nthreads = os.cpu_count()
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(v, str(nthreads))
    c = CONFIGS[args.config or "c2"]
    for _ in range(args.warmup):  # warm BLAS / page in (b=0 only)
        cpu_layer_pass_times(c, bs=(0,))
    samples = []
    for _ in range(args.steps):
        t = cpu_layer_pass_times(c)
        samples.append(extrapolate_rollout_seconds(c, t))
    secs = statistics.mean(samples)
    value = c["blocks"] * FRAMES_PER_BLOCK / secs
    sample = (f"per step: oracle numpy layer-passes at b=0,1 cached blocks, extrapolated linearly "
              f"to the {c['blocks']}-block rollout ({secs:.0f}s/rollout)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded numpy)",
            "config": {"workload": c["desc"], "extrapolated": True},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def _gemm_path(runner) -> str:
    if runner.g1:
        return "G1 (tcgen05, norms / RoPE / page write fused) for every projection"
    if runner.g1_qkv:
        return "QKV on G1 (RoPE + page write fused), others cuBLASLt + RMS kernel"
    return "cuBLASLt + RMS kernel"


def rope_grid(args, c):
    """--rope: 3D RoPE over (frames, latent rows, latent columns) of a block, Wan2.1 480p:
    3 frames x 30 x 52 = 4,680 tokens (the north_star's fused RoPE; the reference has none)."""
    if not args.rope:
        return None
    if c["block_len"] != 4680:
        raise SystemExit("--rope is defined for the 4,680-token (3 x 30 x 52) blocks")
    return (3, 30, 52)


def attn_traffic(cfgname, world):
    """DRAM bytes of one K1 launch of this workload (rank shape at `world` ranks) from an
    ncu --set full capture committed in profiles/attn_traffic.json, or (None, None)."""
    tpath = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if not os.path.exists(tpath):
        return None, None
    with open(tpath) as f:
        recs = json.load(f)
    t_rec = recs.get(cfgname if world == 1 else f"{cfgname}@w{world}")
    if not t_rec:
        return None, None
    return t_rec["dram_bytes_per_launch"], (
        f"{t_rec['launch']}; algorithmic {t_rec['algorithmic_bytes_per_launch']} B; {t_rec['source']}")


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank (NCCL). IFX_DIST_BACKEND=gloo lets several ranks share a GPU to test
    # the multi-rank code path on a 1-GPU box (UlyssesComm stages the a2a through the host).
    backend = os.environ.get("IFX_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1 or args.ulysses:
        if world == 1:  # --ulysses at N = 1: the multi-GPU code path on one rank
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfgname = args.config or "c2"
    c = CONFIGS[cfgname]
    if world > 1 or args.ulysses:
        return run_ulysses_bench(args, c, cfgname, world, rank, local)
    if "prefill" in c:
        return run_host_tier_bench(args, c, cfgname, local)

    from paper_2511_20714_b200 import _device
    from paper_2511_20714_b200 import engine as E

    torch.backends.cuda.matmul.allow_tf32 = False
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0, rope_grid=rope_grid(args, c))
    model = E.build_model(mc, weights=c["weights"])
    T, D = mc.block_len, mc.model_dim
    nb = c["blocks"]
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(nb, E.DenoiseSchedule(STEPS), seed=0)
    host_noise = [E._init_noise(mc, 0, ch) for ch in range(nb)]
    dev_noise = [torch.from_numpy(n).cuda() for n in host_noise]
    eng = E.Engine(model, kvc)
    runner = E._runner(model)

    def rollout_device():
        return eng.generate(req, noise_provider=lambda ch: dev_noise[ch], to_host=False)

    for _ in range(args.warmup):
        rollout_device()
    torch.cuda.synchronize()

    # ---- timed region: K rollouts, inputs resident in HBM
    runner.attn_events = []
    launches0 = _device.LAUNCHES[0]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.cuda.nvtx.range_push("timed")
        h0 = time.perf_counter()
        for _ in range(args.steps):
            rollout_device()
        # host wall time of the loop: no explicit sync inside, but launch back-pressure ties
        # it to the GPU once the queue is full (not a measure of host cost)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        torch.cuda.nvtx.range_pop()
        e1.record()
        torch.cuda.synchronize()
    launches = _device.LAUNCHES[0] - launches0
    ms = e0.elapsed_time(e1) / args.steps
    attn_ms = sum(a.elapsed_time(b) for a, b in runner.attn_events)
    n_attn = len(runner.attn_events)
    runner.attn_events = None
    clocks = clk.summary()
    value = nb * FRAMES_PER_BLOCK / (ms / 1e3)
    flops = attn_flops_per_rollout(c) * args.steps
    achieved = flops / (attn_ms / 1e3) / 1e12
    peak, peak_src = load_peaks()

    # ---- e2e: public API, host noise generated + copied H2D, latents + frames D2H
    rollout_host = lambda: eng.generate(req)  # noqa: E731
    rollout_host()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_each = []
    blocks = None
    for _ in range(args.steps):
        t1 = time.perf_counter()
        # a consumer done with the previous rollout's arrays: their pinned buffers are
        # recycled by torch's host allocator instead of pinning fresh memory every step
        blocks = None
        blocks = rollout_host()  # returns once its latents are on the host
        e2e_each.append((time.perf_counter() - t1) * 1e3)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    h, w = mc.frame_shape
    h2d = nb * T * D * 4 + 3 * mc.prompt_dim * 4
    d2h = nb * (T * D * 4 + T * h * w)
    assert all(np.isfinite(b.latent).all() for b in blocks)

    cpu = None if args.no_cpu_baseline else cpu_baseline(c, cfgname)
    traffic, traffic_note = attn_traffic(cfgname, 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (reference-seeded noise, PCG64 random-init weights)",
        "config": {"workload": c["desc"] + (", 3D RoPE (3 x 30 x 52) fused into the QKV GEMM"
                                            if mc.rope_grid else ""),
                   "rope_grid": mc.rope_grid, "gemm": _gemm_path(runner),
                   "layers": mc.layers, "heads": mc.heads,
                   "head_dim": mc.head_dim, "tokens_per_block": T, "blocks": nb,
                   "denoise_steps": len(STEPS), "kv_cache": "bf16 paged (page_len 16): HBM slot pool + pinned host tier",
                   "l2": "inputs larger than L2 (weights 1.4 GB, KV pool up to 6 GB)",
                   "parallelism": "single GPU"},
        "attention_tflops": achieved,
        "attention_frac_of_peak": achieved / peak,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_launch": traffic_note,
                     "peak_source": peak_src,
                     "kernel": "K1 attn_fwd_kernel<128> (tcgen05/TMEM/TMA)",
                     "launches": n_attn, "kernel_ms_per_step": attn_ms / args.steps,
                     "share_of_step": attn_ms / args.steps / ms},
        "e2e": {"value": nb * FRAMES_PER_BLOCK / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                "ms_each": [round(x, 1) for x in e2e_each]},
        "gpu_launches": launches,
        "host_loop_ms_per_step": host_ms,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    emit(line)
    return 0


def run_host_tier_bench(args, c, cfgname, local):
    """c5: steady state of a rollout whose KV cache exceeds HBM (reference tier semantics:
    device-first allocation with host spill, restore-on-fetch with LRU demotion,
    kvcache.py:126-175). Prefill appends synthetic K/V for `prefill` blocks through the
    cache API; then each timed step generates one block (engine.py:285-312) over the
    whole cache: tier moves at the context fetch (K6), device pages read in place by K1,
    host pages staged H2D on the side stream one layer ahead."""
    import torch

    from paper_2511_20714_b200 import _device
    from paper_2511_20714_b200 import engine as E
    from paper_2511_20714_b200.kvcache import CROSS_ATTN, SELF_ATTN, KvCache

    torch.backends.cuda.matmul.allow_tf32 = False
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0, rope_grid=rope_grid(args, c))
    model = E.build_model(mc, weights=c["weights"])
    T, L, W = mc.block_len, mc.layers, model.attn_width
    pages_blk = -(-T // 16)
    nb_pre, nb = c["prefill"], max(c["blocks"], args.steps)
    # the host tier lives in pinned RAM: size the rollout to what this box can pin
    # (MemAvailable x 0.6), so the run reports the longest cache it can actually hold
    blk_host_bytes = L * pages_blk * 2 * 16 * W * 2
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(x.split()[1]) * 1024 for x in f if x.startswith("MemAvailable"))
        max_host_blocks = int(0.6 * avail // blk_host_bytes)
        nb_pre = max(1, min(nb_pre, c["device_blocks"] + max_host_blocks - nb - 3))
    except (OSError, StopIteration):
        pass
    kvc = E.default_kv_config(mc, capacity_pages_device=c["device_blocks"] * L * pages_blk,
                              capacity_pages_host=(nb_pre + nb + 2) * L * pages_blk)
    cache = KvCache(kvc, dtype=torch.bfloat16, reserve_tokens=T * (c["device_blocks"] + 1), row_width=W)
    host_slots = (nb_pre + nb + 2 - c["device_blocks"]) * L * pages_blk
    t0 = time.perf_counter()
    cache.pool(SELF_ATTN).ensure(0, host_slots)  # pinned + mapped + zeroed once, up front
    host_alloc_s = time.perf_counter() - t0
    emb = E.embed_prompt(model, "a quiet scene")
    for li, (kc, vc) in enumerate(E._cross_kv(model, emb)):
        cache.append_block(li, kc, vc, kind=CROSS_ATTN, chunk_index=0)
    g = torch.Generator(device="cuda").manual_seed(0)
    kv = [torch.randn(T, W, device="cuda", generator=g).bfloat16() for _ in range(2)]
    runner = E._runner(model)
    t0 = time.perf_counter()
    for b in range(nb_pre):  # the cache state of a rollout: each block's context fetch
        with cache.batch():  # (bookkeeping + tier moves, engine.py:297-298), then appends
            E._KvContext(model, cache, runner.stager, 1)
            E._touch_cross(model, cache)
        for li in range(L):
            cache.append_block(li, kv[0], kv[1], kind=SELF_ATTN, chunk_index=b)
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    sched = E.DenoiseSchedule(STEPS)
    noise = torch.randn(T, mc.model_dim, device="cuda", generator=g)
    runner.stager.budget = c.get("stage_budget_gb", 8) << 30  # HBM left after pool + weights

    def block(ch):
        return E.generate_block(model, cache, sched, None, ch, 0, noise=noise.clone(), to_host=False)

    for w in range(min(args.warmup, 1)):  # one warm block (the cache keeps growing)
        block(nb_pre + w)
    torch.cuda.synchronize()
    ch0 = nb_pre + min(args.warmup, 1)
    runner.attn_events = []
    mv0, st0 = list(cache.moved_pages), runner.stager.staged_pages
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            block(ch0 + i)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    attn_ms = sum(a.elapsed_time(b) for a, b in runner.attn_events) / args.steps
    runner.attn_events = None
    P = len(STEPS) + 1
    flops = sum(4.0 * T * (b * T + T) * mc.model_dim * L * P for b in range(ch0, ch0 + args.steps)) / args.steps
    peak, peak_src = load_peaks()
    page_b = 2 * 16 * W * 2  # K + V bytes of one page
    moved = [(a - b) * page_b / args.steps for a, b in zip(cache.moved_pages, mv0)]
    staged = (runner.stager.staged_pages - st0) * page_b / args.steps
    st = cache.memory_stats()
    line = {
        "metric": METRIC, "value": FRAMES_PER_BLOCK / (ms / 1e3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (prefill K/V and noise from torch.randn, random-init weights)",
        "config": {"workload": c["desc"], "step": "one generated block (4 steps + clean pass)",
                   "cached_blocks": [ch0, ch0 + args.steps - 1],
                   "device_pages": st.device_pages_used, "host_pages": st.host_pages_used,
                   "prefill_s": prefill_s, "host_pool_alloc_s": host_alloc_s,
                   "host_pool_GB": host_slots * 2 * 16 * W * 2 / 1e9},
        "roofline": {"bound": "tensor", "achieved": flops / (attn_ms / 1e3) / 1e12, "peak": peak,
                     "unit": "TFLOP/s", "frac": flops / (attn_ms / 1e3) / 1e12 / peak,
                     "traffic": None, "peak_source": peak_src, "kernel": "K1 (paged)",
                     "note": "event window includes each layer's wait for its host pages "
                             "to be staged (PCIe-bound); see tools/attn_probe.py for K1 alone",
                     "kernel_ms_per_step": attn_ms, "share_of_step": attn_ms / ms},
        "host_tier": {"d2h_bytes_per_step": moved[0], "h2d_bytes_per_step": moved[1],
                      "staged_h2d_bytes_per_step": staged,
                      "pcie_GBps_if_serial": (moved[0] + moved[1] + staged) / (ms / 1e3) / 1e9},
        "gpu_launches": None, "clocks": clk.summary(), "cpu_baseline": None,
    }
    emit(line)
    return 0


def head_split(runner) -> str:
    """How a Ulysses rank's attention is split (parallel.py plans)."""
    if runner.grouped is not None:
        g = runner.grouped
        return f"grouped: {g.G} head groups x {g.R} row slices ({g.hl} heads, {g.rows} query rows per rank)"
    if runner.plan is not None:
        return f"balanced: {runner.plan.hl} heads / {len(runner.plan.segs)} segments on rank 0"
    return "whole heads"


def run_ulysses_bench(args, c, cfgname, world, rank, local):
    """bench.py for N > 1: one rollout strong-scaled over N GPUs with Ulysses."""
    import torch
    import torch.distributed as dist

    from paper_2511_20714_b200 import _device
    from paper_2511_20714_b200 import engine as E
    from paper_2511_20714_b200.parallel import UlyssesComm, UlyssesEngine

    torch.backends.cuda.matmul.allow_tf32 = False
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0, rope_grid=rope_grid(args, c))
    # the same model as the N = 1 line (reference PCG64 weights for c1-c3); heads % N != 0
    # use the balanced query split, no padding
    model = E.ToyModel(mc, weights=c["weights"])
    comm = UlyssesComm()
    nb = c["blocks"]
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(nb, E.DenoiseSchedule(STEPS), seed=0)
    # the reference's seeded noise (engine.py:280-282), resident in HBM for `value`
    noise = [torch.from_numpy(E._init_noise(mc, 0, ch)).cuda() for ch in range(nb)]
    exchange = "peer scatter over NVLink (G1 QKV epilogue + K1 O epilogue, peer barriers)"
    try:
        eng = UlyssesEngine(model, comm, kvc, p2p=args.exchange == "p2p")
    except Exception as e:  # e.g. CUDA IPC unavailable in this container: say so, use NCCL
        if args.exchange != "p2p":
            raise
        exchange = f"NCCL all-to-all (peer mesh setup failed: {type(e).__name__}: {e})"
        eng = UlyssesEngine(model, comm, kvc, p2p=False)
    if eng.runner.xch is None and args.exchange == "nccl":
        exchange = "NCCL all-to-all (K5 pack / unpack)"
    roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], gather=False)  # noqa: E731
    for _ in range(args.warmup):
        roll()
    torch.cuda.synchronize()
    dist.barrier()
    # K1 roofline from one extra rollout with per-launch CUDA events (external event nodes
    # inside the pass graphs); the timed region below runs without them
    eng.runner.attn_events = []
    roll()
    torch.cuda.synchronize()
    attn_ms = sum(a.elapsed_time(b) for a, b in eng.runner.attn_events)
    eng.runner.attn_events = None
    dist.barrier()
    l0 = _device.LAUNCHES[0]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            roll()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = _device.LAUNCHES[0] - l0
    peak, peak_src = load_peaks()
    # algorithmic FLOPs of this rank's share (one rollout)
    flops_rank = attn_flops_per_rollout(c) / world
    achieved = flops_rank / (attn_ms / 1e3) / 1e12 if attn_ms > 0 else None
    # e2e: host noise (reference seeding) in, gathered latents out; one untimed rollout
    # first (pinned host buffers are allocated on first use, then cached)
    eng.generate(req, to_host=True)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        host = eng.generate(req, to_host=True)  # gathered latents in pinned host memory
    torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) / args.steps], device="cuda")
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    clocks = clk.summary()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c, cfgname)  # host cores of rank 0's node; other ranks wait
    traffic, traffic_note = attn_traffic(cfgname, world)
    if rank == 0:
        T, D = mc.block_len, mc.model_dim
        line = {"metric": METRIC, "value": nb * FRAMES_PER_BLOCK / (ms / 1e3), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": ("synthetic (reference-seeded noise, PCG64 random-init weights)"
                         if c["weights"] == "reference" else "synthetic (reference-seeded noise, "
                         "torch-seeded random-init weights)"),
                "config": {"workload": c["desc"], "parallelism": f"ulysses{world}",
                           "head_split": head_split(eng.runner), "exchange": exchange,
                           "l2": "inputs larger than L2"},
                "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak if achieved else None, "traffic": traffic,
                             "traffic_launch": traffic_note, "peak_source": peak_src,
                             "scope": "rank 0's K1 launches, one eager rollout with per-launch events"},
                "e2e": {"value": nb * FRAMES_PER_BLOCK / float(e2e.item()), "unit": UNIT,
                        "h2d_bytes_per_step": nb * T * D * 4 // world,
                        "d2h_bytes_per_step": nb * T * D * 4},
                "comm": {"a2a_messages": comm.messages, "a2a_bytes": comm.bytes,
                         "peer_barriers": eng.runner.xch.mesh.barriers if eng.runner.xch else 0},
                "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
                "cuda_graphs": "denoise passes captured once per block, replayed (IFX_CUDA_GRAPHS=0: eager)"}
        emit(line)
    dist.barrier()
    eng.runner.release_graphs()  # captured NCCL work must be freed before the group
    torch.cuda.synchronize()
    dist.destroy_process_group()
    return 0


_JSON_FD = None  # the real stdout when fd 1 is redirected (N > 1)


def emit(line: dict) -> None:
    """Print the run's ONE JSON line on stdout (the real one, see main)."""
    text = json.dumps(line) + "\n"
    if _JSON_FD is None:
        sys.stdout.write(text)
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, text.encode())


def main():
    global _JSON_FD
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or "--ulysses" in sys.argv:
        # NCCL writes its banner ("NCCL version ...") to fd 1 on rank 0: keep stdout to the
        # JSON line by sending everything else written to fd 1 to stderr
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ulysses", action="store_true",
                    help="run the Ulysses (multi-GPU) engine even at N = 1 (exchange overhead probe)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: Ulysses re-shard through NVLink peer memory (scatter epilogues "
                         "+ peer barriers) or NCCL all-to-alls")
    ap.add_argument("--rope", action="store_true",
                    help="3D RoPE on Q/K (3 x 30 x 52 grid), fused into the QKV GEMM epilogue")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
