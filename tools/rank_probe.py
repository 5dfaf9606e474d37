"""Compute-only timing of ONE rank's share of a W-rank Ulysses rollout, on one GPU.

    python tools/rank_probe.py [--configs c2 c4] [--worlds 1 2 4 8] [--ranks 0]

The Ulysses engine runs with a LoopbackComm (parallel.py): rank r of W with exactly the
kernels it launches in the real job (GEMMs on n = T/W rows, the QKV scatter epilogue, K1
over its heads / balanced segments for all T queries, the O scatter, peer barriers), but
every peer arena is local memory and barriers pass at once — no NVLink time, no waiting
for slower ranks. ms_rank is therefore a lower bound of the W-GPU step; W * value_1 /
value_W compares it to perfect strong scaling. Prints one JSON line per (config, W, rank).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def _profile(roll, name, W, r):
    import collections

    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        roll()
        torch.cuda.synchronize()
    path = f"/tmp/rank_trace_{os.getpid()}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    os.unlink(path)
    k = [e for e in ev if e.get("cat") == "kernel" and "dur" in e]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in k:
        n = e["name"]
        if "gemm_kernel" in n:
            key = "G1 " + n[n.index("gemm_kernel"):n.index(">", n.index("gemm_kernel")) + 1]
        elif "nvjet" in n or "cutlass" in n or "cublas" in n.lower() or "gemm" in n.lower():
            key = "cuBLASLt"
        else:
            import re
            m = re.search(r"::(\w+)(<[^()]*>)?\(", n.replace("(anonymous namespace)", "anon"))
            key = (m.group(1) + (m.group(2) or "")) if m else n[:60]
        agg[key][0] += 1
        agg[key][1] += e["dur"]
    busy = sum(v[1] for v in agg.values())
    span = max(e["ts"] + e["dur"] for e in k) - min(e["ts"] for e in k)
    ks = sorted(k, key=lambda e: e["ts"])
    gaps = [b["ts"] - (a["ts"] + a["dur"]) for a, b in zip(ks, ks[1:])]
    hist = {lab: round(sum(g for g in gaps if lo <= g < hi) / 1e3, 2) for lab, lo, hi in
            (("<2us", -1e9, 2), ("2-5us", 2, 5), ("5-20us", 5, 20), ("20-200us", 20, 200),
             (">200us", 200, 1e12))}
    big = sorted(range(len(gaps)), key=lambda i: -gaps[i])[:12]
    t0 = ks[0]["ts"]
    top = [(round(gaps[i], 1), round((ks[i]["ts"] - t0) / 1e3, 2), ks[i]["name"][:40], ks[i + 1]["name"][:40])
           for i in sorted(big)]
    print(json.dumps({"top_gaps_us_at_ms_after_before": top}), flush=True)
    print(json.dumps({"profile": name, "world": W, "rank": r, "span_ms": round(span / 1e3, 2),
                      "kernel_ms": round(busy / 1e3, 2), "launches": len(k), "gap_ms_by_size": hist,
                      "kernels": {n: [c, round(us / 1e3, 2)] for n, (c, us) in
                                  sorted(agg.items(), key=lambda x: -x[1][1])[:14]}}), flush=True)


def _c5_rank(name, c, W, r, steps):
    """c5 (minute-long 14B rollout) as one rank of W: the rank's head shard of a cache with
    `prefill` cached blocks (synthetic K/V through the cache API, the reference's per-block
    fetch bookkeeping), all of it HBM-resident, then `steps` generated blocks timed."""
    import bench
    from paper_2511_20714_b200 import engine as E
    from paper_2511_20714_b200.kvcache import CROSS_ATTN, SELF_ATTN, KvCache
    from paper_2511_20714_b200.parallel import LoopbackComm, UlyssesEngine
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0)
    model = E.ToyModel(mc, weights=c["weights"])
    T, L = mc.block_len, mc.layers
    nb_pre = c["prefill"]
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    eng = UlyssesEngine(model, LoopbackComm(W, r), kvc, p2p=True)
    rn = eng.runner
    cache = KvCache(kvc, dtype=torch.bfloat16, reserve_tokens=T * (nb_pre + steps + 2),
                    row_width=rn.wl, cross_row_width=model.attn_width)
    emb = E.embed_prompt(model, "a quiet scene")
    for li, (kc, vc) in enumerate(E._cross_kv(model, emb)):
        cache.append_block(li, kc, vc, kind=CROSS_ATTN, chunk_index=0)
    g = torch.Generator(device="cuda").manual_seed(0)
    kv = [torch.randn(T, rn.wl, device="cuda", generator=g).bfloat16() for _ in range(2)]
    for b in range(nb_pre):
        with cache.batch():
            E._KvContext(model, cache, rn.stager, 1)
            E._touch_cross(model, cache)
        for li in range(L):
            cache.append_block(li, kv[0], kv[1], kind=SELF_ATTN, chunk_index=b)
    torch.cuda.synchronize()
    sched = E.DenoiseSchedule(bench.STEPS)
    noise = torch.randn(rn.n, mc.model_dim, device="cuda", generator=g)

    def block(ch):
        ctx, cross = E._block_context(model, cache, None, rn.stager, len(bench.STEPS) + 1)
        rn.denoise(noise.clone(), sched, ctx, cross, cache, ch)

    block(nb_pre)  # warm
    torch.cuda.synchronize()
    rn.attn_events = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        block(nb_pre + 1 + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    attn_ms = sum(a.elapsed_time(b) for a, b in rn.attn_events) / steps
    rn.attn_events = None
    P = len(bench.STEPS) + 1
    flops = sum(4.0 * T * (b * T + T) * mc.model_dim * L * P
                for b in range(nb_pre + 1, nb_pre + 1 + steps)) / steps / W
    st = cache.memory_stats()
    print(json.dumps({"config": name, "world": W, "rank": r, "cached_blocks": nb_pre + 1,
                      "ms_per_block_rank": round(ms, 1),
                      "latent_frames_per_s_if_all_ranks_equal": round(3 / (ms / 1e3), 3),
                      "k1_ms": round(attn_ms, 1), "k1_tflops_rank": round(flops / (attn_ms / 1e3) / 1e12, 1),
                      "kv_shard_device_GB": round(st.device_pages_used * 16 * rn.wl * 2 * 2 / 1e9, 2),
                      "host_pages": st.host_pages_used, "head_split": bench.head_split(rn)}), flush=True)
    rn.release_graphs()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "c4"])
    ap.add_argument("--worlds", nargs="+", type=int, default=[1, 2, 4, 8])
    ap.add_argument("--ranks", nargs="+", type=int, default=[0])
    ap.add_argument("--rollouts", type=int, default=2)
    ap.add_argument("--profile", action="store_true",
                    help="also print per-kernel GPU time of one rollout (torch.profiler / CUPTI)")
    args = ap.parse_args()
    import torch.distributed as dist

    import bench
    from paper_2511_20714_b200 import engine as E
    from paper_2511_20714_b200.parallel import LoopbackComm, UlyssesEngine

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    torch.backends.cuda.matmul.allow_tf32 = False
    for name in args.configs:
        c = bench.CONFIGS[name]
        if "prefill" in c:
            for W in args.worlds:
                for r in args.ranks:
                    if W >= 4 and r < W:  # a rank's shard of the 60-block cache fits HBM
                        _c5_rank(name, c, W, r, args.rollouts)
            continue
        mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                           block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                           weight_seed=0)
        model = E.ToyModel(mc, weights=c["weights"])
        nb = c["blocks"]
        kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
        req = E.GenerationRequest(nb, E.DenoiseSchedule(bench.STEPS), seed=0)
        noise = [torch.from_numpy(E._init_noise(mc, 0, ch)).cuda() for ch in range(nb)]
        flops = bench.attn_flops_per_rollout(c)
        base = None
        for W in args.worlds:
            if mc.block_len % W:
                continue
            for r in args.ranks:
                if r >= W:
                    continue
                eng = UlyssesEngine(model, LoopbackComm(W, r), kvc, p2p=True)
                roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], gather=False)  # noqa: E731
                for _ in range(2):
                    roll()
                torch.cuda.synchronize()
                eng.runner.attn_events = []
                roll()
                torch.cuda.synchronize()
                evs = eng.runner.attn_events
                attn_ms = sum(a.elapsed_time(b) for a, b in evs)
                per = len(evs) // nb if len(evs) % nb == 0 else 0
                T_ = mc.block_len
                blk_tf = [round(4.0 * T_ * (b + 1) * T_ * mc.model_dim * c["layers"] * (len(bench.STEPS) + 1) / W
                                / (sum(x.elapsed_time(y) for x, y in evs[b * per:(b + 1) * per]) / 1e3) / 1e12, 1)
                          for b in range(nb)] if per else None
                eng.runner.attn_events = None
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.rollouts):
                    roll()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.rollouts
                value = nb * bench.FRAMES_PER_BLOCK / (ms / 1e3)
                if W == 1 and r == 0:
                    base = value
                print(json.dumps({
                    "config": name, "world": W, "rank": r, "ms_rank": round(ms, 2),
                    "value_if_all_ranks_equal": round(value, 3),
                    "strong_scaling_bound": round(value / (W * base), 3) if base else None,
                    "k1_ms": round(attn_ms, 2), "k1_share": round(attn_ms / ms, 3),
                    "k1_tflops_rank": round(flops / W / (attn_ms / 1e3) / 1e12, 1),
                    "k1_tflops_by_block": blk_tf,
                    "head_split": bench.head_split(eng.runner), "g1_fused_norms": eng.runner.g1_all,
                    "g1_choice_ms": getattr(eng.runner, "g1_choice", None)}), flush=True)
                if args.profile:
                    _profile(roll, name, W, r)
                eng.runner.release_graphs()
                del eng
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
        del model
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
