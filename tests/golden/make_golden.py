"""Generate golden fixtures by running the LIVE reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports the unmodified reference from /root/reference/pkg/src (read-only; no
bytecode written) and freezes its outputs under tests/golden/ so the oracle and
the CUDA path can be checked on machines where the reference is absent (the GPU
box). Nothing here is imported by tests at run time except the fixture files.

Fixtures:
  attention.npz      scaled_dot_attention / partial-merge cases (attention.py:74-180)
  kv_traces.json     random op sequences with the reference KvCache's FULL state
                     (page ids, tiers, filled, start_token, last_access, clock,
                     block entries) after every op + sha256 of fetched bytes
                     (kvcache.py:105-404)
  engine_small.npz   generate_sequence / recompute_reference latents for small
                     configs incl. windowed + prompt switches (engine.py:368-489)
  engine_tiny.npz    the c1 workload (2L, 4H, dh64, 768 tok/block, 3 blocks,
                     4 steps) final latents + final cache state
  parallel.npz/json  ulysses_attention vs dense + predict_communication
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from inferix import attention as RA  # noqa: E402
from inferix import engine as RE  # noqa: E402
from inferix import kvcache as RK  # noqa: E402
from inferix import parallel as RP  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def ref_state(cache) -> dict:
    """Canonical snapshot of a reference KvCache (same schema as oracle.kvcache.state)."""
    return {
        "clock": cache._access_clock,
        "next_page": cache._next_page_id,
        "next_block": cache._next_block_id,
        "device_used": cache._device_used,
        "host_used": cache._host_used,
        "streams": [
            [layer, kind, s.base, s.total,
             [[p.id, int(p.tier == RK.HOST), p.filled, p.start_token, p.last_access]
              for p in s.pages]]
            for (layer, kind), s in cache._streams.items()
        ],
        "blocks": [[e.block_id, e.layer, e.kind, e.token_range[0], e.token_range[1],
                    list(e.page_list), e.chunk_index] for e in cache.block_entries()],
    }


def sha(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


def rows(seed, t, d):
    g = np.random.default_rng(seed)
    return (g.standard_normal((t, d)).astype(np.float32),
            g.standard_normal((t, d)).astype(np.float32))


# ---------------------------------------------------------------------------
def gen_attention():
    out = {}
    cases = [(7, 8, 16, 4, 0.7), (3, 5, 7, 4, 1.0), (11, 6, 9, 8, 1.0), (21, 33, 70, 16, 0.8),
             (5, 128, 300, 64, 1.0), (6, 200, 257, 128, 1.0)]
    for i, (seed, n, m, d, dens) in enumerate(cases):
        g = np.random.default_rng(seed)
        q = g.standard_normal((n, d)).astype(np.float32)
        k = g.standard_normal((m, d)).astype(np.float32)
        v = g.standard_normal((m, d)).astype(np.float32)
        mask = g.random((n, m)) < dens
        mask[:, 0] = True
        out[f"c{i}_q"], out[f"c{i}_k"], out[f"c{i}_v"], out[f"c{i}_mask"] = q, k, v, mask
        out[f"c{i}_out"] = RA.scaled_dot_attention(q, k, v, mask)
        cut = m // 3
        pa = RA.attention_partial(q, k[:cut], v[:cut], mask[:, :cut])
        pb = RA.attention_partial(q, k[cut:], v[cut:], mask[:, cut:])
        pm = RA.merge_partials(pa, pb)
        out[f"c{i}_pa_acc"], out[f"c{i}_pa_max"], out[f"c{i}_pa_den"] = pa.acc, pa.row_max, pa.denom
        out[f"c{i}_merged"] = RA.finalize_partial(pm)
    out["ncases"] = np.array(len(cases))
    for nb, bl, win in [(3, 4, None), (4, 3, 5), (2, 5, 0)]:
        out[f"mask_{nb}_{bl}_{win}"] = RA.windowed_block_causal_mask(nb, bl, win)
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **out)


# ---------------------------------------------------------------------------
def run_kv_sequence(seed, n_ops):
    """Random ops incl. cross appends/clears; record result + full state per op."""
    g = np.random.default_rng(seed)
    cfg = dict(num_layers=2, head_dim=8, page_len=int(g.integers(1, 24)),
               capacity_pages_device=int(g.integers(0, 12)),
               capacity_pages_host=int(g.integers(0, 24)))
    cache = RK.create_cache(RK.KvConfig(**cfg))
    ops, live = [], []
    kinds = ("append", "append", "append_cross", "fetch_range", "fetch_indices",
             "offload", "evict", "clear_cross", "fetch_cross")
    for step in range(n_ops):
        op = kinds[int(g.integers(0, len(kinds)))]
        layer = int(g.integers(0, 2))
        rec = {"op": op, "layer": layer}
        try:
            if op in ("append", "append_cross"):
                t = int(g.integers(1, 40))
                dseed = int(g.integers(0, 2**31))
                k, v = rows(dseed, t, 8)
                kind = RK.SELF_ATTN if op == "append" else RK.CROSS_ATTN
                rec.update(t=t, dseed=dseed)
                e = cache.append_block(layer, k, v, kind=kind, chunk_index=step)
                live.append(e.block_id)
                rec.update(result=[e.block_id, list(e.token_range), e.page_list])
            elif op == "offload":
                ids = [int(x) for x in g.choice(live, size=min(2, len(live)), replace=False)] if live else []
                cur = {b.block_id for b in cache.block_entries()}
                ids = [i for i in ids if i in cur]
                rec.update(ids=ids)
                rec.update(result=cache.offload_blocks(ids))
            elif op == "evict":
                keep = int(g.integers(0, 48))
                rec.update(keep=keep)
                rec.update(result=cache.evict_window(keep))
            elif op == "clear_cross":
                rec.update(result=cache.clear_cross_attention())
            else:
                kind = RK.CROSS_ATTN if op == "fetch_cross" else RK.SELF_ATTN
                base, total = cache.addressable_range(layer, kind)
                if total == base:
                    rec.update(op="noop")
                elif op == "fetch_indices":
                    idx = [int(x) for x in g.integers(base, total, size=int(g.integers(0, 6)))]
                    fk, fv = cache.fetch_indices(layer, idx)
                    rec.update(idx=idx, result=sha(fk, fv))
                else:
                    a = int(g.integers(base, total))
                    b = int(g.integers(a, total)) + 1
                    fk, fv = cache.fetch_range(layer, (a, b), kind)
                    rec.update(op="fetch_range", kind=kind, range=[a, b], result=sha(fk, fv))
        except RK.CapacityError:
            rec["error"] = "CapacityError"
        rec["state"] = ref_state(cache)
        ops.append(rec)
    return {"seed": seed, "config": cfg, "ops": ops}


def gen_kv():
    seqs = [run_kv_sequence(s, 25) for s in range(60)]
    # SURVEY A4 case 1 (known-answer trace)
    cache = RK.create_cache(RK.KvConfig(num_layers=1, head_dim=4, page_len=4,
                                        capacity_pages_device=2, capacity_pages_host=8))
    a4 = []
    k, v = rows(1, 10, 4)
    cache.append_block(0, k, v); a4.append(ref_state(cache))
    cache.fetch_range(0, (8, 10)); a4.append(ref_state(cache))
    cache.fetch_range(0, (0, 2)); a4.append(ref_state(cache))
    k, v = rows(2, 3, 4)
    cache.append_block(0, k, v); a4.append(ref_state(cache))
    cache.evict_window(5); a4.append(ref_state(cache))
    with open(os.path.join(HERE, "kv_traces.json"), "w") as f:
        json.dump({"sequences": seqs, "a4_case1": a4}, f, separators=(",", ":"))


# ---------------------------------------------------------------------------
SMALL_ENGINE_CASES = [
    # (layers, heads, head_dim, block_len, num_blocks, steps, seed, window, prompts, wseed)
    (2, 2, 8, 8, 2, [1.0, 0.5, 0.25], 3, None, [(0, "a quiet scene")], 0),
    (2, 2, 4, 20, 2, [1.0, 0.5], 0, None, [(0, "a b c"), (1, "d e")], 0),
    (3, 4, 8, 16, 3, [1.0, 0.5, 0.25], 5, 16, [(0, "x"), (2, "y z")], 1),
    (1, 1, 8, 32, 4, [1.0, 0.75, 0.5, 0.25], 9, None, [(0, "a quiet scene")], 2),
    (2, 4, 16, 24, 3, [1.0, 0.5], 1, 30, [(0, "red"), (1, "blue sky")], 3),
]


def gen_engine_small():
    out = {}
    for i, (L, H, dh, bl, nb, steps, seed, win, prompts, wseed) in enumerate(SMALL_ENGINE_CASES):
        model = RE.build_model(RE.ModelConfig(layers=L, heads=H, head_dim=dh, block_len=bl,
                                              frame_shape=(8, 8), prompt_dim=8, weight_seed=wseed))
        req = RE.GenerationRequest(num_blocks=nb, schedule=RE.DenoiseSchedule(steps=steps),
                                   seed=seed, prompt_schedule=prompts, kv_window=win)
        eng = RE.Engine(model)
        got = eng.generate(req)
        want = RE.recompute_reference(model, req)
        out[f"e{i}_cached"] = np.stack([b.latent for b in got])
        out[f"e{i}_recompute"] = np.stack([b.latent for b in want])
        out[f"e{i}_frames0"] = np.stack(got[0].frames)
        out[f"e{i}_state"] = np.frombuffer(json.dumps(ref_state(eng.cache)).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "engine_small.npz"), **out)


def gen_engine_tiny():
    """c1: BASELINE.json configs[0]."""
    model = RE.build_model(RE.ModelConfig(layers=2, heads=4, head_dim=64, block_len=768,
                                          frame_shape=(16, 16), prompt_dim=16, weight_seed=0))
    req = RE.GenerationRequest(num_blocks=3, schedule=RE.DenoiseSchedule(steps=[1.0, 0.75, 0.5, 0.25]),
                               seed=0)
    eng = RE.Engine(model)
    got = eng.generate(req)
    np.savez_compressed(
        os.path.join(HERE, "engine_tiny.npz"),
        latents=np.stack([b.latent for b in got]),
        state=np.frombuffer(json.dumps(ref_state(eng.cache)).encode(), np.uint8),
        wq0_sha=np.frombuffer(sha(model.layers[0].wq).encode(), np.uint8),
        wdec_sha=np.frombuffer(sha(model.w_decode).encode(), np.uint8))


# ---------------------------------------------------------------------------
def gen_parallel():
    out, preds = {}, []
    for seq_len in (8, 24, 64):
        for heads in (1, 2, 4):
            for world in (1, 2, 4):
                g = np.random.default_rng(seq_len + 10 * heads + world)
                d = heads * 4
                lens = RP.equal_shards(seq_len, world)
                qs = [g.standard_normal((n, d)).astype(np.float32) for n in lens]
                ks = [g.standard_normal((n, d)).astype(np.float32) for n in lens]
                vs = [g.standard_normal((n, d)).astype(np.float32) for n in lens]
                mask = RA.block_causal_mask(seq_len // 4, 4)
                tag = f"{seq_len}_{heads}_{world}"
                out[f"dense_{tag}"] = np.concatenate(RP.dense_reference(qs, ks, vs, heads, mask))
                if heads % world == 0:
                    grp = RP.WorkerGroup(world)
                    out[f"ulysses_{tag}"] = np.concatenate(
                        RP.ulysses_attention(grp, qs, ks, vs, heads, mask))
                    traced = [t for t in grp.trace if t.sender != t.receiver]
                    out[f"trace_{tag}"] = np.array([len(traced), sum(t.bytes for t in traced)])
                for name, fn in (("ringkv", RP.ring_attention_pass_kv),
                                 ("ringq", RP.ring_attention_pass_q)):
                    grp = RP.WorkerGroup(world)
                    out[f"{name}_{tag}"] = np.concatenate(fn(grp, qs, ks, vs, mask, heads=heads))
                    traced = [t for t in grp.trace if t.sender != t.receiver]
                    out[f"{name}trace_{tag}"] = np.array([len(traced), sum(t.bytes for t in traced)])
                for s in RP.STRATEGIES:
                    if s == "ulysses" and heads % world:
                        continue
                    preds.append([s, lens, heads, 4, world,
                                  list(RP.predict_communication(s, lens, heads, 4, world))])
    np.savez_compressed(os.path.join(HERE, "parallel.npz"), **out)
    chosen = [[sl, h, w, RP.choose_strategy(sl, h, w, RP.LinkCostModel())]
              for sl in (64, 4680) for h in (4, 12, 40) for w in (1, 2, 4, 8)]
    with open(os.path.join(HERE, "parallel.json"), "w") as f:
        json.dump({"predictions": preds, "choices": chosen}, f)


if __name__ == "__main__":
    gen_attention()
    gen_kv()
    gen_engine_small()
    gen_engine_tiny()
    gen_parallel()
    for n in sorted(os.listdir(HERE)):
        print(n, os.path.getsize(os.path.join(HERE, n)))
