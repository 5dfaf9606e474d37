"""Deep golden fixtures from the LIVE reference (build container only; hours of numpy).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_deep.py [acceptance] [c2] [c3]

Like make_golden.py this imports the unmodified reference from /root/reference/pkg/src
(read-only) and freezes its outputs, here at the depths the GPU parity tests need:

  acceptance.npz   the reference's acceptance gates restated as fixtures:
                   * kv_differential: sha256 digest of every observable of the
                     10,000-sequence KV differential (test_acceptance.py:126-134 driving
                     test_kvcache.py:286-331, n_ops=15), driven by tests/kv_differential.py
                   * cache_correctness: the 12 randomized configs of
                     test_acceptance.py:51-81 — cached and recomputed latents per trial
  c2_deep.npz      BASELINE configs[1] at FULL depth: 30 layers x 12 heads x 128, T = 4680,
                   3 blocks x 4 denoise steps (steps 1.0/0.75/0.5/0.25), weight_seed 0,
                   seed 0, "a quiet scene", engine.py:368-411 with capacity_pages_device=1e8.
                   Per block: a row subset of the final latent (first/last 32 rows + every
                   47th), full-tensor float64 moments, and the final cache state (zlib JSON)
  c3_deep.npz      configs[2] length: 21 blocks (20 cached, context 93,600 tokens) at
                   2 layers, 1 denoise step: per-block row subsets + moments + final state
  c4_deep.npz      configs[3] width: the 14B shape (40 heads x 128, D = 5,120, T = 4,680) at
                   3 layers, 2 blocks x 2 denoise steps (1.0 / 0.5): row subsets + moments
                   + final state

Timing on the 8-core build container: acceptance ~2 min, c2 ~80 min, c3 ~75 min, c4 8.5 min.
"""

from __future__ import annotations

import json
import os
import sys
import time
import zlib

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))  # tests/ (kv_differential driver)

import numpy as np  # noqa: E402

from inferix import engine as RE  # noqa: E402
from inferix import kvcache as RK  # noqa: E402

import kv_differential as KD  # noqa: E402
from make_golden import ref_state  # noqa: E402

STEPS = [1.0, 0.75, 0.5, 0.25]


def sample_rows(t: int, edge: int, stride: int) -> np.ndarray:
    mid = np.arange(edge, max(edge, t - edge), stride)
    return np.unique(np.concatenate([np.arange(min(edge, t)), mid, np.arange(max(0, t - edge), t)]))


def moments(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.float64)
    return np.array([x.sum(), (x * x).sum(), np.abs(x).sum(), np.abs(x).max()])


def gen_acceptance():
    t0 = time.time()
    make = lambda **kw: RK.create_cache(RK.KvConfig(**kw))  # noqa: E731
    digests = [KD.run_sequence(make, ref_state, lambda a: a, np.random.default_rng(seed), n_ops=15)
               for seed in range(10_000)]
    out = {"kv_digests": np.array([bytes.fromhex(d) for d in digests], dtype="S32")}
    print(f"kv differential 10000: {time.time() - t0:.1f}s", flush=True)
    # test_acceptance.py:51-81, draw for draw
    rng = np.random.default_rng(2026)
    for trial in range(12):
        layers = int(rng.integers(1, 5))
        heads = int(rng.choice([1, 2, 4]))
        head_dim = int(rng.choice([4, 8]))
        block_len = int(rng.choice([4, 8, 16, 32]))
        num_blocks = int(rng.integers(1, 5))
        windowed = bool(rng.integers(0, 2)) and num_blocks > 1
        cfg = dict(layers=layers, heads=heads, head_dim=head_dim, block_len=block_len,
                   frame_shape=(8, 8), prompt_dim=8, weight_seed=trial)
        req = dict(num_blocks=num_blocks, seed=trial, kv_window=block_len if windowed else None)
        model = RE.build_model(RE.ModelConfig(**cfg))
        mk = lambda: RE.GenerationRequest(schedule=RE.DenoiseSchedule(steps=[1.0, 0.5, 0.25]), **req)  # noqa: E731
        got = RE.generate_sequence(model, mk())
        want = RE.recompute_reference(model, mk())
        out[f"t{trial}_cfg"] = np.frombuffer(json.dumps([cfg, req]).encode(), np.uint8)
        out[f"t{trial}_cached"] = np.stack([b.latent for b in got])
        out[f"t{trial}_recompute"] = np.stack([b.latent for b in want])
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **out)
    print(f"acceptance done: {time.time() - t0:.1f}s", flush=True)


def gen_deep(name, layers, blocks, steps, edge, stride, heads=12):
    t0 = time.time()
    mc = RE.ModelConfig(layers=layers, heads=heads, head_dim=128, block_len=4680, frame_shape=(16, 16),
                        prompt_dim=16, weight_seed=0)
    model = RE.build_model(mc)
    eng = RE.Engine(model, RE.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096))
    rows = sample_rows(mc.block_len, edge, stride)
    out = {"rows": rows, "meta": np.frombuffer(json.dumps(dict(
        layers=layers, heads=heads, head_dim=128, block_len=4680, blocks=blocks, steps=steps,
        frame_shape=[16, 16], prompt_dim=16, weight_seed=0, seed=0,
        prompt="a quiet scene", capacity_pages_device=10**8, capacity_pages_host=4096)).encode(), np.uint8)}

    def sink(block):
        c = block.chunk_index
        out[f"b{c}_rows"] = block.latent[rows]
        out[f"b{c}_moments"] = moments(block.latent)
        out[f"b{c}_frame_rows"] = np.stack([block.frames[r] for r in rows])
        print(f"{name}: block {c} done at {time.time() - t0:.0f}s", flush=True)
        # checkpoint after every block so a partial run is still usable
        np.savez_compressed(os.path.join(HERE, f"{name}.partial.npz"), **out)

    req = RE.GenerationRequest(num_blocks=blocks, schedule=RE.DenoiseSchedule(steps=steps), seed=0)
    eng.generate(req, sinks=[sink])
    st = KD.canon(ref_state(eng.cache))
    out["state_z"] = np.frombuffer(zlib.compress(json.dumps(st, separators=(",", ":")).encode(), 9),
                                   np.uint8)
    out["state_sha"] = np.frombuffer(KD.state_digest(st).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    os.remove(os.path.join(HERE, f"{name}.partial.npz"))
    print(f"{name} done: {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["acceptance", "c2", "c3", "c4"]
    if "acceptance" in what:
        gen_acceptance()
    if "c2" in what:
        gen_deep("c2_deep", layers=30, blocks=3, steps=STEPS, edge=32, stride=47)
    if "c3" in what:
        gen_deep("c3_deep", layers=2, blocks=21, steps=[1.0], edge=16, stride=293)
    if "c4" in what:
        gen_deep("c4_deep", layers=3, blocks=2, steps=[1.0, 0.5], edge=16, stride=97, heads=40)
