"""Pin the CPU oracle against golden vectors frozen from the live reference.

CPU-only; the oracle is the checker used by every GPU parity test, so it must
itself match the reference (tests/golden/make_golden.py) first.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from kv_replay import load_traces, replay

from oracle import attention as OA
from oracle import engine as OE
from oracle import kvcache as OK
from oracle import parallel as OP
from paper_2511_20714_b200.errors import CapacityError, DimensionError, MaskError


@pytest.fixture(scope="module")
def att():
    return np.load(os.path.join(GOLDEN, "attention.npz"))


def test_attention_cases_match_reference(att):
    for i in range(int(att["ncases"])):
        q, k, v, m = (att[f"c{i}_{n}"] for n in ("q", "k", "v", "mask"))
        np.testing.assert_allclose(OA.scaled_dot_attention(q, k, v, m), att[f"c{i}_out"], atol=2e-6)
        cut = k.shape[0] // 3
        pa = OA.attention_partial(q, k[:cut], v[:cut], m[:, :cut])
        np.testing.assert_allclose(pa.acc, att[f"c{i}_pa_acc"], atol=1e-5)
        np.testing.assert_array_equal(pa.row_max, att[f"c{i}_pa_max"])
        pb = OA.attention_partial(q, k[cut:], v[cut:], m[:, cut:])
        np.testing.assert_allclose(OA.finalize_partial(OA.merge_partials(pa, pb)),
                                   att[f"c{i}_merged"], atol=2e-6)


def test_masks_match_reference(att):
    for nb, bl, win in [(3, 4, None), (4, 3, 5), (2, 5, 0)]:
        np.testing.assert_array_equal(OA.windowed_block_causal_mask(nb, bl, win),
                                      att[f"mask_{nb}_{bl}_{win}"])


def test_attention_known_answers_and_errors():
    # test_attention.py:27-39 — single key returns v exactly; tie averages
    v = np.array([[3.0, -1.0]], np.float32)
    out = OA.scaled_dot_attention([[0.3, -2.0]], [[1.0, 5.0]], v, np.ones((1, 1), bool))
    np.testing.assert_array_equal(out, v)
    out = OA.scaled_dot_attention([[1.0, 1.0]], np.eye(2), np.eye(2), np.ones((1, 2), bool))
    np.testing.assert_allclose(out, [[0.5, 0.5]], atol=1e-7)
    with pytest.raises(MaskError):
        OA.scaled_dot_attention(np.ones((2, 4)), np.ones((3, 4)), np.ones((3, 4)),
                                np.array([[1, 1, 1], [0, 0, 0]], bool))
    with pytest.raises(DimensionError):
        OA.scaled_dot_attention(np.ones((2, 4)), np.ones((3, 2)), np.ones((3, 4)), np.ones((2, 3), bool))
    with pytest.raises(DimensionError):
        OA.scaled_dot_attention(np.full((1, 2), np.nan), np.ones((1, 2)), np.ones((1, 2)), np.ones((1, 1), bool))


def test_kv_traces_full_state_bit_exact():
    tr = load_traces()
    for seq in tr["sequences"]:
        replay(seq, lambda c: OK.create_cache(OK.KvConfig(**c)), CapacityError=CapacityError)


def test_kv_survey_a4_case1():
    tr = load_traces()["a4_case1"]
    from kv_replay import rows
    c = OK.create_cache(OK.KvConfig(num_layers=1, head_dim=4, page_len=4,
                                    capacity_pages_device=2, capacity_pages_host=8))
    c.append_block(0, *rows(1, 10, 4)); assert c.state() == tr[0]
    c.fetch_range(0, (8, 10)); assert c.state() == tr[1]
    c.fetch_range(0, (0, 2)); assert c.state() == tr[2]
    c.append_block(0, *rows(2, 3, 4)); assert c.state() == tr[3]
    c.evict_window(5); assert c.state() == tr[4]


SMALL = [
    (2, 2, 8, 8, 2, [1.0, 0.5, 0.25], 3, None, [(0, "a quiet scene")], 0),
    (2, 2, 4, 20, 2, [1.0, 0.5], 0, None, [(0, "a b c"), (1, "d e")], 0),
    (3, 4, 8, 16, 3, [1.0, 0.5, 0.25], 5, 16, [(0, "x"), (2, "y z")], 1),
    (1, 1, 8, 32, 4, [1.0, 0.75, 0.5, 0.25], 9, None, [(0, "a quiet scene")], 2),
    (2, 4, 16, 24, 3, [1.0, 0.5], 1, 30, [(0, "red"), (1, "blue sky")], 3),
]


@pytest.mark.parametrize("i", range(len(SMALL)))
def test_engine_small_matches_reference(i):
    g = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    L, H, dh, bl, nb, steps, seed, win, prompts, wseed = SMALL[i]
    model = OE.ToyModel(OE.ModelConfig(layers=L, heads=H, head_dim=dh, block_len=bl,
                                       frame_shape=(8, 8), prompt_dim=8, weight_seed=wseed))
    req = OE.GenerationRequest(nb, OE.DenoiseSchedule(steps), seed, prompts, win)
    lats, cache = OE.generate_sequence(model, req)
    np.testing.assert_allclose(np.stack(lats), g[f"e{i}_cached"], atol=1e-5)
    assert cache.state() == json.loads(bytes(g[f"e{i}_state"]))
    np.testing.assert_allclose(np.stack(OE.recompute_reference(model, req)), g[f"e{i}_recompute"], atol=1e-5)
    frames = OE.decode_frames(model, lats[0])
    assert np.abs(np.stack(frames).astype(int) - g[f"e{i}_frames0"].astype(int)).max() <= 1


def test_engine_tiny_c1_matches_reference():
    g = np.load(os.path.join(GOLDEN, "engine_tiny.npz"))
    model = OE.ToyModel(OE.ModelConfig(layers=2, heads=4, head_dim=64, block_len=768,
                                       frame_shape=(16, 16), prompt_dim=16, weight_seed=0))
    req = OE.GenerationRequest(3, OE.DenoiseSchedule([1.0, 0.75, 0.5, 0.25]), 0)
    lats, cache = OE.generate_sequence(model, req)
    np.testing.assert_allclose(np.stack(lats), g["latents"], atol=1e-5)
    assert cache.state() == json.loads(bytes(g["state"]))


def test_parameter_count_formula():
    cfg = OE.ModelConfig(layers=2, heads=2, head_dim=16, frame_shape=(8, 8), prompt_dim=16)
    d, p = cfg.model_dim, cfg.prompt_dim
    assert OE.ToyModel(cfg).num_parameters() == 2 * (10 * d * d + 2 * p * d) + d + d * d + d * 64


def test_parallel_matches_reference():
    g = np.load(os.path.join(GOLDEN, "parallel.npz"))
    for seq_len in (8, 24, 64):
        for heads in (1, 2, 4):
            for world in (1, 2, 4):
                r = np.random.default_rng(seq_len + 10 * heads + world)
                d = heads * 4
                lens = OP.equal_shards(seq_len, world)
                qs = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                ks = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                vs = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                mask = OA.block_causal_mask(seq_len // 4, 4)
                tag = f"{seq_len}_{heads}_{world}"
                np.testing.assert_allclose(np.concatenate(OP.dense_reference(qs, ks, vs, heads, mask)),
                                           g[f"dense_{tag}"], atol=1e-6)
                if heads % world == 0:
                    out, trace = OP.ulysses_attention(qs, ks, vs, heads, mask)
                    np.testing.assert_allclose(np.concatenate(out), g[f"ulysses_{tag}"], atol=1e-6)
                    off = [t for t in trace if t[0] != t[1]]
                    assert [len(off), sum(t[2] for t in off)] == g[f"trace_{tag}"].tolist()
                else:
                    with pytest.raises(DimensionError):
                        OP.ulysses_attention(qs, ks, vs, heads, mask)
                for name, fn in (("ringkv", OP.ring_attention_pass_kv), ("ringq", OP.ring_attention_pass_q)):
                    out, trace = fn(qs, ks, vs, mask, heads)
                    np.testing.assert_allclose(np.concatenate(out), g[f"{name}_{tag}"], atol=1e-6)
                    off = [t for t in trace if t[0] != t[1]]
                    assert [len(off), sum(t[2] for t in off)] == g[f"{name}trace_{tag}"].tolist()


def test_comm_predictions_match_reference():
    with open(os.path.join(GOLDEN, "parallel.json")) as f:
        j = json.load(f)
    for s, lens, heads, hd, world, want in j["predictions"]:
        assert list(OP.predict_communication(s, lens, heads, hd, world)) == want
    for sl, h, w, want in j["choices"]:
        got = OP.choose_strategy(sl, h, w)
        assert got["strategy"] == want["strategy"] and got["bytes"] == want["bytes"]
