"""The reference's acceptance gates (/root/reference/pkg/tests/test_acceptance.py) re-run
through the B200 path, against fixtures frozen from the live reference
(tests/golden/make_golden_deep.py -> acceptance.npz).

* KV differential, 10,000 sequences (test_acceptance.py:126-134 driving
  test_kvcache.py:286-331): the same random op sequences, draw for draw
  (tests/kv_differential.py), through the device KvCache — native page table, fp32 HBM and
  pinned-host pools, K2 page writes, K6 tier moves, K7 gathers. Every observable (block
  entries, offload / evict counts, addressable ranges, every fetched byte, the final full
  bookkeeping state) is hashed per sequence and must equal the reference's digest:
  bit-exact. The oracle is pinned on the same digests on CPU.
* Cache correctness, 12 randomized configs (test_acceptance.py:51-81): the B200 engine's
  cached generation vs the reference's cached latents AND the B200 cache-free recompute
  vs the reference's recompute, within the stated bf16/fp32 tolerance (max-abs 2e-2,
  cosine > 0.999); and the B200 engine's own cache == recompute.
"""

import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN
import kv_differential as KD

ATOL_LATENT = 2e-2


def _golden():
    return np.load(os.path.join(GOLDEN, "acceptance.npz"))


def _digests():
    """The 10,000 reference digests (stored as numpy S32, which drops trailing NULs)."""
    return [bytes(d).ljust(32, b"\0") for d in _golden()["kv_digests"]]


def _cos(a, b):
    a, b = a.ravel().astype(np.float64), b.ravel().astype(np.float64)
    return float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))


def test_oracle_kv_differential_10000():
    """CPU: the oracle KvStore reproduces all 10,000 reference digests (pins the oracle)."""
    from oracle import kvcache as OK

    want = _digests()
    make = lambda **kw: OK.create_cache(OK.KvConfig(**kw))  # noqa: E731
    t0 = time.monotonic()
    for seed in range(10_000):
        got = KD.run_sequence(make, lambda c: c.state(), lambda a: a,
                              np.random.default_rng(seed), n_ops=15)
        assert bytes.fromhex(got) == want[seed], f"seed {seed}"
    print(f"oracle kv differential 10000: {time.monotonic() - t0:.1f}s")


@pytest.mark.gpu
def test_kv_differential_10000_gpu():
    """The reference's 10,000-sequence KV differential through the device KvCache: every
    sequence's digest bit-identical to the live reference's."""
    from paper_2511_20714_b200 import kvcache as K

    want = _digests()
    make = lambda **kw: K.create_cache(K.KvConfig(**kw))  # noqa: E731
    to_np = lambda t: t.float().cpu().numpy()  # noqa: E731
    t0 = time.monotonic()
    bad = []
    for seed in range(10_000):
        got = KD.run_sequence(make, lambda c: c.state(), to_np, np.random.default_rng(seed), n_ops=15)
        if bytes.fromhex(got) != want[seed]:
            bad.append(seed)
    print(f"B200 kv differential 10000: {len(bad)} mismatches, {time.monotonic() - t0:.1f}s")
    assert not bad, f"sequences differing from the reference: {bad[:20]}"


def _trials():
    g = _golden()
    for trial in range(12):
        cfg, req = json.loads(bytes(g[f"t{trial}_cfg"]).decode())
        yield trial, cfg, req, g[f"t{trial}_cached"], g[f"t{trial}_recompute"]


@pytest.mark.gpu
def test_cache_correctness_12_configs_gpu():
    """test_acceptance.py:51-81 on device: 12 randomized configs (1-4 layers, 1/2/4 heads of
    width 4/8, blocks of 4-32 tokens, windowed or not)."""
    from paper_2511_20714_b200 import engine as E

    worst = [0.0, 0.0, 0.0]
    for trial, cfg, req, want_cached, want_rec in _trials():
        cfg["frame_shape"] = tuple(cfg["frame_shape"])
        model = E.build_model(E.ModelConfig(**cfg))
        mk = lambda: E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5, 0.25]), **req)  # noqa: E731
        got = np.stack([b.latent for b in E.generate_sequence(model, mk())])
        rec = np.stack([b.latent for b in E.recompute_reference(model, mk())])
        errs = (float(np.abs(got - want_cached).max()), float(np.abs(rec - want_rec).max()),
                float(np.abs(got - rec).max()))
        for i, e in enumerate(errs):
            worst[i] = max(worst[i], e)
        assert errs[0] <= ATOL_LATENT and _cos(got, want_cached) > 0.999, (trial, errs)
        assert errs[1] <= ATOL_LATENT and _cos(rec, want_rec) > 0.999, (trial, errs)
        assert errs[2] <= ATOL_LATENT, (trial, errs)
    print(f"12 configs: cached vs reference {worst[0]:.2e}, recompute vs reference "
          f"{worst[1]:.2e}, B200 cache vs B200 recompute {worst[2]:.2e}")
