"""3D RoPE oracle (no reference counterpart — parity unpinned by the reference, see
oracle/rope.py): algebraic properties and the cache-correctness invariant with RoPE on."""

import numpy as np

from oracle import engine as OE
from oracle.rope import apply_rope, rope_parts, rope_tables


def test_parts_follow_wan_split():
    assert rope_parts(128) == (44, 42, 42)
    assert rope_parts(64) == (24, 20, 20)
    assert sum(rope_parts(96)) == 96


def test_rotation_preserves_pair_norms_and_identity_at_origin():
    g = np.random.default_rng(0)
    x = g.standard_normal((24, 2 * 64)).astype(np.float32)
    cos, sin = rope_tables((2, 3, 4), 5, 64)
    y = apply_rope(x, cos, sin, 2)
    n0 = np.linalg.norm(x.reshape(24, 2, 32, 2), axis=-1)
    n1 = np.linalg.norm(y.reshape(24, 2, 32, 2), axis=-1)
    np.testing.assert_allclose(n0, n1, rtol=1e-5, atol=1e-6)
    c0, s0 = rope_tables((1, 1, 1), 0, 64)  # position (0, 0, 0): no rotation
    np.testing.assert_allclose(apply_rope(x[:1], c0, s0, 2), x[:1], atol=1e-7)


def test_scores_depend_on_relative_frame_only():
    """q.k after RoPE is invariant to shifting every token by the same number of frames."""
    g = np.random.default_rng(1)
    q = g.standard_normal((12, 64)).astype(np.float32)
    k = g.standard_normal((12, 64)).astype(np.float32)
    a = rope_tables((3, 2, 2), 0, 64)
    b = rope_tables((3, 2, 2), 7, 64)
    s_a = apply_rope(q, *a, 1) @ apply_rope(k, *a, 1).T
    s_b = apply_rope(q, *b, 1) @ apply_rope(k, *b, 1).T
    np.testing.assert_allclose(s_a, s_b, atol=2e-4)


def test_cached_generation_equals_recompute_with_rope():
    """The reference's core invariant (test_engine.py:187-218) holds with 3D RoPE: cached
    post-RoPE K at absolute positions == full recompute."""
    for window in (None, 8):
        cfg = OE.ModelConfig(layers=2, heads=2, head_dim=12, block_len=8, frame_shape=(4, 4),
                             prompt_dim=8, rope_grid=(2, 2, 2))
        model = OE.ToyModel(cfg)
        req = OE.GenerationRequest(3, OE.DenoiseSchedule([1.0, 0.5]), seed=4,
                                   prompt_schedule=[(0, "a"), (2, "b c")], kv_window=window)
        lats, _ = OE.generate_sequence(model, req)
        ref = OE.recompute_reference(model, req)
        assert max(float(np.abs(a - b).max()) for a, b in zip(lats, ref)) <= 1e-4
        # and RoPE actually changes the result
        plain = OE.ToyModel(OE.ModelConfig(layers=2, heads=2, head_dim=12, block_len=8,
                                           frame_shape=(4, 4), prompt_dim=8))
        assert np.abs(OE.generate_sequence(plain, req)[0][1] - lats[1]).max() > 1e-3
