"""Host noise generator (csrc/noise_host.cpp) vs the reference's own draw, engine.py:280-282:
np.random.default_rng([seed, chunk]).standard_normal((T, D)).astype(np.float32). Bit-exact,
for any thread count (the parallel parse must reproduce the sequential stream)."""

import numpy as np
import pytest
import torch

from paper_2511_20714_b200.engine import host_normal_f32
from paper_2511_20714_b200.errors import ConfigError, DimensionError


def _ref(seed, chunk, shape):
    return np.random.default_rng([seed, chunk]).standard_normal(shape).astype(np.float32)


@pytest.mark.parametrize("seed,chunk,shape,threads", [
    (7, 0, (4680, 1536), None),    # c2 block (engine.py:280-282 at the bench config)
    (7, 6, (4680, 1536), 5),
    (0, 0, (256, 64), None),       # below the per-thread minimum: sequential path
    (1, 2, (100003,), 3),          # ragged split
    (5, 1, (1,), 8),
    (3, 4, (70000, 3), 64),        # more threads than 64K-normal chunks
    (11, 0, (0, 16), 4),           # empty
])
def test_noise_bit_exact(seed, chunk, shape, threads):
    out = torch.empty(shape, dtype=torch.float32)
    host_normal_f32(np.random.default_rng([seed, chunk]), out, threads=threads)
    ref = _ref(seed, chunk, shape)
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


def test_noise_rejects_used_or_foreign_generators():
    out = torch.empty(8, dtype=torch.float32)
    rng = np.random.default_rng([1, 1])
    rng.integers(0, 2**32, dtype=np.uint32)  # leaves a buffered 32-bit half: not fresh
    with pytest.raises(ConfigError):
        host_normal_f32(rng, out)
    with pytest.raises(ConfigError):
        host_normal_f32(np.random.Generator(np.random.MT19937(1)), out)
    with pytest.raises(DimensionError):
        host_normal_f32(np.random.default_rng(1), torch.empty(8, dtype=torch.float64))
