"""Small end-to-end runs for compute-sanitizer (memcheck): the engine with a host tier
(K6 moves, DMA staging, paged K1 with staging codes), the folded cross-attention, K2/K7,
the few-keys kernel, the persistent K1 with several items per CTA (and split-KV), and the
block copies."""
import numpy as np
import torch

from paper_2511_20714_b200 import engine as E
from paper_2511_20714_b200._device import attn_fwd

E.GRAPHS = False  # keep every launch visible to the tool
kw = dict(layers=3, heads=2, head_dim=64, block_len=48, frame_shape=(4, 4), prompt_dim=8)
kvc = E.KvConfig(num_layers=3, head_dim=128, page_len=16, capacity_pages_device=10,
                 capacity_pages_host=10**4)
eng = E.Engine(E.build_model(E.ModelConfig(**kw)), kvc)
blocks = eng.generate(E.GenerationRequest(4, E.DenoiseSchedule([1.0, 0.5]), 1, [(0, "a b"), (2, "c")]))
assert all(np.isfinite(b.latent).all() for b in blocks)
q = torch.randn(2000, 256, device="cuda").bfloat16()
k = torch.randn(3, 256, device="cuda").bfloat16()
o = torch.empty_like(q)
attn_fwd(q, 2, 128, o, k, k, 0, 3)  # K1s
# persistent K1 with several items per CTA: 12 heads x 20 query tiles = 240 items on 148
# CTAs (contiguous context + own keys); then 5 heads, split-KV partials + K4 combine
q = torch.randn(2500, 12 * 128, device="cuda").bfloat16()
kv = torch.randn(700, 12 * 128, device="cuda").bfloat16()
o = torch.empty_like(q)
attn_fwd(q, 12, 128, o, kv, kv, 0, 700, q, q)
q5 = torch.randn(4680, 5 * 128, device="cuda").bfloat16()
kv5 = torch.randn(9000, 5 * 128, device="cuda").bfloat16()
o5 = torch.empty_like(q5)
attn_fwd(q5, 5, 128, o5, kv5, kv5, 0, 9000, q5, q5)
torch.cuda.synchronize()
print("sanitize probe ok", eng.cache.memory_stats())
