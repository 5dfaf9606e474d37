"""cProfile of the host side of one c2-structured rollout with 256 tokens per block (GPU work
negligible, so the profile is the pure enqueue cost: Python, ctypes, launches)."""
import cProfile
import pstats

import torch

from paper_2511_20714_b200 import engine as E

mc = E.ModelConfig(layers=30, heads=12, head_dim=128, block_len=256, frame_shape=(16, 16), prompt_dim=16)
model = E.build_model(mc, weights="device")
kvc = E.default_kv_config(mc, capacity_pages_device=10**8)
req = E.GenerationRequest(7, E.DenoiseSchedule([1.0, 0.75, 0.5, 0.25]), seed=0)
noise = [torch.randn(mc.block_len, mc.model_dim, device="cuda") for _ in range(7)]
eng = E.Engine(model, kvc)
roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)  # noqa: E731
for _ in range(2):
    roll()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
roll()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
