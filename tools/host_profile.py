"""cProfile of the host side of one c2 rollout (where do the enqueue microseconds go?)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, STEPS  # noqa: E402
from paper_2511_20714_b200 import engine as E  # noqa: E402

c = CONFIGS["c2"]
mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"], block_len=c["block_len"],
                   frame_shape=(16, 16), prompt_dim=16)
model = E.build_model(mc, weights="device")
kvc = E.default_kv_config(mc, capacity_pages_device=10**8)
req = E.GenerationRequest(c["blocks"], E.DenoiseSchedule(STEPS), seed=0)
noise = [torch.randn(mc.block_len, mc.model_dim, device="cuda") for _ in range(c["blocks"])]
eng = E.Engine(model, kvc)
roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)  # noqa: E731
roll()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
roll()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
