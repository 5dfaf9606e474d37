"""Host (Python + launch) cost of one c2-shaped rollout: same 30 layers x 12 heads x 128 and
launch sequence, but 256 tokens per block so the GPU work is negligible; wall time of the
rollout ~ host enqueue cost. Compare with bench.py's ms_per_step to see how close the
engine is to being host-bound."""
import json
import time

import torch

from paper_2511_20714_b200 import engine as E

mc = E.ModelConfig(layers=30, heads=12, head_dim=128, block_len=256, frame_shape=(16, 16), prompt_dim=16)
model = E.build_model(mc, weights="device")
kvc = E.default_kv_config(mc, capacity_pages_device=10**8)
req = E.GenerationRequest(7, E.DenoiseSchedule([1.0, 0.75, 0.5, 0.25]), seed=0)
noise = [torch.randn(mc.block_len, mc.model_dim, device="cuda") for _ in range(7)]
eng = E.Engine(model, kvc)
roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)  # noqa: E731
for _ in range(3):
    roll()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    roll()
torch.cuda.synchronize()
print(json.dumps({"host_ms_per_rollout": round((time.perf_counter() - t0) / 3 * 1e3, 1),
                  "note": "c2 layer/launch structure at 256 tokens per block"}))
