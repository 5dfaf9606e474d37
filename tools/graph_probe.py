"""Feasibility: capture one denoise pass (our ctypes kernels + cuBLAS) in a CUDA graph and
replay it; compare with eager and time both (c2 shape, 1 cached block)."""
import time

import torch

from paper_2511_20714_b200 import engine as E

mc = E.ModelConfig(layers=30, heads=12, head_dim=128, block_len=4680, frame_shape=(16, 16), prompt_dim=16)
model = E.build_model(mc, weights="device")
kvc = E.default_kv_config(mc, capacity_pages_device=10**8)
eng = E.Engine(model, kvc)
req = E.GenerationRequest(2, E.DenoiseSchedule([1.0, 0.75, 0.5, 0.25]), seed=0)
g = torch.Generator(device="cuda").manual_seed(0)
noise = [torch.randn(mc.block_len, mc.model_dim, device="cuda", generator=g) for _ in range(2)]
eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)
cache = eng.cache
runner = E._runner(model)
ctx, cross = E._block_context(model, cache, E.embed_prompt(model, "a quiet scene"), runner.stager, 1)
lat = noise[0].clone()
eps = torch.empty_like(lat)
runner.forward(lat, 1.0, ctx, cross, None, eps_out=eps)  # warm (allocations, attributes)
ref = eps.clone()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    ctx.calls = 0
    with torch.cuda.graph(graph):
        runner.forward(lat, 1.0, ctx, cross, None, eps_out=eps)
torch.cuda.current_stream().wait_stream(s)
eps.zero_()
graph.replay()
torch.cuda.synchronize()
print("graph vs eager max abs diff:", float((eps - ref).abs().max()))
for name, fn in (("eager", lambda: runner.forward(lat, 1.0, ctx, cross, None, eps_out=eps)),
                 ("graph", graph.replay)):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    h = (time.perf_counter() - t0) / 5
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) / 5
    print(f"{name}: host enqueue {h*1e3:.2f} ms, wall {w*1e3:.2f} ms per pass")
