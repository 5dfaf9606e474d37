"""Can torch.distributed NCCL all_to_all_single be captured in a CUDA graph? (world size 1
on the single-GPU box: exercises ProcessGroupNCCL under stream capture.)"""
import os

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
x = torch.randn(1 << 20, device="cuda")
y = torch.empty_like(x)
dist.all_to_all_single(y, x)  # warm (communicator init outside capture)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        z = x * 2
        dist.all_to_all_single(y, z)
        w = y + 1
torch.cuda.current_stream().wait_stream(s)
x.copy_(torch.arange(x.numel(), device="cuda", dtype=torch.float32))
g.replay()
torch.cuda.synchronize()
print("nccl a2a in graph ok:", bool(torch.equal(w, x * 2 + 1)))
# uneven splits (balanced plan style)
sz = [x.numel()]
with torch.cuda.stream(s):
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        dist.all_to_all_single(y, x, sz, sz)
torch.cuda.current_stream().wait_stream(s)
g2.replay()
torch.cuda.synchronize()
print("variable-split a2a in graph ok:", bool(torch.equal(y, x)), flush=True)
import time  # noqa: E402
t0 = time.time()
del g, g2
torch.cuda.synchronize()
dist.destroy_process_group()
print(f"destroy after freeing the graphs: {time.time() - t0:.1f}s", flush=True)
