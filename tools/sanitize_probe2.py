"""compute-sanitizer probe for the r05 paths: the Ulysses engine with the peer-memory
exchange (G1 scatter epilogue, K1 O scatter, peer barriers, K2 page write from the receive
region) in its whole-head and grouped forms, G1 with the norms fused (IFX_G1=all), the
real-rank strategy API (copy-engine pulls, K1 partials, K4 combine), and PDL launches.
World size 1 (in-process gloo group): the mesh maps this rank's own arena."""
import os

os.environ.setdefault("IFX_G1", "all")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29561")

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2511_20714_b200 import engine as E  # noqa: E402
from paper_2511_20714_b200 import parallel as P  # noqa: E402

E.GRAPHS = False  # keep every launch visible to the tool
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=0, world_size=1)
cfg = dict(layers=2, heads=3, head_dim=64, block_len=96, frame_shape=(4, 4), prompt_dim=8,
           rope_grid=(1, 8, 12))
req = E.GenerationRequest(3, E.DenoiseSchedule([1.0, 0.5]), 0, [(0, "a b"), (2, "c")])
eng = P.UlyssesEngine(E.ToyModel(E.ModelConfig(**cfg)), P.UlyssesComm(), p2p=True)
lats = eng.generate(req)
assert all(np.isfinite(x.cpu().numpy()).all() for x in lats)
# the strategy API: unequal shards are impossible at world 1, but every code path runs
r = np.random.default_rng(0)
q = r.standard_normal((40, 128)).astype(np.float32)
k = r.standard_normal((56, 128)).astype(np.float32)
mask = r.random((40, 56)) < 0.7
mask[:, 0] = True
for st in ("ulysses", "ring_pass_kv", "ring_pass_q"):
    out, _ = P.sequence_parallel_attention(P.UlyssesComm(), q, k, k, 2, mask, strategy=st)
    assert np.isfinite(out.cpu().numpy()).all()
torch.cuda.synchronize()
eng.runner.release_graphs()
dist.destroy_process_group()
print("sanitize probe 2 ok")
