"""Debug: engine host-tier parity per staging mode (resident / N rotating buffers)."""
import sys

import numpy as np

from oracle import engine as OE
from paper_2511_20714_b200 import engine as E

L, P, cap = 5, 16, 18
kw = dict(layers=L, heads=2, head_dim=64, block_len=40, frame_shape=(4, 4), prompt_dim=8)
req = dict(num_blocks=5, seed=4, prompt_schedule=[(0, "a b"), (3, "c d e")], kv_window=None)
kvc = dict(num_layers=L, head_dim=128, page_len=P, capacity_pages_device=cap, capacity_pages_host=10**4)
want, ocache = OE.generate_sequence(OE.ToyModel(OE.ModelConfig(**kw)), OE.GenerationRequest(
    schedule=OE.DenoiseSchedule([1.0, 0.5]), **req), OE.KvConfig(**kvc))
orig_prepare = E._KvContext.prepare


def prep(self):
    orig_prepare(self)
    if self.paged and self.jobs and not getattr(self, "_printed", False):
        self._printed = True
        print("  block ctx: jobs", self.jobs, "nbuf", self.nbuf, "resident", self.resident, "R", self.R)


E._KvContext.prepare = prep
for mode in sys.argv[1:] or ("big", "3", "2", "0"):
    model = E.build_model(E.ModelConfig(**kw))
    r = E._runner(model)
    if mode == "big":
        r.stager.buffers, r.stager.budget = None, 1 << 30
    else:
        r.stager.buffers, r.stager.budget = (int(mode) if mode != "0" else None), 0
    eng = E.Engine(model, E.KvConfig(**kvc))
    got = eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5]), **req))
    errs = [float(np.abs(g.latent - w).max()) for g, w in zip(got, want)]
    print(mode, ["%.3g" % e for e in errs], eng.cache.state() == ocache.state(), flush=True)
