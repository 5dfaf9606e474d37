"""Time the host noise generator (csrc/noise_host.cpp) against numpy's sequential draw."""
import os
import time

import numpy as np
import torch

from paper_2511_20714_b200.engine import host_normal_f32

T, D = 4680, 1536
print("cpu_count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for rep in range(2):
    t = time.perf_counter()
    ref = np.random.default_rng([7, rep]).standard_normal((T, D)).astype(np.float32)
    print(f"numpy sequential: {(time.perf_counter() - t) * 1e3:.1f} ms")
pinned = torch.empty((T, D), dtype=torch.float32, pin_memory=torch.cuda.is_available())
for th in (1, 4, 8, 15, 16, 32, None):
    best = 1e9
    for rep in range(3):
        t = time.perf_counter()
        host_normal_f32(np.random.default_rng([7, 1]), pinned, threads=th)
        best = min(best, time.perf_counter() - t)
    print(f"native threads={th}: {best * 1e3:.2f} ms")
