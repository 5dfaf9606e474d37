"""Run-to-run spread of the end-to-end c2 rollout (public API, host noise, latents to host).

    python tools/e2e_probe.py [--n 6]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_20714_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6)
    args = ap.parse_args()
    c = bench.CONFIGS["c2"]
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0)
    model = E.build_model(mc, weights=c["weights"])
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(c["blocks"], E.DenoiseSchedule(bench.STEPS), seed=0)
    eng = E.Engine(model, kvc)
    for graphs in (True, False, True):
        E.GRAPHS = graphs
        eng.generate(req)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.n):
            t0 = time.perf_counter()
            eng.generate(req)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"graphs={graphs}: ms per rollout", [round(t * 1e3, 1) for t in ts],
              f"fps {[round(21 / t, 2) for t in ts]}", flush=True)


if __name__ == "__main__":
    main()
