"""Per-kernel GPU time of one warm block (4 denoise passes + clean pass) of the c2 / c4
workload: torch.profiler (CUPTI) kernel records grouped by kernel name. Run with IFX_G1=0/1
to compare the cuBLASLt + RMS-kernel path with G1's fused epilogues.

    python tools/pass_profile.py [c2|c4] [--cached N]
"""
import argparse
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_20714_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--blocks", type=int, default=2)
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0)
    model = E.build_model(mc, weights="device")
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(args.blocks, E.DenoiseSchedule(bench.STEPS), seed=0)
    g = torch.Generator(device="cuda").manual_seed(0)
    noise = [torch.randn(mc.block_len, mc.model_dim, device="cuda", generator=g) for _ in range(args.blocks)]
    eng = E.Engine(model, kvc)

    def roll():
        return eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)

    for _ in range(2):
        roll()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        roll()
        torch.cuda.synchronize()
    path = f"gpurun_out/pass_trace_{os.getpid()}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    os.unlink(path)
    k = [e for e in ev if e.get("cat") == "kernel" and "dur" in e]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in k:
        n = e["name"]
        key = ("G1 " + n[n.index("gemm_kernel"):n.index(">", n.index("gemm_kernel")) + 1] + " grid " +
               str(e.get("args", {}).get("grid")) if "gemm_kernel" in n else
               "cuBLASLt" if ("nvjet" in n or "cutlass" in n or "sm100" in n or "gemm" in n.lower()) else n[:60])
        agg[key][0] += 1
        agg[key][1] += e["dur"]
    tot = sum(v[1] for v in agg.values())
    print(json.dumps({"config": args.config, "g1": os.environ.get("IFX_G1", "1"),
                      "blocks": args.blocks, "kernel_ms": tot / 1e3}))
    for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{us / 1e3:9.2f} ms {n:6d}  {100 * us / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main()
