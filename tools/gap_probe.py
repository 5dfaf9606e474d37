"""Where the GPU idles inside a c2 rollout: torch.profiler (CUPTI) timeline of one warm
rollout, GPU gaps > 20 us listed with the host op that was running when each gap began.

    python tools/gap_probe.py [--blocks N]
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
    ap.add_argument("--out", default="gpurun_out/gap_trace.json")
    args = ap.parse_args()
    c = bench.CONFIGS["c2"]
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0)
    model = E.build_model(mc, weights=c["weights"])
    nb = c["blocks"]
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(nb, E.DenoiseSchedule(bench.STEPS), seed=0)
    noise = [torch.from_numpy(E._init_noise(mc, 0, ch)).cuda() for ch in range(nb)]
    eng = E.Engine(model, kvc)

    def roll():
        return eng.generate(req, noise_provider=lambda ch: noise[ch], to_host=False)

    for _ in range(3):
        roll()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
        roll()
        torch.cuda.synchronize()
    prof.export_chrome_trace(args.out)
    ev = json.load(open(args.out))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")
                  and "dur" in e], key=lambda e: e["ts"])
    cpu = [e for e in ev if e.get("cat") in ("cpu_op", "python_function", "user_annotation")
           and "dur" in e]
    t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
    busy = 0.0
    end = t0
    gaps = []
    for e in gpu:
        if e["ts"] > end + 20:
            gaps.append((e["ts"] - end, end, e["name"][:60]))
        busy += max(0.0, e["ts"] + e["dur"] - max(e["ts"], end))
        end = max(end, e["ts"] + e["dur"])
    span = t1 - t0
    print(f"GPU span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms ({busy / span:.1%}), "
          f"{len(gaps)} gaps > 20 us totalling {sum(g[0] for g in gaps) / 1e3:.1f} ms")

    def host_at(ts):
        best = None
        for e in cpu:
            if e["ts"] <= ts <= e["ts"] + e["dur"] and e.get("cat") != "user_annotation":
                if best is None or e["dur"] < best["dur"]:
                    best = e
        return best["name"][:70] if best else "?"

    agg = collections.defaultdict(lambda: [0, 0.0])
    for g, ts, nxt in gaps:
        k = (host_at(ts), nxt)
        agg[k][0] += 1
        agg[k][1] += g
    for (h, nxt), (n, tot) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{tot / 1e3:8.2f} ms  {n:4d} gaps  host: {h}  -> next kernel: {nxt}")


if __name__ == "__main__":
    main()
