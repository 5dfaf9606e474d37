"""Where a Ulysses rank's host time goes at W ranks (loopback mesh, one GPU): torch.profiler
with CPU + CUDA activity over one rollout; prints the largest GPU idle gaps with the host
ops running during each gap, and the top host functions by total time.

    python tools/host_gap_probe.py [--config c2] [--world 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--world", type=int, default=8)
    args = ap.parse_args()
    import cProfile
    import pstats

    import torch.distributed as dist

    import bench
    from paper_2511_20714_b200 import engine as E
    from paper_2511_20714_b200.parallel import LoopbackComm, UlyssesEngine
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29542")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    c = bench.CONFIGS[args.config]
    mc = E.ModelConfig(layers=c["layers"], heads=c["heads"], head_dim=c["head_dim"],
                       block_len=c["block_len"], frame_shape=c["frame_shape"], prompt_dim=16,
                       weight_seed=0)
    model = E.ToyModel(mc, weights=c["weights"])
    nb = c["blocks"]
    kvc = E.default_kv_config(mc, capacity_pages_device=10**8, capacity_pages_host=4096)
    req = E.GenerationRequest(nb, E.DenoiseSchedule(bench.STEPS), seed=0)
    noise = [torch.from_numpy(E._init_noise(mc, 0, ch)).cuda() for ch in range(nb)]
    eng = UlyssesEngine(model, LoopbackComm(args.world, 0), kvc, p2p=True)
    roll = lambda: eng.generate(req, noise_provider=lambda ch: noise[ch], gather=False)  # noqa: E731
    for _ in range(2):
        roll()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    roll()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("cumulative").print_stats(45)
    st.sort_stats("tottime").print_stats(30)
    eng.runner.release_graphs()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
