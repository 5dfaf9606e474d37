"""QKV projection of one Ulysses rank: cuBLASLt (then pack for the all-to-all), G1 plain, and
G1 with the peer-scatter epilogue (destinations in local memory, the layout of rank 0 of
W), at the c2 / c4 rank shapes M = T/W. CUDA events, 20 calls after 5 warm-up.

    python tools/scatter_probe.py
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_20714_b200 import _device as D  # noqa: E402
from paper_2511_20714_b200.parallel import P2PExchange  # noqa: E402


def timed(fn, n=20):
    for _ in range(5):
        fn()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(n):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / n


def main():
    T, dhp = 4680, 128
    for cfg, H, D_ in (("c2", 12, 1536), ("c4", 40, 5120)):
        for W in (1, 2, 4, 8):
            balanced = H % W != 0
            n = T // W
            a = torch.randn(n, D_, device="cuda").bfloat16()
            b = (torch.randn(D_, 3 * H * dhp, device="cuda") / D_ ** 0.5).bfloat16()
            out = torch.empty(n, 3 * H * dhp, device="cuda", dtype=torch.bfloat16)
            rb = P2PExchange.region_bytes(H, T, W, dhp, balanced)
            s_off = max(rb) // 256 * 256 + 256
            stride = (s_off + n * H * dhp * 2 + 255) // 256 * 256
            arena = torch.empty(stride * W, device="cuda", dtype=torch.uint8)
            base = arena.data_ptr()
            table, _ = P2PExchange.layout(H, T, W, 0, dhp, balanced, lambda p, o: base + p * stride + o, s_off)
            t = torch.from_numpy(table.reshape(3 * H, 8)).cuda()
            flops = 2.0 * n * D_ * 3 * H * dhp
            lt = timed(lambda: D.gemm(a, b, out))
            g1 = timed(lambda: D.gemm_fused(a, b, out))
            sc = timed(lambda: D.gemm_fused(a, b, None, scatter=(t, dhp)))
            print(json.dumps({"cfg": cfg, "world": W, "M": n, "N": 3 * H * dhp, "K": D_,
                              "cublaslt_us": round(lt * 1e3, 1), "g1_us": round(g1 * 1e3, 1),
                              "g1_scatter_us": round(sc * 1e3, 1),
                              "scatter_tflops": round(flops / sc / 1e9, 1),
                              "cublaslt_tflops": round(flops / lt / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
