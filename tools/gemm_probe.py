"""G1 (tcgen05 GEMM, csrc/gemm_sm100.cu) vs cuBLASLt (ifx_gemm_bf16) on the engine's
projection shapes. Each shape: 5 warm-up calls, then 20 timed calls with CUDA events on
the current stream, both libraries alternating in rounds; prints one JSON line per shape.

    python tools/gemm_probe.py [c2|c4|all] [--ranks W]

--ranks W: the shapes of one Ulysses rank at W ranks (M = T / W rows).
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_20714_b200 import _device as D  # noqa: E402

SHAPES = {
    "c2": [("qkv", 4680, 4608, 1536, "bf16"), ("wo", 4680, 1536, 1536, "f32+"),
           ("w1", 4680, 3072, 1536, "relu"), ("w2", 4680, 1536, 3072, "f32+"),
           ("eps", 4680, 1536, 1536, "f32")],
    "c4": [("qkv", 4680, 15360, 5120, "bf16"), ("wo", 4680, 5120, 5120, "f32+"),
           ("w1", 4680, 10240, 5120, "relu"), ("w2", 4680, 5120, 10240, "f32+")],
}


def timed(fn, n=20):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(n):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / n


def main():
    which = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "all"
    W = int(sys.argv[sys.argv.index("--ranks") + 1]) if "--ranks" in sys.argv else 1
    cfgs = ["c2", "c4"] if which == "all" else [which]
    g = torch.Generator(device="cuda").manual_seed(0)
    for cfg in cfgs:
        for name, M, N, K, mode in SHAPES[cfg]:
            M //= W
            a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
            b = (torch.randn(K, N, device="cuda", generator=g) / K ** 0.5).bfloat16()
            f32 = mode.startswith("f32")
            out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
            beta = 1.0 if mode == "f32+" else 0.0
            relu = mode == "relu"
            norm = None
            if mode == "f32+":  # the engine's residual GEMMs also emit the next norm's stats
                norm = D.RowNorm(torch.empty(M, N, device="cuda", dtype=torch.bfloat16),
                                 torch.empty(M, D.gemm_tiles_n(M, N, K), device="cuda"), 0, N)
            g1 = lambda: D.gemm_fused(a, b, out, beta=beta, relu=relu, norm_out=norm)  # noqa: E731
            lt = lambda: D.gemm(a, b, out, beta=beta, relu=relu)  # noqa: E731
            for _ in range(5):
                g1()
                lt()
            torch.cuda.synchronize()
            t_g1, t_lt = [], []
            for _ in range(3):
                t_g1.append(timed(g1))
                t_lt.append(timed(lt))
            fl = 2.0 * M * N * K
            rec = {"cfg": cfg, "ranks": W, "gemm": name, "M": M, "N": N, "K": K, "epilogue": mode,
                   "g1_us": min(t_g1) * 1e3, "cublaslt_us": min(t_lt) * 1e3,
                   "g1_tflops": fl / (min(t_g1) * 1e-3) / 1e12,
                   "cublaslt_tflops": fl / (min(t_lt) * 1e-3) / 1e12,
                   "tiles_n": D.gemm_tiles_n(M, N, K)}
            rec["g1_vs_lt"] = rec["cublaslt_us"] / rec["g1_us"]
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
