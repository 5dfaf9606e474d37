"""One projection shape through G1 (or cuBLASLt with `lt`) a few times, for ncu captures.

    ncu --set full -k regex:gemm_kernel -s 2 -c 1 python tools/ncu_gemm.py qkv [lt]

Shapes: qkv/w1 (bf16 out), wo/w2 (fp32 residual out + next-norm statistics, as in the
engine), qkv14 (the 14B QKV).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_20714_b200 import _device as D  # noqa: E402

SHAPES = {"qkv": (4680, 4608, 1536), "wo": (4680, 1536, 1536), "w1": (4680, 3072, 1536),
          "w2": (4680, 1536, 3072), "qkv14": (4680, 15360, 5120)}
name = sys.argv[1]
M, N, K = SHAPES[name]
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
b = (torch.randn(K, N, device="cuda", generator=g) / K ** 0.5).bfloat16()
resid = name in ("wo", "w2")
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if resid else torch.bfloat16)
norm = None
if resid:
    norm = D.RowNorm(torch.empty(M, N, device="cuda", dtype=torch.bfloat16),
                     torch.empty(M, 2 * -(-N // 64), device="cuda"), 0, N)
for _ in range(4):
    if len(sys.argv) > 2 and sys.argv[2] == "lt":
        D.gemm(a, b, out, beta=1.0 if resid else 0.0)
    else:
        D.gemm_fused(a, b, out, beta=1.0 if resid else 0.0, norm_out=norm)
torch.cuda.synchronize()
