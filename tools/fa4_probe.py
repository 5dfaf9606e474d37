"""Comparison ceiling (NOT part of the product): the in-box FA4 CuTe-DSL sm100 forward
(vllm.vllm_flash_attn.cute) on K1's c2 shapes: T = 4680 queries, 12 heads x 128, b cached
blocks (C = b*T context keys + T own keys), non-causal. Same FLOP accounting as
tools/attn_probe.py: 4*T*(C+T)*D / CUDA-event time."""
import json
import sys

import torch

from vllm.vllm_flash_attn.cute.interface import flash_attn_func

T, dh = 4680, 128
H = int(sys.argv[sys.argv.index("--heads") + 1]) if "--heads" in sys.argv else 12
NQ = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else T
D = H * dh
for b in (0, 1, 3, 6, 20):
    C = b * T
    q = torch.randn(1, NQ, H, dh, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, C + T, H, dh, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, C + T, H, dh, device="cuda", dtype=torch.bfloat16)
    f = lambda: flash_attn_func(q, k, v, causal=False)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"impl": "fa4-cute (vllm, reference ceiling)", "b": b, "ms": round(ms, 4),
                      "heads": H, "rows": NQ,
                      "tflops": round(4.0 * NQ * (C + T) * D / ms / 1e9, 1)}), flush=True)
