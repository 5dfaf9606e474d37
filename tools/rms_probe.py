"""Fused RMS-norm (x + t*tvec -> bf16) timing at the c2 / c4 widths, x L2-resident as in the
engine (written by the previous GEMM). CUDA events over 200 launches."""
import torch

from paper_2511_20714_b200._device import rms_bf16

for width in (1536, 5120):
    x = torch.randn(4680, width, device="cuda")
    tv = torch.randn(width, device="cuda")
    y = torch.empty(4680, width, device="cuda", dtype=torch.bfloat16)
    xo = torch.empty_like(x)
    for _ in range(20):
        rms_bf16(x, y, tv, 0.5, xo)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        rms_bf16(x, y, tv, 0.5, xo)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 200 * 1e3
    gb = 4680 * width * (4 + 4 + 2) / 1e9
    print(f"width {width}: {us:.2f} us per launch, {gb / us * 1e6 / 1e3:.2f} TB/s algorithmic (x read, x_out + y written)")
