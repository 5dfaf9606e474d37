"""One K1 launch at the c2 shape with b cached blocks, for `ncu --set full` (-k regex:attn)."""
import sys

import torch

from paper_2511_20714_b200._device import attn_fwd

b = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T, H, dh = 4680, 12, 128
D = H * dh
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
ks = torch.randn(max(b * T, 1), D, device="cuda").bfloat16()
vs = torch.randn(max(b * T, 1), D, device="cuda").bfloat16()
out = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    attn_fwd(qkv[:, :D], H, dh, out, ks, vs, 0, b * T, qkv[:, D:2 * D], qkv[:, 2 * D:])
torch.cuda.synchronize()
