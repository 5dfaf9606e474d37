"""One K1 launch at the c2 shape with b cached blocks, for `ncu --set full` (-k regex:attn).

    python tools/ncu_attn.py [b] [--paged] [--heads H] [--rows N]

--heads / --rows: one Ulysses rank's launch (its heads, its query rows; keys of the whole
block and context), e.g. 8 ranks of the 12-head shape (grouped plan): --heads 3 --rows 2340.

--paged: the context comes through a page_len-16 slot table (engine layout, consecutive
slots), i.e. the attn_fwd_kernel<128, true> variant."""
import sys

import torch

from paper_2511_20714_b200._device import attn_fwd

b = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
paged = "--paged" in sys.argv
def _opt(name, default):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


T, dh, P = 4680, 128, 16
H = _opt("--heads", 12)
NQ = _opt("--rows", T)
D = H * dh
C = b * T
rows = -(-max(C, 1) // P) * P
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
ks = torch.randn(rows, D, device="cuda").bfloat16()
vs = torch.randn(rows, D, device="cuda").bfloat16()
out = torch.empty(NQ, D, device="cuda", dtype=torch.bfloat16)
kw = {}
if paged and C:
    import numpy as np

    from paper_2511_20714_b200._device import tile_run_codes
    kw = dict(ctx_slots=torch.arange(rows // P, device="cuda", dtype=torch.int32), page_len=P,
              first_token=0, tile_runs=torch.from_numpy(
                  tile_run_codes(np.arange(rows // P, dtype=np.int32), P)).cuda())
for _ in range(3):
    attn_fwd(qkv[:NQ, :D], H, dh, out, ks, vs, 0, C, qkv[:, D:2 * D], qkv[:, 2 * D:], **kw)
torch.cuda.synchronize()
