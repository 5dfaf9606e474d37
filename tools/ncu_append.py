"""K2 page writes at the c2 shape (4680 x 1536 bf16 K and V from the strided QKV buffer into
consecutive page slots of an HBM pool, page_len 16), for `ncu --set full -k regex:append`.
The pool (8 blocks, 230 MB) exceeds what one write leaves in L2 across launches."""
import ctypes

import torch

from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200._device import stream_ptr

T, D, P = 4680, 1536, 16
pages = -(-T // P)
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
ks = torch.zeros(8 * pages * P, D, device="cuda", dtype=torch.bfloat16)
vs = torch.zeros_like(ks)
pool = _abi.KvPool()
pool.dev_k, pool.dev_v, pool.width, pool.page_len, pool.type = ks.data_ptr(), vs.data_ptr(), D, P, _abi.BF16
L = _abi.lib()
for i in range(4):
    slots = torch.arange(i * pages, (i + 1) * pages, device="cuda", dtype=torch.int32)
    _abi.check(L.ifx_kv_append(qkv[:, D:].data_ptr(), qkv[:, 2 * D:].data_ptr(), 3 * D, _abi.BF16,
                               ctypes.byref(pool), slots.data_ptr(), 0, 0, T, stream_ptr()))
torch.cuda.synchronize()
