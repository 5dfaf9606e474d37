"""K2 page writes at the c2 shape (4680 x 1536 bf16 K and V from the strided QKV buffer into
consecutive page slots of an HBM pool, page_len 16), for `ncu --set full -k regex:append`.

The destination cycles through a pool of N_BLOCKS blocks (default 16: 920 MB of K + V, 7x
the 126 MB L2), one block per launch, so by launch 10 the L2 is full of the earlier
launches' dirty pages and this launch's writes evict them to HBM: capture that launch with
`--cache-control none -s 9 -c 1` to see the HBM writes (r04); ncu's default cache flush
leaves the destination L2-resident (r03: 0.28 MB of DRAM writes).

    python tools/ncu_append.py [N_BLOCKS] [LAUNCHES]
"""
import sys
import ctypes

import torch

from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200._device import stream_ptr

T, D, P = 4680, 1536, 16
pages = -(-T // P)
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
NB = int(sys.argv[1]) if len(sys.argv) > 1 else 16
LAUNCHES = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ks = torch.zeros(NB * pages * P, D, device="cuda", dtype=torch.bfloat16)
vs = torch.zeros_like(ks)
pool = _abi.KvPool()
pool.dev_k, pool.dev_v, pool.width, pool.page_len, pool.type = ks.data_ptr(), vs.data_ptr(), D, P, _abi.BF16
L = _abi.lib()
all_slots = [torch.arange(i * pages, (i + 1) * pages, device="cuda", dtype=torch.int32)
             for i in range(NB)]
for i in range(LAUNCHES):
    slots = all_slots[i % NB]
    _abi.check(L.ifx_kv_append(qkv[:, D:].data_ptr(), qkv[:, 2 * D:].data_ptr(), 3 * D, _abi.BF16,
                               ctypes.byref(pool), slots.data_ptr(), 0, 0, T, stream_ptr()))
torch.cuda.synchronize()
