"""K2 page write / K7 gather / K6 page moves at the c2 shape (CUDA events, warm, > L2 traffic).

Algorithmic bytes: read + write of 2 x T x D bf16 (K and V of one layer-block). K2 writes
into page slots of a 40-block HBM pool (page_len 16, consecutive slots like the engine's
appends); K6 moves the same pages HBM -> mapped pinned host -> HBM (PCIe)."""
import ctypes
import json

import torch

from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200._device import stream_ptr
from paper_2511_20714_b200.kvcache import _HostBuf

T, D, P = 4680, 1536, 16
L = _abi.lib()
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
pages = -(-T // P)
pool_k = torch.zeros(40 * pages * P, D, device="cuda", dtype=torch.bfloat16)  # 575 MB > L2
pool_v = torch.zeros_like(pool_k)
host_k, host_v = _HostBuf(pages * P * D * 2), _HostBuf(pages * P * D * 2)
pool = _abi.KvPool()
pool.dev_k, pool.dev_v, pool.host_k, pool.host_v = pool_k.data_ptr(), pool_v.data_ptr(), host_k.ptr, host_v.ptr
pool.width, pool.page_len, pool.type = D, P, _abi.BF16
slots = [torch.arange(i * pages, (i + 1) * pages, device="cuda", dtype=torch.int32) for i in range(40)]
out_k = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
out_v = torch.empty_like(out_k)
moves = torch.stack([torch.arange(pages), torch.arange(pages)], 1).cuda()


def timed(fn, n=40):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


nbytes = 2 * 2 * T * D * 2
pb = ctypes.byref(pool)
app = lambda i: L.ifx_kv_append(qkv[:, D:].data_ptr(), qkv[:, 2 * D:].data_ptr(), 3 * D, _abi.BF16,  # noqa
                                pb, slots[i % 40].data_ptr(), 0, 0, T, stream_ptr())
gat = lambda i: L.ifx_kv_gather(pb, slots[i % 40].data_ptr(), 0, None, 0, T,  # noqa
                                out_k.data_ptr(), out_v.data_ptr(), stream_ptr())
d2h = lambda i: L.ifx_kv_move_pages(pb, moves.data_ptr(), pages, 0, stream_ptr())  # noqa
h2d = lambda i: L.ifx_kv_move_pages(pb, moves.data_ptr(), pages, 1, stream_ptr())  # noqa
for name, fn, nb in (("K2 append", app, nbytes), ("K7 gather", gat, nbytes),
                     ("K6 D2H (PCIe)", d2h, nbytes // 2), ("K6 H2D (PCIe)", h2d, nbytes // 2)):
    us = timed(fn, 40 if "K6" not in name else 10)
    print(json.dumps({"kernel": name, "us": round(us, 2), "GB/s": round(nb / us / 1e3, 1),
                      "bytes": nb}))
