"""K2 page write / K7 gather bandwidth at the c2 shape (CUDA events, warm, > L2 traffic).

Algorithmic bytes: read + write of 2 x T x D bf16 (K and V of one layer-block)."""
import json

import torch

from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200._device import stream_ptr

T, D = 4680, 1536
L = _abi.lib()
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
slab_k = torch.zeros(40 * T, D, device="cuda", dtype=torch.bfloat16)  # 575 MB: > L2 per sweep
slab_v = torch.zeros_like(slab_k)
out_k = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
out_v = torch.empty_like(out_k)


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
app = lambda i: L.ifx_kv_append(qkv[:, D:].data_ptr(), qkv[:, 2 * D:].data_ptr(), 3 * D, _abi.BF16,  # noqa
                                slab_k.data_ptr(), slab_v.data_ptr(), D, _abi.BF16, (i % 40) * T, T, D,
                                stream_ptr())
gat = lambda i: L.ifx_kv_gather(slab_k.data_ptr(), slab_v.data_ptr(), D, _abi.BF16, None,  # noqa
                                (i % 40) * T, T, D, out_k.data_ptr(), out_v.data_ptr(), stream_ptr())
for name, fn in (("K2 append", app), ("K7 gather", gat)):
    us = timed(fn)
    print(json.dumps({"kernel": name, "us": round(us, 2), "GB/s": round(nbytes / us / 1e3, 1),
                      "bytes": nbytes}))
