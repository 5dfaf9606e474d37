"""One K2 page write at the c2 shape (4680 x 1536 bf16 K and V, strided QKV source)."""
import torch

from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200._device import stream_ptr

T, D = 4680, 1536
qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
ks = torch.zeros(8 * T, D, device="cuda", dtype=torch.bfloat16)
vs = torch.zeros_like(ks)
L = _abi.lib()
for i in range(4):
    _abi.check(L.ifx_kv_append(qkv[:, D:].data_ptr(), qkv[:, 2 * D:].data_ptr(), 3 * D, _abi.BF16,
                               ks.data_ptr(), vs.data_ptr(), D, _abi.BF16, i * T, T, D, stream_ptr()))
torch.cuda.synchronize()
