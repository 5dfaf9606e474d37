"""Which torch/cuBLAS call shapes fuse the engine's residual add and ReLU (c2 shapes)."""
import time
import torch

T, D = 4680, 1536
a = torch.randn(T, D, device="cuda").bfloat16()
w = torch.randn(D, D, device="cuda").bfloat16() * 0.02
w1 = torch.randn(D, 2 * D, device="cuda").bfloat16() * 0.02
x = torch.randn(T, D, device="cuda")
tmp = torch.empty_like(x)
bias = torch.zeros(2 * D, device="cuda", dtype=torch.bfloat16)
f = torch.empty(T, 2 * D, device="cuda", dtype=torch.bfloat16)


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def mm_add():
    torch.mm(a, w, out_dtype=torch.float32, out=tmp)
    x.add_(tmp)


print("mm(out_dtype=f32)+add_ us", timeit(mm_add))
try:
    ref = x + (a.float() @ w.float())
    x2 = x.clone()
    torch.addmm(x2, a, w, out_dtype=torch.float32, out=x2)
    print("addmm inplace ok, err", (x2 - ref).abs().max().item())
    print("addmm(out=x) us", timeit(lambda: torch.addmm(x, a, w, out_dtype=torch.float32, out=x)))
except Exception as e:
    print("addmm inplace failed:", repr(e)[:300])
try:
    y = torch._addmm_activation(bias, a, w1, use_gelu=False)
    print("addmm_activation ok", y.dtype, (y.float() - torch.relu(a.float() @ w1.float())).abs().max().item())
    print("mm+relu_ us", timeit(lambda: torch.mm(a, w1, out=f).relu_()))
    print("_addmm_activation us", timeit(lambda: torch._addmm_activation(bias, a, w1, use_gelu=False, out=f)))
except Exception as e:
    print("addmm_activation failed:", repr(e)[:300])
