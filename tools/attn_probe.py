"""Quick K1 timing at the Wan-1.3B shape (T=4680, H=12, dh=128) for b cached blocks.

    python tools/attn_probe.py [--quick]

Prints algorithmic TFLOP/s = 4*T*(C+T)*D / kernel time (CUDA events, warm, inputs > L2).
"""

import argparse
import json

import torch

from paper_2511_20714_b200._device import attn_fwd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--no-split", action="store_true")
    ap.add_argument("--paged", action="store_true", help="context through a page_len-16 slot table")
    ap.add_argument("--cross", type=int, default=0, help="n prompt keys only (cross-attention)")
    ap.add_argument("--rows", type=int, default=0, help="query rows (default T; e.g. 2340 = "
                    "one rank of 8 at the 12-head shape, grouped plan)")
    args = ap.parse_args()
    T, H, dh = 4680, args.heads, 128
    D = H * dh
    res = []
    for b in ((0, 1, 3, 6, 20) if not args.quick and not args.cross else (3,)):
        C = b * T
        if args.cross:  # q over a few prompt keys, no own-block keys
            k3 = torch.randn(args.cross, D, device="cuda").bfloat16()
            out = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
            q = torch.randn(T, D, device="cuda").bfloat16()
            f = lambda: attn_fwd(q, H, dh, out, k3, k3, 0, args.cross)  # noqa: E731
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.iters):
                f()
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"cross_keys": args.cross, "us": round(e0.elapsed_time(e1) / args.iters * 1e3, 2)}))
            return
        qkv = torch.randn(T, 3 * D, device="cuda").bfloat16()
        ks = torch.randn(max(C, 1), D, device="cuda").bfloat16()
        vs = torch.randn(max(C, 1), D, device="cuda").bfloat16()
        NQ = args.rows or T
        out = torch.empty(NQ, D, device="cuda", dtype=torch.bfloat16)
        kw = {}
        if args.paged and C:  # engine layout: page k of the stream in slot k (appends are in order)
            P = 16
            n_pages = -(-C // P)
            ks = torch.randn(n_pages * P, D, device="cuda").bfloat16()
            vs = torch.randn(n_pages * P, D, device="cuda").bfloat16()
            import numpy as np

            from paper_2511_20714_b200._device import tile_run_codes
            kw = dict(ctx_slots=torch.arange(n_pages, device="cuda", dtype=torch.int32), page_len=P,
                      first_token=0, tile_runs=torch.from_numpy(
                          tile_run_codes(np.arange(n_pages, dtype=np.int32), P)).cuda())
        f = lambda: attn_fwd(qkv[:NQ, :D], H, dh, out, ks, vs, 0, C, qkv[:, D:2 * D], qkv[:, 2 * D:],  # noqa: E731
                             split_kv=not args.no_split, **kw)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        flops = 4.0 * NQ * (C + T) * D
        res.append({"b": b, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1)})
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
