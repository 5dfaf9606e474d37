"""Ulysses re-shard host logic over a real 2-rank `gloo` group on CPU.

The CUDA pack/unpack kernels are swapped for test-local torch permutes (the same index
map as csrc/kv_ops.cu:ulysses_transpose) so the collective plumbing of
paper_2511_20714_b200.parallel.UlyssesComm — split order, head ownership, sequence
reassembly, byte accounting — runs on CPU. Attention is the oracle's numpy restatement.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _pack_ref(src, groups, world, chunk):
    n = src.shape[0]
    return src[:, :groups * world * chunk].reshape(n, groups, world, chunk).permute(2, 0, 1, 3).contiguous()


def _unpack_ref(src, out, groups, world, chunk):
    n = out.shape[0]
    out[:, :groups * world * chunk] = src.view(world, n, groups, chunk).permute(1, 2, 0, 3).reshape(n, -1)
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, heads, dh, T, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.attention import multi_head
        from oracle.parallel import predict_communication
        from paper_2511_20714_b200.parallel import UlyssesComm

        comm = UlyssesComm(pack=_pack_ref, unpack=_unpack_ref)
        D = heads * dh
        n = T // world
        g = np.random.default_rng(123)
        full = g.standard_normal((T, 3 * D)).astype(np.float32)  # same on every rank
        mine = torch.from_numpy(full[rank * n:(rank + 1) * n])
        qkv_h = comm.seq_to_head(mine, 3)
        hl = heads // world
        w = hl * dh
        cols = slice(rank * w, (rank + 1) * w)
        want = np.concatenate([full[:, :D][:, cols], full[:, D:2 * D][:, cols], full[:, 2 * D:][:, cols]], 1)
        assert np.array_equal(qkv_h.numpy(), want)
        # local-head attention (oracle), then back to sequence sharding
        qh, kh, vh = (qkv_h[:, i * w:(i + 1) * w].numpy() for i in range(3))
        o_h = torch.from_numpy(multi_head(qh, kh, vh, hl, np.ones((T, T), bool)))
        out = torch.empty(n, D)
        comm.head_to_seq(o_h, out)
        dense = multi_head(full[:, :D], full[:, D:2 * D], full[:, 2 * D:], heads, np.ones((T, T), bool))
        err = float(np.abs(out.numpy() - dense[rank * n:(rank + 1) * n]).max())
        msgs, nbytes = predict_communication("ulysses", [n] * world, heads, dh, world)
        q.put((rank, err, comm.messages * world, comm.bytes * world, msgs, nbytes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,heads", [(2, 4), (2, 2)])
def test_ulysses_comm_two_ranks_gloo(world, heads):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, heads, 8, 24, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, msgs, nbytes, pmsgs, pbytes in res:
        assert err <= 1e-5, (rank, err)
        # traced traffic (summed over ranks) == the reference cost model (parallel.py:317-333)
        assert (msgs, nbytes) == (pmsgs, pbytes)
