"""Ulysses on the GPU: the reference-API simulation vs the reference's golden outputs, and
the real multi-process UlyssesEngine (2 ranks sharing cuda:0 over a gloo group; NCCL is
used when each rank has its own GPU) vs the single-GPU engine."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_reference_api_ulysses_and_ring_vs_golden():
    from paper_2511_20714_b200 import parallel as P
    from paper_2511_20714_b200.attention import block_causal_mask

    g = np.load(os.path.join(GOLDEN, "parallel.npz"))
    for seq_len in (8, 24, 64):
        for heads in (1, 2, 4):
            for world in (1, 2, 4):
                r = np.random.default_rng(seq_len + 10 * heads + world)
                d = heads * 4
                lens = P.equal_shards(seq_len, world)
                qs = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                ks = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                vs = [r.standard_normal((n, d)).astype(np.float32) for n in lens]
                mask = block_causal_mask(seq_len // 4, 4)
                tag = f"{seq_len}_{heads}_{world}"
                dense = torch.cat(P.dense_reference(qs, ks, vs, heads, mask)).cpu().numpy()
                assert np.abs(dense - g[f"dense_{tag}"]).max() <= 2e-2
                if heads % world == 0:
                    grp = P.WorkerGroup(world)
                    out = torch.cat(P.ulysses_attention(grp, qs, ks, vs, heads, mask)).cpu().numpy()
                    assert np.abs(out - g[f"ulysses_{tag}"]).max() <= 2e-2
                    traced = [t for t in grp.trace if t.sender != t.receiver]
                    assert [len(traced), sum(t.bytes for t in traced)] == g[f"trace_{tag}"].tolist()
                    assert P.predict_communication("ulysses", lens, heads, 4, world) == \
                        (len(traced), sum(t.bytes for t in traced))
                for name, fn, strat in (("ringkv", P.ring_attention_pass_kv, "ring_pass_kv"),
                                        ("ringq", P.ring_attention_pass_q, "ring_pass_q")):
                    grp = P.WorkerGroup(world)
                    out = torch.cat(fn(grp, qs, ks, vs, mask, heads=heads)).cpu().numpy()
                    assert np.abs(out - g[f"{name}_{tag}"]).max() <= 2e-2, (name, tag)
                    traced = [t for t in grp.trace if t.sender != t.receiver]
                    got = [len(traced), sum(t.bytes for t in traced)]
                    assert got == g[f"{name}trace_{tag}"].tolist(), (name, tag)
                    assert P.predict_communication(strat, lens, heads, 4, world) == tuple(got)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFG = dict(layers=2, heads=4, head_dim=64, block_len=256, frame_shape=(8, 8), prompt_dim=16)
REQ = dict(num_blocks=3, seed=0, prompt_schedule=[(0, "a quiet scene"), (2, "rain")])


def _rank(rank, world, port, q, cfg=None, kvc=None, pad=True, p2p=False, g1=None):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if g1 is not None:
        os.environ["IFX_G1"] = g1  # read when the engine module is imported (below)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20714_b200 import engine as E
        from paper_2511_20714_b200.parallel import UlyssesComm, UlyssesEngine

        model = E.ToyModel(E.ModelConfig(**(cfg or CFG)), head_multiple=world if pad else 1)
        eng = UlyssesEngine(model, UlyssesComm(), E.KvConfig(**kvc) if kvc else None, p2p=p2p)
        lats = eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5]), **REQ))
        moved = eng.runner.xch.mesh.barriers if p2p else eng.comm.bytes
        eng.runner.release_graphs()
        torch.cuda.synchronize()
        q.put((rank, [l.cpu().numpy() for l in lats], eng.cache.state(), moved))
    finally:
        dist.destroy_process_group()


CFG_ROPE = dict(CFG, rope_grid=(1, 16, 16), heads=3)  # 3 heads on 2 ranks: dummy-head padding


# device capacity below the working set: each rank's head shard spills to its own pinned
# host pool, restores / demotions move data per rank, host pages are staged for K1
KV_SPILL = dict(num_layers=2, head_dim=256, page_len=16, capacity_pages_device=40,
                capacity_pages_host=10**4)


@pytest.mark.parametrize("world,cfg", [(2, CFG), (2, CFG_ROPE)])
def test_ulysses_p2p_fused_norm_path(world, cfg):
    """The peer-exchange rank with every projection on G1 and the RMS norms fused into the
    epilogues (IFX_G1=all; chosen automatically at small per-rank row counts) vs the
    single-GPU engine and the oracle (grouped plan for 3 heads on 2 ranks)."""
    from oracle import engine as OE
    from paper_2511_20714_b200 import engine as E

    ref = E.Engine(E.build_model(E.ModelConfig(**cfg))).generate(
        E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5]), **REQ))
    want, _ = OE.generate_sequence(OE.ToyModel(OE.ModelConfig(**cfg)),
                                   OE.GenerationRequest(schedule=OE.DenoiseSchedule([1.0, 0.5]), **REQ))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, cfg, None, False, True, "all"))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lats, state, _ in res:
        for a, b, w in zip(lats, ref, want):
            assert np.abs(a - b.latent).max() <= 2e-2, rank
            assert np.abs(a - w).max() <= 2e-2, rank


@pytest.mark.parametrize("p2p", [False, True], ids=["a2a", "p2p"])
@pytest.mark.parametrize("world,cfg,kvc,pad", [(2, CFG, None, True), (2, CFG_ROPE, None, True),
                                              (2, CFG, KV_SPILL, True),
                                              (2, CFG_ROPE, None, False),  # balanced: 1.5 heads/rank
                                              (2, dict(CFG, heads=3), dict(KV_SPILL, head_dim=192), False),
                                              (3, dict(CFG, block_len=192), None, False)])  # 4 heads / 3 ranks
def test_ulysses_engine_matches_single_gpu(world, cfg, kvc, pad, p2p):
    """2-3 ranks sharing cuda:0 (gloo group). a2a: pack -> all-to-all (host-staged) ->
    unpack. p2p: no all-to-all — G1's QKV epilogue and K1's epilogue store into the other
    processes' arenas (CUDA IPC mappings), ordered by ifx_peer_barrier."""
    from paper_2511_20714_b200 import engine as E

    ref_model = E.build_model(E.ModelConfig(**cfg))
    ref_eng = E.Engine(ref_model, E.KvConfig(**kvc) if kvc else None)
    ref = ref_eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5]), **REQ))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, cfg, kvc, pad, p2p))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # directly against the numpy oracle (the reference restated, pinned by the golden
    # fixtures), not only against the single-GPU engine
    from oracle import engine as OE
    ocfg = dict(cfg)
    oreq = OE.GenerationRequest(schedule=OE.DenoiseSchedule([1.0, 0.5]), **REQ)
    okv = None
    if kvc:
        from oracle.kvcache import KvConfig as OKv
        okv = OKv(**kvc)
    want, _ = OE.generate_sequence(OE.ToyModel(OE.ModelConfig(**ocfg)), oreq, kv_config=okv)
    for rank, lats, state, nbytes in res:
        for a, b, w in zip(lats, ref, want):
            assert np.abs(a - b.latent).max() <= 2e-2, rank
            assert np.abs(a - w).max() <= 2e-2, rank
        # replicated page table == single-GPU page table == reference semantics
        assert state == ref_eng.cache.state()
        assert nbytes > 0  # bytes through the all-to-alls, or peer barriers
    if kvc:
        assert ref_eng.cache.memory_stats().host_pages_used > 0


GRAPH_STEPS = [1.0, 0.75, 0.5]


def _a2a_var_capture(port, q):
    """NCCL's variable-size all-to-all (the balanced plan's re-shard) inside a CUDA graph
    capture on a world-1 group: recorded once, replayed with new data."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2511_20714_b200.parallel import UlyssesComm
        comm = UlyssesComm()
        send = torch.zeros(1000, device="cuda", dtype=torch.bfloat16)
        recv = torch.zeros(1000, device="cuda", dtype=torch.bfloat16)
        comm.a2a_var(send, [1000], recv, [1000])  # warm-up outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g.capture_begin()
            comm.a2a_var(send, [1000], recv, [1000])
            g.capture_end()
        ok = []
        for i in range(3):
            send.copy_(torch.arange(1000, device="cuda").to(torch.bfloat16) * (i + 1))
            g.replay()
            torch.cuda.synchronize()
            ok.append(bool(torch.equal(recv, send)))
        del g
        torch.cuda.synchronize()
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_ulysses_a2a_var_nccl_graph_capture_world1():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_a2a_var_capture, args=(_free_port(), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0 and ok == [True, True, True]


def _rank_nccl(port, q, p2p=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2511_20714_b200 import engine as E
        from paper_2511_20714_b200.parallel import UlyssesComm, UlyssesEngine

        eng = UlyssesEngine(E.ToyModel(E.ModelConfig(**CFG)), UlyssesComm(), p2p=p2p)
        # 3 steps: a block's first pass may run eagerly (idle GPU), the rest are captured
        lats = eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule(GRAPH_STEPS), **REQ))
        q.put(([l.cpu().numpy() for l in lats], eng.cache.state(), eng.runner._graph is not None))
        eng.runner.release_graphs()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def _auto_fallback(port, q):
    """UlyssesEngine's default exchange when the peer mesh cannot be built (CUDA IPC refused,
    simulated): every rank falls back to the NCCL all-to-alls instead of failing."""
    import warnings

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ.pop("IFX_ULYSSES", None)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2511_20714_b200 import engine as E
        from paper_2511_20714_b200 import parallel as P
        from paper_2511_20714_b200.errors import ConfigError

        def refuse(self, *a, **k):
            raise ConfigError("peer mesh: cudaIpcOpenMemHandle refused (test)")
        P.PeerMesh.__init__ = refuse
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            eng = P.UlyssesEngine(E.build_model(E.ModelConfig(**CFG)), P.UlyssesComm())
        lats = [b.cpu().numpy() for b in eng.generate(E.GenerationRequest(
            schedule=E.DenoiseSchedule(GRAPH_STEPS), **REQ))]
        q.put((eng.runner.xch is None, any("NCCL" in str(x.message) for x in w), lats))
        eng.runner.release_graphs()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def test_ulysses_auto_exchange_falls_back_to_nccl():
    from paper_2511_20714_b200 import engine as E

    ref = E.Engine(E.build_model(E.ModelConfig(**CFG))).generate(
        E.GenerationRequest(schedule=E.DenoiseSchedule(GRAPH_STEPS), **REQ))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_auto_fallback, args=(_free_port(), q))
    p.start()
    nccl, warned, lats = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0 and nccl and warned
    for a, b in zip(lats, ref):
        assert np.abs(a - b.latent).max() <= 2e-2


@pytest.mark.parametrize("p2p", [False, True], ids=["a2a", "p2p"])
def test_ulysses_nccl_graph_capture_world1(p2p):
    """The NCCL path of the Ulysses runner on one GPU: its denoise passes are captured as
    CUDA graphs with the all-to-alls inside (world size 1 exercises ProcessGroupNCCL under
    stream capture) — or, p2p, with the scatter epilogues and peer barriers inside — and
    match the single-GPU engine."""
    from paper_2511_20714_b200 import engine as E

    ref_eng = E.Engine(E.build_model(E.ModelConfig(**CFG)))
    ref = ref_eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule(GRAPH_STEPS), **REQ))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_rank_nccl, args=(_free_port(), q, p2p))
    p.start()
    lats, state, graphed = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0 and graphed
    for a, b in zip(lats, ref):
        assert np.abs(a - b.latent).max() <= 2e-2
    assert state == ref_eng.cache.state()


C2W = dict(layers=2, heads=12, head_dim=128, block_len=4680, frame_shape=(4, 4), prompt_dim=16,
           weight_seed=0)
C2REQ = dict(num_blocks=2, seed=0, prompt_schedule=[(0, "a quiet scene")])


def _rank_c2(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20714_b200 import engine as E
        from paper_2511_20714_b200.parallel import UlyssesComm, UlyssesEngine

        eng = UlyssesEngine(E.build_model(E.ModelConfig(**C2W)), UlyssesComm(), p2p=True)
        lats = eng.generate(E.GenerationRequest(schedule=E.DenoiseSchedule([1.0, 0.5]), **C2REQ))
        plan = ("grouped" if eng.runner.grouped is not None else
                "balanced" if eng.runner.plan is not None else "whole")
        eng.runner.release_graphs()
        torch.cuda.synchronize()
        q.put((rank, [x.cpu().numpy() for x in lats], eng.cache.state(), plan))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_ulysses_p2p_c2_shape_vs_oracle(world):
    """The peer-exchange Ulysses engine at the benchmark's width and block length (12 heads
    x 128, 4,680 tokens, reference PCG64 weights and seeded noise; 2 layers, 2 blocks) on
    `world` rank processes sharing cuda:0 — 2 ranks: whole heads (6 per rank); 8 ranks: the
    grouped plan the 8-GPU bench runs (4 head groups x 2 row slices) — vs the numpy oracle:
    max-abs <= 2e-2, cosine > 0.999, page table identical on every rank."""
    from oracle import engine as OE

    want, ocache = OE.generate_sequence(OE.ToyModel(OE.ModelConfig(**C2W)), OE.GenerationRequest(
        schedule=OE.DenoiseSchedule([1.0, 0.5]), **C2REQ))
    want = np.stack(want)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_c2, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, lats, state, plan in res:
        got = np.stack(lats)
        a, b = got.ravel().astype(np.float64), want.ravel().astype(np.float64)
        cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
        assert np.abs(got - want).max() <= 2e-2 and cos > 0.999, (rank, float(np.abs(got - want).max()))
        assert state == ocache.state()
        assert plan == ("whole" if world == 2 else "grouped")


def _rank_c4(rank, world, port, q, meta, rows):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20714_b200 import engine as E
        from paper_2511_20714_b200.parallel import UlyssesComm, UlyssesEngine

        mc = E.ModelConfig(layers=meta["layers"], heads=meta["heads"], head_dim=meta["head_dim"],
                           block_len=meta["block_len"], frame_shape=tuple(meta["frame_shape"]),
                           prompt_dim=meta["prompt_dim"], weight_seed=meta["weight_seed"])
        kvc = E.default_kv_config(mc, capacity_pages_device=meta["capacity_pages_device"],
                                  capacity_pages_host=meta["capacity_pages_host"])
        eng = UlyssesEngine(E.build_model(mc), UlyssesComm(), kvc, p2p=True)
        lats = eng.generate(E.GenerationRequest(meta["blocks"], E.DenoiseSchedule(meta["steps"]),
                                                seed=meta["seed"], prompt_schedule=[(0, meta["prompt"])]))
        out = [x.cpu().numpy()[rows] for x in lats]
        eng.runner.release_graphs()
        torch.cuda.synchronize()
        q.put((rank, out, eng.cache.state(), eng.runner.xch is not None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_ulysses_p2p_c4_width_vs_reference(world):
    """The 14B width the scaling configs name (c4: 40 heads x 128, D = 5,120, T = 4,680;
    3 layers x 2 blocks x 2 steps) on `world` rank processes sharing cuda:0 through the
    peer-exchange engine (10 / 5 whole heads per rank) vs the LIVE reference's latents
    (tests/golden/c4_deep.npz): max-abs <= 2e-2, cosine > 0.999 on every block, and every
    rank's page table equal to the reference's, bit for bit."""
    import json
    import zlib

    import kv_differential as KD

    path = os.path.join(GOLDEN, "c4_deep.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c4_deep.npz not generated")
    g = np.load(path)
    meta = json.loads(bytes(g["meta"]).decode())
    rows = g["rows"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_c4, args=(r, world, port, q, meta, rows)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want_state = json.loads(zlib.decompress(bytes(g["state_z"])).decode())
    worst = (0.0, 1.0)
    for rank, lats, state, p2p in res:
        assert p2p
        for c, got in enumerate(lats):
            want = g[f"b{c}_rows"]
            a, b = got.ravel().astype(np.float64), want.ravel().astype(np.float64)
            cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
            err = float(np.abs(got - want).max())
            assert err <= 2e-2 and cos > 0.999, (rank, c, err, cos)
            worst = (max(worst[0], err), min(worst[1], cos))
        assert KD.canon(state) == want_state
    print(f"c4 width, {world} ranks: worst max-abs {worst[0]:.3e}, cosine {worst[1]:.7f}; "
          "page table bit-exact on every rank")
