"""CPU check of the physical tier logic in the native page table (csrc/pagetable.cpp):
slot assignment and the drained page-move batches.

A Python model of the two pools stands in for HBM / pinned host memory: each page's
payload is written into its slot on append (as K2 does), each drained batch is executed
as K6 would (every move of a batch concurrently), and after every call every live page's
payload must sit in the slot of the tier the page table reports. Each batch must also be
hazard-free (no slot both read and written, no slot written twice), which is what lets K6
run a batch as one launch."""

import numpy as np
import pytest

from paper_2511_20714_b200.kvcache import KvConfig, PageTable


def _check_batches(mv):
    for key in np.unique(mv[:, 0] * 4 + mv[:, 2] * 2 + mv[:, 1]):
        b = mv[mv[:, 0] * 4 + mv[:, 2] * 2 + mv[:, 1] == key]
        d = int(b[0, 2])
        src = b[:, 4] if d == 1 else b[:, 3]
        dst = b[:, 3] if d == 1 else b[:, 4]
        assert len(set(dst.tolist())) == len(dst), "slot written twice in one batch"
        # reads and writes of one batch are on different tiers, so they cannot collide;
        # the sources must be distinct pages too
        assert len(set(src.tolist())) == len(src)


def _run(seed):
    rng = np.random.default_rng(seed)
    P = int(rng.integers(1, 6))
    cfg = KvConfig(num_layers=2, head_dim=4, page_len=P,
                   capacity_pages_device=int(rng.integers(0, 7)), capacity_pages_host=60)
    pt = PageTable(cfg)
    pools = {(k, t): {} for k in (0, 1) for t in (0, 1)}  # (kind, tier) -> slot -> payload
    payload = {}  # page id -> token-start tag (what its rows hold)
    kinds = ("self_attn", "cross_attn")

    def execute():
        mv = pt.drain_moves()
        if len(mv):
            _check_batches(mv)
            key = mv[:, 0] * 4 + mv[:, 2] * 2 + mv[:, 1]
            cuts = np.flatnonzero(np.diff(key)) + 1
            for lo, hi in zip(np.r_[0, cuts], np.r_[cuts, len(mv)]):
                b = mv[lo:hi]
                kind, d = int(b[0, 1]), int(b[0, 2])
                srct, dstt = (0, 1) if d == 0 else (1, 0)
                vals = [pools[(kind, srct)].get(int(r[3] if d == 0 else r[4])) for r in b]
                for r, val in zip(b, vals):
                    pools[(kind, dstt)][int(r[4] if d == 0 else r[3])] = val

    def verify():
        st = pt.state()
        for layer, kind, base, total, pages in st["streams"]:
            if not pages:
                continue
            k = 0 if kind == "self_attn" else 1
            codes, first = pt.slots(layer, kind, pages[0][3], total)
            assert len(codes) == len(pages)
            for (pid, tier, filled, start, _la), c in zip(pages, codes):
                assert (c < 0) == (tier == 1)
                slot = int(c) if c >= 0 else -1 - int(c)
                assert pools[(k, tier)].get(slot) == payload[pid], (seed, pid)
        ext = pt.pool_extent()
        n_dev = sum(1 for s in st["streams"] for p in s[4] if p[1] == 0)
        assert ext[0] + ext[2] <= max(cfg.capacity_pages_device, 0) + 2 * n_dev + 8

    for _ in range(40):
        op = rng.integers(0, 10)
        layer, kind = int(rng.integers(0, 2)), kinds[int(rng.random() < 0.25)]
        if op < 4:
            rc, bid, start, written, pages = pt.append(layer, kind, int(rng.integers(1, 12)), 0)
            if written:  # also after a CapacityError: rows already packed are written
                k = 0 if kind == "self_attn" else 1
                codes_all, first = pt.slots(layer, kind, start, start + written)
                ids = [s for s in pt.state()["streams"] if s[0] == layer and s[1] == kind][0][4]
                for p in ids:
                    if p[0] not in payload:
                        payload[p[0]] = (p[0], p[3])
                for p, c in zip([p for p in ids if p[3] >= first], codes_all):
                    tier = 0 if c >= 0 else 1
                    slot = int(c) if c >= 0 else -1 - int(c)
                    pools[(k, tier)][slot] = payload[p[0]]  # K2 writes the page's rows
            execute()
        elif op == 4 and rng.random() < 0.5:  # a batch of fetches (one epoch), drained once
            pt.batch_begin()
            for _ in range(int(rng.integers(1, 6))):
                li, kd = int(rng.integers(0, 2)), kinds[int(rng.random() < 0.25)]
                base, total = pt.range(li, kd)
                if total > base:
                    a = int(rng.integers(base, total))
                    pt.touch_range(li, kd, a, int(rng.integers(a, total + 1)))
            pt.batch_end()
            execute()
        elif op < 8:
            base, total = pt.range(layer, kind)
            if total > base:
                if op == 7:
                    pt.touch_indices(layer, kind, [int(x) for x in rng.integers(base, total, size=6)])
                else:
                    a = int(rng.integers(base, total))
                    pt.touch_range(layer, kind, a, int(rng.integers(a, total + 1)))
            execute()
        elif op == 8:
            st = pt.state()
            ids = [b[0] for b in st["blocks"]]
            if ids:
                try:
                    pt.offload([int(x) for x in rng.choice(ids, size=min(3, len(ids)), replace=False)])
                except Exception:
                    pass
            execute()
        else:
            pt.evict_window(int(rng.integers(0, 25)))
            execute()
        verify()


@pytest.mark.parametrize("seed", range(200))
def test_tier_moves_keep_every_page_in_its_slot(seed):
    _run(seed)


def test_tile_run_codes():
    """K1's per-tile run table (_device.tile_run_codes): a tile is one TMA box iff its pages
    are consecutive slots of one pool; partial last tiles never are."""
    from paper_2511_20714_b200._device import tile_run_codes

    NO = np.iinfo(np.int32).min
    assert list(tile_run_codes(np.arange(20, dtype=np.int32), 16)) == [0, 8, NO]
    codes = np.array([-1, -2, -3, -4, 5, 6, 7, 9, -5, -6, -7, -8, -9, -10, -11, -12], np.int32)
    assert list(tile_run_codes(codes, 16)) == [NO, -5]
    assert list(tile_run_codes(codes, 64)) == [-1, -3, 5, NO, -5, -7, -9, -11]
    assert list(tile_run_codes(np.array([3], np.int32), 128)) == [3]


def test_batched_context_fetch_cancels_lru_churn():
    """The engine's per-block context fetch (every layer's whole range, layer order) over a
    cache larger than the device tier: call by call, LRU demotion makes almost every page
    round-trip; as one batch the churn cancels and only net tier changes move."""
    L, P, per_block, blocks, cap = 6, 4, 5, 12, 150

    def run(batched):
        pt = PageTable(KvConfig(num_layers=L, head_dim=4, page_len=P, capacity_pages_device=cap,
                                capacity_pages_host=10**5))
        moved = []
        for b in range(blocks):
            n = 0
            if batched:
                pt.batch_begin()
            for li in range(L):
                base, total = pt.range(li, "self_attn")
                if total > base:
                    pt.touch_range(li, "self_attn", base, total)
                    if not batched:
                        n += len(pt.drain_moves())
            if batched:
                pt.batch_end()
                n += len(pt.drain_moves())
            for li in range(L):
                pt.append(li, "self_attn", per_block * P, b)
            moved.append(n)
            # host slots are only held by pages really on the host (plus this batch's slack)
            assert pt.pool_extent()[1] <= pt.state()["host_used"] + 2 * L * per_block
        return moved, pt.state()

    per_call, st1 = run(False)
    batched, st2 = run(True)
    assert st1 == st2  # bookkeeping is identical either way
    total_pages = L * blocks * per_block
    assert total_pages > 2 * cap
    assert sum(per_call[-3:]) > 6 * sum(batched[-3:])
    assert max(batched[-3:]) <= 2 * L * per_block  # ~ the pages whose tier really changes


def test_drain_refused_inside_open_batch():
    """A drain inside an open batch would clear the move log while the batch's pages still
    index it (a later restore in the batch would retarget an unrelated move): refused."""
    from paper_2511_20714_b200.errors import ConfigError

    pt = PageTable(KvConfig(num_layers=1, head_dim=4, page_len=1, capacity_pages_device=1,
                            capacity_pages_host=8))
    for _ in range(4):
        pt.append(0, "self_attn", 1, 0)
    pt.drain_moves()
    pt.batch_begin()
    pt.touch_indices(0, "self_attn", [1])
    with pytest.raises(ConfigError):
        pt.drain_moves()
    pt.touch_indices(0, "self_attn", [2])
    pt.touch_indices(0, "self_attn", [0])
    pt.batch_end()
    mv = pt.drain_moves()
    _check_batches(mv)
    # the churn cancels inside the batch: page 0 is back on the device tier in its own slot
    # (whose data never left), pages 1-3 stay on the host tier, and no move is left to run
    st = pt.state()
    assert [p[1] for p in st["streams"][0][4]] == [0, 1, 1, 1]
    assert pt.slots(0, "self_attn", 0, 1)[0].tolist() == [0]
    assert len(mv) == 0


def test_cache_calls_inside_batch_keep_the_move_log():
    """KvCache.fetch_indices inside batch() raises (data only consistent after the batch)
    and offload_blocks inside batch() defers its moves to the batch's end."""
    from paper_2511_20714_b200.kvcache import KvCache

    cache = KvCache(KvConfig(num_layers=1, head_dim=4, page_len=1, capacity_pages_device=2,
                             capacity_pages_host=8))
    pt = cache.page_table
    with _nullbatch(cache):
        with pytest.raises(RuntimeError):
            cache.fetch_indices(0, [])
        cache.offload_blocks([])  # no drain inside the open batch
        assert cache._batch == 1
    assert cache._batch == 0
    del pt


class _nullbatch:
    """Opens the cache's batch bookkeeping without executing moves on exit (no GPU here)."""

    def __init__(self, cache):
        self.cache = cache

    def __enter__(self):
        self.cache._pt.batch_begin()
        self.cache._batch += 1

    def __exit__(self, *exc):
        self.cache._batch -= 1
        self.cache._pt.batch_end()
