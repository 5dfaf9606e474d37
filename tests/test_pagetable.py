"""Native page table (csrc/pagetable.cpp) vs the LIVE reference's full bookkeeping state.

CPU-only: drives libinferix_b200.so's ifx_pt_* entry points (no device memory) through the
golden traces frozen from /root/reference (tests/golden/kv_traces.json): page ids, tiers,
filled counts, start tokens, per-page last_access, the global access clock and block
entries must be bit-identical after every op, including partially failed appends.
Also a randomized differential against the oracle over many more sequences.
"""

import numpy as np
import pytest

from kv_replay import load_traces

from oracle import kvcache as OK
from paper_2511_20714_b200 import _abi
from paper_2511_20714_b200.errors import CapacityError, ConfigError, OutOfRangeError
from paper_2511_20714_b200.kvcache import KvConfig, PageTable


class BookkeepingCache:
    """Reference KvCache API over the native page table, data-less (fetch returns None)."""

    def __init__(self, cfg: dict):
        self.pt = PageTable(KvConfig(**cfg))

    def append_block(self, layer, k, v, kind="self_attn", chunk_index=0):
        rc, bid, start, written, pages = self.pt.append(layer, kind, k.shape[0], chunk_index)
        _abi.check(rc)

        class E:
            pass
        e = E()
        e.block_id, e.token_range, e.page_list = bid, (start, start + k.shape[0]), pages
        return e

    def offload_blocks(self, ids):
        return self.pt.offload(ids)

    def evict_window(self, keep):
        return self.pt.evict_window(keep)

    def clear_cross_attention(self):
        return self.pt.clear_cross()

    def fetch_range(self, layer, rng, kind="self_attn"):
        self.pt.touch_range(layer, kind, rng[0], rng[1])
        return None, None

    def fetch_indices(self, layer, idx, kind="self_attn"):
        self.pt.touch_indices(layer, kind, list(idx))
        return None, None

    def state(self):
        return self.pt.state()


def test_golden_traces_full_state_bit_exact():
    tr = load_traces()
    n_ops = 0
    for seq in tr["sequences"]:
        cache = BookkeepingCache(seq["config"])
        for i, rec in enumerate(seq["ops"]):
            op, layer = rec["op"], rec["layer"]
            err = None
            try:
                if op in ("append", "append_cross"):
                    k = np.zeros((rec["t"], 8), np.float32)
                    kind = "self_attn" if op == "append" else "cross_attn"
                    e = cache.append_block(layer, k, k, kind=kind, chunk_index=i)
                    got = [e.block_id, list(e.token_range), e.page_list]
                    assert got == rec["result"], (seq["seed"], i)
                elif op == "offload":
                    assert cache.offload_blocks(rec["ids"]) == rec["result"]
                elif op == "evict":
                    assert cache.evict_window(rec["keep"]) == rec["result"]
                elif op == "clear_cross":
                    assert cache.clear_cross_attention() == rec["result"]
                elif op == "fetch_indices":
                    cache.fetch_indices(layer, rec["idx"])
                elif op == "fetch_range":
                    cache.fetch_range(layer, rec["range"], rec["kind"])
            except CapacityError:
                err = "CapacityError"
            assert err == rec.get("error"), (seq["seed"], i)
            assert cache.state() == rec["state"], (seq["seed"], i, op)
            n_ops += 1
    assert n_ops == 60 * 25


def test_survey_a4_known_answer_trace():
    tr = load_traces()["a4_case1"]
    c = BookkeepingCache(dict(num_layers=1, head_dim=4, page_len=4, capacity_pages_device=2,
                              capacity_pages_host=8))
    z = lambda n: np.zeros((n, 4), np.float32)  # noqa: E731
    c.append_block(0, z(10), z(10)); assert c.state() == tr[0]
    c.fetch_range(0, (8, 10)); assert c.state() == tr[1]
    c.fetch_range(0, (0, 2)); assert c.state() == tr[2]
    c.append_block(0, z(3), z(3)); assert c.state() == tr[3]
    c.evict_window(5); assert c.state() == tr[4]


def _random_ops(seed, n_ops, make):
    """Random op sequence applied to `make(cfg)`; yields the state after each op."""
    g = np.random.default_rng(seed)
    cfg = dict(num_layers=int(g.integers(1, 4)), head_dim=4, page_len=int(g.integers(1, 20)),
               capacity_pages_device=int(g.integers(0, 16)), capacity_pages_host=int(g.integers(0, 32)))
    c = make(cfg)
    live = []
    for i in range(n_ops):
        op = int(g.integers(0, 8))
        L = cfg["num_layers"]
        layer = int(g.integers(0, L))
        kind = "cross_attn" if g.integers(0, 4) == 0 else "self_attn"
        try:
            if op <= 2:
                t = int(g.integers(1, 50))
                e = c.append_block(layer, np.zeros((t, 4), np.float32), np.zeros((t, 4), np.float32),
                                   kind=kind, chunk_index=i)
                live.append(e.block_id)
            elif op == 3 and live:
                c.offload_blocks([live[int(g.integers(0, len(live)))]])
            elif op == 4:
                c.evict_window(int(g.integers(0, 60)))
            elif op == 5 and g.integers(0, 3) == 0:
                c.clear_cross_attention()
            else:
                st = c.state()
                s = [x for x in st["streams"] if x[0] == layer and x[1] == kind][0]
                base, total = s[2], s[3]
                if total > base:
                    a = int(g.integers(base, total))
                    b = int(g.integers(a, total)) + 1
                    if op == 6:
                        c.fetch_range(layer, (a, b), kind)
                    else:
                        c.fetch_indices(layer, [int(x) for x in g.integers(base, total, size=4)], kind)
        except (CapacityError, OutOfRangeError):
            pass
        yield c.state()


@pytest.mark.parametrize("chunk", range(4))
def test_randomized_differential_vs_oracle(chunk):
    """400 extra random sequences (3 layers, cross streams, tiny capacities) vs the oracle."""
    for seed in range(chunk * 100, chunk * 100 + 100):
        mine = _random_ops(seed, 30, BookkeepingCache)
        ref = _random_ops(seed, 30, lambda cfg: OK.create_cache(OK.KvConfig(**cfg)))
        for step, (a, b) in enumerate(zip(mine, ref)):
            assert a == b, (seed, step)


def test_config_errors():
    with pytest.raises(ConfigError):
        PageTable(KvConfig(num_layers=1, head_dim=8, page_len=0))
    with pytest.raises(ConfigError):
        PageTable(KvConfig(num_layers=1, head_dim=8, capacity_pages_device=-1))
    pt = PageTable(KvConfig(num_layers=1, head_dim=8, capacity_pages_device=0, capacity_pages_host=0))
    rc, *_ = pt.append(0, "self_attn", 4, 0)
    assert rc == _abi.ECAPACITY
    with pytest.raises(OutOfRangeError):
        pt.touch_range(0, "self_attn", 0, 1)
    with pytest.raises(OutOfRangeError):
        pt.offload([99])
    with pytest.raises(ConfigError):
        pt.evict_window(-1)


def test_large_stream_touch_is_fast():
    """c3-scale bookkeeping: 21 blocks x 4680 tokens x 30 layers, one context touch per
    layer per block (engine.py:228-237) must stay far below the GPU block time."""
    import time
    pt = PageTable(KvConfig(num_layers=30, head_dim=1536, page_len=16,
                            capacity_pages_device=10**7, capacity_pages_host=10**7))
    t0 = time.perf_counter()
    for b in range(21):
        for l in range(30):
            base, total = pt.range(l, "self_attn")
            if total > base:
                pt.touch_range(l, "self_attn", base, total)
        for l in range(30):
            rc, *_ = pt.append(l, "self_attn", 4680, b)
            assert rc == 0
    dt = time.perf_counter() - t0
    assert pt.state()["clock"] == 30 * 4680 * sum(range(21))
    assert dt < 5.0, dt
