"""Replay the golden KV op traces (tests/golden/kv_traces.json) on any cache
implementation exposing the reference KvCache API plus `state()`.

Used to pin the oracle (test_oracle.py) and the native page table
(test_pagetable.py) against the live reference's full bookkeeping state.
"""

import hashlib
import json
import os

import numpy as np

from conftest import GOLDEN


def load_traces():
    with open(os.path.join(GOLDEN, "kv_traces.json")) as f:
        return json.load(f)


def rows(seed, t, d):
    g = np.random.default_rng(seed)
    return (g.standard_normal((t, d)).astype(np.float32),
            g.standard_normal((t, d)).astype(np.float32))


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(np.asarray(a), np.float32).tobytes())
    return h.hexdigest()


def replay(seq, make_cache, to_numpy=lambda a: a, CapacityError=Exception):
    """Run one recorded sequence; assert result + full state after every op."""
    cache = make_cache(seq["config"])
    for i, rec in enumerate(seq["ops"]):
        op, layer = rec["op"], rec["layer"]
        got = None
        err = None
        try:
            if op in ("append", "append_cross"):
                k, v = rows(rec["dseed"], rec["t"], 8)
                kind = "self_attn" if op == "append" else "cross_attn"
                e = cache.append_block(layer, k, v, kind=kind, chunk_index=i)
                got = [e.block_id, list(e.token_range), list(e.page_list)]
            elif op == "offload":
                got = cache.offload_blocks(rec["ids"])
            elif op == "evict":
                got = cache.evict_window(rec["keep"])
            elif op == "clear_cross":
                got = cache.clear_cross_attention()
            elif op == "fetch_indices":
                fk, fv = cache.fetch_indices(layer, rec["idx"])
                got = sha(to_numpy(fk), to_numpy(fv))
            elif op == "fetch_range":
                fk, fv = cache.fetch_range(layer, tuple(rec["range"]), rec["kind"])
                got = sha(to_numpy(fk), to_numpy(fv))
        except CapacityError:
            err = "CapacityError"
        where = f"seed {seq['seed']} op {i} ({op})"
        assert err == rec.get("error"), where
        if err is None and "result" in rec:
            assert got == rec["result"], where
        assert cache.state() == rec["state"], where
