"""Cache-agnostic driver for the reference's KV differential acceptance gate.

Mirrors `TestDifferential.run_sequence` (/root/reference/pkg/tests/test_kvcache.py:286-331)
draw for draw — the same numpy Generator calls in the same order — so a sequence seeded
`default_rng(seed)` performs exactly the ops the reference's 10,000-sequence gate
(`test_acceptance.py:126-134`, n_ops=15) performs. Instead of asserting against the naive
contiguous store inline, every observable (block entries, offload/evict counts, the
addressable range, every fetched byte, and the final full bookkeeping state) is folded into
one sha256 per sequence. `tests/golden/make_golden_deep.py` records those digests from the
LIVE reference KvCache; `tests/test_acceptance_gpu.py` recomputes them through the B200
KvCache (native page table + device pools + tier moves) and requires equality.

Test infrastructure only: imported by tests/ and the golden generator, never by the package.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np

OPS = ("append", "fetch_range", "fetch_indices", "offload", "evict")


def canon(x):
    """Plain-python canonical form (ints, lists) of a state snapshot for hashing."""
    if isinstance(x, dict):
        return {str(k): canon(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [canon(v) for v in x]
    if isinstance(x, (np.integer,)):
        return int(x)
    if isinstance(x, (np.floating,)):
        return float(x)
    return x


def state_digest(state) -> str:
    return hashlib.sha256(json.dumps(canon(state), separators=(",", ":")).encode()).hexdigest()


def run_sequence(make_cache, state_of, to_numpy, rng, n_ops=15, head_dim=8, page_len=None) -> str:
    """One differential sequence (test_kvcache.py:286-331); returns its digest."""
    page_len = page_len or int(rng.integers(1, 24))
    cap_dev = int(rng.integers(1, 12))
    cache = make_cache(num_layers=2, head_dim=head_dim, page_len=page_len,
                       capacity_pages_device=cap_dev, capacity_pages_host=4096)
    h = hashlib.sha256()
    appended = []
    for _ in range(n_ops):
        op = OPS[rng.integers(0, len(OPS))]
        layer = int(rng.integers(0, 2))
        if op == "append":
            t = int(rng.integers(1, 40))
            k = rng.standard_normal((t, head_dim)).astype(np.float32)
            v = rng.standard_normal((t, head_dim)).astype(np.float32)
            e = cache.append_block(layer, k, v)
            appended.append(e.block_id)
            h.update(repr(("A", int(e.block_id), [int(x) for x in e.token_range],
                           [int(p) for p in e.page_list])).encode())
        elif op == "offload" and appended:
            ids = rng.choice(appended, size=min(2, len(appended)), replace=False)
            live = [b.block_id for b in cache.block_entries()]
            n = cache.offload_blocks([int(i) for i in ids if i in live])
            h.update(repr(("O", int(n))).encode())
        elif op == "evict":
            keep = int(rng.integers(0, 48))
            n = cache.evict_window(keep)
            h.update(repr(("E", int(n))).encode())
        else:
            base, total = cache.addressable_range(layer)
            h.update(repr(("R", int(base), int(total))).encode())
            if total == base:
                continue
            if op == "fetch_range":
                a = int(rng.integers(base, total))
                b = int(rng.integers(a, total)) + 1
                got = cache.fetch_range(layer, (a, b))
            else:
                n = rng.integers(0, 6)
                idx = rng.integers(base, total, size=n).tolist()
                got = cache.fetch_indices(layer, idx)
            for arr in got:
                h.update(np.ascontiguousarray(to_numpy(arr), np.float32).tobytes())
    h.update(state_digest(state_of(cache)).encode())
    return h.hexdigest()
