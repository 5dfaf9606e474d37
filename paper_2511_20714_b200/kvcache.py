"""Paged, tiered, block-wise KV cache — drop-in for `inferix.kvcache` on B200.

Reference: /root/reference/pkg/src/inferix/kvcache.py (KvConfig :33-58, KvCache :105-404).

Split of responsibilities:
  * bookkeeping (page ids, tiers, LRU, access clock, eviction, block entries) is the
    native page table in libinferix_b200.so (csrc/pagetable.cpp), bit-exact with the
    reference (tests/test_pagetable.py replays the reference's full state);
  * data lives in HBM: one K slab and one V slab per (layer, kind), rows addressed by
    stream position (token id - origin), written by K2 (`ifx_kv_append`, 128-bit stores)
    and read either in place by the attention kernel K1 or through K7 (`ifx_kv_gather`)
    for `fetch_range` / `fetch_indices`.

Storage dtype is fp32 (bit-exact API parity, the default) or bf16 (the engine's choice:
K1 reads bf16 tiles). Returned fetches are new CUDA tensors.
"""

from __future__ import annotations

import ctypes
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._device import count_launch, dtype_code, require_cuda, row_ld, stream_ptr
from .errors import ConfigError, DimensionError, OutOfRangeError

DUMP_MAGIC = b"INFKV1"  # kvcache.py:22
DEVICE, HOST = "device", "host"  # kvcache.py:72-73
SELF_ATTN, CROSS_ATTN = "self_attn", "cross_attn"  # kvcache.py:75-76
_KIND = {SELF_ATTN: _abi.SELF_ATTN, CROSS_ATTN: _abi.CROSS_ATTN}
_KIND_NAME = {v: k for k, v in _KIND.items()}


@dataclass
class LatentConfig:
    """kvcache.py:26-31 — MLA-style latent store (down on append, up on fetch)."""
    latent_dim: int
    down_proj: object  # [head_dim, latent_dim]
    up_proj: object    # [latent_dim, head_dim]


@dataclass
class KvConfig:
    """kvcache.py:33-58."""
    num_layers: int
    head_dim: int
    page_len: int = 16
    latent: LatentConfig | None = None
    capacity_pages_device: int = 1024
    capacity_pages_host: int = 1024

    def validate(self):
        if self.num_layers < 1 or self.head_dim < 1 or self.page_len < 1:
            raise ConfigError("num_layers, head_dim, page_len must be >= 1")
        if self.capacity_pages_device < 0 or self.capacity_pages_host < 0:
            raise ConfigError("capacities must be >= 0")
        lat = self.latent
        if lat is not None:
            if not 1 <= lat.latent_dim <= self.head_dim:
                raise ConfigError("latent_dim must be in [1, head_dim]")
            if tuple(lat.down_proj.shape) != (self.head_dim, lat.latent_dim):
                raise ConfigError("down_proj must be [head_dim, latent_dim]")
            if tuple(lat.up_proj.shape) != (lat.latent_dim, self.head_dim):
                raise ConfigError("up_proj must be [latent_dim, head_dim]")

    @property
    def stored_width(self) -> int:
        return self.latent.latent_dim if self.latent is not None else self.head_dim


@dataclass
class BlockEntry:
    """kvcache.py:79-86."""
    block_id: int
    layer: int
    token_range: tuple
    page_list: list
    kind: str
    chunk_index: int


@dataclass
class KvStats:
    """kvcache.py:89-95."""
    device_pages_used: int
    host_pages_used: int
    total_tokens: int
    blocks_per_layer: dict
    bytes_logical: int


class _Slab:
    """Device K/V rows of one (layer, kind) stream: row = token - origin.

    Grows geometrically; when it must grow and tokens below the stream base are dead
    (window eviction), live rows are compacted to the front instead (origin moves)."""

    def __init__(self, width: int, dtype: torch.dtype, rows: int):
        self.width, self.dtype = width, dtype
        self.origin = 0
        rows = max(16, rows)
        dev = require_cuda()
        self.k = torch.zeros(rows, width, device=dev, dtype=dtype)
        self.v = torch.zeros(rows, width, device=dev, dtype=dtype)

    def reset(self):
        self.origin = 0

    def ensure(self, base: int, end: int, page_len: int):
        """Make rows for tokens [base, end) addressable. Rows from the start of the page
        holding `base` are kept (a partially evicted page stays readable for dump())."""
        need = end - self.origin
        if need <= self.k.shape[0]:
            return
        keep = base - base % page_len
        if end - keep <= self.k.shape[0] // 2 and keep > self.origin:  # compact in place
            live0 = keep - self.origin
            n = max(0, min(self.k.shape[0], end - self.origin) - live0)
            if n:
                self.k[:n].copy_(self.k[live0:live0 + n].clone())
                self.v[:n].copy_(self.v[live0:live0 + n].clone())
            self.origin = keep
            return
        rows = max(need, 2 * self.k.shape[0])
        k = torch.zeros(rows, self.width, device=self.k.device, dtype=self.dtype)
        v = torch.zeros_like(k)
        k[:self.k.shape[0]].copy_(self.k)
        v[:self.v.shape[0]].copy_(self.v)
        self.k, self.v = k, v


class PageTable:
    """ctypes handle of the native bit-exact page table (csrc/pagetable.cpp). Host-only:
    no device memory, usable without a GPU (tests/test_pagetable.py)."""

    def __init__(self, config: KvConfig):
        config.validate()
        self.config = config
        h = ctypes.c_void_p()
        _abi.check(_abi.lib().ifx_pt_create(config.num_layers, config.head_dim, config.page_len,
                                             config.capacity_pages_device,
                                             config.capacity_pages_host, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _abi.lib().ifx_pt_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    @staticmethod
    def kind_code(kind) -> int:
        if kind not in _KIND:
            raise ConfigError(f"unknown kind {kind!r}")
        return _KIND[kind]

    def append(self, layer: int, kind: str, t: int, chunk_index: int):
        """-> (rc, block_id, start, written, page_ids); rc != 0 keeps `written` rows."""
        bid, start, written, npages = (ctypes.c_int64() for _ in range(4))
        cap = t // self.config.page_len + 2
        pages = (ctypes.c_int64 * cap)()
        rc = _abi.lib().ifx_pt_append(self._h, layer, self.kind_code(kind), t, chunk_index,
                                      ctypes.byref(bid), ctypes.byref(start), ctypes.byref(written),
                                      pages, cap, ctypes.byref(npages))
        return rc, bid.value, start.value, written.value, list(pages[:npages.value])

    def offload(self, block_ids) -> int:
        ids = [int(b) for b in block_ids]
        arr = (ctypes.c_int64 * max(1, len(ids)))(*ids)
        moved = ctypes.c_int64()
        _abi.check(_abi.lib().ifx_pt_offload(self._h, arr, len(ids), ctypes.byref(moved)))
        return moved.value

    def evict_window(self, keep: int) -> int:
        freed = ctypes.c_int64()
        _abi.check(_abi.lib().ifx_pt_evict_window(self._h, int(keep), ctypes.byref(freed)))
        return freed.value

    def clear_cross(self) -> int:
        n = ctypes.c_int64()
        _abi.check(_abi.lib().ifx_pt_clear_cross(self._h, ctypes.byref(n)))
        return n.value

    def touch_range(self, layer: int, kind: str, a: int, b: int) -> None:
        _abi.check(_abi.lib().ifx_pt_touch_range(self._h, layer, self.kind_code(kind), a, b))

    def touch_indices(self, layer: int, kind: str, idx) -> None:
        arr = (ctypes.c_int64 * max(1, len(idx)))(*idx)
        _abi.check(_abi.lib().ifx_pt_touch_indices(self._h, layer, self.kind_code(kind), arr,
                                                   len(idx)))

    def range(self, layer: int, kind: str):
        base, total = ctypes.c_int64(), ctypes.c_int64()
        _abi.check(_abi.lib().ifx_pt_range(self._h, layer, self.kind_code(kind),
                                           ctypes.byref(base), ctypes.byref(total)))
        return base.value, total.value

    def stats(self) -> list:
        L = self.config.num_layers
        out = (ctypes.c_int64 * (3 + L))()
        _abi.check(_abi.lib().ifx_pt_stats(self._h, out, 3 + L))
        return list(out)

    def state(self) -> dict:
        """Canonical full bookkeeping state (same schema as oracle.kvcache.KvStore.state)."""
        n = ctypes.c_int64()
        _abi.check(_abi.lib().ifx_pt_snapshot(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_int64 * n.value)()
        _abi.check(_abi.lib().ifx_pt_snapshot(self._h, buf, n.value, ctypes.byref(n)))
        it = iter(buf)
        nx = lambda: next(it)  # noqa: E731
        st = {"clock": nx(), "next_page": nx(), "next_block": nx(), "device_used": nx(),
              "host_used": nx()}
        streams = []
        for _ in range(nx()):
            layer, kind, base, total, npg = nx(), nx(), nx(), nx(), nx()
            pages = [[nx(), nx(), nx(), nx(), nx()] for _ in range(npg)]
            streams.append([layer, _KIND_NAME[kind], base, total, pages])
        blocks = []
        for _ in range(nx()):
            bid, layer, kind, a, b, chunk, npg = (nx() for _ in range(7))
            blocks.append([bid, layer, _KIND_NAME[kind], a, b, [nx() for _ in range(npg)], chunk])
        st["streams"], st["blocks"] = streams, blocks
        return st


class KvCache:
    """Drop-in for `inferix.kvcache.KvCache` (kvcache.py:105-404); create via create_cache().

    Extra keyword arguments (B200 only): `dtype` of the device slabs (torch.float32 for
    bit-exact API parity, torch.bfloat16 for the engine), `reserve_tokens` rows to
    pre-allocate per self-attention stream, `row_width` of the device rows when it
    differs from head_dim (the engine stores per-head zero-padded rows; a Ulysses rank
    stores only its heads), `cross_row_width` likewise for the cross-attention streams."""

    def __init__(self, config: KvConfig, dtype: torch.dtype = torch.float32,
                 reserve_tokens: int = 0, row_width: int | None = None,
                 cross_row_width: int | None = None):
        config.validate()
        self.config = config
        self.dtype = dtype
        self._lock = threading.RLock()
        self._pt = PageTable(config)
        if row_width is not None and config.latent is not None:
            raise ConfigError("row_width override is not supported in latent mode")
        w = row_width or config.stored_width
        wc = cross_row_width or w
        self._row_width = {SELF_ATTN: w, CROSS_ATTN: wc}
        self._slabs = {}
        for layer in range(config.num_layers):
            self._slabs[(layer, SELF_ATTN)] = _Slab(w, dtype, reserve_tokens)
            self._slabs[(layer, CROSS_ATTN)] = _Slab(wc, dtype, 64)
        self._latent_down = self._latent_up = None
        if config.latent is not None:
            dev = require_cuda()
            self._latent_down = torch.as_tensor(np.asarray(config.latent.down_proj, np.float32)).to(dev)
            self._latent_up = torch.as_tensor(np.asarray(config.latent.up_proj, np.float32)).to(dev)

    @property
    def page_table(self) -> PageTable:
        return self._pt

    def slab(self, layer: int, kind: str = SELF_ATTN) -> _Slab:
        """Device rows of a stream (the engine's K1 reads them in place)."""
        return self._slabs[(layer, kind)]

    @staticmethod
    def _as_rows(x) -> torch.Tensor:
        if isinstance(x, torch.Tensor):
            t = x if x.is_cuda else x.to(require_cuda())
            return t if t.dtype in (torch.float32, torch.bfloat16) else t.float()
        a = np.asarray(x, dtype=np.float32)
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(require_cuda()) if a.ndim == 2 else t

    # -- mutations ------------------------------------------------------------------------
    def append_block(self, layer: int, k, v, kind: str = SELF_ATTN, chunk_index: int = 0,
                     stream=None) -> BlockEntry:
        """kvcache.py:179-234: validate, (latent down-proj), page bookkeeping, K2 page write."""
        cfg = self.config
        k, v = self._as_rows(k), self._as_rows(v)
        if k.dim() != 2 or tuple(k.shape) != tuple(v.shape):
            raise DimensionError("k and v must be equal-shaped [t, head_dim]")
        t, d = k.shape
        if t < 1:
            raise DimensionError("append needs at least one token")
        if d != cfg.head_dim and d != self._row_width.get(kind):
            raise DimensionError(f"width {d} != head_dim {cfg.head_dim}")
        if not 0 <= layer < cfg.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        PageTable.kind_code(kind)
        if self._latent_down is not None:
            k = (k.float() @ self._latent_down).contiguous()
            v = (v.float() @ self._latent_down).contiguous()
        if k.stride(1) != 1 or v.stride(1) != 1 or k.stride(0) != v.stride(0):
            k, v = k.contiguous(), v.contiguous()
        with self._lock:
            rc, bid, start, written, pages = self._pt.append(layer, kind, t, chunk_index)
            if written > 0:  # rows already packed even if allocation then failed (kvcache.py:210-223)
                base, total = self._pt.range(layer, kind)
                s = self._slabs[(layer, kind)]
                s.ensure(base, total, cfg.page_len)
                _abi.check(_abi.lib().ifx_kv_append(
                    k.data_ptr(), v.data_ptr(), row_ld(k), dtype_code(k.dtype),
                    s.k.data_ptr(), s.v.data_ptr(), s.width, dtype_code(s.dtype),
                    total - written - s.origin, written, s.width, stream_ptr(stream)), "kv_append")
                count_launch()
            _abi.check(rc, "append_block")
            return BlockEntry(bid, layer, (start, start + t), pages, kind, chunk_index)

    def offload_blocks(self, block_ids) -> int:
        """kvcache.py:236-256 (tier bookkeeping; data stays resident in HBM)."""
        with self._lock:
            return self._pt.offload(block_ids)

    def evict_window(self, keep_last_n_tokens: int) -> int:
        """kvcache.py:258-285."""
        with self._lock:
            return self._pt.evict_window(keep_last_n_tokens)

    def clear_cross_attention(self) -> int:
        """kvcache.py:287-299."""
        with self._lock:
            n = self._pt.clear_cross()
            for layer in range(self.config.num_layers):
                self._slabs[(layer, CROSS_ATTN)].reset()
            return n

    # -- reads ----------------------------------------------------------------------------
    def touch_range(self, layer: int, token_range, kind: str = SELF_ATTN) -> None:
        """Bookkeeping half of fetch_range (restore-on-read + per-token access clock,
        kvcache.py:303-339) without moving data — what the engine calls before K1 reads
        the slab in place."""
        a, b = token_range
        with self._lock:
            self._pt.touch_range(layer, kind, a, b)

    def _gather(self, layer, kind, rows: torch.Tensor | None, first: int, n: int):
        s = self._slabs[(layer, kind)]
        ko = torch.empty(n, s.width, device=s.k.device, dtype=s.dtype)
        vo = torch.empty_like(ko)
        if n:
            _abi.check(_abi.lib().ifx_kv_gather(
                s.k.data_ptr(), s.v.data_ptr(), s.width, dtype_code(s.dtype),
                None if rows is None else rows.data_ptr(), first - s.origin, n, s.width,
                ko.data_ptr(), vo.data_ptr(), stream_ptr()), "kv_gather")
            count_launch()
        if self._latent_up is not None:
            ko, vo = ko.float() @ self._latent_up, vo.float() @ self._latent_up
        return ko, vo

    def fetch_range(self, layer: int, token_range, kind: str = SELF_ATTN):
        """kvcache.py:328-339 -> (k, v) new CUDA tensors [end-start, head_dim]."""
        a, b = token_range
        if not 0 <= layer < self.config.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        with self._lock:
            self._pt.touch_range(layer, kind, a, b)
            return self._gather(layer, kind, None, a, b - a)

    def fetch_indices(self, layer: int, indices, kind: str = SELF_ATTN):
        """kvcache.py:341-353 (order and duplicates preserved; empty -> (0, head_dim))."""
        idx = [int(i) for i in indices]
        if not 0 <= layer < self.config.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        with self._lock:
            self._pt.touch_indices(layer, kind, idx)
            if not idx:
                w, dev = self.config.head_dim, require_cuda()
                return (torch.empty(0, w, device=dev), torch.empty(0, w, device=dev))
            s = self._slabs[(layer, kind)]
            rows = torch.tensor(idx, dtype=torch.int64).to(s.k.device) - s.origin
            return self._gather(layer, kind, rows, 0, len(idx))

    def addressable_range(self, layer: int, kind: str = SELF_ATTN):
        """kvcache.py:355-357."""
        return self._pt.range(layer, kind)

    def memory_stats(self) -> KvStats:
        """kvcache.py:359-372 (bytes_logical counts fp32 K+V like the reference)."""
        with self._lock:
            out = self._pt.stats()
        tokens = out[2]
        L = self.config.num_layers
        return KvStats(out[0], out[1], tokens, {l: out[3 + l] for l in range(L)},
                       tokens * self.config.stored_width * 4 * 2)

    def state(self) -> dict:
        with self._lock:
            return self._pt.state()

    def block_entries(self) -> list:
        """kvcache.py:374-376."""
        return [BlockEntry(b[0], b[1], (b[3], b[4]), b[5], b[2], b[6]) for b in self.state()["blocks"]]

    def dump(self, path) -> None:
        """kvcache.py:380-404 — INFKV1 snapshot (fp32 rows, pages sorted by id)."""
        cfg = self.config
        pages = []
        for layer, kind, _base, _total, pgs in self.state()["streams"]:
            for pid, tier, filled, start, _la in pgs:
                pages.append((pid, tier, filled, start, layer, kind))
        pages.sort()
        with open(path, "wb") as f:
            f.write(DUMP_MAGIC)
            f.write(struct.pack("<5I", cfg.num_layers, cfg.head_dim, cfg.page_len,
                                cfg.capacity_pages_device, cfg.capacity_pages_host))
            f.write(struct.pack("<I", len(pages)))
            for pid, tier, filled, start, layer, kind in pages:
                f.write(struct.pack("<IBII", pid, tier, filled, start))
                s = self._slabs[(layer, kind)]
                r0 = start - s.origin
                f.write(s.k[r0:r0 + filled].float().cpu().numpy().tobytes())
                f.write(s.v[r0:r0 + filled].float().cpu().numpy().tobytes())


def create_cache(config: KvConfig, **kw) -> KvCache:
    """kvcache.py:407-408."""
    return KvCache(config, **kw)
