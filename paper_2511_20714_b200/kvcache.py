"""Paged, tiered, block-wise KV cache — drop-in for `inferix.kvcache` on B200.

Reference: /root/reference/pkg/src/inferix/kvcache.py (KvConfig :33-58, KvCache :105-404).

Split of responsibilities:
  * bookkeeping (page ids, tiers, LRU, access clock, eviction, block entries) is the
    native page table in libinferix_b200.so (csrc/pagetable.cpp), bit-exact with the
    reference (tests/test_pagetable.py replays the reference's full state);
  * data placement follows the tiers exactly: every page owns a slot (page_len rows) in
    the HBM pool (tier device) or in the mapped pinned-host pool (tier host) of its kind;
    the tier moves a call makes (restore-on-read with LRU demotion, offload) are drained
    from the page table and executed as whole-page copies (K6 `ifx_kv_move_pages`);
  * K2 (`ifx_kv_append`) writes appended rows straight into their pages' slots (device
    or host), K7 (`ifx_kv_gather`) serves fetch_range / fetch_indices, and the attention
    kernel K1 reads device pages in place through the slot table (engine.py).

Storage dtype is fp32 (bit-exact API parity, the default) or bf16 (the engine's choice:
K1 reads bf16 tiles). Returned fetches are new CUDA tensors.
"""

from __future__ import annotations

import contextlib
import ctypes
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._device import count_launch, dtype_code, gemm, require_cuda, row_ld, stream_ptr
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
class KvPage:
    """kvcache.py:68-76 — one page of a stream. k_data / v_data are the page's stored rows
    ([filled, stored_width] CUDA tensors, read from whichever tier holds them); `slot` is
    the B200 physical slot in that tier's pool."""
    id: int
    tier: str
    k_data: object
    v_data: object
    filled: int = 0
    start_token: int = 0
    last_access: int = 0
    slot: int = -1


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


class _HostBuf:
    """Pinned host memory mapped into the device address space (ifx_host_alloc): K2/K6/K7
    address it directly (UVA). Zero-filled so partially filled pages stay finite."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _abi.check(_abi.lib().ifx_host_alloc(int(nbytes), ctypes.byref(p)), "host_alloc")
        self.ptr, self.nbytes = p.value or 0, int(nbytes)
        if self.ptr:
            self.bytes_view().zero_()

    def bytes_view(self) -> torch.Tensor:
        """CPU uint8 tensor aliasing the buffer (valid while self is alive)."""
        return torch.frombuffer((ctypes.c_uint8 * self.nbytes).from_address(self.ptr),
                                dtype=torch.uint8)

    def __del__(self):
        if getattr(self, "ptr", 0):
            try:
                _abi.lib().ifx_host_free(ctypes.c_void_p(self.ptr))
            except Exception:  # interpreter shutdown
                pass
            self.ptr = 0


class _Pool:
    """Slot pools of one kind (self / cross): HBM [slots * page_len, width] K and V, and
    the pinned host tier alike. Grown geometrically as the page table's high-water marks
    rise (device growth is a stream-ordered copy; host growth synchronises first)."""

    def __init__(self, width: int, dtype: torch.dtype, page_len: int, max_dev: int, max_host: int):
        self.width, self.dtype, self.page_len = width, dtype, page_len
        self.max_dev, self.max_host = max(4, max_dev), max(4, max_host)  # tier capacities
        self.esz = torch.finfo(dtype).bits // 8
        self.dev_slots = self.host_slots = 0
        self.dev_k = self.dev_v = None
        self.host_k = self.host_v = None
        self._abi = None

    @property
    def slot_bytes(self) -> int:
        return self.page_len * self.width * self.esz

    def ensure(self, dev_slots: int, host_slots: int) -> None:
        P, W = self.page_len, self.width
        if dev_slots > self.dev_slots:  # geometric growth, never past the tier's capacity
            n = max(dev_slots, min(2 * self.dev_slots, self.max_dev), 4)
            dev = require_cuda()
            k = torch.zeros(n * P, W, device=dev, dtype=self.dtype)
            v = torch.zeros_like(k)
            if self.dev_slots:
                k[:self.dev_slots * P].copy_(self.dev_k)
                v[:self.dev_slots * P].copy_(self.dev_v)
            self.dev_k, self.dev_v, self.dev_slots = k, v, n
            self._abi = None
        if host_slots > self.host_slots:
            n = max(host_slots, min(2 * self.host_slots, self.max_host), 4)
            k, v = _HostBuf(n * self.slot_bytes), _HostBuf(n * self.slot_bytes)
            if self.host_slots:
                torch.cuda.synchronize()  # no kernel may still address the old buffers
                used = self.host_slots * self.slot_bytes
                k.bytes_view()[:used].copy_(self.host_k.bytes_view()[:used])
                v.bytes_view()[:used].copy_(self.host_v.bytes_view()[:used])
            self.host_k, self.host_v, self.host_slots = k, v, n
            self._abi = None

    def abi(self) -> _abi.KvPool:
        if self._abi is None:
            p = _abi.KvPool()
            p.dev_k = self.dev_k.data_ptr() if self.dev_k is not None else None
            p.dev_v = self.dev_v.data_ptr() if self.dev_v is not None else None
            p.host_k = self.host_k.ptr if self.host_k is not None else None
            p.host_v = self.host_v.ptr if self.host_v is not None else None
            p.width, p.page_len, p.type = self.width, self.page_len, dtype_code(self.dtype)
            self._abi = p
        return self._abi

    def host_rows(self, which: str) -> torch.Tensor:
        """CPU [host_slots * page_len, width] view of the host tier (tests, dump)."""
        buf = self.host_k if which == "k" else self.host_v
        return buf.bytes_view().view(self.dtype).view(-1, self.width)


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

    def drain_moves(self) -> np.ndarray:
        """Logged tier moves as int64 [n, 5] (epoch, kind, dir, device slot, host slot), in
        execution order."""
        n = ctypes.c_int64()
        L = _abi.lib()
        _abi.check(L.ifx_pt_drain_moves(self._h, None, 0, ctypes.byref(n)))
        if n.value == 0:
            return np.zeros((0, 5), np.int64)
        out = np.empty((n.value, 5), np.int64)
        _abi.check(L.ifx_pt_drain_moves(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        out.size, ctypes.byref(n)))
        return out

    def batch_begin(self) -> None:
        _abi.check(_abi.lib().ifx_pt_batch_begin(self._h))

    def batch_end(self) -> None:
        _abi.check(_abi.lib().ifx_pt_batch_end(self._h))

    def pending(self, max_layer: int = -1) -> tuple:
        """(live moves, demotions waiting for a host slot, those of them on self streams of
        layers <= max_layer) of the open epoch."""
        out = (ctypes.c_int64 * 3)()
        _abi.check(_abi.lib().ifx_pt_pending(self._h, max_layer, out))
        return out[0], out[1], out[2]

    def pool_extent(self) -> list:
        """Slots ever used: [self device, self host, cross device, cross host]."""
        out = (ctypes.c_int64 * 4)()
        _abi.check(_abi.lib().ifx_pt_pool_extent(self._h, out))
        return list(out)

    def slots(self, layer: int, kind: str, start: int, end: int):
        """(int32 slot codes of the pages covering [start, end), first page's start token);
        code >= 0 device slot, < 0 host slot -1-code."""
        n, first = ctypes.c_int64(), ctypes.c_int64()
        L = _abi.lib()
        k = self.kind_code(kind)
        _abi.check(L.ifx_pt_slots(self._h, layer, k, start, end, None, 0, ctypes.byref(first),
                                  ctypes.byref(n)))
        out = np.empty(n.value, np.int32)
        if n.value:
            _abi.check(L.ifx_pt_slots(self._h, layer, k, start, end, out.ctypes.data, n.value,
                                      ctypes.byref(first), ctypes.byref(n)))
        return out, first.value

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


class _PendingAppend:
    """An append whose bookkeeping ran (KvCache.append_reserve) and whose rows are written
    by the caller's kernel (`page`) or, failing that, by K2 in `finish`."""

    __slots__ = ("cache", "layer", "kind", "chunk", "t", "rc", "bid", "start", "written",
                 "pages", "slots", "page")

    def __init__(self, cache, layer, kind, chunk, t, rc, bid, start, written, pages):
        self.cache, self.layer, self.kind, self.chunk, self.t = cache, layer, kind, chunk, t
        self.rc, self.bid, self.start, self.written, self.pages = rc, bid, start, written, pages
        self.slots = self.page = None

    def finish(self, k=None, v=None, stream=None) -> "BlockEntry":
        c = self.cache
        if self.page is None and self.written > 0:  # rows the producer could not write
            k, v = c._as_rows(k), c._as_rows(v)
            if c._latent_down is None:
                k, v = c._pad_rows(self.kind, k, v)
            with c._lock:
                c._write_rows(self.layer, self.kind, self.start, self.written, k, v, stream)
        _abi.check(self.rc, "append_block")
        return BlockEntry(self.bid, self.layer, (self.start, self.start + self.t), self.pages,
                          self.kind, self.chunk)


class KvCache:
    """Drop-in for `inferix.kvcache.KvCache` (kvcache.py:105-404); create via create_cache().

    Extra keyword arguments (B200 only): `dtype` of the pools (torch.float32 for bit-exact
    API parity, torch.bfloat16 for the engine), `reserve_tokens` per self-attention stream
    to pre-size the HBM pool for, `row_width` of the pool rows when it differs from
    head_dim (the engine stores per-head zero-padded rows; a Ulysses rank stores only its
    heads), `cross_row_width` likewise for the cross-attention streams."""

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
        # pool rows are a multiple of 16 bytes (K2/K7 move rows in 16-byte vectors): widths
        # the reference accepts but that do not align are zero-padded in the pool and
        # trimmed on every read, so no call fails after its bookkeeping is recorded
        esz = torch.finfo(dtype).bits // 8
        w = row_width or -(-config.stored_width * esz // 16) * 16 // esz
        wc = cross_row_width or w
        self._row_width = {SELF_ATTN: w, CROSS_ATTN: wc}
        self._logical_width = {SELF_ATTN: config.stored_width if row_width is None else w,
                               CROSS_ATTN: config.stored_width if row_width is None else wc}
        cd, ch = config.capacity_pages_device, config.capacity_pages_host
        self._pools = {SELF_ATTN: _Pool(w, dtype, config.page_len, cd, ch),
                       CROSS_ATTN: _Pool(wc, dtype, config.page_len, cd, ch)}
        self.moved_pages = [0, 0]  # pages copied device->host, host->device (tier moves)
        self._batch = 0  # depth of open batch() contexts
        # bumped by every call that can change cross-attention rows (append / clear / evict):
        # the engine reuses its per-block fold of the prompt K/V while it is unchanged
        self.cross_version = 0
        self.fold_memo = None
        if reserve_tokens:
            per_layer = -(-reserve_tokens // config.page_len) + 1
            self._pools[SELF_ATTN].ensure(min(config.capacity_pages_device,
                                              per_layer * config.num_layers), 0)
        self._latent_down = self._latent_up = self._latent_up_bf16 = None
        if config.latent is not None:
            dev = require_cuda()
            # row-major fp32 on the device (K2L / K7L index them as [rows, cols])
            self._latent_down = torch.as_tensor(np.ascontiguousarray(config.latent.down_proj, np.float32)).to(dev)
            self._latent_up = torch.as_tensor(np.ascontiguousarray(config.latent.up_proj, np.float32)).to(dev)

    @property
    def page_table(self) -> PageTable:
        return self._pt

    def pool(self, kind: str = SELF_ATTN) -> _Pool:
        """Slot pools of a kind (the engine's K1 reads device pages in place)."""
        return self._pools[kind]

    @staticmethod
    def _as_rows(x) -> torch.Tensor:
        if isinstance(x, torch.Tensor):
            t = x if x.is_cuda else x.to(require_cuda())
            return t if t.dtype in (torch.float32, torch.bfloat16) else t.float()
        a = np.asarray(x, dtype=np.float32)
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(require_cuda()) if a.ndim == 2 else t

    # -- physical placement ---------------------------------------------------------------
    def _sync(self, stream=None) -> None:
        """Grow the pools to the page table's slot high-water marks, then execute the tier
        moves its last call logged (K6: device->host batch, then host->device batch)."""
        mv = self._pt.drain_moves()  # first: the drain assigns demotions' host slots
        ext = self._pt.pool_extent()
        self._pools[SELF_ATTN].ensure(ext[0], ext[1])
        self._pools[CROSS_ATTN].ensure(ext[2], ext[3])
        if not len(mv):
            return
        for kind_code, pool in ((0, self._pools[SELF_ATTN]), (1, self._pools[CROSS_ATTN])):
            sel = mv[:, 1] == kind_code
            if sel.any() and (mv[sel, 3].max() >= pool.dev_slots or mv[sel, 4].max() >= pool.host_slots
                              or mv[sel, 3:5].min() < 0):
                raise RuntimeError("page move outside the pools (page table / pool size mismatch)")
        dev = require_cuda()
        pairs = torch.from_numpy(np.ascontiguousarray(mv[:, 3:5])).to(dev, non_blocking=True)
        # consecutive records with the same (epoch, dir, kind) form one hazard-free launch
        key = mv[:, 0] * 4 + mv[:, 2] * 2 + mv[:, 1]
        cuts = np.flatnonzero(np.diff(key)) + 1
        for lo, hi in zip(np.r_[0, cuts], np.r_[cuts, len(mv)]):
            kind = _KIND_NAME[int(mv[lo, 1])]
            d = int(mv[lo, 2])
            p = self._pools[kind]
            _abi.check(_abi.lib().ifx_kv_move_pages(ctypes.byref(p.abi()), pairs[lo].data_ptr(),
                                                   int(hi - lo), d, stream_ptr(stream)), "kv_move_pages")
            count_launch()
            self.moved_pages[d] += int(hi - lo)

    @contextlib.contextmanager
    def batch(self, stream=None):
        """Bookkeeping calls inside share one move batch; the moves run (K6) at exit. The
        data of pages touched inside is only consistent after exit (the engine fetches the
        whole context this way, then builds K1's slot tables)."""
        with self._lock:
            self._pt.batch_begin()
            self._batch += 1
            try:
                yield self
            finally:
                self._batch -= 1
                self._pt.batch_end()
                if self._batch == 0:
                    self._sync(stream)

    def batch_checkpoint(self, fetched_layer: int = 10**9, stream=None) -> None:
        """Inside a layer-ordered context fetch in batch(): if the demotions that will not be
        undone before the batch ends (pages of layers <= fetched_layer) would outgrow the
        pinned host pool already allocated, run this batch's moves now and continue in a
        fresh one. Bounds the host footprint of a fetch whose tiers change a lot (e.g. the
        first fetch after a long prefill) without splitting the steady-state fetch, whose
        mid-fetch demotions of later layers are all undone."""
        if self._batch != 1:  # nested batches: only the outermost may run its moves
            return
        _, _, lazy = self._pt.pending(fetched_layer)
        ext = self._pt.pool_extent()
        spare = []
        for pool, used in ((self._pools[SELF_ATTN], ext[1]), (self._pools[CROSS_ATTN], ext[3])):
            free = pool.host_slots - used
            if pool.host_slots * pool.slot_bytes < (4 << 30):  # small pools may still double
                free = max(free, pool.host_slots)
            spare.append(free)
        if lazy > max(min(spare), 0):
            self._pt.batch_end()
            try:
                self._sync(stream)
            finally:
                self._pt.batch_begin()

    def _no_batch(self, what: str) -> None:
        if self._batch:
            raise RuntimeError(f"{what} inside KvCache.batch(): page data is only consistent "
                               f"after the batch's moves ran")

    def slot_table(self, layer: int, kind: str, start: int, end: int):
        """(int32 slot codes of the pages covering tokens [start, end), first page's start)."""
        return self._pt.slots(layer, kind, start, end)

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
        if self._latent_down is None:
            k, v = self._pad_rows(kind, k, v)
        with self._lock:
            self._no_batch("append_block")
            if kind == CROSS_ATTN:
                self.cross_version += 1
            rc, bid, start, written, pages = self._pt.append(layer, kind, t, chunk_index)
            self._sync(stream)
            if written > 0:  # rows already packed even if allocation then failed (kvcache.py:210-223)
                self._write_rows(layer, kind, start, written, k, v, stream)
            _abi.check(rc, "append_block")
            return BlockEntry(bid, layer, (start, start + t), pages, kind, chunk_index)

    def _pad_rows(self, kind: str, k, v):
        """Rows as the pool stores them: zero-padded to the pool width (16-byte rows)."""
        pad = self._row_width[kind] - k.shape[1]
        if pad > 0 and k.shape[1] == self._logical_width[kind]:  # unaligned width: zero-pad rows
            k = torch.nn.functional.pad(k, (0, pad))
            v = torch.nn.functional.pad(v, (0, pad))
        if k.stride(1) != 1 or v.stride(1) != 1 or k.stride(0) != v.stride(0):
            k, v = k.contiguous(), v.contiguous()
        return k, v

    def _write_rows(self, layer: int, kind: str, start: int, n: int, k, v, stream=None) -> None:
        """The page write of tokens [start, start + n): K2, or in latent mode K2L (the rows
        down-projected inside the page-write kernel, kvcache.py:201-203)."""
        codes, first = self._pt.slots(layer, kind, start, start + n)
        slots = torch.from_numpy(codes).to(k.device, non_blocking=True)
        p = self._pools[kind]
        if self._latent_down is not None:
            if k.stride(1) != 1 or v.stride(1) != 1 or k.stride(0) != v.stride(0):
                k, v = k.contiguous(), v.contiguous()
            lat = self.config.latent
            _abi.check(_abi.lib().ifx_kv_append_latent(
                k.data_ptr(), v.data_ptr(), row_ld(k), dtype_code(k.dtype), k.shape[1],
                self._latent_down.data_ptr(), lat.latent_dim, ctypes.byref(p.abi()),
                slots.data_ptr(), first, start, n, stream_ptr(stream)), "kv_append_latent")
        else:
            _abi.check(_abi.lib().ifx_kv_append(
                k.data_ptr(), v.data_ptr(), row_ld(k), dtype_code(k.dtype), ctypes.byref(p.abi()),
                slots.data_ptr(), first, start, n, stream_ptr(stream)), "kv_append")
        count_launch()

    def append_reserve(self, layer: int, t: int, kind: str = SELF_ATTN, chunk_index: int = 0,
                       stream=None) -> "_PendingAppend":
        """append_block (kvcache.py:179-234) split in two for a producer kernel that writes
        the rows itself (G1's QKV epilogue on the clean pass): the page bookkeeping runs NOW,
        in the reference's order; the returned object's `page` is the page-write spec for
        `gemm_fused` (None: the caller must use `finish(k, v)`, which then runs K2), and
        `finish` returns the BlockEntry or raises the bookkeeping's error (CapacityError
        after the rows the reference would have packed were written)."""
        cfg = self.config
        if t < 1:
            raise DimensionError("append needs at least one token")
        if not 0 <= layer < cfg.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        PageTable.kind_code(kind)
        with self._lock:
            self._no_batch("append_block")
            if kind == CROSS_ATTN:
                self.cross_version += 1
            rc, bid, start, written, pages = self._pt.append(layer, kind, t, chunk_index)
            self._sync(stream)
            pend = _PendingAppend(self, layer, kind, chunk_index, t, rc, bid, start, written, pages)
            pool = self._pools[kind]
            if (rc == _abi.OK and self._latent_down is None and pool.dtype == torch.bfloat16
                    and self._row_width[kind] == self._logical_width[kind]):
                codes, first = self._pt.slots(layer, kind, start, start + written)
                pend.slots = torch.from_numpy(codes).to(require_cuda(), non_blocking=True)
                pend.page = (pool.abi(), pend.slots, first, start)
            return pend

    def offload_blocks(self, block_ids) -> int:
        """kvcache.py:236-256: demote the blocks' device pages; their data moves to the
        pinned host pool (K6) even when a later block id fails (partial, like the
        reference)."""
        with self._lock:
            try:
                return self._pt.offload(block_ids)
            finally:
                if not self._batch:  # inside batch(): the moves run when the batch ends
                    self._sync()

    def evict_window(self, keep_last_n_tokens: int) -> int:
        """kvcache.py:258-285 (freed pages return their slots to the pools)."""
        with self._lock:
            self._no_batch("evict_window")
            self.cross_version += 1
            return self._pt.evict_window(keep_last_n_tokens)

    def clear_cross_attention(self) -> int:
        """kvcache.py:287-299."""
        with self._lock:
            self._no_batch("clear_cross_attention")
            self.cross_version += 1
            return self._pt.clear_cross()

    # -- reads ----------------------------------------------------------------------------
    def touch_range(self, layer: int, token_range, kind: str = SELF_ATTN, stream=None) -> None:
        """Bookkeeping half of fetch_range (restore-on-read + per-token access clock,
        kvcache.py:303-339) with the data moves it implies, without gathering — what the
        engine calls before K1 reads the pages in place."""
        a, b = token_range
        with self._lock:
            try:
                self._pt.touch_range(layer, kind, a, b)
            finally:
                if not self._batch:
                    self._sync(stream)

    def _gather(self, layer, kind, tokens: torch.Tensor | None, first: int, n: int, lo: int, hi: int,
                raw: bool = False):
        self._no_batch("a fetch")
        p = self._pools[kind]
        dev = require_cuda()
        if self._latent_up is not None and not raw:  # K7L: gather + up-projection, fp32
            lat = self.config.latent
            d = self.config.head_dim
            ko = torch.empty(n, d, device=dev, dtype=torch.float32)
            vo = torch.empty_like(ko)
            if n:
                codes, first_tok = self._pt.slots(layer, kind, lo, hi)
                slots = torch.from_numpy(codes).to(dev, non_blocking=True)
                _abi.check(_abi.lib().ifx_kv_gather_latent(
                    ctypes.byref(p.abi()), slots.data_ptr(), first_tok,
                    None if tokens is None else tokens.data_ptr(), first, n, lat.latent_dim,
                    self._latent_up.data_ptr(), d, ko.data_ptr(), vo.data_ptr(), d, _abi.F32,
                    stream_ptr()), "kv_gather_latent")
                count_launch()
            return ko, vo
        ko = torch.empty(n, p.width, device=dev, dtype=p.dtype)
        vo = torch.empty_like(ko)
        if n:
            codes, first_tok = self._pt.slots(layer, kind, lo, hi)
            slots = torch.from_numpy(codes).to(dev, non_blocking=True)
            _abi.check(_abi.lib().ifx_kv_gather(
                ctypes.byref(p.abi()), slots.data_ptr(), first_tok,
                None if tokens is None else tokens.data_ptr(), first, n,
                ko.data_ptr(), vo.data_ptr(), stream_ptr()), "kv_gather")
            count_launch()
        lw = self._logical_width[kind]
        if p.width != lw:  # padded pool rows (alignment)
            ko, vo = ko[:, :lw].contiguous(), vo[:, :lw].contiguous()
        return ko, vo

    def gather_expanded(self, layer: int, kind: str, lo: int, hi: int):
        """Rows [lo, hi) as bf16 [n, head_dim] for attention (no access-clock tick: the
        caller did the fetch bookkeeping). In latent mode the stored rows are gathered (K7)
        and up-projected on the tensor cores (one bf16 GEMM each for K and V, fp32
        accumulation); otherwise the rows themselves."""
        ko, vo = self._gather(layer, kind, None, lo, hi - lo, lo, hi, raw=True)
        if self._latent_up is None:
            return ko, vo
        if self._latent_up_bf16 is None:
            self._latent_up_bf16 = self._latent_up.to(torch.bfloat16).contiguous()
        d = self.config.head_dim
        outs = []
        for x in (ko, vo):
            y = torch.empty(x.shape[0], d, device=x.device, dtype=torch.bfloat16)
            if x.shape[0]:
                gemm(x.to(torch.bfloat16).contiguous(), self._latent_up_bf16, y)
            outs.append(y)
        return outs[0], outs[1]

    def fetch_range(self, layer: int, token_range, kind: str = SELF_ATTN):
        """kvcache.py:328-339 -> (k, v) new CUDA tensors [end-start, head_dim]."""
        a, b = token_range
        if not 0 <= layer < self.config.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        with self._lock:
            self.touch_range(layer, (a, b), kind)
            return self._gather(layer, kind, None, a, b - a, a, b)

    def fetch_indices(self, layer: int, indices, kind: str = SELF_ATTN):
        """kvcache.py:341-353 (order and duplicates preserved; empty -> (0, head_dim))."""
        idx = [int(i) for i in indices]
        if not 0 <= layer < self.config.num_layers:
            raise OutOfRangeError(f"layer {layer} out of range")
        with self._lock:
            self._no_batch("a fetch")
            try:
                self._pt.touch_indices(layer, kind, idx)
            finally:
                self._sync()
            if not idx:
                w, dev = self.config.head_dim, require_cuda()
                return (torch.empty(0, w, device=dev), torch.empty(0, w, device=dev))
            toks = torch.tensor(idx, dtype=torch.int64).to(require_cuda(), non_blocking=True)
            return self._gather(layer, kind, toks, 0, len(idx), min(idx), max(idx) + 1)

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

    def pages(self, layer: int, kind: str = SELF_ATTN) -> list:
        """The pages of a stream in token order as KvPage records (kvcache.py:98-101), with
        their rows gathered from their tier (no access-clock tick, like dump())."""
        with self._lock:
            for lay, knd, _base, total, pgs in self.state()["streams"]:
                if lay == layer and knd == kind and pgs:
                    s0 = pgs[0][3]
                    k, v = self._gather(layer, kind, None, s0, total - s0, s0, total, raw=True)
                    codes, _ = self._pt.slots(layer, kind, s0, total)
                    return [KvPage(pid, DEVICE if tier == 0 else HOST, k[st - s0:st - s0 + f],
                                   v[st - s0:st - s0 + f], f, st, la,
                                   int(c) if c >= 0 else -1 - int(c))
                            for (pid, tier, f, st, la), c in zip(pgs, codes)]
            return []

    def block_entries(self) -> list:
        """kvcache.py:374-376."""
        return [BlockEntry(b[0], b[1], (b[3], b[4]), b[5], b[2], b[6]) for b in self.state()["blocks"]]

    def dump(self, path) -> None:
        """kvcache.py:380-404 — INFKV1 snapshot (fp32 rows, pages sorted by id). Reads every
        page where it lives (device or host pool) without touching the access clock."""
        cfg = self.config
        pages, rows = [], {}
        for layer, kind, _base, total, pgs in self.state()["streams"]:
            if not pgs:
                continue
            s0 = pgs[0][3]
            k, v = self._gather(layer, kind, None, s0, total - s0, s0, total, raw=True)
            rows[(layer, kind)] = (s0, k.float().cpu().numpy(), v.float().cpu().numpy())
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
                s0, k, v = rows[(layer, kind)]
                f.write(k[start - s0:start - s0 + filled].tobytes())
                f.write(v[start - s0:start - s0 + filled].tobytes())


def create_cache(config: KvConfig, **kw) -> KvCache:
    """kvcache.py:407-408."""
    return KvCache(config, **kw)
