// pagetable.cpp — bit-exact host bookkeeping of the paged two-tier KV cache.
//
// Behaviour restated from /root/reference/pkg/src/inferix/kvcache.py:105-404; every quirk in
// SURVEY.md §7.4 item 4 is reproduced and pinned by tests/test_pagetable.py against the
// live reference's full state (tests/golden/kv_traces.json):
//   * page ids / block ids are global monotone counters, never reused (kvcache.py:141,232)
//   * allocation is device-first, spills to host, CapacityError when both full (:128-138),
//     and an append that fails keeps the pages it already packed (:210-223)
//   * the access clock ticks once per token fetched (:156-158,319)
//   * restore demotes the device page with the smallest last_access; ties go to the first
//     page in (layer, self/cross) stream order then page order (:166-169)
//   * evict_window frees only FULL pages wholly below the new base (:272-278)
//   * clear_cross_attention resets the cross streams' total to 0 (:298)
//
// B200 design notes (DESIGN.md §Page table):
//   * Within a stream, page k covers tokens [s0 + k*page_len, ...) where s0 is the first
//     page's start — pages fill completely before the next is created and start_token ==
//     stream.total at creation (kvcache.py:211-214). So token -> page is O(1) arithmetic
//     and the device slab can be addressed by stream position.
//   * The LRU index (ordered set keyed (last_access, stream, page id)) is only maintained
//     while some page lives on the host tier; without host pages no restore can happen,
//     so the common no-spill case touches pages in O(pages) with no tree updates.
//   * Physical placement follows the tiers exactly: every page owns a SLOT in the device
//     pool (tier 0) or the pinned host pool (tier 1) of its kind (self / cross; a slot is
//     page_len rows). Tier changes inside one call (restore, demote) are logged as page
//     moves and drained by the caller as two hazard-free batches executed in order: all
//     device->host copies, then all host->device copies (K6, ifx_kv_move_pages). Within a
//     call, host slots freed by a restore are only recycled at the drain (so no D2H of the
//     batch overwrites a host page an H2D of the batch still has to read), and a page that
//     is restored and demoted again (or the reverse) in the same call cancels its pending
//     move instead of chaining a second one.
//
// Snapshot record (ifx_pt_snapshot), all int64:
//   clock, next_page, next_block, device_used, host_used, n_streams,
//   per stream: layer, kind, base, total, n_pages, per page: id, tier(0 dev/1 host), filled,
//               start_token, last_access
//   n_blocks, per block (ascending id): id, layer, kind, start, end, chunk, n_pages, ids...

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ifx_abi.h"
#include "common_host.h"

namespace {

struct Page {
  int64_t id;
  int tier;  // 0 device, 1 host
  int64_t filled;
  int64_t start;
  int64_t last_access;
  int stream;
  int64_t slot = -1;      // row block in the pool of (kind, tier)
  int64_t pending = -1;   // index of this call's live move that brought it to its tier
  int64_t prev_slot = -1; // the slot that move copies from (still holds the data)
};

// slot allocator of one (kind, tier) pool: LIFO free list + high-water mark; frees of
// host slots made during a call are deferred to the drain (see header)
struct SlotPool {
  // free slots ordered: take() returns the smallest, so pages allocated or moved together
  // get ascending consecutive slots (one TMA box per key tile in K1, one DMA per run when
  // staging host pages)
  std::set<int64_t> free_set;
  std::vector<Page*> holder;  // page in each slot (device pools)
  std::vector<int64_t> deferred;
  std::vector<char> is_deferred;
  int64_t hwm = 0;
  void grow(int64_t s) {
    if ((int64_t)holder.size() <= s) holder.resize(s + 1, nullptr);
  }
  int64_t take() {
    if (!free_set.empty()) {
      const int64_t s = *free_set.begin();
      free_set.erase(free_set.begin());
      return s;
    }
    grow(hwm);
    return hwm++;
  }
  bool take_specific(int64_t s) { return free_set.erase(s) > 0; }
  void give(int64_t s) {
    grow(s);
    holder[s] = nullptr;
    free_set.insert(s);
  }
  void defer(int64_t s) {
    if ((int64_t)is_deferred.size() <= s) is_deferred.resize(s + 1, 0);
    is_deferred[s] = 1;
    deferred.push_back(s);
  }
  bool reclaim(int64_t s) {  // take back a deferred slot (its data is still there)
    if (s < (int64_t)is_deferred.size() && is_deferred[s]) {
      is_deferred[s] = 0;
      return true;
    }
    return false;
  }
  void flush() {
    for (int64_t s : deferred)
      if (s < (int64_t)is_deferred.size() && is_deferred[s]) {
        is_deferred[s] = 0;
        give(s);
      }
    deferred.clear();
  }
};

struct Move {
  int64_t epoch;  // the call that logged it: batches execute per call, in call order
  int kind;
  int dir;  // 0 device -> host (demote), 1 host -> device (restore)
  int64_t dev_slot, host_slot;  // a demotion's host slot is assigned when its epoch ends
  bool live;
};

struct Stream {
  std::deque<Page*> pages;
  int64_t total = 0;
  int64_t base = 0;
};

struct Block {
  int64_t id, layer;
  int kind;
  int64_t start, end, chunk;
  std::vector<int64_t> pages;
};

using LruKey = std::tuple<int64_t, int, int64_t>;  // (last_access, stream idx, page id)

}  // namespace

struct ifx_pagetable {
  int64_t num_layers, head_dim, page_len, cap_dev, cap_host;
  std::vector<Stream> streams;  // index = layer*2 + kind  (dict order of kvcache.py:112-116)
  std::map<int64_t, Block> blocks;
  std::map<int64_t, Page*> live;  // all allocated pages by id
  int64_t next_block = 0, next_page = 0, dev_used = 0, host_used = 0, clock = 0;
  bool lru_on = false;
  std::set<LruKey> lru;  // device pages, maintained only while host_used > 0
  SlotPool pools[2][2];  // [kind][tier]
  std::vector<Move> moves;
  std::vector<Page*> pend_pages;  // pages with a move pending in the current call
  int64_t epoch = 0;
  int batch_depth = 0;  // > 0: calls share one epoch (ifx_pt_batch_begin / _end)
  std::mutex mu;

  // start of every mutating call: moves of earlier calls are final (they execute before
  // this call's), host slots they freed may be recycled. Inside a batch every call belongs
  // to the batch's epoch, so a page restored by one call and demoted again by a later one
  // (the LRU churn of a whole-context fetch) cancels instead of moving twice.
  void begin_call() {
    if (batch_depth > 0) return;
    finalize_epoch();
    epoch++;
    for (Page* p : pend_pages) p->pending = -1;
    pend_pages.clear();
    for (auto& k : pools)
      for (auto& t : k) t.flush();
  }

  ~ifx_pagetable() {
    for (auto& kv : live) delete kv.second;
  }

  // -- LRU index -------------------------------------------------------------------------
  void lru_sync() {
    bool want = host_used > 0;
    if (want == lru_on) return;
    lru.clear();
    lru_on = want;
    if (!want) return;
    for (auto& kv : live)
      if (kv.second->tier == 0) lru.insert(key(kv.second));
  }
  static LruKey key(const Page* p) { return LruKey(p->last_access, p->stream, p->id); }

  // -- allocation (kvcache.py:126-158) ---------------------------------------------------
  Page* alloc(int s, int64_t start) {
    int tier;
    if (dev_used < cap_dev) {
      tier = 0;
      dev_used++;
    } else if (host_used < cap_host) {
      tier = 1;
      host_used++;
    } else {
      return nullptr;
    }
    Page* p = new Page{next_page++, tier, 0, start, 0, s};
    p->slot = pools[s & 1][tier].take();
    if (tier == 0) pools[s & 1][0].holder[p->slot] = p;
    live[p->id] = p;
    if (tier == 0 && lru_on) lru.insert(key(p));
    lru_sync();
    return p;
  }

  void release(Page* p) {  // no call leaves pending moves, so the slot is free at once
    pools[p->stream & 1][p->tier].give(p->slot);
    if (p->tier == 0) {
      dev_used--;
      if (lru_on) lru.erase(key(p));
    } else {
      host_used--;
    }
    live.erase(p->id);
    delete p;
    lru_sync();
  }

  // End of an epoch: pages still demoted get their host slot now. Assigning it lazily
  // means a page demoted and restored again within the epoch never holds one, so a batch
  // whose LRU churn cycles the whole device tier needs host slots only for the pages
  // whose tier really changed (not for every page in flight). Host slots freed by this
  // epoch's restores are still deferred here, so no H2D source is handed out.
  void finalize_epoch() {
    for (Page* p : pend_pages)
      if (p->tier == 1 && p->slot < 0 && p->pending >= 0) {
        const int64_t hs = pools[p->stream & 1][1].take();
        moves[p->pending].host_slot = hs;
        p->slot = hs;
      }
  }

  // Make device slot s available to a page being restored in the epoch that demoted it:
  // free -> take it; held by a page whose H2D into s is still pending -> retarget that H2D.
  bool reclaim_device_slot(SlotPool& dp, int64_t s) {
    if (dp.take_specific(s)) return true;
    if (s >= (int64_t)dp.holder.size()) return false;
    Page* h = dp.holder[s];
    if (h == nullptr || h->pending < 0 || moves[h->pending].dir != 1 || !moves[h->pending].live)
      return false;
    const int64_t ds = dp.take();
    moves[h->pending].dev_slot = ds;
    h->slot = ds;
    dp.holder[ds] = h;
    dp.holder[s] = nullptr;
    return true;
  }

  void demote(Page* p) {  // device -> host
    if (lru_on) lru.erase(key(p));
    const int k = p->stream & 1;
    if (p->pending >= 0 && pools[k][1].reclaim(p->prev_slot)) {
      // restored earlier in this call: its data never left the host slot it came from
      moves[p->pending].live = false;
      pools[k][0].give(p->slot);
      p->slot = p->prev_slot;
      p->pending = -1;
    } else {
      moves.push_back(Move{epoch, k, 0, p->slot, -1, true});  // host slot: finalize_epoch()
      pools[k][0].give(p->slot);  // read by the D2H batch before any H2D may refill it
      p->pending = (int64_t)moves.size() - 1;
      p->prev_slot = p->slot;
      p->slot = -1;
      pend_pages.push_back(p);
    }
    p->tier = 1;
    dev_used--;
    host_used++;
    lru_sync();
  }

  // kvcache.py:160-175
  void restore(Page* p) {
    if (cap_dev == 0) return;  // read in place
    if (dev_used >= cap_dev) {
      // lru_on is guaranteed: p itself lives on the host
      Page* victim = live.at(std::get<2>(*lru.begin()));
      demote(victim);
    }
    const int k = p->stream & 1;
    SlotPool& dp = pools[k][0];
    if (p->pending >= 0 && reclaim_device_slot(dp, p->prev_slot)) {
      // demoted earlier in this epoch: its data never left its device slot, which it gets
      // back (a page restored into that slot meanwhile is pointed at another one before its
      // H2D runs) -- the demotion's D2H is cancelled, nothing moves
      moves[p->pending].live = false;  // (no host slot was assigned to it yet)
      p->pending = -1;
      p->slot = p->prev_slot;
      dp.holder[p->slot] = p;
      p->tier = 0;
      host_used--;
      dev_used++;
      if (lru_on) lru.insert(key(p));
      lru_sync();
      return;
    }
    const int64_t ds = dp.take();
    dp.holder[ds] = p;
    if (p->slot < 0) {  // demoted in this epoch and its device slot could not be reclaimed:
      p->slot = pools[k][1].take();  // round trip through a host slot (D2H before H2D)
      moves[p->pending].host_slot = p->slot;
    }
    {
      // (a demotion earlier in this call, if any, stays live: D2H runs before H2D)
      moves.push_back(Move{epoch, k, 1, ds, p->slot, true});
      pools[k][1].defer(p->slot);
      p->pending = (int64_t)moves.size() - 1;
      p->prev_slot = p->slot;
      pend_pages.push_back(p);
    }
    p->slot = ds;
    p->tier = 0;
    host_used--;
    dev_used++;
    if (lru_on) lru.insert(key(p));
    lru_sync();
  }

  void touch(Page* p, int64_t ticks) {
    if (lru_on && p->tier == 0) lru.erase(key(p));
    clock += ticks;
    p->last_access = clock;
    if (lru_on && p->tier == 0) lru.insert(key(p));
  }

  Page* page_of(Stream& st, int64_t pos) {
    if (st.pages.empty()) return nullptr;
    int64_t k = (pos - st.pages.front()->start) / page_len;
    if (pos < st.pages.front()->start || k >= (int64_t)st.pages.size()) return nullptr;
    Page* p = st.pages[k];
    if (pos < p->start || pos >= p->start + p->filled) return nullptr;
    return p;
  }
};

extern "C" {

int ifx_pt_create(int64_t num_layers, int64_t head_dim, int64_t page_len, int64_t cap_dev,
                  int64_t cap_host, ifx_pagetable** out) {
  if (num_layers < 1 || head_dim < 1 || page_len < 1)
    return ifx::fail(IFX_ECONFIG, "num_layers, head_dim, page_len must be >= 1");
  if (cap_dev < 0 || cap_host < 0) return ifx::fail(IFX_ECONFIG, "capacities must be >= 0");
  auto* pt = new ifx_pagetable();
  pt->num_layers = num_layers;
  pt->head_dim = head_dim;
  pt->page_len = page_len;
  pt->cap_dev = cap_dev;
  pt->cap_host = cap_host;
  pt->streams.resize(num_layers * 2);
  *out = pt;
  return IFX_OK;
}

void ifx_pt_destroy(ifx_pagetable* pt) { delete pt; }

static int check_stream(const ifx_pagetable* pt, int64_t layer, int kind) {
  if (layer < 0 || layer >= pt->num_layers) return ifx::fail(IFX_ERANGE, "layer out of range");
  if (kind != IFX_SELF_ATTN && kind != IFX_CROSS_ATTN)
    return ifx::fail(IFX_ECONFIG, "unknown kind");
  return IFX_OK;
}

int ifx_pt_append(ifx_pagetable* pt, int64_t layer, int kind, int64_t t, int64_t chunk_index,
                  int64_t* out_block_id, int64_t* out_start, int64_t* out_written,
                  int64_t* out_pages, int64_t page_cap, int64_t* out_npages) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  *out_written = 0;
  if (t < 1) return ifx::fail(IFX_EDIM, "append needs at least one token");
  if (int rc = check_stream(pt, layer, kind)) return rc;
  const int s = (int)(layer * 2 + kind);
  Stream& st = pt->streams[s];
  const int64_t start = st.total;
  *out_start = start;  // also on CapacityError: the caller copies the rows already packed
  std::vector<int64_t> ids;
  int64_t written = 0;
  while (written < t) {  // kvcache.py:210-223
    Page* p = st.pages.empty() ? nullptr : st.pages.back();
    if (p == nullptr || p->filled == pt->page_len) {
      p = pt->alloc(s, st.total);
      if (!p) {
        *out_written = written;
        return ifx::fail(IFX_ECAPACITY, "both tiers full (device=" + std::to_string(pt->cap_dev) +
                                            ", host=" + std::to_string(pt->cap_host) + " pages)");
      }
      st.pages.push_back(p);
    }
    int64_t n = std::min(pt->page_len - p->filled, t - written);
    p->filled += n;
    st.total += n;
    written += n;
    if (ids.empty() || ids.back() != p->id) ids.push_back(p->id);
  }
  Block b{pt->next_block++, layer, kind, start, start + t, chunk_index, ids};
  pt->blocks[b.id] = b;
  *out_written = written;
  *out_block_id = b.id;
  *out_start = start;
  *out_npages = (int64_t)ids.size();
  for (int64_t i = 0; i < (int64_t)ids.size() && i < page_cap; ++i) out_pages[i] = ids[i];
  return IFX_OK;
}

int ifx_pt_offload(ifx_pagetable* pt, const int64_t* block_ids, int64_t n, int64_t* out_moved) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  *out_moved = 0;
  std::vector<Page*> order;  // dict insertion order of kvcache.py:238-245
  std::set<int64_t> seen;
  for (int64_t i = 0; i < n; ++i) {
    auto it = pt->blocks.find(block_ids[i]);
    if (it == pt->blocks.end())
      return ifx::fail(IFX_ERANGE, "unknown block id " + std::to_string(block_ids[i]));
    const Block& b = it->second;
    std::set<int64_t> want(b.pages.begin(), b.pages.end());
    for (Page* p : pt->streams[b.layer * 2 + b.kind].pages)
      if (want.count(p->id) && seen.insert(p->id).second) order.push_back(p);
  }
  for (Page* p : order) {  // kvcache.py:246-256
    if (p->tier != 0) continue;
    if (pt->host_used >= pt->cap_host) return ifx::fail(IFX_ECAPACITY, "host tier full, cannot offload");
    pt->demote(p);
    (*out_moved)++;
  }
  return IFX_OK;
}

int ifx_pt_evict_window(ifx_pagetable* pt, int64_t keep, int64_t* out_freed) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  if (keep < 0) return ifx::fail(IFX_ECONFIG, "keep_last_n_tokens must be >= 0");
  int64_t freed = 0;
  for (int64_t l = 0; l < pt->num_layers; ++l) {  // kvcache.py:263-278
    Stream& st = pt->streams[l * 2 + IFX_SELF_ATTN];
    int64_t nb = std::max(st.base, st.total - keep);
    freed += nb - st.base;
    st.base = nb;
    std::deque<Page*> keepers;
    for (Page* p : st.pages) {
      if (p->start + p->filled <= nb && p->filled == pt->page_len)
        pt->release(p);
      else
        keepers.push_back(p);
    }
    st.pages.swap(keepers);
  }
  for (auto it = pt->blocks.begin(); it != pt->blocks.end();) {  // kvcache.py:280-284
    const Block& b = it->second;
    if (b.kind == IFX_SELF_ATTN && b.end <= pt->streams[b.layer * 2 + IFX_SELF_ATTN].base)
      it = pt->blocks.erase(it);
    else
      ++it;
  }
  *out_freed = freed;
  return IFX_OK;
}

int ifx_pt_clear_cross(ifx_pagetable* pt, int64_t* out_cleared) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  int64_t cleared = 0;
  for (auto it = pt->blocks.begin(); it != pt->blocks.end();) {
    if (it->second.kind == IFX_CROSS_ATTN) {
      it = pt->blocks.erase(it);
      cleared++;
    } else {
      ++it;
    }
  }
  for (int64_t l = 0; l < pt->num_layers; ++l) {
    Stream& st = pt->streams[l * 2 + IFX_CROSS_ATTN];
    for (Page* p : st.pages) pt->release(p);
    st = Stream();
  }
  *out_cleared = cleared;
  return IFX_OK;
}

int ifx_pt_touch_range(ifx_pagetable* pt, int64_t layer, int kind, int64_t start, int64_t end) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  if (int rc = check_stream(pt, layer, kind)) return rc;
  Stream& st = pt->streams[layer * 2 + kind];
  if (start < st.base || end > st.total || start > end)
    return ifx::fail(IFX_ERANGE, "range [" + std::to_string(start) + ", " + std::to_string(end) +
                                     ") outside addressable [" + std::to_string(st.base) + ", " +
                                     std::to_string(st.total) + ")");
  int64_t pos = start;
  while (pos < end) {  // one step per page run: restore at its first token, then tick
    Page* p = pt->page_of(st, pos);
    if (!p) return ifx::fail(IFX_ERANGE, "token " + std::to_string(pos) + " not stored");
    int64_t run = std::min(end, p->start + p->filled) - pos;
    if (p->tier == 1) pt->restore(p);
    pt->touch(p, run);
    pos += run;
  }
  return IFX_OK;
}

int ifx_pt_touch_indices(ifx_pagetable* pt, int64_t layer, int kind, const int64_t* idx,
                         int64_t n) {
  std::lock_guard<std::mutex> g(pt->mu);
  pt->begin_call();
  if (int rc = check_stream(pt, layer, kind)) return rc;
  Stream& st = pt->streams[layer * 2 + kind];
  for (int64_t i = 0; i < n; ++i)  // validation precedes any mutation (kvcache.py:346-349)
    if (idx[i] < st.base || idx[i] >= st.total)
      return ifx::fail(IFX_ERANGE, "index " + std::to_string(idx[i]) + " not stored");
  for (int64_t i = 0; i < n; ++i) {
    Page* p = pt->page_of(st, idx[i]);
    if (!p) return ifx::fail(IFX_ERANGE, "token " + std::to_string(idx[i]) + " not stored");
    if (p->tier == 1) pt->restore(p);
    pt->touch(p, 1);
  }
  return IFX_OK;
}

int ifx_pt_range(const ifx_pagetable* pt, int64_t layer, int kind, int64_t* base, int64_t* total) {
  if (int rc = check_stream(pt, layer, kind)) return rc;
  const Stream& st = pt->streams[layer * 2 + kind];
  *base = st.base;
  *total = st.total;
  return IFX_OK;
}

int ifx_pt_stats(const ifx_pagetable* pt, int64_t* out, int64_t cap) {
  if (cap < 3 + pt->num_layers) return ifx::fail(IFX_EDIM, "stats buffer too small");
  out[0] = pt->dev_used;
  out[1] = pt->host_used;
  int64_t tok = 0;
  for (const Stream& st : pt->streams) tok += st.total - st.base;
  out[2] = tok;
  for (int64_t l = 0; l < pt->num_layers; ++l) out[3 + l] = 0;
  for (const auto& kv : pt->blocks) out[3 + kv.second.layer]++;
  return IFX_OK;
}

int ifx_pt_snapshot(const ifx_pagetable* pt, int64_t* out, int64_t cap, int64_t* out_len) {
  std::vector<int64_t> r = {pt->clock, pt->next_page, pt->next_block, pt->dev_used,
                            pt->host_used, (int64_t)pt->streams.size()};
  for (size_t s = 0; s < pt->streams.size(); ++s) {
    const Stream& st = pt->streams[s];
    r.insert(r.end(), {(int64_t)(s / 2), (int64_t)(s % 2), st.base, st.total,
                       (int64_t)st.pages.size()});
    for (const Page* p : st.pages)
      r.insert(r.end(), {p->id, (int64_t)p->tier, p->filled, p->start, p->last_access});
  }
  r.push_back((int64_t)pt->blocks.size());
  for (const auto& kv : pt->blocks) {
    const Block& b = kv.second;
    r.insert(r.end(), {b.id, b.layer, (int64_t)b.kind, b.start, b.end, b.chunk,
                       (int64_t)b.pages.size()});
    r.insert(r.end(), b.pages.begin(), b.pages.end());
  }
  *out_len = (int64_t)r.size();
  if (out == nullptr) return IFX_OK;
  if (cap < (int64_t)r.size()) return ifx::fail(IFX_EDIM, "snapshot buffer too small");
  std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
  return IFX_OK;
}

int ifx_pt_batch_begin(ifx_pagetable* pt) {
  std::lock_guard<std::mutex> g(pt->mu);
  if (pt->batch_depth == 0) pt->begin_call();
  pt->batch_depth++;
  return IFX_OK;
}

int ifx_pt_batch_end(ifx_pagetable* pt) {
  std::lock_guard<std::mutex> g(pt->mu);
  if (pt->batch_depth == 0) return ifx::fail(IFX_ECONFIG, "batch_end without batch_begin");
  pt->batch_depth--;
  return IFX_OK;
}

int ifx_pt_pending(const ifx_pagetable* pt, int64_t max_layer, int64_t* out3) {
  int64_t live = 0, lazy = 0, committed = 0;
  for (const Move& m : pt->moves) live += m.live ? 1 : 0;
  std::set<const Page*> seen;
  for (const Page* p : pt->pend_pages)
    if (p->tier == 1 && p->slot < 0 && p->pending >= 0 && seen.insert(p).second) {
      lazy++;
      if (p->stream % 2 == IFX_SELF_ATTN && p->stream / 2 <= max_layer) committed++;
    }
  out3[0] = live;
  out3[1] = lazy;
  out3[2] = committed;
  return IFX_OK;
}

int ifx_pt_drain_moves(ifx_pagetable* pt, int64_t* out, int64_t cap, int64_t* n_records) {
  std::lock_guard<std::mutex> g(pt->mu);
  // a drain clears the move log, but pages of an open batch still index it (pending):
  // later restores / demotions of the batch would then retarget or cancel the wrong move
  if (pt->batch_depth > 0) return ifx::fail(IFX_ECONFIG, "drain_moves inside an open batch");
  pt->finalize_epoch();
  std::vector<const Move*> live;
  for (const Move& m : pt->moves)
    if (m.live) live.push_back(&m);
  // execution order: per call (epoch), every device->host copy before any host->device one
  std::stable_sort(live.begin(), live.end(), [](const Move* a, const Move* b) {
    return a->epoch != b->epoch ? a->epoch < b->epoch : a->dir < b->dir;
  });
  *n_records = (int64_t)live.size();
  if (out == nullptr) return IFX_OK;
  if (cap < 5 * (int64_t)live.size()) return ifx::fail(IFX_EDIM, "move buffer too small");
  for (size_t i = 0; i < live.size(); ++i) {
    const Move& m = *live[i];
    int64_t* r = out + 5 * i;
    r[0] = m.epoch;
    r[1] = m.kind;
    r[2] = m.dir;
    r[3] = m.dev_slot;
    r[4] = m.host_slot;
  }
  pt->moves.clear();
  return IFX_OK;
}

int ifx_pt_pool_extent(const ifx_pagetable* pt, int64_t* out4) {
  for (int k = 0; k < 2; ++k)
    for (int t = 0; t < 2; ++t) out4[k * 2 + t] = pt->pools[k][t].hwm;
  return IFX_OK;
}

int ifx_pt_slots(ifx_pagetable* pt, int64_t layer, int kind, int64_t start, int64_t end,
                 int32_t* out, int64_t cap, int64_t* first_token, int64_t* n) {
  std::lock_guard<std::mutex> g(pt->mu);
  if (int rc = check_stream(pt, layer, kind)) return rc;
  Stream& st = pt->streams[layer * 2 + kind];
  pt->finalize_epoch();
  *n = 0;
  *first_token = start;
  if (start >= end) return IFX_OK;
  if (st.pages.empty() || start < st.pages.front()->start || end > st.total)
    return ifx::fail(IFX_ERANGE, "slot range outside the stored pages");
  const int64_t s0 = st.pages.front()->start;
  const int64_t k0 = (start - s0) / pt->page_len, k1 = (end - 1 - s0) / pt->page_len + 1;
  *first_token = s0 + k0 * pt->page_len;
  *n = k1 - k0;
  if (out == nullptr) return IFX_OK;
  if (cap < k1 - k0) return ifx::fail(IFX_EDIM, "slot buffer too small");
  for (int64_t k = k0; k < k1; ++k) {
    const Page* p = st.pages[k];
    if (p->slot > INT32_MAX - 1) return ifx::fail(IFX_EDIM, "slot index exceeds int32");
    out[k - k0] = p->tier == 0 ? (int32_t)p->slot : (int32_t)(-1 - p->slot);
  }
  return IFX_OK;
}

}  // extern "C"
