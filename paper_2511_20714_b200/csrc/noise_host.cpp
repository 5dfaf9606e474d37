// noise_host.cpp — multi-threaded, bit-exact host generator of the per-block initial noise
// of the generate loop: np.random.default_rng([seed, chunk]).standard_normal((T, D))
// .astype(np.float32)  (reference engine.py:280-282).
//
// The reference draws T*D float64 normals from one PCG64 (XSL-RR 128/64) stream with
// numpy's 256-layer ziggurat, sequentially: ~0.1-0.2 s per c2 block on one core, which is
// longer than the GPU needs for the whole block. Dependency, pinned: numpy 2.3 — we link
// its own `random_standard_normal` (numpy/random/lib/libnpyrandom.a, the C routine behind
// Generator.standard_normal) so the ziggurat tables and rejection logic are numpy's, and
// drive it with our PCG64 implementation, which can jump ahead (LCG advance).
//
// Parallel parse of one sequential stream. A normal consumes a variable number of raw
// 64-bit draws (1 in ~99% of cases, more on ziggurat rejection), so the raw stream is cut
// into T chunks [P_k, P_{k+1}) and thread k parses from P_k as if a normal started there,
// recording the raw start position of its first normals. Parses are self-synchronising: the
// true parse enters chunk k at E_{k-1} (the end of chunk k-1's last normal, which is >= P_k)
// and, after at most a few normals, lands on a position thread k also started a normal at;
// from there both produce the same normals. A sequential stitch walks the chunks, re-parses
// the few normals before the meeting point, and the outputs are concatenated. Every value
// is produced by the same numpy routine from the same raw draws, hence bit-identical.
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <thread>
#include <vector>

#include "common_host.h"
#include "ifx_abi.h"

extern "C" {
// numpy/random/bitgen.h (numpy 2.3) — layout of the generator handle numpy's
// distributions take.
typedef struct ifx_np_bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} ifx_np_bitgen;
double random_standard_normal(ifx_np_bitgen* bitgen_state);  // libnpyrandom.a
}

namespace {

typedef unsigned __int128 u128;

const u128 kMult = (static_cast<u128>(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

struct Pcg64 {
  u128 state, inc;
  uint64_t pos;  // raw draws consumed since the generator's initial state
};

inline uint64_t pcg_next(void* p) {
  Pcg64* g = static_cast<Pcg64*>(p);
  g->state = g->state * kMult + g->inc;
  g->pos++;
  const uint64_t hi = static_cast<uint64_t>(g->state >> 64), lo = static_cast<uint64_t>(g->state);
  const unsigned rot = static_cast<unsigned>(g->state >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
uint32_t pcg_next32(void* p) { return static_cast<uint32_t>(pcg_next(p)); }  // unused by normals
double pcg_next_double(void* p) { return static_cast<double>(pcg_next(p) >> 11) * (1.0 / 9007199254740992.0); }

// state after `delta` more LCG steps (O(log delta) multiplies)
u128 advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kMult, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

struct Stream {
  Pcg64 g;
  ifx_np_bitgen bg;
  Stream(u128 s0, u128 inc, uint64_t at) {
    g.state = advance(s0, inc, at);
    g.inc = inc;
    g.pos = at;
    bg.state = &g;
    bg.next_uint64 = pcg_next;
    bg.next_uint32 = pcg_next32;
    bg.next_double = pcg_next_double;
    bg.next_raw = pcg_next;
  }
  float normal() { return static_cast<float>(random_standard_normal(&bg)); }
};

constexpr int kHead = 64;  // start positions recorded per chunk for the stitch

struct Chunk {
  uint64_t p0, p1;                // raw range whose positions may start a normal
  std::vector<float> v;           // speculative normals
  uint64_t starts[kHead];         // raw start of v[0..kHead)
  uint64_t end;                   // raw position after the last normal
  // stitch result
  std::vector<float> fix;         // true normals before the meeting point
  size_t skip = 0;                // v[skip..] are true normals
  bool synced = false;
};

void parse(Chunk& c, u128 s0, u128 inc) {
  Stream st(s0, inc, c.p0);
  c.v.clear();
  c.v.reserve(static_cast<size_t>(c.p1 - c.p0) + 16);
  while (st.g.pos < c.p1) {
    if (c.v.size() < static_cast<size_t>(kHead)) c.starts[c.v.size()] = st.g.pos;
    c.v.push_back(st.normal());
  }
  c.end = st.g.pos;
}

std::mutex g_mu;             // one call at a time reuses the chunk buffers
std::vector<Chunk> g_chunks;

}  // namespace

extern "C" int ifx_noise_normal_f32(const uint64_t pcg_state[4], int64_t n, float* out,
                                    int threads) {
  if (n < 0 || (n > 0 && out == nullptr) || pcg_state == nullptr)
    return ifx::fail(IFX_EDIM, "noise: bad arguments");
  if (n == 0) return IFX_OK;
  const u128 s0 = (static_cast<u128>(pcg_state[0]) << 64) | pcg_state[1];
  const u128 inc = (static_cast<u128>(pcg_state[2]) << 64) | pcg_state[3];
  int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  T = std::max(1, std::min<int>(T, static_cast<int>(std::max<int64_t>(1, n / 65536))));
  if (T == 1) {
    Stream st(s0, inc, 0);
    for (int64_t i = 0; i < n; ++i) out[i] = st.normal();
    return IFX_OK;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_chunks.resize(T);
  // ~1.2% of normals take extra draws; cover n normals with ~2% spare raw positions
  const uint64_t raw = static_cast<uint64_t>(n) + static_cast<uint64_t>(n) / 50 + 1024;
  const uint64_t per = (raw + T - 1) / T;
  for (int k = 0; k < T; ++k) {
    g_chunks[k].p0 = per * k;
    g_chunks[k].p1 = per * (k + 1);
  }
  {
    std::vector<std::thread> pool;
    for (int k = 1; k < T; ++k) pool.emplace_back(parse, std::ref(g_chunks[k]), s0, inc);
    parse(g_chunks[0], s0, inc);
    for (auto& t : pool) t.join();
  }
  // stitch: chunk 0 starts at raw 0, the true start
  g_chunks[0].skip = 0;
  g_chunks[0].fix.clear();
  g_chunks[0].synced = true;
  uint64_t entry = g_chunks[0].end;
  for (int k = 1; k < T; ++k) {
    Chunk& c = g_chunks[k];
    c.fix.clear();
    c.synced = false;
    const size_t nh = std::min(c.v.size(), static_cast<size_t>(kHead));
    Stream st(s0, inc, entry);
    while (st.g.pos < c.p1) {
      const uint64_t* hit = std::lower_bound(c.starts, c.starts + nh, st.g.pos);
      if (hit != c.starts + nh && *hit == st.g.pos) {
        c.skip = static_cast<size_t>(hit - c.starts);
        c.synced = true;
        break;
      }
      c.fix.push_back(st.normal());
    }
    if (!c.synced) c.skip = c.v.size();  // never met: the re-parse produced the whole chunk
    entry = c.synced ? c.end : st.g.pos;
  }
  // output offsets, parallel copy, sequential tail if the spare raw range fell short
  std::vector<int64_t> off(T + 1, 0);
  for (int k = 0; k < T; ++k)
    off[k + 1] = off[k] + static_cast<int64_t>(g_chunks[k].fix.size() + g_chunks[k].v.size() - g_chunks[k].skip);
  auto emit = [&](int k) {
    const Chunk& c = g_chunks[k];
    int64_t o = off[k];
    for (size_t i = 0; i < c.fix.size() && o < n; ++i) out[o++] = c.fix[i];
    if (o < n) {
      const size_t cnt = std::min(c.v.size() - c.skip, static_cast<size_t>(n - o));
      std::copy(c.v.begin() + c.skip, c.v.begin() + c.skip + cnt, out + o);
    }
  };
  {
    std::vector<std::thread> pool;
    for (int k = 1; k < T; ++k) pool.emplace_back(emit, k);
    emit(0);
    for (auto& t : pool) t.join();
  }
  if (off[T] < n) {
    Stream st(s0, inc, entry);
    for (int64_t i = off[T]; i < n; ++i) out[i] = st.normal();
  }
  return IFX_OK;
}
