// device_common.cuh -- shared device building blocks for the sm_100a hull.
//
// Everything here is written for Blackwell (sm_100a): 32-wide warps, warp
// vote/shuffle for intra-warp ranks, shared memory for block scans,
// decoupled look-back over relaxed/acquire gpu-scope loads for single-pass
// device-wide scans, and FP64 predicates with explicit round-to-nearest
// intrinsics (no FMA contraction; the library is also compiled -fmad=false).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hull_kernels.cuh"

#define SH_DEV __device__ __forceinline__

// Kernel-boundary probes (tools/prof_once.py with TRACE_ROUND=255): compiled
// in only with -DSHB_PROBES, so the production kernels carry no extra code.
#ifdef SHB_PROBES
#define SHB_PROBE(...) __VA_ARGS__
#else
#define SHB_PROBE(...)
#endif

namespace shb {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// Geometry: geometry.hpp:17-27 restated with explicit RN intrinsics so the
// operation order and rounding are exactly the reference's:
//   cross(a,b,c) = (b.x-a.x)*(c.y-a.y) - (b.y-a.y)*(c.x-a.x)
// The per-edge differences (b.x-a.x), (b.y-a.y) are hoisted: same ops.

struct Edge {
  double ax, ay, ex, ey;
};

SH_DEV Edge make_edge(double ax, double ay, double bx, double by) {
  Edge e;
  e.ax = ax;
  e.ay = ay;
  e.ex = __dsub_rn(bx, ax);
  e.ey = __dsub_rn(by, ay);
  return e;
}

SH_DEV double cross_e(const Edge& e, double px, double py) {
  return __dsub_rn(__dmul_rn(e.ex, __dsub_rn(py, e.ay)), __dmul_rn(e.ey, __dsub_rn(px, e.ax)));
}

// outward_distance (geometry.hpp:25-27): positive iff p is strictly right of a->b
SH_DEV double outward_e(const Edge& e, double px, double py) { return -cross_e(e, px, py); }

// hull.cpp:47-49: double comparisons, so -0.0 == +0.0
SH_DEV bool lex_less(double ax, double ay, double bx, double by) {
  return ax != bx ? ax < bx : ay < by;
}

// ---------------------------------------------------------------------------
// Farthest-point candidate and its total order:
// larger outward distance first; equal distance -> earlier in the
// reference's chain order (lower chain: lex-smallest; upper chain:
// lex-largest); equal coordinates -> lowest id.  Only d > 0 candidates exist
// (a segment is splittable iff its max d > 0, hull.cpp:190), so d == 0 with
// id == NONE is the empty record.


SH_DEV Cand empty_cand() {
  Cand c;
  c.d = 0.0;
  c.x = 0.0;
  c.y = 0.0;
  c.id = NONE;
  c.pos = NONE;
  return c;
}

SH_DEV bool cand_better(const Cand& a, const Cand& b, bool lower) {
  if (a.d != b.d) return a.d > b.d;
  if (a.x != b.x) return lower ? a.x < b.x : a.x > b.x;
  if (a.y != b.y) return lower ? a.y < b.y : a.y > b.y;
  return a.id < b.id;
}

SH_DEV Cand shfl_cand(const Cand& c, int src) {
  Cand o;
  o.d = __shfl_sync(FULL, c.d, src);
  o.x = __shfl_sync(FULL, c.x, src);
  o.y = __shfl_sync(FULL, c.y, src);
  o.id = __shfl_sync(FULL, c.id, src);
  o.pos = __shfl_sync(FULL, c.pos, src);
  return o;
}

SH_DEV Cand shfl_xor_cand(const Cand& c, int m) {
  Cand o;
  o.d = __shfl_xor_sync(FULL, c.d, m);
  o.x = __shfl_xor_sync(FULL, c.x, m);
  o.y = __shfl_xor_sync(FULL, c.y, m);
  o.id = __shfl_xor_sync(FULL, c.id, m);
  o.pos = __shfl_xor_sync(FULL, c.pos, m);
  return o;
}

// Order-preserving integer key of a finite double under FP comparison: -0.0
// and +0.0 compare equal, so both get the key of +0.0.  Integer compares of
// keys are short-latency and branch-free, unlike chains of FP64 compares.
SH_DEV unsigned long long fkey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  b = (b << 1) == 0ull ? 0ull : b;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// cand_better on keys, branch-free (same order: candidates' d are > 0 or the
// empty 0.0, whose bit patterns order like the values)
SH_DEV bool cand_better_k(const Cand& a, const Cand& b, bool lower) {
  const unsigned long long da = (unsigned long long)__double_as_longlong(a.d);
  const unsigned long long db = (unsigned long long)__double_as_longlong(b.d);
  const unsigned long long ax = fkey(a.x), bx = fkey(b.x), ay = fkey(a.y), by = fkey(b.y);
  const bool xl = lower ? ax < bx : ax > bx, yl = lower ? ay < by : ay > by;
  return (da > db) | ((da == db) & (xl | ((ax == bx) & (yl | ((ay == by) & (a.id < b.id))))));
}

// warp-wide minimum of a 64-bit key (two 32-bit redux steps)
SH_DEV unsigned long long warp_min_u64(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_min_sync(FULL, hi);
  const uint32_t ml = __reduce_min_sync(FULL, hi == mh ? (uint32_t)v : 0xFFFFFFFFu);
  return ((unsigned long long)mh << 32) | ml;
}

// CTA-wide lexicographic argmin, per slot, of the key tuples the threads
// offer (smaller is better at every level; invalid offers are skipped):
// one warp min + one shared atomicMin per warp per level, and a barrier per
// level -- no FP64 compare chains, no block-wide shuffles of records.
// s_best[NSL][NK] is scratch; on return win[s] tells whether this thread's
// tuple equals the slot's minimum (several threads only for equal tuples,
// so the last key should make tuples unique) and s_best holds the minima
// (all ~0 for a slot without offers).
template <int NSL, int NK>
SH_DEV void cta_lexmin(const unsigned long long (&key)[NSL][NK], const bool (&valid)[NSL],
                       unsigned long long (*s_best)[NK], bool (&win)[NSL]) {
  __syncthreads();  // s_best may still be read from a previous use
  if (threadIdx.x < NSL * NK) s_best[threadIdx.x / NK][threadIdx.x % NK] = ~0ull;
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NSL; ++s) win[s] = valid[s];
#pragma unroll
  for (int l = 0; l < NK; ++l) {
#pragma unroll
    for (int s = 0; s < NSL; ++s) {
      const unsigned long long v = warp_min_u64(win[s] ? key[s][l] : ~0ull);
      if ((threadIdx.x & 31) == 0 && v != ~0ull) atomicMin(&s_best[s][l], v);
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < NSL; ++s) win[s] = win[s] && key[s][l] == s_best[s][l];
  }
}

// Lexicographic keys (smaller is better) of a farthest-point candidate under
// cand_better: larger d, then the chain's lex direction, then lower id; the
// index makes the tuple unique.
SH_DEV void cand_keys(const Cand& a, bool lower, unsigned long long (&key)[4]) {
  const unsigned long long kx = fkey(a.x), ky = fkey(a.y);
  key[0] = ~(unsigned long long)__double_as_longlong(a.d);
  key[1] = lower ? kx : ~kx;
  key[2] = lower ? ky : ~ky;
  key[3] = ((unsigned long long)a.id << 32) | a.pos;
}

// full-warp argmax of one chain's candidates (all lanes end with the winner)
SH_DEV Cand warp_best(Cand c, bool lower) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const Cand o = shfl_xor_cand(c, m);
    if (cand_better_k(o, c, lower)) c = o;
  }
  return c;
}

// ---------------------------------------------------------------------------
// Memory-model helpers (gpu scope).

SH_DEV unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

SH_DEV void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

SH_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

SH_DEV uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

SH_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (sm_90+): the next kernel in the stream may be
// scheduled now / this kernel waits for its predecessor's completion + memory.
SH_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
SH_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// The value, hidden from the optimiser: keeps it from unswitching code on a
// data-dependent index with few possible values (e.g. computing a point's
// route for both chains and selecting afterwards).
SH_DEV uint32_t opaque_u32(uint32_t v) {
  asm("" : "+r"(v));
  return v;
}

SH_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// Farthest-point slot {dbits, SlotRec}: a 64-bit atomicMax on the distance
// bits (positive doubles order like their bit patterns) filters contention;
// only contenders that reach the running maximum take the record's lock and
// apply the full comparator.  Works on global and shared slots (generic
// atomics).  The lock loop keeps the critical section inside the loop body,
// which is starvation-free under independent thread scheduling even when two
// lanes of one warp contend.
// SHARED: the record lives in shared memory (CTA-scope ordering suffices);
// otherwise gpu scope with acquire/release fences (not the sequentially
// consistent __threadfence, which also invalidates L1).
SH_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

SH_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// lock word: acquire-CAS to take it, release-store to drop it (no full
// fences: the critical section only touches the record itself)
template <bool SHARED>
SH_DEV bool lock_try(uint32_t* l) {
  uint32_t old;
  if (SHARED)
    asm volatile("atom.acquire.cta.shared::cta.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "r"(smem_u32(l)) : "memory");
  else
    asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(l) : "memory");
  return old == 0u;
}
template <bool SHARED>
SH_DEV void lock_release(uint32_t* l) {
  if (SHARED)
    asm volatile("st.release.cta.shared::cta.u32 [%0], 0;" ::"r"(smem_u32(l)) : "memory");
  else
    asm volatile("st.release.gpu.global.u32 [%0], 0;" ::"l"(l) : "memory");
}

template <bool SHARED>
SH_DEV void rec_update(SlotRec* rec, const Cand& c, bool lower) {
  bool done = false;
  while (!done) {
    if (lock_try<SHARED>(&rec->lock)) {
      volatile SlotRec* v = rec;
      Cand o;
      o.id = v->id;
      o.d = v->d;
      o.x = v->x;
      o.y = v->y;
      if (o.id == NONE || cand_better(c, o, lower)) {
        v->d = c.d;
        v->x = c.x;
        v->y = c.y;
        v->id = c.id;
      }
      lock_release<SHARED>(&rec->lock);
      done = true;
    }
  }
}

// relaxed gpu-scope atomic add issued from one lane: inline PTX so the
// compiler cannot turn it into a warp-aggregated atomic whose result is
// shuffled (and therefore waited for) right away
// shared-memory atomic add from one lane: inline PTX, because the compiler
// expands `if (lane == 0) atomicAdd(...)` into its warp-aggregation sequence
// (vote, find-leader, popc, shuffle: ~15 instructions per call)
SH_DEV uint32_t atom_add_shared(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

SH_DEV uint32_t atom_add_relaxed(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// (a CTA's shared slots keep only the high word of the distance bits: a
// positive double's high word orders like the value, and 32-bit shared max is
// a native atomic where the 64-bit one is a compare-and-swap loop)
SH_DEV void rec_clear(uint32_t* dhi, SlotRec* rec) {
  *dhi = 0u;
  rec->d = 0.0;
  rec->x = 0.0;
  rec->y = 0.0;
  rec->id = NONE;
  rec->lock = 0u;
}

SH_DEV void rec_clear(unsigned long long* dbits, SlotRec* rec) {
  *dbits = 0ull;
  rec->d = 0.0;
  rec->x = 0.0;
  rec->y = 0.0;
  rec->id = NONE;
  rec->lock = 0u;
}

// ---------------------------------------------------------------------------
// Grid barrier for a cooperative launch (all CTAs co-resident).  The
// generation word is read before arriving, so a fast CTA re-entering the
// next barrier cannot be confused with the current one.
SH_DEV void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

SH_DEV void grid_barrier(uint32_t* count, uint32_t* gen, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t g;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    fence_acq_rel_gpu();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *(volatile uint32_t*)count = 0u;
      fence_acq_rel_gpu();
      st_release_u32(gen, g + 1);
    } else {
      uint32_t v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
        if (v != g) break;
        __nanosleep(20);
      }
    }
    fence_acq_rel_gpu();
  }
  __syncthreads();
}

// Grid barrier on a monotone arrival counter: each participating CTA adds 1
// (release) and waits until the counter reaches `target` (acquire), the
// running total of participants over all barriers so far -- the last arrival
// completes the barrier itself, with no reset and no second word to publish.
SH_DEV void grid_barrier_ctr(unsigned long long* ctr, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single-pass device-wide exclusive scan of per-tile
// counts).  Status words pack (epoch:30 | flag:2) << 32 | value:32; a word
// whose epoch differs from the launch's is "not yet published", so the
// status array never needs clearing between launches.

constexpr uint32_t LB_AGG = 1u, LB_PRE = 2u;

SH_DEV unsigned long long lb_pack(uint32_t epoch, uint32_t flag, uint32_t value) {
  return ((unsigned long long)((epoch << 2) | flag) << 32) | value;
}

// Executed by one full warp.  Returns the exclusive prefix of `tile`.
SH_DEV uint32_t lookback_warp(unsigned long long* status, uint32_t tile, uint32_t aggregate,
                              uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status + 0, lb_pack(epoch, LB_PRE, aggregate));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, lb_pack(epoch, LB_AGG, aggregate));
  uint32_t exclusive = 0;
  long long idx = (long long)tile - 1;
  while (true) {
    const long long t = idx - lane;
    uint32_t flag = 0, val = 0;
    if (t >= 0) {
      unsigned long long w;
      do {
        w = ld_relaxed_u64(status + t);
      } while ((uint32_t)(w >> 34) != epoch || ((uint32_t)(w >> 32) & 3u) == 0);
      flag = (uint32_t)(w >> 32) & 3u;
      val = (uint32_t)w;
    }
    __syncwarp();
    const unsigned pmask = __ballot_sync(FULL, flag == LB_PRE);
    uint32_t contrib;
    if (pmask) {
      const int first = __ffs(pmask) - 1;
      contrib = lane <= first ? val : 0u;
    } else {
      contrib = val;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) contrib += __shfl_xor_sync(FULL, contrib, m);
    exclusive += contrib;
    if (pmask) break;
    idx -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, lb_pack(epoch, LB_PRE, exclusive + aggregate));
  return exclusive;
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024).
// `warp_sums` must hold blockDim.x/32 + 1 entries.  Returns the exclusive
// prefix; *total receives the block total.  Contains __syncthreads.
SH_DEV uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nwarps ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nwarps) warp_sums[lane] = w;  // inclusive warp prefix
    if (lane == nwarps - 1) warp_sums[nwarps] = w;
  }
  __syncthreads();
  const uint32_t before = warp == 0 ? 0u : warp_sums[warp - 1];
  *total = warp_sums[nwarps];
  const uint32_t r = before + x - v;
  __syncthreads();
  return r;
}

}  // namespace shb

// ---------------------------------------------------------------------------
// TMA bulk-copy ring (sm_90+/sm_100a `cp.async.bulk` + mbarrier transaction
// counts).  One elected thread streams fixed-size tiles of the SoA input into
// NS shared-memory stages; every thread consumes a stage after waiting on its
// mbarrier phase.  The memory system always has NS-1 tiles in flight per CTA
// regardless of how long the consumers compute, which is what the latency-
// bound register-load versions of K1/K2/K3 lacked (ncu: 0.5-0.7 eligible
// warps per scheduler at 25-37% occupancy).
namespace shb {


SH_DEV void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

SH_DEV void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

SH_DEV void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SH_DEV void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

SH_DEV void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

SH_DEV void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Ring of NS stages of T points (x, y f64 and optionally ids u32).
// T % 64 == 0; the global arrays must be 16-byte aligned (the host stages
// unaligned inputs).  A tile's last (cnt % 4) points are not copied (bulk
// copies move multiples of 16 bytes); consumers read those from global.
template <int T, int NS, bool IDS, int AUX = 0, int NCW = 15>
struct TileRing {
  // AUX: bytes per 64-point chunk of an optional side stream (K3: the chain bits)
  static constexpr size_t kAuxBytes = (size_t)(T / 64) * AUX;
  static constexpr size_t kStageBytes = (size_t)T * (16 + (IDS ? 4 : 0)) + kAuxBytes;
  static constexpr size_t kBytes = NS * kStageBytes + 2 * NS * sizeof(unsigned long long);
  double* xs;                 // [NS][T]
  double* ys;                 // [NS][T]
  uint32_t* is;               // [NS][T] when IDS
  unsigned char* aux;         // [NS][kAuxBytes]
  unsigned long long* bar;    // [NS] full: the stage's bytes landed
  unsigned long long* ebar;   // [NS] empty: every consumer warp is done with it

  SH_DEV void carve(unsigned char* base) {
    xs = reinterpret_cast<double*>(base);
    ys = xs + NS * T;
    is = reinterpret_cast<uint32_t*>(ys + NS * T);
    aux = reinterpret_cast<unsigned char*>(is + (IDS ? NS * T : 0));
    bar = reinterpret_cast<unsigned long long*>(base + NS * kStageBytes);
    ebar = bar + NS;
  }
  SH_DEV void init() {  // thread 0, followed by __syncthreads by the caller
    for (int s = 0; s < NS; ++s) {
      mbar_init(bar + s, 1);
      mbar_init(ebar + s, NCW);
    }
    mbar_fence_init();
  }
  // thread 0: stream points [first, first + cnt) into stage s
  SH_DEV void issue(int s, const double* X, const double* Y, const uint32_t* I, uint32_t first,
                    uint32_t cnt, const unsigned char* A = nullptr, bool with_aux = true) {
    const uint32_t c4 = cnt & ~3u;
    const uint32_t ab = AUX ? ((cnt + 63) / 64) * AUX : 0u;
    if (c4 == 0 && ab == 0) {  // nothing to copy: complete the phase with a plain arrival
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar + s))
                   : "memory");
      return;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // stage was read by threads
    mbar_expect_tx(bar + s, c4 * (16u + (IDS ? 4u : 0u)) + ab);
    if (c4) {
      tma_load_1d(xs + s * T, X + first, c4 * 8u, bar + s);
      tma_load_1d(ys + s * T, Y + first, c4 * 8u, bar + s);
      if (IDS) tma_load_1d(is + s * T, I + first, c4 * 4u, bar + s);
    }
    if (ab && with_aux) tma_load_1d(aux + s * kAuxBytes, A + (size_t)(first / 64) * AUX, ab, bar + s);
  }
  // the aux bytes of a stage whose point bytes (and expected count) were issued
  SH_DEV void issue_aux(int s, uint32_t first, uint32_t cnt, const unsigned char* A) {
    const uint32_t ab = AUX ? ((cnt + 63) / 64) * AUX : 0u;
    if (ab) tma_load_1d(aux + s * kAuxBytes, A + (size_t)(first / 64) * AUX, ab, bar + s);
  }
  SH_DEV void wait(int s, uint32_t parity) { mbar_wait(bar + s, parity); }
  // one arrival per warp when the warp no longer reads stage s
  SH_DEV void release(int s) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(ebar + s);
  }
};

}  // namespace shb

namespace shb {

// The tiles this CTA streams: b, b+G, ... (mapped to ntiles-1-t when `reverse`).
template <int T>
struct TileWalk {
  uint32_t ntiles, mine;
  bool reverse;
  SH_DEV TileWalk(uint32_t n, bool rev) : reverse(rev) {
    ntiles = (n + T - 1) / T;
    mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  }
  SH_DEV uint32_t first(uint32_t k) const {
    const uint32_t t = blockIdx.x + k * gridDim.x;
    return (reverse ? ntiles - 1 - t : t) * T;
  }
};

// Producer lane, before the kernel's griddepcontrol.wait: start the ring on
// the first min(NS, mine) tiles of inputs that do not depend on the previous
// kernel (the point arrays; with_aux = false leaves out the aux bytes, which
// stream_input issues for these stages once the wait returned).  Returns the
// number of tiles started; every thread computes the same value.
template <int T, int NS, bool IDS, int AUX, int NCW>
SH_DEV uint32_t stream_prefetch(TileRing<T, NS, IDS, AUX, NCW>& R, uint32_t n, const double* X,
                                const double* Y, const uint32_t* I, bool reverse, bool with_aux) {
  const TileWalk<T> w(n, reverse);
#ifndef SHB_PREFETCH
#define SHB_PREFETCH 16
#endif
  // stages started before griddepcontrol.wait: they overlap the wait, but a
  // full ring also queues ahead of the partials the prologue must read next
  const uint32_t pre = min(w.mine, (uint32_t)min(NS, SHB_PREFETCH));
  if ((int)(threadIdx.x >> 5) == NCW && (threadIdx.x & 31) == 0) {
    for (uint32_t k = 0; k < pre; ++k) {
      const uint32_t first = w.first(k);
      R.issue((int)k, X, Y, I, first, min((uint32_t)T, n - first), nullptr, with_aux);
    }
  }
  return pre;
}

// A CTA that started tiles but leaves early waits for their bulk copies.
template <int T, int NS, bool IDS, int AUX, int NCW>
SH_DEV void stream_drain(TileRing<T, NS, IDS, AUX, NCW>& R, uint32_t pre) {
  if (threadIdx.x == 0)
    for (uint32_t k = 0; k < pre; ++k) R.wait((int)k, 0u);
  __syncthreads();
}

// As stream_drain, for stages prefetched without their aux bytes: those are
// issued first (the stage's expected byte count includes them).
template <int T, int NS, bool IDS, int AUX, int NCW>
SH_DEV void stream_drain_points(TileRing<T, NS, IDS, AUX, NCW>& R, uint32_t pre, uint32_t n,
                                const unsigned char* A) {
  const TileWalk<T> w(n, false);
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < pre; ++k) {
      const uint32_t first = w.first(k);
      R.issue_aux((int)k, first, min((uint32_t)T, n - first), A);
    }
    for (uint32_t k = 0; k < pre; ++k) R.wait((int)k, 0u);
  }
  __syncthreads();
}

// Streams this CTA's share of the input through the ring: tiles b, b+G, ...
// (mapped to ntiles-1-t when `reverse`), calling body(stage, first, cnt) in
// the NCW consumer warps for each tile after its bytes landed.  Warp
// NCW is a dedicated producer: it refills a stage as soon as every
// consumer warp released it (empty mbarrier), so no consumer ever waits for
// another consumer and no CTA-wide barrier is needed per tile.  `pre` tiles
// were already started by stream_prefetch (without their aux bytes when
// aux_pending).  The caller initialised the ring (+ __syncthreads); a
// __syncthreads ends the stream.
template <int T, int NS, bool IDS, int AUX, int NCW, class Body>
SH_DEV void stream_input(TileRing<T, NS, IDS, AUX, NCW>& R, uint32_t n, const double* X,
                         const double* Y, const uint32_t* I, const unsigned char* A, bool reverse,
                         const Body& body, uint32_t pre = 0, bool aux_pending = false) {
  const TileWalk<T> w(n, reverse);
  const uint32_t mine = w.mine;
  if ((int)(threadIdx.x >> 5) == NCW) {  // producer warp
    if ((threadIdx.x & 31) == 0) {
      for (uint32_t k = 0; k < pre && aux_pending; ++k) {
        const uint32_t first = w.first(k);
        R.issue_aux((int)k, first, min((uint32_t)T, n - first), A);
      }
      for (uint32_t k = pre; k < mine; ++k) {
        const int s = (int)(k % NS);
        if (k >= (uint32_t)NS) mbar_wait(R.ebar + s, ((k / NS) - 1) & 1u);
        const uint32_t first = w.first(k);
        R.issue(s, X, Y, I, first, min((uint32_t)T, n - first), A);
      }
    }
  } else {
    for (uint32_t k = 0; k < mine; ++k) {
      const int s = (int)(k % NS);
      R.wait(s, (k / NS) & 1u);
      const uint32_t first = w.first(k);
      body(s, first, min((uint32_t)T, n - first));
      R.release(s);
    }
  }
  __syncthreads();
}

}  // namespace shb
