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

#define SH_DEV __device__ __forceinline__

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

struct Cand {
  double d, x, y;
  uint32_t id, pos;
};

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

// full-warp argmax of one chain's candidates (all lanes end with the winner)
SH_DEV Cand warp_best(Cand c, bool lower) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const Cand o = shfl_xor_cand(c, m);
    if (cand_better(o, c, lower)) c = o;
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

SH_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// Farthest-point slot {dbits, win}: a 64-bit atomicMax on the distance bits
// (positive doubles order like their bit patterns) filters contention, then a
// CAS loop on the winner's position applies the full comparator.  The
// incumbent's distance is recomputed from its stored coordinates against the
// slot's edge -- every contender of a slot belongs to the same new segment,
// so the caller's own edge IS the slot's edge and the recomputed value is
// bit-identical to the one the incumbent offered.
//   LD : functor (pos) -> (x, y, id) reading the array the positions index
// Callers must have made the candidate's own row visible (__threadfence)
// before offering.  Works on global and on shared slots (generic atomics).
template <class LD>
SH_DEV void slot_offer(unsigned long long* dbits, uint32_t* win, const Cand& c, bool lower,
                       const Edge& e, const LD& ld) {
  const unsigned long long mine = (unsigned long long)__double_as_longlong(c.d);
  if (mine < *(volatile unsigned long long*)dbits) return;
  const unsigned long long old = atomicMax(dbits, mine);
  if (mine < old) return;
  uint32_t cur = *(volatile uint32_t*)win;
  while (true) {
    if (cur != NONE) {
      Cand o;
      ld(cur, o.x, o.y, o.id);
      o.d = outward_e(e, o.x, o.y);
      o.pos = cur;
      if (!cand_better(c, o, lower)) return;
    }
    const uint32_t prev = atomicCAS(win, cur, c.pos);
    if (prev == cur) return;
    cur = prev;
  }
}

// (x, y, id) of a position in SoA input arrays (ids null => id == position)
struct LoadSoA {
  const double* x;
  const double* y;
  const uint32_t* id;
  SH_DEV void operator()(uint32_t p, double& ox, double& oy, uint32_t& oid) const {
    ox = __ldcg(x + p);
    oy = __ldcg(y + p);
    oid = id ? __ldcg(id + p) : p;
  }
};

// (x, y, id) of a position in a live set
struct LoadLive {
  const double2* xy;
  const uint2* is;
  SH_DEV void operator()(uint32_t p, double& ox, double& oy, uint32_t& oid) const {
    const double2 v = __ldcg(xy + p);
    ox = v.x;
    oy = v.y;
    oid = __ldcg(&is[p].x);
  }
};

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
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *(volatile uint32_t*)count = 0u;
      __threadfence();
      st_release_u32(gen, g + 1);
    } else {
      uint32_t v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
        if (v != g) break;
        __nanosleep(20);
      }
    }
    __threadfence();
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
