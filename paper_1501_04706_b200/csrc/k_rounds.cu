// k_rounds.cu -- the refinement rounds of the sm_100a QuickHull
// (hull.cpp:264-282; SURVEY.md section 7.3 "lex routing").
//
//   K3 k3_round1  round 1 straight from the input + K2's class bits: route
//                 every member of the two chains to the A->C or C->B edge of
//                 its chain's farthest point C, keep iff strictly outside
//                 (hull.cpp:196-201), compact the survivors into the live set
//                 and fuse the farthest-point search of round 2
//   KR k_rounds   every later round in ONE persistent cooperative launch:
//                 per round a segment-table phase (rebuilt redundantly in each
//                 CTA's shared memory for small tables, a grid-wide scan for
//                 large ones), a point phase (route, keep, compact, offer) and
//                 one grid barrier; once the live set is small, CTA 0 finishes
//                 the remaining rounds alone with __syncthreads only
//   K5 k5_emit    copy the final heads (the hull, CCW from P0) to the caller
//
// Compaction is order-free: the hull and the per-round stats depend only on
// segment membership and on the total order of the farthest-point
// comparator, never on where a survivor lands, so every tile reserves its
// output range with ONE atomicAdd and no scan/look-back is needed.
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

// ===========================================================================
// shared pieces
// ===========================================================================

SH_DEV Route ldcg_route(const Route* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldcg(q), b = __ldcg(q + 1), cc = __ldcg(q + 2);
  const uint4 t = __ldcg(reinterpret_cast<const uint4*>(q + 3));
  Route r;
  r.ax = a.x; r.ay = a.y; r.cx = b.x; r.cy = b.y; r.bx = cc.x; r.by = cc.y;
  r.cid = t.x; r.ns = t.y; r.flags = t.z; r.pad = t.w;
  return r;
}

// Route one member (x, y, id) of old segment r:
//   left = lower ? lex(p) < lex(C) : lex(C) < lex(p)
//   d    = outward_distance(left ? (A, C) : (C, B), p); keep iff d > 0
// Returns false when the member is dropped outright (segment not splittable,
// or p is C itself).
SH_DEV bool route_point(const Route& r, double x, double y, uint32_t id, double& d,
                        uint32_t& nseg, bool& left) {
  if (!(r.flags & RT_SPLIT) || id == r.cid) return false;
  const bool lower = r.flags & RT_LOWER;
  left = lower ? lex_less(x, y, r.cx, r.cy) : lex_less(r.cx, r.cy, x, y);
  const Edge e = left ? make_edge(r.ax, r.ay, r.cx, r.cy) : make_edge(r.cx, r.cy, r.bx, r.by);
  d = outward_e(e, x, y);
  nseg = r.ns + (left ? 0u : 1u);
  return d > 0.0;  // hull.cpp:199 keep iff d > 0 (heads are not members)
}

SH_DEV Edge route_edge(const Route& r, bool left) {
  return left ? make_edge(r.ax, r.ay, r.cx, r.cy) : make_edge(r.cx, r.cy, r.bx, r.by);
}

// Block-contiguous output reservation for one tile.  keepm bit j says point
// j of this thread survives; positions are written to pos[j].  Contains two
// __syncthreads.  One atomicAdd per tile on the round's survivor counter.
template <int NP, int NW>
SH_DEV void reserve_tile(uint32_t keepm, uint32_t (&pos)[NP], uint32_t* counter,
                         uint32_t* s_wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bal[NP];
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    bal[j] = __ballot_sync(FULL, (keepm >> j) & 1u);
    tot += __popc(bal[j]);
  }
  if (lane == 0) s_wcnt[warp] = tot;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < NW ? s_wcnt[lane] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t all = __shfl_sync(FULL, incl, 31);
    uint32_t base = 0;
    if (lane == 0 && all) base = atomicAdd(counter, all);
    base = __shfl_sync(FULL, base, 0);
    if (lane < NW) s_wcnt[lane] = base + incl - v;
  }
  __syncthreads();
  uint32_t off = s_wcnt[warp];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    pos[j] = off + __popc(bal[j] & lt);
    off += __popc(bal[j]);
  }
}

// Shared-memory farthest slots of one CTA (small next tables).
//   phase A (per kept point): atomicMax on the distance bits
//   __syncthreads (all of the tile's rows are now visible block-wide)
//   phase B (points at the block maximum): CAS on the winner with the full
//   comparator, incumbent read back from the live set
// then, once per round, flush_slots() offers each CTA record to the global slot.
template <int NP, class EdgeOf>
SH_DEV void offer_tile_smem(unsigned long long* s_db, uint32_t* s_win, uint32_t keepm,
                            const double (&px)[NP], const double (&py)[NP],
                            const double (&pd)[NP], const uint32_t (&pid)[NP],
                            const uint32_t (&pseg)[NP], const uint32_t (&pos)[NP],
                            const EdgeOf& edge_of, uint32_t lowmask, const LoadLive& ld) {
  uint32_t candm = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if ((keepm >> j) & 1u) {
      const unsigned long long db = (unsigned long long)__double_as_longlong(pd[j]);
      if (db >= *(volatile unsigned long long*)&s_db[pseg[j]]) {
        const unsigned long long old = atomicMax(&s_db[pseg[j]], db);
        if (db >= old) candm |= 1u << j;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if ((candm >> j) & 1u) {
      const unsigned long long db = (unsigned long long)__double_as_longlong(pd[j]);
      if (db == *(volatile unsigned long long*)&s_db[pseg[j]]) {
        Cand me;
        me.d = pd[j]; me.x = px[j]; me.y = py[j]; me.id = pid[j]; me.pos = pos[j];
        slot_offer(&s_db[pseg[j]], &s_win[pseg[j]], me, (lowmask >> j) & 1u, edge_of(j), ld);
      }
    }
  }
}

// ===========================================================================
// K3: round 1 straight from the input
// ===========================================================================

constexpr int K3_U = 4;                   // 64-point chunks per warp per tile
constexpr int K3_NP = 2 * K3_U;           // points per thread per tile
constexpr int K3_CHUNKS = WARPS * K3_U;   // chunks per tile (2048 points)

template <bool VEC>
SH_DEV double2 ldcs_pair(const double* __restrict__ a, uint32_t q) {
  if (VEC) return __ldcs(reinterpret_cast<const double2*>(a) + q);
  return make_double2(__ldcs(a + 2 * q), __ldcs(a + 2 * q + 1));
}

template <bool IDS, bool VEC>
__global__ void __launch_bounds__(TPB) k3_round1(Bufs B) {
  __shared__ Route s_rt[2];
  __shared__ unsigned long long s_db[4];
  __shared__ uint32_t s_win[4], s_from[4];
  __shared__ uint32_t s_wcnt[WARPS];
  __shared__ uint32_t s_Sn, s_Slon;
  __shared__ int s_last;
  Ctl* c = B.ctl;
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  double2* Oxy = B.Lxy[1];
  uint2* Ois = B.Lis[1];

  // ---- table phase (S = 2: the lower chain P0->Pr and the upper chain Pr->P0) ----
  if (threadIdx.x == 0) {
    uint32_t ns = 0, Slon = 1;
    for (int s = 0; s < 2; ++s) {
      const uint32_t w = __ldcg(B.Sw[0] + s);
      const bool split = w != NONE;
      Route r;
      r.ax = __ldcg(B.Tx[0] + s);
      r.ay = __ldcg(B.Ty[0] + s);
      r.bx = __ldcg(B.Tx[0] + (s ^ 1));
      r.by = __ldcg(B.Ty[0] + (s ^ 1));
      r.cx = split ? __ldcg(X + w) : 0.0;
      r.cy = split ? __ldcg(Y + w) : 0.0;
      r.cid = split ? (I ? __ldcg(I + w) : w) : NONE;
      r.ns = ns;
      r.flags = (split ? RT_SPLIT : 0u) | (s == 0 ? RT_LOWER : 0u);
      r.pad = 0;
      s_rt[s] = r;
      s_from[ns] = s;
      if (blockIdx.x == 0) {
        B.Tx[1][ns] = r.ax;
        B.Ty[1][ns] = r.ay;
        B.Tid[1][ns] = __ldcg(B.Tid[0] + s);
      }
      if (split) {
        s_from[ns + 1] = s | 0x80000000u;
        if (blockIdx.x == 0) {
          B.Tx[1][ns + 1] = r.cx;
          B.Ty[1][ns + 1] = r.cy;
          B.Tid[1][ns + 1] = r.cid;
        }
      }
      ns += split ? 2 : 1;
      if (s == 0) Slon = ns;
    }
    s_Sn = ns;
    s_Slon = Slon;
    for (int t = 0; t < 4; ++t) {
      s_db[t] = 0ull;
      s_win[t] = NONE;
    }
    if (blockIdx.x == 0) {  // clear round 2's slots and counter
      for (int t = 0; t < 8; ++t) {
        B.Sd[2][t] = 0ull;
        B.Sw[2][t] = NONE;
      }
      c->out_cnt[2] = 0;
    }
  }
  __syncthreads();
  const Route rlo = s_rt[0], rup = s_rt[1];
  const uint32_t Sn = s_Sn, Slon = s_Slon;
  const LoadLive ld{Oxy, Ois};

  // ---- point phase ----
  const uint32_t nchunks = (n + 63) >> 6;
  const uint32_t ntiles = (nchunks + K3_CHUNKS - 1) / K3_CHUNKS;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    double px[K3_NP], py[K3_NP], pd[K3_NP];
    uint32_t pid[K3_NP], pseg[K3_NP], pos[K3_NP];
    uint32_t keepm = 0, lowm = 0, leftm = 0;
    uint4 bits[K3_U];
#pragma unroll
    for (int u = 0; u < K3_U; ++u) {
      const uint32_t ch = tile * K3_CHUNKS + u * WARPS + warp;
      bits[u] = make_uint4(0u, 0u, 0u, 0u);
      double2 xv = make_double2(0.0, 0.0), yv = xv;
      if (ch < nchunks) {
        bits[u] = __ldg(B.bits + ch);
        const uint32_t q = ch * 32 + lane;
        if (2 * q + 1 < n) {
          xv = ldcs_pair<VEC>(X, q);
          yv = ldcs_pair<VEC>(Y, q);
        } else if (2 * q < n) {
          xv.x = __ldcs(X + 2 * q);
          yv.x = __ldcs(Y + 2 * q);
        }
      }
      px[2 * u] = xv.x; px[2 * u + 1] = xv.y;
      py[2 * u] = yv.x; py[2 * u + 1] = yv.y;
    }
#pragma unroll
    for (int u = 0; u < K3_U; ++u) {
      const uint32_t ch = tile * K3_CHUNKS + u * WARPS + warp;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * u + h;
        const uint32_t lw = ((h ? bits[u].y : bits[u].x) >> lane) & 1u;
        const uint32_t uw = ((h ? bits[u].w : bits[u].z) >> lane) & 1u;
        pd[j] = 0.0;
        pseg[j] = 0;
        const uint32_t i = ch * 64 + 2 * lane + h;
        pid[j] = 0;
        if (lw | uw) {
          pid[j] = IDS ? __ldg(I + i) : i;
          const Route& r = lw ? rlo : rup;
          bool left = false;
          if (route_point(r, px[j], py[j], pid[j], pd[j], pseg[j], left)) {
            keepm |= 1u << j;
            if (left) leftm |= 1u << j;
            if (lw) lowm |= 1u << j;
          }
        }
      }
    }
    reserve_tile<K3_NP, WARPS>(keepm, pos, &c->out_cnt[1], s_wcnt);
#pragma unroll
    for (int j = 0; j < K3_NP; ++j) {
      if ((keepm >> j) & 1u) {
        Oxy[pos[j]] = make_double2(px[j], py[j]);
        Ois[pos[j]] = make_uint2(pid[j], pseg[j]);
      }
    }
    offer_tile_smem<K3_NP>(s_db, s_win, keepm, px, py, pd, pid, pseg, pos,
                           [&](int j) {
                             return route_edge(((lowm >> j) & 1u) ? rlo : rup, (leftm >> j) & 1u);
                           },
                           lowm, ld);
  }

  // ---- flush the CTA's slots to the global slots of round 2's argmax ----
  __syncthreads();
  __threadfence();
  if (threadIdx.x < Sn) {
    const uint32_t t = threadIdx.x;
    const uint32_t w = s_win[t];
    if (w != NONE) {
      Cand me;
      ld(w, me.x, me.y, me.id);
      me.d = __longlong_as_double((long long)s_db[t]);
      me.pos = w;
      const uint32_t f = s_from[t];
      const Route& r = s_rt[f & 1u];
      slot_offer(B.Sd[1] + t, B.Sw[1] + t, me, t < Slon, route_edge(r, (f >> 31) == 0u),
                 ld);
    }
  }

  // ---- last CTA closes round 1 ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  c->ticket = 0;
  const uint32_t mn = *(volatile uint32_t*)&c->out_cnt[1];
  const uint32_t before = c->S_cur + c->m_cur;
  StatRec st;
  st.segments = Sn;
  st.points_remaining = Sn + mn;
  st.points_removed = before - (Sn + mn);
  st.pad = 0;
  B.stats[0] = st;
  c->round = 1;
  c->S_cur = Sn;
  c->Slo_cur = Slon;
  c->m_cur = mn;
  if (mn == 0) c->status = ST_DONE;
  __threadfence();
}

// ===========================================================================
// KR: rounds >= 2, one persistent cooperative launch
// ===========================================================================

constexpr int RW = RTPB / 32;          // warps per CTA
constexpr int KR_U = 4;                // live points per thread per tile
constexpr int KR_TILE = RTPB * KR_U;   // 2048

struct RoundSmem {
  Route rt[SMALL_S];               // route entries of a small table   64 KB
  unsigned long long db[NSLOT];    // CTA farthest slots: distance bits 16 KB
  uint32_t win[NSLOT];             //                     winner pos     8 KB
  uint32_t from[NSLOT];            // new segment -> (old segment, side) 8 KB
};

// Barrier over the CTAs still working on the rounds.
SH_DEV void rounds_barrier(Ctl* c, uint32_t P) {
  if (P > 1) grid_barrier(&c->bar_count, &c->bar_gen, P);
  else __syncthreads();
}

// Small table (S <= SMALL_S), rebuilt by every participating CTA in smem.
// CTA 0 also writes the next head table.  Returns S', S'lo.
SH_DEV void table_small(const Bufs& B, RoundSmem& sm, uint32_t S, uint32_t Slo, uint32_t pin,
                        uint32_t pout, uint32_t sin, uint32_t* s_ws, uint32_t& Sn,
                        uint32_t& Slon) {
  const double2* Cxy = B.Lxy[pin];
  const uint2* Cis = B.Lis[pin];
  const double* Tx = B.Tx[pin];
  const double* Ty = B.Ty[pin];
  const uint32_t* Ti = B.Tid[pin];
  const bool heads = blockIdx.x == 0;
  uint32_t running = 0, lower_splits = 0;
  for (uint32_t s0 = 0; s0 < S; s0 += RTPB) {
    const uint32_t s = s0 + threadIdx.x;
    const uint32_t w = s < S ? __ldcg(B.Sw[sin] + s) : NONE;
    const uint32_t split = (s < S && w != NONE) ? 1u : 0u;
    uint32_t total;
    const uint32_t pre = block_exclusive_scan(split, s_ws, &total);
    lower_splits += (uint32_t)__syncthreads_count(split && s < Slo);
    if (s < S) {
      const uint32_t ns = s + running + pre;
      const uint32_t sb = s + 1 == S ? 0u : s + 1;
      Route r;
      r.ax = __ldcg(Tx + s);
      r.ay = __ldcg(Ty + s);
      r.bx = __ldcg(Tx + sb);
      r.by = __ldcg(Ty + sb);
      r.ns = ns;
      r.flags = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
      r.pad = 0;
      if (split) {
        const double2 cv = __ldcg(Cxy + w);
        r.cx = cv.x;
        r.cy = cv.y;
        r.cid = __ldcg(&Cis[w].x);
      } else {
        r.cx = 0.0;
        r.cy = 0.0;
        r.cid = NONE;
      }
      sm.rt[s] = r;
      sm.from[ns] = s;
      if (split) sm.from[ns + 1] = s | 0x80000000u;
      if (heads) {
        B.Tx[pout][ns] = r.ax;
        B.Ty[pout][ns] = r.ay;
        B.Tid[pout][ns] = __ldcg(Ti + s);
        if (split) {
          B.Tx[pout][ns + 1] = r.cx;
          B.Ty[pout][ns + 1] = r.cy;
          B.Tid[pout][ns + 1] = r.cid;
        }
      }
    }
    running += total;
  }
  Sn = S + running;
  Slon = Slo + lower_splits;
  for (uint32_t t = threadIdx.x; t < Sn; t += RTPB) {
    sm.db[t] = 0ull;
    sm.win[t] = NONE;
  }
  __syncthreads();
}

// Large table: a grid-wide two-step scan over the P participating CTAs.
// Returns false on segment-table overflow (every CTA returns consistently).
SH_DEV bool table_large(const Bufs& B, uint32_t S, uint32_t Slo, uint32_t pin, uint32_t pout,
                        uint32_t sin, uint32_t P, uint32_t* s_ws, uint32_t& Sn,
                        uint32_t& Slon) {
  Ctl* c = B.ctl;
  const uint32_t per = (S + P - 1) / P;
  const uint32_t lo = blockIdx.x * per, hi = min(S, lo + per);
  // T1: splittable counts of this CTA's range (total and lower chain)
  uint32_t cnt = 0, cnt_lo = 0;
  for (uint32_t s = lo + threadIdx.x; s < hi; s += RTPB) {
    const bool split = __ldcg(B.Sw[sin] + s) != NONE;
    cnt += split;
    cnt_lo += split && s < Slo;
  }
  {
    uint32_t t1, t2;
    block_exclusive_scan(cnt, s_ws, &t1);
    block_exclusive_scan(cnt_lo, s_ws, &t2);
    if (threadIdx.x == 0) {
      B.blk_cnt[blockIdx.x] = t1;
      B.blk_cnt[MAX_ROUND_BLOCKS + blockIdx.x] = t2;
    }
  }
  rounds_barrier(c, P);
  // T2: prefix of this CTA + totals
  uint32_t pre = 0, tot = 0, tot_lo = 0;
  for (uint32_t b = threadIdx.x; b < P; b += RTPB) {
    const uint32_t v = __ldcg(B.blk_cnt + b);
    tot += v;
    if (b < blockIdx.x) pre += v;
    tot_lo += __ldcg(B.blk_cnt + MAX_ROUND_BLOCKS + b);
  }
  uint32_t pre_all, tot_all, tot_lo_all;
  block_exclusive_scan(pre, s_ws, &pre_all);
  block_exclusive_scan(tot, s_ws, &tot_all);
  block_exclusive_scan(tot_lo, s_ws, &tot_lo_all);
  Sn = S + tot_all;
  Slon = Slo + tot_lo_all;
  if (Sn > B.s_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) c->status = ST_OVERFLOW;
    return false;
  }
  const double2* Cxy = B.Lxy[pin];
  const uint2* Cis = B.Lis[pin];
  const double* Tx = B.Tx[pin];
  const double* Ty = B.Ty[pin];
  const uint32_t* Ti = B.Tid[pin];
  uint32_t running = pre_all;
  for (uint32_t s0 = lo; s0 < hi; s0 += RTPB) {
    const uint32_t s = s0 + threadIdx.x;
    const uint32_t w = s < hi ? __ldcg(B.Sw[sin] + s) : NONE;
    const uint32_t split = (s < hi && w != NONE) ? 1u : 0u;
    uint32_t total;
    const uint32_t p = block_exclusive_scan(split, s_ws, &total);
    if (s < hi) {
      const uint32_t ns = s + running + p;
      const uint32_t sb = s + 1 == S ? 0u : s + 1;
      Route r;
      r.ax = __ldcg(Tx + s);
      r.ay = __ldcg(Ty + s);
      r.bx = __ldcg(Tx + sb);
      r.by = __ldcg(Ty + sb);
      r.ns = ns;
      r.flags = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
      r.pad = 0;
      if (split) {
        const double2 cv = __ldcg(Cxy + w);
        r.cx = cv.x;
        r.cy = cv.y;
        r.cid = __ldcg(&Cis[w].x);
      } else {
        r.cx = 0.0;
        r.cy = 0.0;
        r.cid = NONE;
      }
      B.route[s] = r;
      B.Tx[pout][ns] = r.ax;
      B.Ty[pout][ns] = r.ay;
      B.Tid[pout][ns] = __ldcg(Ti + s);
      if (split) {
        B.Tx[pout][ns + 1] = r.cx;
        B.Ty[pout][ns + 1] = r.cy;
        B.Tid[pout][ns + 1] = r.cid;
      }
    }
    running += total;
  }
  rounds_barrier(c, P);
  return true;
}

__global__ void __launch_bounds__(RTPB, 1) k_rounds(Bufs B) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RoundSmem& sm = *reinterpret_cast<RoundSmem*>(smem_raw);
  __shared__ uint32_t s_ws[RW + 1];
  __shared__ uint32_t s_wcnt[RW];
  Ctl* c = B.ctl;
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  uint32_t r = *(volatile uint32_t*)&c->round + 1;
  uint32_t S = *(volatile uint32_t*)&c->S_cur;
  uint32_t Slo = *(volatile uint32_t*)&c->Slo_cur;
  uint32_t m = *(volatile uint32_t*)&c->m_cur;
  const uint32_t n = B.n;
  uint32_t P = gridDim.x;

  while (true) {
    if (P > 1 && m <= TAIL_M) {  // every CTA sees the same m: consistent
      P = 1;
      if (blockIdx.x != 0) return;
    }
    const uint32_t pin = (r - 1) & 1u, pout = r & 1u;
    const uint32_t sin = (r - 1) % 3u, sout = r % 3u, sres = (r + 1) % 3u;
    const bool small = S <= (uint32_t)SMALL_S;
    uint32_t Sn, Slon;
    if (small) {
      table_small(B, sm, S, Slo, pin, pout, sin, s_ws, Sn, Slon);
    } else if (!table_large(B, S, Slo, pin, pout, sin, P, s_ws, Sn, Slon)) {
      return;
    }
    // clear round r+1's farthest slots (at most 2 Sn segments) and counter
    {
      const uint32_t lim = min(2 * Sn, B.s_cap);
      for (uint32_t t = blockIdx.x * RTPB + threadIdx.x; t < lim; t += P * RTPB) {
        B.Sd[sres][t] = 0ull;
        B.Sw[sres][t] = NONE;
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) c->out_cnt[sres] = 0;
    }

    // ---- point phase ----
    const double2* Ixy = B.Lxy[pin];
    const uint2* Iis = B.Lis[pin];
    double2* Oxy = B.Lxy[pout];
    uint2* Ois = B.Lis[pout];
    const LoadLive ld{Oxy, Ois};
    unsigned long long* Sd = B.Sd[sout];
    uint32_t* Sw = B.Sw[sout];
    const uint32_t ntiles = (m + KR_TILE - 1) / KR_TILE;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += P) {
      double px[KR_U], py[KR_U], pd[KR_U];
      uint32_t pid[KR_U], pseg[KR_U], pos[KR_U];
      uint32_t keepm = 0, lowm = 0, leftm = 0;
      uint32_t oseg[KR_U];
#pragma unroll
      for (int u = 0; u < KR_U; ++u) {
        const uint32_t e = tile * KR_TILE + u * RTPB + threadIdx.x;
        px[u] = py[u] = 0.0;
        pid[u] = 0;
        oseg[u] = NONE;
        if (e < m) {
          const double2 v = __ldcs(Ixy + e);
          const uint2 is = __ldcs(Iis + e);
          px[u] = v.x;
          py[u] = v.y;
          pid[u] = is.x;
          oseg[u] = is.y;
        }
      }
#pragma unroll
      for (int u = 0; u < KR_U; ++u) {
        pd[u] = 0.0;
        pseg[u] = 0;
        if (oseg[u] != NONE) {
          const Route rr = small ? sm.rt[oseg[u]] : ldcg_route(B.route + oseg[u]);
          bool left = false;
          if (route_point(rr, px[u], py[u], pid[u], pd[u], pseg[u], left)) {
            keepm |= 1u << u;
            if (left) leftm |= 1u << u;
            if (rr.flags & RT_LOWER) lowm |= 1u << u;
          }
        }
      }
      reserve_tile<KR_U, RW>(keepm, pos, &c->out_cnt[sout], s_wcnt);
#pragma unroll
      for (int u = 0; u < KR_U; ++u) {
        if ((keepm >> u) & 1u) {
          Oxy[pos[u]] = make_double2(px[u], py[u]);
          Ois[pos[u]] = make_uint2(pid[u], pseg[u]);
        }
      }
      auto edge_of = [&](int u) {
        const Route rr = small ? sm.rt[oseg[u]] : ldcg_route(B.route + oseg[u]);
        return route_edge(rr, (leftm >> u) & 1u);
      };
      if (small) {
        offer_tile_smem<KR_U>(sm.db, sm.win, keepm, px, py, pd, pid, pseg, pos, edge_of, lowm,
                              ld);
      } else if (keepm) {
        __threadfence();
#pragma unroll
        for (int u = 0; u < KR_U; ++u) {
          if ((keepm >> u) & 1u) {
            Cand me;
            me.d = pd[u]; me.x = px[u]; me.y = py[u]; me.id = pid[u]; me.pos = pos[u];
            slot_offer(Sd + pseg[u], Sw + pseg[u], me, (lowm >> u) & 1u, edge_of(u), ld);
          }
        }
      }
    }
    if (small) {  // flush the CTA's slots
      __syncthreads();
      __threadfence();
      for (uint32_t t = threadIdx.x; t < Sn; t += RTPB) {
        const uint32_t w = sm.win[t];
        if (w != NONE) {
          Cand me;
          ld(w, me.x, me.y, me.id);
          me.d = __longlong_as_double((long long)sm.db[t]);
          me.pos = w;
          const uint32_t f = sm.from[t];
          const Route& rr = sm.rt[f & 0x7FFFFFFFu];
          slot_offer(Sd + t, Sw + t, me, t < Slon, route_edge(rr, (f >> 31) == 0u), ld);
        }
      }
    }
    rounds_barrier(c, P);

    // ---- close round r (every participating CTA computes the same) ----
    const uint32_t mn = __ldcg(&c->out_cnt[sout]);
    if (blockIdx.x == 0 && threadIdx.x == 0 && r <= (uint32_t)STATS_CAP) {
      StatRec st;
      st.segments = Sn;
      st.points_remaining = Sn + mn;
      st.points_removed = (S + m) - (Sn + mn);
      st.pad = 0;
      B.stats[r - 1] = st;
    }
    S = Sn;
    Slo = Slon;
    m = mn;
    if (mn == 0 || r + 1 > n) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->round = r;
        c->S_cur = S;
        c->Slo_cur = Slo;
        c->m_cur = m;
        c->status = mn == 0 ? ST_DONE : ST_INTERNAL;  // hull.cpp:265-267
        __threadfence();
      }
      return;
    }
    ++r;
  }
}

// ===========================================================================
// K5: emit the hull (segment heads in table order) into caller device memory
// ===========================================================================

__global__ void k5_emit(Bufs B, double* ox, double* oy, long long* oidx, uint64_t cap) {
  const Ctl* c = B.ctl;
  if (c->status != ST_DONE) return;
  const uint32_t par = c->round & 1u;
  const uint32_t h = c->S_cur;
  const uint32_t lim = h < cap ? h : (uint32_t)cap;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += gridDim.x * blockDim.x) {
    if (ox) ox[i] = B.Tx[par][i];
    if (oy) oy[i] = B.Ty[par][i];
    if (oidx) oidx[i] = (long long)B.Tid[par][i];
  }
}

// ===========================================================================
// host-side launch wrappers
// ===========================================================================

size_t rounds_smem_bytes() { return sizeof(RoundSmem); }

cudaError_t configure_round_kernels() {
  return cudaFuncSetAttribute(k_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(RoundSmem));
}

int rounds_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_rounds, RTPB, sizeof(RoundSmem));
  return b < 1 ? 1 : b;
}

int k3_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_round1<false, true>, TPB, 0);
  return b < 1 ? 1 : b;
}

void launch_k3(const Bufs& B, bool ids, bool vec, int grid, cudaStream_t s) {
  if (ids) {
    if (vec) k3_round1<true, true><<<grid, TPB, 0, s>>>(B);
    else k3_round1<true, false><<<grid, TPB, 0, s>>>(B);
  } else {
    if (vec) k3_round1<false, true><<<grid, TPB, 0, s>>>(B);
    else k3_round1<false, false><<<grid, TPB, 0, s>>>(B);
  }
}

cudaError_t launch_rounds(const Bufs& B, int grid, cudaStream_t s) {
  Bufs b = B;
  void* args[] = {&b};
  return cudaLaunchCooperativeKernel((const void*)k_rounds, dim3(grid), dim3(RTPB), args,
                                     sizeof(RoundSmem), s);
}

void launch_k5(const Bufs& B, double* ox, double* oy, long long* oidx, uint64_t cap,
               cudaStream_t s) {
  k5_emit<<<16, 256, 0, s>>>(B, ox, oy, oidx, cap);
}

}  // namespace shb
