// k_pre.cu -- the two full-input passes of the sm_100a QuickHull.
//
//   K1 k1_extremes  four directional extremes + first non-finite index
//                   (hull.cpp:25-45, 221-237); the last CTA derives the
//                   quadrilateral (hull.cpp:58-74)
//   K2 k2_classify  quadrilateral filter (hull.cpp:76-91), collinearity flag
//                   (hull.cpp:238-248), chain classification (hull.cpp:114-118)
//                   and the round-1 farthest point of both chains
//                   (hull.cpp:160-184) -- no point is written: the class of
//                   every point leaves as 2 bits in `bits`
//
// Both are pure HBM streams over SoA f64 x/y: every thread keeps U
// independent 16-byte loads per array in flight (double2 = a pair of
// consecutive points), grids are a multiple of the SM count, and K2 walks
// the input backwards so it starts on the tail K1 just left in L2 (and ends
// on the head, where K3 starts).
#include <cuda_runtime.h>

#include <type_traits>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

// ===========================================================================
// helpers
// ===========================================================================

// Total order of doubles as u64 keys (-0.0 sorts just below +0.0; a
// threshold only has to bound the final extreme, so that is harmless).
SH_DEV unsigned long long okey(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
SH_DEV double okey_dec(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

SH_DEV bool nonfinite(double v) {
  return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}

// ===========================================================================
// K1: extremes with directional ties (hull.cpp:25-45) + first non-finite index
// ===========================================================================

template <int DIR>
SH_DEV bool ext_better(const ExtRec& a, const ExtRec& b) {
  if (b.pos == NONE) return a.pos != NONE;
  if (a.pos == NONE) return false;
  if (DIR == 0) {  // left: min x, then min y
    if (a.x != b.x) return a.x < b.x;
    if (a.y != b.y) return a.y < b.y;
  } else if (DIR == 1) {  // bottom: min y, then max x
    if (a.y != b.y) return a.y < b.y;
    if (a.x != b.x) return a.x > b.x;
  } else if (DIR == 2) {  // right: max x, then max y
    if (a.x != b.x) return a.x > b.x;
    if (a.y != b.y) return a.y > b.y;
  } else {  // top: max y, then min x
    if (a.y != b.y) return a.y > b.y;
    if (a.x != b.x) return a.x < b.x;
  }
  return a.id < b.id;  // exact duplicates: lowest index (strict compares)
}

SH_DEV ExtRec shfl_ext(const ExtRec& e, int m) {
  ExtRec o;
  o.x = __shfl_xor_sync(FULL, e.x, m);
  o.y = __shfl_xor_sync(FULL, e.y, m);
  o.id = __shfl_xor_sync(FULL, e.id, m);
  o.pos = __shfl_xor_sync(FULL, e.pos, m);
  return o;
}

SH_DEV void warp_reduce_ext(ExtRec* e, unsigned long long& bad) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    ExtRec o;
    o = shfl_ext(e[0], m);
    if (ext_better<0>(o, e[0])) e[0] = o;
    o = shfl_ext(e[1], m);
    if (ext_better<1>(o, e[1])) e[1] = o;
    o = shfl_ext(e[2], m);
    if (ext_better<2>(o, e[2])) e[2] = o;
    o = shfl_ext(e[3], m);
    if (ext_better<3>(o, e[3])) e[3] = o;
    const unsigned long long ob = __shfl_xor_sync(FULL, bad, m);
    bad = ob < bad ? ob : bad;
  }
}

// reduce (e, bad) over the block; result valid in thread 0
SH_DEV void block_reduce_ext(ExtRec* e, unsigned long long& bad) {
  __shared__ ExtRec s_e[4][MAXW];
  __shared__ unsigned long long s_bad[MAXW];
  const int nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_reduce_ext(e, bad);
  if (lane == 0) {
    for (int k = 0; k < 4; ++k) s_e[k][warp] = e[k];
    s_bad[warp] = bad;
  }
  __syncthreads();
  if (warp == 0) {
    for (int k = 0; k < 4; ++k) {
      if (lane < nw) {
        e[k] = s_e[k][lane];
      } else {
        e[k].pos = NONE;
      }
    }
    bad = lane < nw ? s_bad[lane] : ~0ull;
    warp_reduce_ext(e, bad);
  }
  __syncthreads();
}

// One point, visited in increasing index order within a thread, so strict
// comparisons keep the lowest index among exact duplicates (hull.cpp:39-43).
// With caller ids (shard merge) the id decides exact duplicates explicitly.
template <bool IDS>
SH_DEV void ext_visit(ExtRec (&e)[4], unsigned long long& bad, double x, double y, uint32_t id,
                      uint32_t pos) {
  if (nonfinite(x) || nonfinite(y)) {
    if (bad == ~0ull) bad = pos;
    return;
  }
  if (x <= e[0].x && (x < e[0].x || y < e[0].y || (IDS && y == e[0].y && id < e[0].id))) {
    e[0].x = x; e[0].y = y; e[0].id = id; e[0].pos = pos;
  }
  if (y <= e[1].y && (y < e[1].y || x > e[1].x || (IDS && x == e[1].x && id < e[1].id))) {
    e[1].x = x; e[1].y = y; e[1].id = id; e[1].pos = pos;
  }
  if (x >= e[2].x && (x > e[2].x || y > e[2].y || (IDS && y == e[2].y && id < e[2].id))) {
    e[2].x = x; e[2].y = y; e[2].id = id; e[2].pos = pos;
  }
  if (y >= e[3].y && (y > e[3].y || x < e[3].x || (IDS && x == e[3].x && id < e[3].id))) {
    e[3].x = x; e[3].y = y; e[3].id = id; e[3].pos = pos;
  }
}

// Thread 0, once the four extremes and the first bad index are known:
// degenerate statuses (hull.cpp:222-237) and the quadrilateral (hull.cpp:58-74).
SH_DEV void finalize_extremes(const Bufs& B, const ExtRec (&e)[4], unsigned long long bad) {
  Ctl* c = B.ctl;
  c->ticket = 0;
  c->bad_index = bad;
  // round-0 farthest slots (K2 offers into Slot[0]; hull_kernels.cuh)
  rec_clear(&B.Sd[0][0], &B.Srec[0][0]);
  rec_clear(&B.Sd[0][1], &B.Srec[0][1]);
  c->mark[0] = globaltimer_ns() - c->t0_ns;
  if (bad != ~0ull) {
    c->status = ST_NONFINITE;
    return;
  }
  for (int k = 0; k < 4; ++k) {
    c->ext_x[k] = e[k].x;
    c->ext_y[k] = e[k].y;
    c->ext_id[k] = e[k].id;
    c->ext_pos[k] = e[k].pos;
  }
  if (e[0].x == e[2].x && e[0].y == e[2].y) {  // hull.cpp:234-237
    c->status = ST_SINGLE;
    return;
  }
  // hull.cpp:58-74: corners [left, bottom, right, top], distinct count and
  // the edges between consecutive non-equal corners (with wrap-around)
  int distinct = 0;
  for (int a = 0; a < 4; ++a) {
    bool seen = false;
    for (int b = 0; b < a; ++b) seen |= (e[a].x == e[b].x && e[a].y == e[b].y);
    if (!seen) ++distinct;
  }
  int ne = 0;
  for (int a = 0; a < 4; ++a) {
    const ExtRec& p = e[a];
    const ExtRec& qq = e[(a + 1) & 3];
    if (!(p.x == qq.x && p.y == qq.y)) {
      const Edge ed = make_edge(p.x, p.y, qq.x, qq.y);
      c->edges[ne][0] = ed.ax;
      c->edges[ne][1] = ed.ay;
      c->edges[ne][2] = ed.ex;
      c->edges[ne][3] = ed.ey;
      ++ne;
    }
  }
  for (int k = ne; k < 4; ++k)
    for (int j = 0; j < 4; ++j) c->edges[k][j] = 0.0;
  c->distinct = distinct;
  c->nedges = ne;
  c->mark[0] = globaltimer_ns() - c->t0_ns;
}

template <bool IDS>
using Ring1 = TileRing<Cfg1::T, Cfg1::NS, IDS, 0, Cfg1::CW>;

template <bool IDS>
__global__ void __launch_bounds__(Cfg1::TPB, 1) k1_extremes(Bufs B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring1<IDS> R;
  R.carve(smem_raw);
  Ctl* c = B.ctl;
  const uint32_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  ExtRec e[4];
  e[0].x = INF;  e[0].y = INF;   // left
  e[1].x = -INF; e[1].y = INF;   // bottom
  e[2].x = -INF; e[2].y = -INF;  // right
  e[3].x = INF;  e[3].y = -INF;  // top
  for (int k = 0; k < 4; ++k) e[k].id = e[k].pos = NONE;
  unsigned long long bad = ~0ull;
  pdl_launch_dependents();  // K2 may be scheduled on SMs this kernel frees
  if (blockIdx.x == 0 && threadIdx.x == 0) c->t0_ns = globaltimer_ns();
  // CTA-wide thresholds for the branch-free filter: a point can only become
  // an extreme if it is at least as extreme as the CTA's running extreme
  // (which bounds the final one).  Keys: min x, min y, max x, max y.
  __shared__ unsigned long long s_thr[4];
  if (threadIdx.x == 0) {
    R.init();
    s_thr[0] = okey(INF);
    s_thr[1] = okey(INF);
    s_thr[2] = okey(-INF);
    s_thr[3] = okey(-INF);
  }
  __syncthreads();

  // forward over the input; within a thread indices only grow, so strict
  // comparisons keep the lowest index among exact duplicates
  stream_input(R, n, X, Y, I, nullptr, false, [&](int s, uint32_t first, uint32_t cnt) {
    const double* xs = R.xs + s * Cfg1::T;
    const double* ys = R.ys + s * Cfg1::T;
    const uint32_t* is = R.is + s * Cfg1::T;
    const double t0 = okey_dec(*(volatile unsigned long long*)&s_thr[0]);
    const double t1 = okey_dec(*(volatile unsigned long long*)&s_thr[1]);
    const double t2 = okey_dec(*(volatile unsigned long long*)&s_thr[2]);
    const double t3 = okey_dec(*(volatile unsigned long long*)&s_thr[3]);
    bool moved = false;
    if (cnt == (uint32_t)Cfg1::T) {
#pragma unroll
      for (int k = 0; k < Cfg1::T / 2 / Cfg1::CT; ++k) {
        const uint32_t p = k * Cfg1::CT + threadIdx.x;
        const double2 xv = reinterpret_cast<const double2*>(xs)[p];
        const double2 yv = reinterpret_cast<const double2*>(ys)[p];
        // can either point reach an extreme, or is it non-finite (exponent
        // all ones)?  Rare once the CTA thresholds have settled.
        const uint32_t M = 0x7ff00000u;
        const uint32_t hm = max(max((uint32_t)__double2hiint(xv.x) & M, (uint32_t)__double2hiint(xv.y) & M),
                                max((uint32_t)__double2hiint(yv.x) & M, (uint32_t)__double2hiint(yv.y) & M));
        const bool cand = (hm == M) | (xv.x <= t0) | (xv.y <= t0) | (yv.x <= t1) | (yv.y <= t1) |
                          (xv.x >= t2) | (xv.y >= t2) | (yv.x >= t3) | (yv.y >= t3);
        if (cand) {
          uint2 iv = make_uint2(0u, 0u);
          if (IDS) iv = reinterpret_cast<const uint2*>(is)[p];
          const uint32_t i = first + 2 * p;
          ext_visit<IDS>(e, bad, xv.x, yv.x, IDS ? iv.x : i, i);
          ext_visit<IDS>(e, bad, xv.y, yv.y, IDS ? iv.y : i + 1, i + 1);
          moved = true;
        }
      }
    } else {
      const uint32_t c4 = cnt & ~3u;
      for (uint32_t j = threadIdx.x; j < cnt; j += Cfg1::CT) {
        const uint32_t i = first + j;
        const bool sm = j < c4;
        const double x = sm ? xs[j] : __ldg(X + i);
        const double y = sm ? ys[j] : __ldg(Y + i);
        const uint32_t id = IDS ? (sm ? is[j] : __ldg(I + i)) : i;
        ext_visit<IDS>(e, bad, x, y, id, i);
      }
      moved = true;
    }
    if (moved) {  // publish this thread's extremes as CTA thresholds
      if (e[0].pos != NONE) atomicMin(&s_thr[0], okey(e[0].x));
      if (e[1].pos != NONE) atomicMin(&s_thr[1], okey(e[1].y));
      if (e[2].pos != NONE) atomicMax(&s_thr[2], okey(e[2].x));
      if (e[3].pos != NONE) atomicMax(&s_thr[3], okey(e[3].y));
    }
  });

  block_reduce_ext(e, bad);
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    K1Partial pt;
    for (int k = 0; k < 4; ++k) pt.e[k] = e[k];
    pt.bad = bad;
    B.k1part[blockIdx.x] = pt;
    __threadfence();
    s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // last CTA: combine the per-CTA partials
  for (int k = 0; k < 4; ++k) e[k].pos = NONE;
  bad = ~0ull;
  for (uint32_t p = threadIdx.x; p < gridDim.x; p += blockDim.x) {
    const K1Partial* qp = B.k1part + p;
    ExtRec o[4];
    for (int k = 0; k < 4; ++k) {
      o[k].x = __ldcg(&qp->e[k].x);
      o[k].y = __ldcg(&qp->e[k].y);
      o[k].id = __ldcg(&qp->e[k].id);
      o[k].pos = __ldcg(&qp->e[k].pos);
    }
    if (ext_better<0>(o[0], e[0])) e[0] = o[0];
    if (ext_better<1>(o[1], e[1])) e[1] = o[1];
    if (ext_better<2>(o[2], e[2])) e[2] = o[2];
    if (ext_better<3>(o[3], e[3])) e[3] = o[3];
    const unsigned long long ob = __ldcg(&qp->bad);
    bad = ob < bad ? ob : bad;
  }
  block_reduce_ext(e, bad);
  if (threadIdx.x != 0) return;

  finalize_extremes(B, e, bad);
}

// ===========================================================================
// K2: filter + classification + round-0 farthest points (no point writes).
// ===========================================================================

SH_DEV void cand_visit(Cand& a, double d, double x, double y, uint32_t id, uint32_t pos,
                       bool lower) {
  if (d > 0.0 && d >= a.d) {
    Cand cc;
    cc.d = d; cc.x = x; cc.y = y; cc.id = id; cc.pos = pos;
    if (cand_better(cc, a, lower)) a = cc;
  }
}

template <bool FILTER, bool IDS>
__global__ void __launch_bounds__(Cfg2::TPB, 1) k2_classify(Bufs B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileRing<Cfg2::T, Cfg2::NS, IDS, 0, Cfg2::CW> R;
  R.carve(smem_raw);
  Ctl* c = B.ctl;
  pdl_wait();               // K1's extremes are complete and visible
  pdl_launch_dependents();  // K3 may be scheduled on SMs this kernel frees
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) c->mark[1] = globaltimer_ns() - c->t0_ns;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  const uint32_t p0 = c->ext_pos[0], pr = c->ext_pos[2];
  const double x0 = c->ext_x[0], y0 = c->ext_y[0], xr = c->ext_x[2], yr = c->ext_y[2];
  const Edge E01 = make_edge(x0, y0, xr, yr);  // lower chain base line P0 -> Pr
  const Edge E10 = make_edge(xr, yr, x0, y0);  // upper chain base line Pr -> P0 (wrap)
  const bool filt = FILTER && c->distinct >= 3;
  const int ne = filt ? c->nedges : 0;
  Edge Q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Q[k].ax = c->edges[k][0];
    Q[k].ay = c->edges[k][1];
    Q[k].ex = c->edges[k][2];
    Q[k].ey = c->edges[k][3];
  }
  Cand a0 = empty_cand(), a1 = empty_cand();
  uint32_t kept = 0;
  bool noncol = false;
  // CTA-wide running maxima of the two chains' distances (positive doubles
  // order like their bits): a point below them cannot be the CTA's farthest,
  // so the per-point candidate branch is almost never taken
  __shared__ unsigned long long s_dmax[2];
  if (threadIdx.x == 0) {
    R.init();
    s_dmax[0] = s_dmax[1] = 0ull;
  }
  __syncthreads();

  // With 4 distinct corners, edge q starts at corner q (left, bottom, right,
  // top) and the chain base lines start at left (P0) and right (Pr), so the
  // per-point differences p - corner are shared by the 6 cross products:
  // the same RN operations as cross() (geometry.hpp:17-19), computed once.
  const bool quad4 = filt && ne == 4 && c->distinct == 4;
  const double cxL = c->ext_x[0], cyL = c->ext_y[0], cxB = c->ext_x[1], cyB = c->ext_y[1];
  const double cxR = c->ext_x[2], cyR = c->ext_y[2], cxT = c->ext_x[3], cyT = c->ext_y[3];
  auto xprod = [](double ex, double ey, double dx, double dy) {
    return __dsub_rn(__dmul_rn(ex, dy), __dmul_rn(ey, dx));
  };

  // backwards over the input: K1 just left the tail in L2, K3 starts at the head
  constexpr int NCH = Cfg2::T / 64 / Cfg2::CW;  // chunks per consumer warp per tile
  constexpr int NP = 2 * NCH;                  // points per thread per tile
#ifndef SHB_K2_REVERSE
#define SHB_K2_REVERSE 1
#endif
  // One tile; FULLT: cnt == T (no bounds checks anywhere).  All decisions are
  // bitwise predicates; the rare candidate updates sit behind one
  // warp-uniform branch.
  // QK: 1 = the 4-corner quadrilateral, 2 = a degenerate one (<= 3 edges),
  // 0 = no filter -- a compile-time choice, so the hot path carries no
  // predicated-off arithmetic of the other variants
  auto tile = [&](auto fullt, auto qk, int s, uint32_t first, uint32_t cnt) {
    constexpr bool FULLT = decltype(fullt)::value;
    constexpr int QK = decltype(qk)::value;
    const double* xs = R.xs + s * Cfg2::T;
    const double* ys = R.ys + s * Cfg2::T;
    const uint32_t* is = R.is + s * Cfg2::T;
    const uint32_t c4 = cnt & ~3u;
    double px[NP], py[NP];
    uint32_t pid[NP];
    bool pv[NP];
    // ---- gather the thread's points (pairs of one 64-point chunk) ----
#pragma unroll
    for (int kk = 0; kk < NCH; ++kk) {
      const uint32_t cc = kk * Cfg2::CW + warp;  // chunk of 64 points within the tile
      const uint32_t j = cc * 64 + 2 * lane;   // this lane's pair
      double2 xv = make_double2(0.0, 0.0), yv = xv;
      uint2 iv = make_uint2(0u, 0u);
      if (FULLT || j + 1 < c4) {
        xv = reinterpret_cast<const double2*>(xs)[j >> 1];
        yv = reinterpret_cast<const double2*>(ys)[j >> 1];
        if (IDS) iv = reinterpret_cast<const uint2*>(is)[j >> 1];
      } else {
        for (int h = 0; h < 2; ++h) {
          const uint32_t jj = j + h;
          if (jj < cnt) {
            const bool sm = jj < c4;
            (h ? xv.y : xv.x) = sm ? xs[jj] : __ldg(X + first + jj);
            (h ? yv.y : yv.x) = sm ? ys[jj] : __ldg(Y + first + jj);
            if (IDS) (h ? iv.y : iv.x) = sm ? is[jj] : __ldg(I + first + jj);
          }
        }
      }
      px[2 * kk] = xv.x; px[2 * kk + 1] = xv.y;
      py[2 * kk] = yv.x; py[2 * kk + 1] = yv.y;
      pid[2 * kk] = IDS ? iv.x : first + j;
      pid[2 * kk + 1] = IDS ? iv.y : first + j + 1;
      pv[2 * kk] = FULLT || j < cnt;
      pv[2 * kk + 1] = FULLT || j + 1 < cnt;
    }
    // ---- arithmetic of all NP points in one branch-free block ----
    // (the RN operations of cross(), geometry.hpp:17-19, with the per-point
    // differences to the 4 corners shared by the 6 cross products)
    double cl[NP], du[NP];
    bool ins[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double x = px[q], y = py[q];
      const double dxL = __dsub_rn(x, cxL), dyL = __dsub_rn(y, cyL);
      const double dxR = __dsub_rn(x, cxR), dyR = __dsub_rn(y, cyR);
      cl[q] = xprod(E01.ex, E01.ey, dxL, dyL);         // cross(P0, Pr, p)
      du[q] = -xprod(E10.ex, E10.ey, dxR, dyR);        // outward_distance(Pr, P0, p)
      bool inside = false;
      if (QK == 1) {  // hull.cpp:80-90: discard iff cross > 0 for every edge
        const double dxB = __dsub_rn(x, cxB), dyB = __dsub_rn(y, cyB);
        const double dxT = __dsub_rn(x, cxT), dyT = __dsub_rn(y, cyT);
        inside = (xprod(Q[0].ex, Q[0].ey, dxL, dyL) > 0.0) &
                 (xprod(Q[1].ex, Q[1].ey, dxB, dyB) > 0.0) &
                 (xprod(Q[2].ex, Q[2].ey, dxR, dyR) > 0.0) &
                 (xprod(Q[3].ex, Q[3].ey, dxT, dyT) > 0.0);
      } else if (QK == 2) {  // degenerate quadrilateral (3 distinct corners)
        inside = true;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          if (qq < ne) inside = inside & (cross_e(Q[qq], x, y) > 0.0);
      }
      ins[q] = inside;
    }
    // ---- bookkeeping: classes, ballots, farthest candidates ----
    const double m0 = fmax(a0.d, __longlong_as_double(*(volatile long long*)&s_dmax[0]));
    const double m1 = fmax(a1.d, __longlong_as_double(*(volatile long long*)&s_dmax[1]));
    const double ad0 = a0.d, ad1 = a1.d;
    uint32_t lwm = 0, upm = 0, c0m = 0, c1m = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const uint32_t i = first + (q >> 1) * (64 * Cfg2::CW) + warp * 64 + 2 * lane + (q & 1);
      const bool keep = pv[q] & !ins[q];
      noncol = noncol | (pv[q] & (cl[q] != 0.0));
      const bool member = keep & (i != p0) & (i != pr);
      const bool neg = cl[q] < 0.0;          // hull.cpp:115-117
      const bool lw = member & neg, up = member & !neg;
      kept += keep;
      lwm |= (uint32_t)lw << q;
      upm |= (uint32_t)up << q;
      // a candidate only when d reaches the running maximum (dl = -cl > 0 for lw)
      c0m |= (uint32_t)(lw & (-cl[q] >= m0)) << q;
      c1m |= (uint32_t)(up & (du[q] > 0.0) & (du[q] >= m1)) << q;
    }
    if (__any_sync(FULL, c0m | c1m)) {  // rare after a CTA's first tiles
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const uint32_t i = first + (q >> 1) * (64 * Cfg2::CW) + warp * 64 + 2 * lane + (q & 1);
        if ((c0m >> q) & 1u) cand_visit(a0, -cl[q], px[q], py[q], pid[q], i, true);
        if ((c1m >> q) & 1u) cand_visit(a1, du[q], px[q], py[q], pid[q], i, false);
      }
    }
#pragma unroll
    for (int kk = 0; kk < NCH; ++kk) {
      const uint32_t cc = kk * Cfg2::CW + warp;
      if (!FULLT && cc * 64 >= cnt) break;  // warp-uniform
      const uint32_t le = __ballot_sync(FULL, (lwm >> (2 * kk)) & 1u);
      const uint32_t lodd = __ballot_sync(FULL, (lwm >> (2 * kk + 1)) & 1u);
      const uint32_t ue = __ballot_sync(FULL, (upm >> (2 * kk)) & 1u);
      const uint32_t uodd = __ballot_sync(FULL, (upm >> (2 * kk + 1)) & 1u);
      if (lane == 0) B.bits[(first >> 6) + cc] = make_uint4(le, lodd, ue, uodd);
    }
    // publish improvements of this thread's candidates as CTA thresholds
    if (a0.d > ad0) atomicMax(&s_dmax[0], (unsigned long long)__double_as_longlong(a0.d));
    if (a1.d > ad1) atomicMax(&s_dmax[1], (unsigned long long)__double_as_longlong(a1.d));
  };
  auto pass = [&](auto qk) {
    stream_input(R, n, X, Y, I, nullptr, SHB_K2_REVERSE != 0, [&](int s, uint32_t first, uint32_t cnt) {
      if (cnt == (uint32_t)Cfg2::T)
        tile(std::true_type{}, qk, s, first, cnt);
      else
        tile(std::false_type{}, qk, s, first, cnt);
    });
  };
  if (quad4)
    pass(std::integral_constant<int, 1>{});
  else if (filt)
    pass(std::integral_constant<int, 2>{});
  else
    pass(std::integral_constant<int, 0>{});

  // block reduction of the two chains' farthest candidates
  __shared__ Cand s_a[2][MAXW];
  __shared__ uint32_t s_kept[MAXW];
  const int nwb = blockDim.x >> 5;
  __shared__ int s_last;
  a0 = warp_best(a0, true);
  a1 = warp_best(a1, false);
  const bool nc_any = __any_sync(FULL, noncol);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) kept += __shfl_xor_sync(FULL, kept, m);
  if (lane == 0) {
    s_a[0][warp] = a0;
    s_a[1][warp] = a1;
    s_kept[warp] = kept | (nc_any ? 0x80000000u : 0u);
  }
  __syncthreads();
  if (warp == 0) {
    a0 = lane < nwb ? s_a[0][lane] : empty_cand();
    a1 = lane < nwb ? s_a[1][lane] : empty_cand();
    a0 = warp_best(a0, true);
    a1 = warp_best(a1, false);
    if (lane == 0) {
      unsigned long long kb = 0;
      bool nc = false;
      for (int w = 0; w < nwb; ++w) {
        kb += s_kept[w] & 0x7FFFFFFFu;
        nc = nc || (s_kept[w] >> 31);
      }
      if (kb) atomicAdd(&c->kept, kb);
      if (nc) atomicOr(&c->noncollinear, 1u);
      if (a0.d > 0.0) rec_offer(&B.Sd[0][0], &B.Srec[0][0], a0, true);
      if (a1.d > 0.0) rec_offer(&B.Sd[0][1], &B.Srec[0][1], a1, false);
      __threadfence();
      s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  c->ticket = 0;
  // round-1 farthest slots (round 1 offers into Slot[1]; its table has <= 4 entries)
  for (int t = 0; t < 4; ++t) rec_clear(&B.Sd[1][t], &B.Srec[1][t]);
  if (!*(volatile uint32_t*)&c->noncollinear) {
    c->status = ST_COLLINEAR;  // hull.cpp:238-248
  } else {
    // first split (hull.cpp:101-158): P0 heads the lower chain, Pr the upper
    B.Tx[0][0] = x0;
    B.Ty[0][0] = y0;
    B.Tid[0][0] = c->ext_id[0];
    B.Tx[0][1] = xr;
    B.Ty[0][1] = yr;
    B.Tid[0][1] = c->ext_id[2];
    const unsigned long long kept_all = *(volatile unsigned long long*)&c->kept;
    c->S_cur = 2;
    c->Slo_cur = 1;
    c->m_cur = (uint32_t)(kept_all - 2);
    c->round = 0;
    if (kept_all == 2) c->status = ST_DONE;
  }
  c->mark[2] = globaltimer_ns() - c->t0_ns;
  __threadfence();
}

// ===========================================================================
// KS: small inputs (n <= SMALL_N) -- K1 + K2 + the round-0 compaction in ONE
// CTA, handing a dense live set straight to the round kernel at round 1.
// Used for the shard-hull merge of the multi-GPU path (~50 x N points) and
// other tiny inputs, where four launches and multi-CTA tails dominate.
// ===========================================================================

template <bool FILTER, bool IDS>
__global__ void __launch_bounds__(1024, 1) k_small_pre(Bufs B) {
  Ctl* c = B.ctl;
  const uint32_t n = B.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  if (threadIdx.x == 0) c->t0_ns = globaltimer_ns();

  // ---- extremes (hull.cpp:25-45); indices grow within a thread ----
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  ExtRec e[4];
  e[0].x = INF;  e[0].y = INF;
  e[1].x = -INF; e[1].y = INF;
  e[2].x = -INF; e[2].y = -INF;
  e[3].x = INF;  e[3].y = -INF;
  for (int k = 0; k < 4; ++k) e[k].id = e[k].pos = NONE;
  unsigned long long bad = ~0ull;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
    ext_visit<IDS>(e, bad, __ldg(X + i), __ldg(Y + i), IDS ? __ldg(I + i) : i, i);
  block_reduce_ext(e, bad);
  if (threadIdx.x == 0) finalize_extremes(B, e, bad);
  __syncthreads();
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;

  // ---- filter + classes + round-0 farthest + dense member list (K2) ----
  const uint32_t p0 = c->ext_pos[0], pr = c->ext_pos[2];
  const double x0 = c->ext_x[0], y0 = c->ext_y[0], xr = c->ext_x[2], yr = c->ext_y[2];
  const Edge E01 = make_edge(x0, y0, xr, yr);
  const Edge E10 = make_edge(xr, yr, x0, y0);
  const bool filt = FILTER && c->distinct >= 3;
  const int ne = filt ? c->nedges : 0;
  Edge Q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Q[k].ax = c->edges[k][0];
    Q[k].ay = c->edges[k][1];
    Q[k].ex = c->edges[k][2];
    Q[k].ey = c->edges[k][3];
  }
  __shared__ uint32_t s_off;
  __shared__ Cand s_a[2][MAXW];
  __shared__ uint32_t s_kept[MAXW];
  if (threadIdx.x == 0) s_off = 0;
  __syncthreads();
  double2* Oxy = B.Lxy[0];
  uint2* Ois = B.Lis[0];
  Cand a0 = empty_cand(), a1 = empty_cand();
  uint32_t kept = 0;
  bool noncol = false;
  for (uint32_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const uint32_t i = b0 + threadIdx.x;
    const bool valid = i < n;
    double x = 0.0, y = 0.0;
    uint32_t id = 0;
    if (valid) {
      x = __ldg(X + i);
      y = __ldg(Y + i);
      id = IDS ? __ldg(I + i) : i;
    }
    const double cl = cross_e(E01, x, y);  // cross(P0, Pr, p)
    bool inside = false;
    if (filt) {  // hull.cpp:80-90
      inside = valid;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
        if (qq < ne) inside = inside && (cross_e(Q[qq], x, y) > 0.0);
    }
    const bool keep = valid && !inside;
    kept += keep;
    noncol = noncol || (valid && cl != 0.0);
    const bool member = keep && i != p0 && i != pr;
    const bool lw = member && cl < 0.0;  // hull.cpp:115-117
    if (lw) cand_visit(a0, -cl, x, y, id, i, true);
    else if (member) cand_visit(a1, outward_e(E10, x, y), x, y, id, i, false);
    // dense append: seg 0 = lower chain, 1 = upper chain
    const uint32_t bal = __ballot_sync(FULL, member);
    uint32_t off = 0;
    if (lane == 0 && bal) off = atomicAdd(&s_off, (uint32_t)__popc(bal));
    off = __shfl_sync(FULL, off, 0);
    if (member) {
      const uint32_t p = off + __popc(bal & lanemask_lt());
      Oxy[p] = make_double2(x, y);
      Ois[p] = make_uint2(id, lw ? 0u : 1u);
    }
  }
  a0 = warp_best(a0, true);
  a1 = warp_best(a1, false);
  const bool nc_any = __any_sync(FULL, noncol);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) kept += __shfl_xor_sync(FULL, kept, m);
  if (lane == 0) {
    s_a[0][warp] = a0;
    s_a[1][warp] = a1;
    s_kept[warp] = kept | (nc_any ? 0x80000000u : 0u);
  }
  __syncthreads();
  if (warp != 0) return;
  const int nwb = blockDim.x >> 5;
  a0 = lane < nwb ? s_a[0][lane] : empty_cand();
  a1 = lane < nwb ? s_a[1][lane] : empty_cand();
  a0 = warp_best(a0, true);
  a1 = warp_best(a1, false);
  if (lane != 0) return;
  unsigned long long kb = 0;
  bool nc = false;
  for (int w = 0; w < nwb; ++w) {
    kb += s_kept[w] & 0x7FFFFFFFu;
    nc = nc || (s_kept[w] >> 31);
  }
  const uint32_t m = s_off;
  c->kept = kb;
  // round-1 farthest records (Slot[0]) and cleared round-1 offer slots (Slot[1])
  const Cand* ab[2] = {&a0, &a1};
  for (int t = 0; t < 2; ++t) {
    rec_clear(&B.Sd[0][t], &B.Srec[0][t]);
    if (ab[t]->d > 0.0) {
      B.Sd[0][t] = (unsigned long long)__double_as_longlong(ab[t]->d);
      B.Srec[0][t].d = ab[t]->d;
      B.Srec[0][t].x = ab[t]->x;
      B.Srec[0][t].y = ab[t]->y;
      B.Srec[0][t].id = ab[t]->id;
    }
  }
  for (int t = 0; t < 4; ++t) rec_clear(&B.Sd[1][t], &B.Srec[1][t]);
  if (!nc) {
    c->status = ST_COLLINEAR;  // hull.cpp:238-248
  } else {
    B.Tx[0][0] = x0;
    B.Ty[0][0] = y0;
    B.Tid[0][0] = c->ext_id[0];
    B.Tx[0][1] = xr;
    B.Ty[0][1] = yr;
    B.Tid[0][1] = c->ext_id[2];
    if (m & 1u) {  // pad the run to an even length
      Oxy[m] = make_double2(0.0, 0.0);
      Ois[m] = make_uint2(NONE, NONE);
    }
    B.run_cnt[0][0] = m;
    c->nruns = 1;
    c->S_cur = 2;
    c->Slo_cur = 1;
    c->m_cur = m;
    c->round = 0;
    if (m == 0) c->status = ST_DONE;
  }
  c->mark[2] = globaltimer_ns() - c->t0_ns;
  c->mark[4] = c->mark[2];
  __threadfence();
}

// ===========================================================================
// host-side launch wrappers
// ===========================================================================

template <bool IDS>
using Ring2 = TileRing<Cfg2::T, Cfg2::NS, IDS, 0, Cfg2::CW>;

cudaError_t configure_stream_kernels_pre() {
  cudaError_t e;
  e = cudaFuncSetAttribute(k1_extremes<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring1<false>::kBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k1_extremes<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring1<true>::kBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k2_classify<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring2<false>::kBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k2_classify<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring2<false>::kBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k2_classify<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring2<true>::kBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k2_classify<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ring2<true>::kBytes);
}

void launch_small(const Bufs& B, bool filter, bool ids, cudaStream_t s) {
  if (filter) {
    if (ids) k_small_pre<true, true><<<1, 1024, 0, s>>>(B);
    else k_small_pre<true, false><<<1, 1024, 0, s>>>(B);
  } else {
    if (ids) k_small_pre<false, true><<<1, 1024, 0, s>>>(B);
    else k_small_pre<false, false><<<1, 1024, 0, s>>>(B);
  }
}

void launch_k1(const Bufs& B, bool ids, int grid, cudaStream_t s) {
  if (ids) k1_extremes<true><<<grid, Cfg1::TPB, Ring1<true>::kBytes, s>>>(B);
  else k1_extremes<false><<<grid, Cfg1::TPB, Ring1<false>::kBytes, s>>>(B);
}

// launch with programmatic stream serialization (PDL): the kernel's own
// griddepcontrol.wait orders it after its predecessor
template <class K>
static cudaError_t launch_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t s,
                              const Bufs& B, bool cooperative = false) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  if (cooperative) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, B);
}

void launch_k2(const Bufs& B, bool filter, bool ids, int grid, cudaStream_t s) {
  if (filter) {
    if (ids) launch_pdl(k2_classify<true, true>, grid, Cfg2::TPB, Ring2<true>::kBytes, s, B);
    else launch_pdl(k2_classify<true, false>, grid, Cfg2::TPB, Ring2<false>::kBytes, s, B);
  } else {
    if (ids) launch_pdl(k2_classify<false, true>, grid, Cfg2::TPB, Ring2<true>::kBytes, s, B);
    else launch_pdl(k2_classify<false, false>, grid, Cfg2::TPB, Ring2<false>::kBytes, s, B);
  }
}

}  // namespace shb
