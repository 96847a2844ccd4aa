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

// The extremes' consequences (hull.cpp:222-237 statuses, hull.cpp:58-74
// quadrilateral), computed from the four extremes and the first bad index.
struct Fin {
  uint32_t status;
  int distinct, nedges;
  unsigned long long bad;
  ExtRec e[4];
  double edges[4][4];  // (ax, ay, ex, ey)
};

SH_DEV void compute_fin(Fin& f, const ExtRec (&e)[4], unsigned long long bad) {
  f.status = ST_RUNNING;
  f.bad = bad;
  f.distinct = 0;
  f.nedges = 0;
  for (int k = 0; k < 4; ++k) {
    f.e[k] = e[k];
    for (int j = 0; j < 4; ++j) f.edges[k][j] = 0.0;
  }
  if (bad != ~0ull) {
    f.status = ST_NONFINITE;
    return;
  }
  if (e[0].x == e[2].x && e[0].y == e[2].y) {  // hull.cpp:234-237
    f.status = ST_SINGLE;
    return;
  }
  // corners [left, bottom, right, top], distinct count and the edges between
  // consecutive non-equal corners (with wrap-around)
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
      f.edges[ne][0] = ed.ax;
      f.edges[ne][1] = ed.ay;
      f.edges[ne][2] = ed.ex;
      f.edges[ne][3] = ed.ey;
      ++ne;
    }
  }
  f.distinct = distinct;
  f.nedges = ne;
}

// one thread publishes Fin in the control block (later kernels, the host)
SH_DEV void write_fin(Ctl* c, const Fin& f) {
  c->bad_index = f.bad;
  for (int k = 0; k < 4; ++k) {
    c->ext_x[k] = f.e[k].x;
    c->ext_y[k] = f.e[k].y;
    c->ext_id[k] = f.e[k].id;
    c->ext_pos[k] = f.e[k].pos;
    for (int j = 0; j < 4; ++j) c->edges[k][j] = f.edges[k][j];
  }
  c->distinct = f.distinct;
  c->nedges = f.nedges;
  if (f.status != ST_RUNNING) c->status = f.status;
}

// Thread 0 of a single-CTA path: extremes -> control block.
SH_DEV void finalize_extremes(const Bufs& B, const ExtRec (&e)[4], unsigned long long bad) {
  Ctl* c = B.ctl;
  Fin f;
  compute_fin(f, e, bad);
  write_fin(c, f);
  c->mark[0] = globaltimer_ns() - c->t0_ns;
}

// Lexicographic keys (smaller is better) of the four directional extremes
// (hull.cpp:25-45): left = min x, min y; bottom = min y, max x; right = max x,
// max y; top = max y, min x; then the id (caller id or index), then the index.
SH_DEV void ext_keys(const ExtRec (&e)[4], unsigned long long (&key)[4][3], bool (&valid)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned long long kx = fkey(e[k].x), ky = fkey(e[k].y);
    key[k][0] = k == 0 ? kx : k == 1 ? ky : k == 2 ? ~kx : ~ky;
    key[k][1] = k == 0 ? ky : k == 1 ? ~kx : k == 2 ? ~ky : kx;
    key[k][2] = ((unsigned long long)e[k].id << 32) | e[k].pos;
    valid[k] = e[k].pos != NONE;
  }
}

// CTA-wide extremes + first bad index of the records the threads hold; the
// winners are copied to out[] (shared or global), a direction without any
// record gets pos = NONE.  Contains barriers.
SH_DEV void cta_extremes(const ExtRec (&e)[4], unsigned long long bad, ExtRec* out,
                         unsigned long long* out_bad) {
  __shared__ unsigned long long s_best[4][3];
  __shared__ unsigned long long s_bad;
  unsigned long long key[4][3];
  bool valid[4], win[4];
  ext_keys(e, key, valid);
  if (threadIdx.x == 0) s_bad = ~0ull;
  cta_lexmin<4, 3>(key, valid, s_best, win);  // starts with a barrier
  if (bad != ~0ull) atomicMin(&s_bad, bad);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (win[k]) out[k] = e[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k)
      if (s_best[k][0] == ~0ull) out[k].pos = NONE;
    *out_bad = s_bad;
  }
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
  if (threadIdx.x == 0 && c->tl_round == 255u) B.dbg[blockIdx.x] = globaltimer_ns() - c->t0_ns;

  // this CTA's extremes -> its partial (the next kernel combines them)
  K1Partial* part = B.k1part + blockIdx.x;
  cta_extremes(e, bad, part->e, &part->bad);
  SHB_PROBE(if (threadIdx.x == 0 && c->tl_round == 255u) B.dbg[1024 + blockIdx.x] = globaltimer_ns());
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

// Every CTA of the kernel after K1 combines K1's per-CTA extremes into the
// quadrilateral (Fin, in shared memory); with `publish`, CTA 0 also writes it
// to the control block and clears round 1's farthest slots.  Contains barriers.
SH_DEV void combine_k1(const Bufs& B, Fin& s_fin, bool publish) {
  Ctl* c = B.ctl;
  ExtRec e[4];
  unsigned long long bad = ~0ull;
  for (int k = 0; k < 4; ++k) e[k].id = e[k].pos = NONE;
  if (threadIdx.x < B.k1_grid) {
    const K1Partial* qp = B.k1part + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e[k].x = __ldcg(&qp->e[k].x);
      e[k].y = __ldcg(&qp->e[k].y);
      e[k].id = __ldcg(&qp->e[k].id);
      e[k].pos = __ldcg(&qp->e[k].pos);
    }
    bad = __ldcg(&qp->bad);
  }
  __shared__ ExtRec s_ext[4];
  __shared__ unsigned long long s_bad;
  SHB_PROBE(const bool probe = blockIdx.x == 0 && threadIdx.x == 0 && c->tl_round == 255u);
  SHB_PROBE(if (probe) B.dbg[1608] = globaltimer_ns() + (unsigned long long)(e[0].x == -1.0));
  cta_extremes(e, bad, s_ext, &s_bad);
  __syncthreads();
  SHB_PROBE(if (probe) B.dbg[1609] = globaltimer_ns());
  if (threadIdx.x == 0) {
    const ExtRec ee[4] = {s_ext[0], s_ext[1], s_ext[2], s_ext[3]};
    compute_fin(s_fin, ee, s_bad);
    if (publish && blockIdx.x == 0) {
      write_fin(c, s_fin);
      SHB_PROBE(if (c->tl_round == 255u) B.dbg[1610] = globaltimer_ns());
      const unsigned long long now = globaltimer_ns() - c->t0_ns;
      c->mark[0] = now;
      c->mark[1] = now;
      // round 1 (K3) offers its farthest points into Slot[1] (<= 4 segments)
      for (int t = 0; t < 4; ++t) rec_clear(&B.Sd[1][t], &B.Srec[1][t]);
    }
  }
  __syncthreads();
}

template <bool FILTER, bool IDS>
__global__ void __launch_bounds__(Cfg2::TPB, 1) k2_classify(Bufs B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileRing<Cfg2::T, Cfg2::NS, IDS, 0, Cfg2::CW> R;
  R.carve(smem_raw);
  Ctl* c = B.ctl;
#ifndef SHB_K2_REVERSE
#define SHB_K2_REVERSE 1
#endif
  // CTA-wide running maxima of the two chains' distances (positive doubles
  // order like their bits): a point below them cannot be the CTA's farthest,
  // so the per-point candidate branch is almost never taken
  __shared__ unsigned long long s_dmax[2];
  if (threadIdx.x == 0) {
    R.init();
    s_dmax[0] = s_dmax[1] = 0ull;
  }
  __syncthreads();
  // the points do not depend on K1: start the ring before waiting for it
  const uint32_t pre = stream_prefetch(R, B.n, B.in_x, B.in_y, B.in_id, SHB_K2_REVERSE != 0, true);
  SHB_PROBE(const bool probe = blockIdx.x == 0 && threadIdx.x == 0 && c->tl_round == 255u);
  SHB_PROBE(if (probe) B.dbg[1600] = globaltimer_ns());
  pdl_wait();               // K1's partial extremes are complete and visible
  SHB_PROBE(if (probe) B.dbg[1601] = globaltimer_ns());
  pdl_launch_dependents();  // K3 may be scheduled on SMs this kernel frees
  // ---- every CTA combines K1's per-CTA extremes (no serial last-CTA step) ----
  __shared__ Fin s_fin;
  combine_k1(B, s_fin, true);
  if (s_fin.status != ST_RUNNING) {
    stream_drain(R, pre);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  const uint32_t p0 = s_fin.e[0].pos, pr = s_fin.e[2].pos;
  const double x0 = s_fin.e[0].x, y0 = s_fin.e[0].y, xr = s_fin.e[2].x, yr = s_fin.e[2].y;
  const Edge E01 = make_edge(x0, y0, xr, yr);  // lower chain base line P0 -> Pr
  const Edge E10 = make_edge(xr, yr, x0, y0);  // upper chain base line Pr -> P0 (wrap)
  const bool filt = FILTER && s_fin.distinct >= 3;
  const int ne = filt ? s_fin.nedges : 0;
  Edge Q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Q[k].ax = s_fin.edges[k][0];
    Q[k].ay = s_fin.edges[k][1];
    Q[k].ex = s_fin.edges[k][2];
    Q[k].ey = s_fin.edges[k][3];
  }
  Cand a0 = empty_cand(), a1 = empty_cand();
  uint32_t kept = 0;
  bool noncol = false;

  // With 4 distinct corners, edge q starts at corner q (left, bottom, right,
  // top) and the chain base lines start at left (P0) and right (Pr), so the
  // per-point differences p - corner are shared by the 6 cross products:
  // the same RN operations as cross() (geometry.hpp:17-19), computed once.
  const bool quad4 = filt && ne == 4 && s_fin.distinct == 4;
  const double cxL = s_fin.e[0].x, cyL = s_fin.e[0].y, cxB = s_fin.e[1].x, cyB = s_fin.e[1].y;
  const double cxR = s_fin.e[2].x, cyR = s_fin.e[2].y, cxT = s_fin.e[3].x, cyT = s_fin.e[3].y;
  auto xprod = [](double ex, double ey, double dx, double dy) {
    return __dsub_rn(__dmul_rn(ex, dy), __dmul_rn(ey, dx));
  };

  // backwards over the input: K1 just left the tail in L2, K3 starts at the head
  constexpr int NCH = Cfg2::T / 64 / Cfg2::CW;  // chunks per consumer warp per tile
  constexpr int NP = 2 * NCH;                  // points per thread per tile
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
      // outward_distance(Pr, P0, p) = -cross: RN is symmetric, so swapping the
      // products gives the same value (up to the sign of a zero, which the
      // d > 0 tests ignore) without the extra negation
      du[q] = __dsub_rn(__dmul_rn(E10.ey, dxR), __dmul_rn(E10.ex, dyR));
      bool inside = false;
      if (QK == 1 || QK == 3) {  // hull.cpp:80-90: discard iff no cross <= 0
        const double dxB = __dsub_rn(x, cxB), dyB = __dsub_rn(y, cyB);
        const double dxT = __dsub_rn(x, cxT), dyT = __dsub_rn(y, cyT);
        const double q0 = xprod(Q[0].ex, Q[0].ey, dxL, dyL), q1 = xprod(Q[1].ex, Q[1].ey, dxB, dyB);
        const double q2 = xprod(Q[2].ex, Q[2].ey, dxR, dyR), q3 = xprod(Q[3].ex, Q[3].ey, dxT, dyT);
        if (QK == 3)  // a wide box: a product may overflow and a cross be NaN, which the
                      // reference's `cross <= 0` test counts as inside
          inside = !(q0 <= 0.0) & !(q1 <= 0.0) & !(q2 <= 0.0) & !(q3 <= 0.0);
        else          // every product is finite: no NaN, and > 0 is the same test
          inside = (q0 > 0.0) & (q1 > 0.0) & (q2 > 0.0) & (q3 > 0.0);
      } else if (QK == 2) {  // degenerate quadrilateral (3 distinct corners)
        inside = true;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          if (qq < ne) inside = inside & !(cross_e(Q[qq], x, y) <= 0.0);
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
    }, pre);
  };
  // box extents below 2^500: every product of two coordinate differences is finite
  const bool wide = !(((s_fin.e[2].x - s_fin.e[0].x) + (s_fin.e[3].y - s_fin.e[1].y)) < 0x1p500);
  if (quad4 && wide)
    pass(std::integral_constant<int, 3>{});
  else if (quad4)
    pass(std::integral_constant<int, 1>{});
  else if (filt)
    pass(std::integral_constant<int, 2>{});
  else
    pass(std::integral_constant<int, 0>{});
  if (threadIdx.x == 0 && c->tl_round == 255u) B.dbg[256 + blockIdx.x] = globaltimer_ns() - c->t0_ns;

  // this CTA's farthest candidates of both chains, kept count and
  // collinearity -> its partial (K3 combines the partials)
  {
    __shared__ unsigned long long s_best2[2][4];
    __shared__ unsigned long long s_kb;
    __shared__ uint32_t s_nc;
    unsigned long long key[2][4];
    bool valid[2], win[2];
    cand_keys(a0, true, key[0]);
    cand_keys(a1, false, key[1]);
    valid[0] = a0.d > 0.0;
    valid[1] = a1.d > 0.0;
    if (threadIdx.x == 0) {
      s_kb = 0;
      s_nc = 0;
    }
    cta_lexmin<2, 4>(key, valid, s_best2, win);  // starts with a barrier
    const uint32_t wk = __reduce_add_sync(FULL, kept);
    const bool wnc = __any_sync(FULL, noncol);
    if (lane == 0) {
      if (wk) atomicAdd(&s_kb, (unsigned long long)wk);
      if (wnc) s_nc = 1u;
    }
    K2Partial* part = B.k2part + blockIdx.x;
    if (win[0]) part->a[0] = a0;
    if (win[1]) part->a[1] = a1;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_best2[0][0] == ~0ull) part->a[0] = empty_cand();
      if (s_best2[1][0] == ~0ull) part->a[1] = empty_cand();
      part->kept = s_kb;
      part->noncol = s_nc;
      if (blockIdx.x == 0) c->mark[2] = globaltimer_ns() - c->t0_ns;
      SHB_PROBE(if (c->tl_round == 255u) B.dbg[1200 + blockIdx.x] = globaltimer_ns());
    }
  }
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
  const uint32_t n = B.n_dev ? *B.n_dev : B.n;  // the merge input's count is device-written
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
  {
    __shared__ ExtRec s_ext[4];
    __shared__ unsigned long long s_bad;
    cta_extremes(e, bad, s_ext, &s_bad);
    __syncthreads();
    if (threadIdx.x == 0) {
      const ExtRec ee[4] = {s_ext[0], s_ext[1], s_ext[2], s_ext[3]};
      finalize_extremes(B, ee, s_bad);
    }
    __syncthreads();
  }
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
        if (qq < ne) inside = inside && !(cross_e(Q[qq], x, y) <= 0.0);
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
  for (int t = 0; t < 4; ++t) {
    rec_clear(&B.Sd[1][t], &B.Srec[1][t]);
    B.Wn[1][t] = NONE;  // round 1 runs in the round kernel
  }
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

// ===========================================================================
// KP: hull::preprocess as a device API (hull.hpp:61-64, hull.cpp:53-99):
// K1's extremes, then every point outside the quadrilateral's strict interior
// is kept, compacted STABLY (input order, like stable_partition_by_flag) with
// a decoupled look-back over 2048-point tiles taken from a tile counter.
// Degenerate quadrilaterals (< 3 distinct corners) keep every point.
// ===========================================================================

constexpr int KP_TPB = 256, KP_ITEMS = 8, KP_TILE = KP_TPB * KP_ITEMS;

__global__ void __launch_bounds__(KP_TPB) k_preprocess(Bufs B, double* ox, double* oy,
                                                        unsigned long long cap) {
  Ctl* c = B.ctl;
  __shared__ Fin s_fin;
  combine_k1(B, s_fin, false);
  const uint32_t st = s_fin.status;
  if (st == ST_NONFINITE) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      c->status = ST_NONFINITE;
      c->bad_index = s_fin.bad;
    }
    return;
  }
  const bool filt = st == ST_RUNNING && s_fin.distinct >= 3;
  const int ne = filt ? s_fin.nedges : 0;
  Edge Q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Q[k].ax = s_fin.edges[k][0];
    Q[k].ay = s_fin.edges[k][1];
    Q[k].ex = s_fin.edges[k][2];
    Q[k].ey = s_fin.edges[k][3];
  }
  __shared__ uint32_t s_cnt[KP_ITEMS * (KP_TPB / 32)];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int W = KP_TPB / 32;
  const uint32_t epoch = *(volatile uint32_t*)B.epoch;
  const uint32_t n = B.n;
  const uint32_t ntiles = (n + KP_TILE - 1) / KP_TILE;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    double px[KP_ITEMS], py[KP_ITEMS];
    uint32_t keep = 0, rank[KP_ITEMS];
#pragma unroll
    for (int j = 0; j < KP_ITEMS; ++j) {
      const uint32_t i = tile * KP_TILE + j * KP_TPB + threadIdx.x;
      if (i < n) {
        px[j] = __ldcs(B.in_x + i);
        py[j] = __ldcs(B.in_y + i);
        bool inside = filt;  // hull.cpp:80-90: discard iff cross > 0 for every edge
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < ne) inside = inside & !(cross_e(Q[k], px[j], py[j]) <= 0.0);
        if (!inside) keep |= 1u << j;
      }
      const unsigned bal = __ballot_sync(FULL, (keep >> j) & 1u);
      if (lane == 0) s_cnt[j * W + warp] = __popc(bal);
      rank[j] = __popc(bal & lanemask_lt());
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the KP_ITEMS x W warp counts (j-major)
      uint32_t v[KP_ITEMS * W / 32];
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < KP_ITEMS * W / 32; ++q) {
        v[q] = s_cnt[lane * (KP_ITEMS * W / 32) + q];
        sum += v[q];
      }
      uint32_t incl = sum;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int q = 0; q < KP_ITEMS * W / 32; ++q) {
        s_cnt[lane * (KP_ITEMS * W / 32) + q] = run;
        run += v[q];
      }
      const uint32_t agg = __shfl_sync(FULL, incl, 31);
      const uint32_t p = lookback_warp(B.tile_status, tile, agg, epoch);
      if (lane == 0) {
        s_prefix = p;
        if (tile == ntiles - 1) c->m_next = p + agg;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KP_ITEMS; ++j) {
      if ((keep >> j) & 1u) {
        const unsigned long long o = (unsigned long long)s_prefix + s_cnt[j * W + warp] + rank[j];
        if (o < cap) {
          ox[o] = px[j];
          oy[o] = py[j];
        }
      }
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    c->ticket = 0;
    c->tile_ctr = 0;
    *B.epoch = epoch + 1;
    __threadfence();
  }
}

void launch_preprocess(const Bufs& B, double* ox, double* oy, unsigned long long cap, int grid,
                       cudaStream_t s) {
  k_preprocess<<<grid, KP_TPB, 0, s>>>(B, ox, oy, cap);
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
