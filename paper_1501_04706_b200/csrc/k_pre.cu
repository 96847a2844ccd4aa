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

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

// ===========================================================================
// helpers
// ===========================================================================

SH_DEV bool nonfinite(double v) {
  return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}

// pair q = points (2q, 2q+1) of a SoA array
template <bool VEC>
SH_DEV double2 load_pair(const double* __restrict__ a, uint32_t q) {
  if (VEC) return __ldg(reinterpret_cast<const double2*>(a) + q);
  return make_double2(__ldg(a + 2 * q), __ldg(a + 2 * q + 1));
}

template <bool VEC>
SH_DEV uint2 load_pair_id(const uint32_t* __restrict__ a, uint32_t q) {
  if (VEC) return __ldg(reinterpret_cast<const uint2*>(a) + q);
  return make_uint2(__ldg(a + 2 * q), __ldg(a + 2 * q + 1));
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
  __shared__ ExtRec s_e[4][WARPS];
  __shared__ unsigned long long s_bad[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_reduce_ext(e, bad);
  if (lane == 0) {
    for (int k = 0; k < 4; ++k) s_e[k][warp] = e[k];
    s_bad[warp] = bad;
  }
  __syncthreads();
  if (warp == 0) {
    for (int k = 0; k < 4; ++k) {
      if (lane < WARPS) {
        e[k] = s_e[k][lane];
      } else {
        e[k].pos = NONE;
      }
    }
    bad = lane < WARPS ? s_bad[lane] : ~0ull;
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

constexpr int K1_U = 4;  // pairs per thread per iteration: 4 x 2 x 16 B in flight

template <bool IDS, bool VEC>
__global__ void __launch_bounds__(TPB) k1_extremes(Bufs B) {
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

  const uint32_t npairs = n >> 1;
  const uint32_t stride = gridDim.x * TPB;
  uint32_t q = blockIdx.x * TPB + threadIdx.x;
  for (; q + (K1_U - 1) * stride < npairs; q += K1_U * stride) {
    double2 xv[K1_U], yv[K1_U];
    uint2 iv[K1_U];
#pragma unroll
    for (int u = 0; u < K1_U; ++u) {
      xv[u] = load_pair<VEC>(X, q + u * stride);
      yv[u] = load_pair<VEC>(Y, q + u * stride);
      if (IDS) iv[u] = load_pair_id<VEC>(I, q + u * stride);
    }
#pragma unroll
    for (int u = 0; u < K1_U; ++u) {
      const uint32_t p = 2 * (q + u * stride);
      ext_visit<IDS>(e, bad, xv[u].x, yv[u].x, IDS ? iv[u].x : p, p);
      ext_visit<IDS>(e, bad, xv[u].y, yv[u].y, IDS ? iv[u].y : p + 1, p + 1);
    }
  }
  for (; q < npairs; q += stride) {
    const double2 xv = load_pair<VEC>(X, q), yv = load_pair<VEC>(Y, q);
    const uint32_t p = 2 * q;
    ext_visit<IDS>(e, bad, xv.x, yv.x, IDS ? __ldg(I + p) : p, p);
    ext_visit<IDS>(e, bad, xv.y, yv.y, IDS ? __ldg(I + p + 1) : p + 1, p + 1);
  }
  if ((n & 1u) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t p = n - 1;
    ext_visit<IDS>(e, bad, __ldg(X + p), __ldg(Y + p), IDS ? __ldg(I + p) : p, p);
  }

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
  for (uint32_t p = threadIdx.x; p < gridDim.x; p += TPB) {
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

  c->ticket = 0;
  c->bad_index = bad;
  // round-0 farthest slots (K2 offers into Slot[0]; hull_kernels.cuh)
  B.Sd[0][0] = 0ull;
  B.Sd[0][1] = 0ull;
  B.Sw[0][0] = NONE;
  B.Sw[0][1] = NONE;
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
}

// ===========================================================================
// K2: filter + classification + round-0 farthest points (no point writes).
// ===========================================================================

constexpr int K2_U = 2;  // 64-point chunks per warp per iteration (8 x 16 B per lane in flight)

SH_DEV void cand_visit(Cand& a, double d, double x, double y, uint32_t id, uint32_t pos,
                       bool lower) {
  if (d > 0.0 && d >= a.d) {
    Cand cc;
    cc.d = d; cc.x = x; cc.y = y; cc.id = id; cc.pos = pos;
    if (cand_better(cc, a, lower)) a = cc;
  }
}

template <bool FILTER, bool IDS, bool VEC>
__global__ void __launch_bounds__(TPB) k2_classify(Bufs B) {
  Ctl* c = B.ctl;
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
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
  const uint32_t nchunks = (n + 63) >> 6;
  const uint32_t nw = gridDim.x * WARPS;
  Cand a0 = empty_cand(), a1 = empty_cand();
  uint32_t kept = 0;
  bool noncol = false;

  for (uint32_t k0 = blockIdx.x * WARPS + warp; k0 < nchunks; k0 += K2_U * nw) {
    double2 xv[K2_U], yv[K2_U];
    uint2 iv[K2_U];
    uint32_t cidx[K2_U];
#pragma unroll
    for (int u = 0; u < K2_U; ++u) {
      const uint32_t k = k0 + u * nw;
      cidx[u] = k < nchunks ? nchunks - 1 - k : NONE;  // backwards over the input
      xv[u] = yv[u] = make_double2(0.0, 0.0);
      iv[u] = make_uint2(0u, 0u);
      if (cidx[u] != NONE) {
        const uint32_t q = cidx[u] * 32 + lane;  // pair index
        if (2 * q + 1 < n) {
          xv[u] = load_pair<VEC>(X, q);
          yv[u] = load_pair<VEC>(Y, q);
          if (IDS) iv[u] = load_pair_id<VEC>(I, q);
        } else if (2 * q < n) {
          xv[u].x = __ldg(X + 2 * q);
          yv[u].x = __ldg(Y + 2 * q);
          if (IDS) iv[u].x = __ldg(I + 2 * q);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < K2_U; ++u) {
      if (cidx[u] == NONE) continue;  // warp-uniform
      uint32_t lo2 = 0, up2 = 0, kp2 = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t i = cidx[u] * 64 + 2 * lane + h;
        const bool valid = i < n;
        const double x = h ? xv[u].y : xv[u].x;
        const double y = h ? yv[u].y : yv[u].x;
        const double cl = cross_e(E01, x, y);
        bool inside = false;
        if (filt) {  // hull.cpp:80-90: discard iff cross > 0 for every edge
          inside = valid;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            if (qq < ne) inside = inside && (cross_e(Q[qq], x, y) > 0.0);
        }
        const bool keep = valid && !inside;
        noncol = noncol || (valid && cl != 0.0);
        const bool member = keep && i != p0 && i != pr;
        const bool lw = member && cl < 0.0;  // hull.cpp:115-117
        const bool up = member && !(cl < 0.0);
        lo2 |= (uint32_t)lw << h;
        up2 |= (uint32_t)up << h;
        kp2 |= (uint32_t)keep << h;
        const uint32_t id = IDS ? (h ? iv[u].y : iv[u].x) : i;
        if (lw) {
          cand_visit(a0, -cl, x, y, id, i, true);  // outward_distance(P0, Pr, p)
        } else if (up) {
          cand_visit(a1, outward_e(E10, x, y), x, y, id, i, false);  // outward_distance(Pr, P0, p)
        }
      }
      const uint32_t le = __ballot_sync(FULL, lo2 & 1u), lodd = __ballot_sync(FULL, lo2 & 2u);
      const uint32_t ue = __ballot_sync(FULL, up2 & 1u), uodd = __ballot_sync(FULL, up2 & 2u);
      kept += __popc(kp2);
      if (lane == 0) B.bits[cidx[u]] = make_uint4(le, lodd, ue, uodd);
    }
  }

  // block reduction of the two chains' farthest candidates
  __shared__ Cand s_a[2][WARPS];
  __shared__ uint32_t s_kept[WARPS];
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
    a0 = lane < WARPS ? s_a[0][lane] : empty_cand();
    a1 = lane < WARPS ? s_a[1][lane] : empty_cand();
    a0 = warp_best(a0, true);
    a1 = warp_best(a1, false);
    if (lane == 0) {
      unsigned long long kb = 0;
      bool nc = false;
      for (int w = 0; w < WARPS; ++w) {
        kb += s_kept[w] & 0x7FFFFFFFu;
        nc = nc || (s_kept[w] >> 31);
      }
      if (kb) atomicAdd(&c->kept, kb);
      if (nc) atomicOr(&c->noncollinear, 1u);
      const LoadSoA ld{X, Y, I};
      if (a0.d > 0.0) slot_offer(&B.Sd[0][0], &B.Sw[0][0], a0, true, E01, ld);
      if (a1.d > 0.0) slot_offer(&B.Sd[0][1], &B.Sw[0][1], a1, false, E10, ld);
      __threadfence();
      s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  c->ticket = 0;
  // round-1 farthest slots (round 1 offers into Slot[1]; its table has <= 4 entries)
  for (int t = 0; t < 4; ++t) {
    B.Sd[1][t] = 0ull;
    B.Sw[1][t] = NONE;
  }
  c->out_cnt[1] = 0;
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
  __threadfence();
}

// ===========================================================================
// host-side launch wrappers
// ===========================================================================

void launch_k1(const Bufs& B, bool ids, bool vec, int grid, cudaStream_t s) {
  if (ids) {
    if (vec) k1_extremes<true, true><<<grid, TPB, 0, s>>>(B);
    else k1_extremes<true, false><<<grid, TPB, 0, s>>>(B);
  } else {
    if (vec) k1_extremes<false, true><<<grid, TPB, 0, s>>>(B);
    else k1_extremes<false, false><<<grid, TPB, 0, s>>>(B);
  }
}

template <bool FILTER>
static void launch_k2_t(const Bufs& B, bool ids, bool vec, int grid, cudaStream_t s) {
  if (ids) {
    if (vec) k2_classify<FILTER, true, true><<<grid, TPB, 0, s>>>(B);
    else k2_classify<FILTER, true, false><<<grid, TPB, 0, s>>>(B);
  } else {
    if (vec) k2_classify<FILTER, false, true><<<grid, TPB, 0, s>>>(B);
    else k2_classify<FILTER, false, false><<<grid, TPB, 0, s>>>(B);
  }
}

int k1_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_extremes<false, true>, TPB, 0);
  return b < 1 ? 1 : b;
}

int k2_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k2_classify<true, false, true>, TPB, 0);
  return b < 1 ? 1 : b;
}

void launch_k2(const Bufs& B, bool filter, bool ids, bool vec, int grid, cudaStream_t s) {
  if (filter) launch_k2_t<true>(B, ids, vec, grid, s);
  else launch_k2_t<false>(B, ids, vec, grid, s);
}

}  // namespace shb
