// hull_kernels.cu -- sm_100a kernels of the segment-based 2D QuickHull.
//
// Pipeline:
//   K1 k1_extremes     extremes + finite check           (hull.cpp:25-45, 221-237)
//   K2 k2_classify     quad filter + collinear flag + chain class + round-0
//                      distance + farthest point of both chains, no writes
//                      of points (hull.cpp:53-99, 101-158, 160-184, 238-248)
//   K3 k3_route<true>  round 1 straight from the input: route each member to
//                      A->C or C->B by lex order against C, keep iff strictly
//                      outside, stable single-pass compaction, fused farthest
//                      point of the next round (hull.cpp:186-217)
//   K4 k4_table        segment-table update (exclusive scan of "splittable")
//                      for large tables; small tables are built by the last
//                      block of the preceding kernel (build_table_block)
//   K3 k3_route<false> every later round on the compacted live set
// All round bookkeeping stays in the device control block (Ctl).
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

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

SH_DEV bool finite_bits(double v) {
  return (((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FFull) != 0x7FFull;
}

__global__ void __launch_bounds__(TPB) k1_extremes(Bufs B) {
  Ctl* c = B.ctl;
  const uint64_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;
  ExtRec e[4];
  for (int k = 0; k < 4; ++k) e[k].pos = NONE;
  unsigned long long bad = ~0ull;
  const uint64_t stride = (uint64_t)gridDim.x * TPB;
  uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x;
  if (i < n) {
    ExtRec r;
    r.x = __ldg(X + i);
    r.y = __ldg(Y + i);
    r.id = I ? __ldg(I + i) : (uint32_t)i;
    r.pos = (uint32_t)i;
    if (!(finite_bits(r.x) && finite_bits(r.y))) bad = i;
    e[0] = e[1] = e[2] = e[3] = r;
    i += stride;
  }
  constexpr int U = 4;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double xs[U], ys[U];
    uint32_t ids[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xs[u] = __ldg(X + i + u * stride);
      ys[u] = __ldg(Y + i + u * stride);
      ids[u] = I ? __ldg(I + i + u * stride) : (uint32_t)(i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double x = xs[u], y = ys[u];
      const uint32_t id = ids[u];
      if (!(finite_bits(x) && finite_bits(y)) && bad == ~0ull) bad = i + u * stride;
      const uint32_t pos = (uint32_t)(i + u * stride);
      if (x < e[0].x || (x == e[0].x && (y < e[0].y || (y == e[0].y && id < e[0].id)))) {
        e[0].x = x; e[0].y = y; e[0].id = id; e[0].pos = pos;
      }
      if (y < e[1].y || (y == e[1].y && (x > e[1].x || (x == e[1].x && id < e[1].id)))) {
        e[1].x = x; e[1].y = y; e[1].id = id; e[1].pos = pos;
      }
      if (x > e[2].x || (x == e[2].x && (y > e[2].y || (y == e[2].y && id < e[2].id)))) {
        e[2].x = x; e[2].y = y; e[2].id = id; e[2].pos = pos;
      }
      if (y > e[3].y || (y == e[3].y && (x < e[3].x || (x == e[3].x && id < e[3].id)))) {
        e[3].x = x; e[3].y = y; e[3].id = id; e[3].pos = pos;
      }
    }
  }
  for (; i < n; i += stride) {
    const double x = __ldg(X + i), y = __ldg(Y + i);
    const uint32_t id = I ? __ldg(I + i) : (uint32_t)i;
    if (!(finite_bits(x) && finite_bits(y)) && bad == ~0ull) bad = i;
    const uint32_t pos = (uint32_t)i;
    if (x < e[0].x || (x == e[0].x && (y < e[0].y || (y == e[0].y && id < e[0].id)))) {
      e[0].x = x; e[0].y = y; e[0].id = id; e[0].pos = pos;
    }
    if (y < e[1].y || (y == e[1].y && (x > e[1].x || (x == e[1].x && id < e[1].id)))) {
      e[1].x = x; e[1].y = y; e[1].id = id; e[1].pos = pos;
    }
    if (x > e[2].x || (x == e[2].x && (y > e[2].y || (y == e[2].y && id < e[2].id)))) {
      e[2].x = x; e[2].y = y; e[2].id = id; e[2].pos = pos;
    }
    if (y > e[3].y || (y == e[3].y && (x < e[3].x || (x == e[3].x && id < e[3].id)))) {
      e[3].x = x; e[3].y = y; e[3].id = id; e[3].pos = pos;
    }
  }

  block_reduce_ext(e, bad);
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    K1Partial p;
    for (int k = 0; k < 4; ++k) p.e[k] = e[k];
    p.bad = bad;
    B.k1part[blockIdx.x] = p;
    __threadfence();
    s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // last block: combine the per-block partials
  for (int k = 0; k < 4; ++k) e[k].pos = NONE;
  bad = ~0ull;
  for (uint32_t p = threadIdx.x; p < gridDim.x; p += TPB) {
    const K1Partial* q = B.k1part + p;
    for (int k = 0; k < 4; ++k) {
      ExtRec o;
      o.x = __ldcg(&q->e[k].x);
      o.y = __ldcg(&q->e[k].y);
      o.id = __ldcg(&q->e[k].id);
      o.pos = __ldcg(&q->e[k].pos);
      const bool b = k == 0 ? ext_better<0>(o, e[0])
                   : k == 1 ? ext_better<1>(o, e[1])
                   : k == 2 ? ext_better<2>(o, e[2])
                            : ext_better<3>(o, e[3]);
      if (b) e[k] = o;
    }
    const unsigned long long ob = __ldcg(&q->bad);
    bad = ob < bad ? ob : bad;
  }
  block_reduce_ext(e, bad);
  if (threadIdx.x != 0) return;

  c->ticket = 0;
  c->bad_index = bad;
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
    const ExtRec& q = e[(a + 1) & 3];
    if (!(p.x == q.x && p.y == q.y)) {
      const Edge ed = make_edge(p.x, p.y, q.x, q.y);
      c->edges[ne][0] = ed.ax;
      c->edges[ne][1] = ed.ay;
      c->edges[ne][2] = ed.ex;
      c->edges[ne][3] = ed.ey;
      ++ne;
    }
  }
  c->distinct = distinct;
  c->nedges = ne;
  // farthest-point slots of the two round-1 segments
  B.Sd[0][0] = 0ull;
  B.Sd[0][1] = 0ull;
  B.Sw[0][0] = NONE;
  B.Sw[0][1] = NONE;
}

// ===========================================================================
// Segment-table update for one round, executed by a single block.
//   splittable(s) <=> a farthest candidate exists (max d > 0, hull.cpp:190)
//   ns(s) = s + #splittable segments before s
//   next table: A at ns, C at ns+1 (when splittable)  (hull.cpp:186-194)
// Also writes the Route entry (A, C, B) each member of s is routed by.
// ===========================================================================

SH_DEV void build_table_block(const Bufs& B) {
  __shared__ uint32_t s_ws[WARPS + 1];
  __shared__ int s_overflow;
  Ctl* c = B.ctl;
  volatile Ctl* vc = c;
  const uint32_t S = vc->S_cur, Slo = vc->Slo_cur, par = vc->parity;
  const bool first = vc->round == 0;
  const double* sx = first ? B.in_x : B.Lx[par];
  const double* sy = first ? B.in_y : B.Ly[par];
  const uint32_t* sid = first ? B.in_id : B.Lid[par];
  const double* Tx = B.Tx[par];
  const double* Ty = B.Ty[par];
  const uint32_t* Ti = B.Tid[par];
  double* Nx = B.Tx[par ^ 1];
  double* Ny = B.Ty[par ^ 1];
  uint32_t* Ni = B.Tid[par ^ 1];
  const uint32_t* Sw = B.Sw[par];
  unsigned long long* Ndn = B.Sd[par ^ 1];
  uint32_t* Nwn = B.Sw[par ^ 1];
  if (threadIdx.x == 0) s_overflow = 0;
  __syncthreads();
  uint32_t running = 0, lower_splits = 0;
  for (uint32_t base = 0; base < S; base += TPB) {
    const uint32_t s = base + threadIdx.x;
    const uint32_t w = s < S ? __ldcg(Sw + s) : NONE;
    const uint32_t split = (s < S && w != NONE) ? 1u : 0u;
    uint32_t total;
    const uint32_t pre = block_exclusive_scan(split, s_ws, &total);
    lower_splits += (uint32_t)__syncthreads_count(split && s < Slo);
    if (s < S) {
      const uint32_t ns = s + running + pre;
      const uint32_t sb = s + 1 == S ? 0u : s + 1;
      Route r;
      r.ax = Tx[s];
      r.ay = Ty[s];
      r.bx = Tx[sb];
      r.by = Ty[sb];
      r.ns = ns;
      r.flags = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
      r.pad = 0;
      if (split) {
        r.cx = __ldcg(sx + w);
        r.cy = __ldcg(sy + w);
        r.cid = sid ? __ldcg(sid + w) : w;
      } else {
        r.cx = 0.0;
        r.cy = 0.0;
        r.cid = NONE;
      }
      B.route[s] = r;
      if (ns + split >= B.s_cap) {
        s_overflow = 1;
      } else {
        Nx[ns] = r.ax;
        Ny[ns] = r.ay;
        Ni[ns] = Ti[s];
        Ndn[ns] = 0ull;
        Nwn[ns] = NONE;
        if (split) {
          Nx[ns + 1] = r.cx;
          Ny[ns + 1] = r.cy;
          Ni[ns + 1] = r.cid;
          Ndn[ns + 1] = 0ull;
          Nwn[ns + 1] = NONE;
        }
      }
    }
    running += total;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    c->S_next = S + running;
    c->Slo_next = Slo + lower_splits;
    c->table_ready = 1;
    if (s_overflow) c->status = ST_OVERFLOW;
  }
  __threadfence();
  __syncthreads();
}

// ===========================================================================
// K2: filter + classification + round-0 farthest points (no point writes).
// ===========================================================================

template <bool FILTER>
__global__ void __launch_bounds__(TPB) k2_classify(Bufs B, int reverse) {
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
  int ne = 0;
  Edge Q[4];
  if (FILTER && c->distinct >= 3) {
    ne = c->nedges;
    for (int k = 0; k < 4; ++k) {
      Q[k].ax = c->edges[k][0];
      Q[k].ay = c->edges[k][1];
      Q[k].ex = c->edges[k][2];
      Q[k].ey = c->edges[k][3];
    }
  }
  const uint32_t nchunks = (n + 31) / 32;
  const uint32_t nw = gridDim.x * WARPS;
  Cand a0 = empty_cand(), a1 = empty_cand();
  uint32_t kept = 0;
  bool noncol = false;
  for (uint32_t k = blockIdx.x * WARPS + warp; k < nchunks; k += nw) {
    const uint32_t chunk = reverse ? nchunks - 1 - k : k;
    const uint32_t i = chunk * 32 + lane;
    const bool valid = i < n;
    double x = 0.0, y = 0.0;
    if (valid) {
      x = __ldg(X + i);
      y = __ldg(Y + i);
    }
    const double cl = cross_e(E01, x, y);
    bool inside = false;
    if (FILTER && ne > 0) {  // hull.cpp:80-90: discard iff cross > 0 for every edge
      inside = valid;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < ne) inside = inside && (cross_e(Q[q], x, y) > 0.0);
    }
    const bool keep = valid && !inside;
    noncol = noncol || (valid && cl != 0.0) || inside;
    const bool member = keep && i != p0 && i != pr;
    const bool lw = member && cl < 0.0;           // hull.cpp:115-117
    const bool up = member && !(cl < 0.0);
    const unsigned blo = __ballot_sync(FULL, lw);
    const unsigned bup = __ballot_sync(FULL, up);
    const unsigned bk = __ballot_sync(FULL, keep);
    if (lane == 0) {
      B.bits_lo[chunk] = blo;
      B.bits_up[chunk] = bup;
      kept += __popc(bk);
    }
    if (lw) {
      const double d = -cl;  // outward_distance(P0, Pr, p)
      if (d > 0.0 && d >= a0.d) {
        Cand cc;
        cc.d = d; cc.x = x; cc.y = y; cc.id = I ? __ldg(I + i) : i; cc.pos = i;
        if (cand_better(cc, a0, true)) a0 = cc;
      }
    } else if (up) {
      const double d = outward_e(E10, x, y);  // outward_distance(Pr, P0, p)
      if (d > 0.0 && d >= a1.d) {
        Cand cc;
        cc.d = d; cc.x = x; cc.y = y; cc.id = I ? __ldg(I + i) : i; cc.pos = i;
        if (cand_better(cc, a1, false)) a1 = cc;
      }
    }
  }

  // block reduction of the two chains' farthest candidates
  __shared__ Cand s_a[2][WARPS];
  __shared__ uint32_t s_kept[WARPS];
  __shared__ int s_last;
  a0 = warp_best(a0, true);
  a1 = warp_best(a1, false);
  const bool nc_any = __any_sync(FULL, noncol);
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
      if (a0.d > 0.0) slot_offer(&B.Sd[0][0], &B.Sw[0][0], a0, true, E01, X, Y, I);
      if (a1.d > 0.0) slot_offer(&B.Sd[0][1], &B.Sw[0][1], a1, false, E10, X, Y, I);
      __threadfence();
      s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    c->ticket = 0;
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
      c->parity = 0;
    }
    __threadfence();
  }
  __syncthreads();
  if (*(volatile uint32_t*)&c->status == ST_RUNNING) build_table_block(B);
}

// ===========================================================================
// K4: segment-table update for large tables (decoupled look-back scan).
// ===========================================================================

constexpr int K4_ITEMS = 8;
constexpr int K4_TILE = TPB * K4_ITEMS;

__global__ void __launch_bounds__(TPB) k4_table(Bufs B) {
  Ctl* c = B.ctl;
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  if (*(volatile uint32_t*)&c->table_ready) return;
  __shared__ uint32_t s_ws[WARPS + 1];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ int s_last;
  const uint32_t epoch = *(volatile uint32_t*)B.epoch;
  const uint32_t S = c->S_cur, Slo = c->Slo_cur, par = c->parity;
  const bool first = c->round == 0;
  const double* sx = first ? B.in_x : B.Lx[par];
  const double* sy = first ? B.in_y : B.Ly[par];
  const uint32_t* sid = first ? B.in_id : B.Lid[par];
  const double* Tx = B.Tx[par];
  const double* Ty = B.Ty[par];
  const uint32_t* Ti = B.Tid[par];
  double* Nx = B.Tx[par ^ 1];
  double* Ny = B.Ty[par ^ 1];
  uint32_t* Ni = B.Tid[par ^ 1];
  const uint32_t* Sw = B.Sw[par];
  unsigned long long* Ndn = B.Sd[par ^ 1];
  uint32_t* Nwn = B.Sw[par ^ 1];
  const uint32_t ntiles = (S + K4_TILE - 1) / K4_TILE;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t s0 = tile * K4_TILE + threadIdx.x * K4_ITEMS;
    uint32_t w[K4_ITEMS];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < K4_ITEMS; ++j) {
      const uint32_t s = s0 + j;
      w[j] = s < S ? __ldcg(Sw + s) : NONE;
      cnt += (s < S && w[j] != NONE) ? 1u : 0u;
    }
    uint32_t total;
    const uint32_t pre = block_exclusive_scan(cnt, s_ws, &total);
    if (threadIdx.x < 32) {
      const uint32_t p = lookback_warp(B.tile_status, tile, total, epoch);
      if (threadIdx.x == 0) {
        s_prefix = p;
        if (tile == ntiles - 1) c->S_next = S + p + total;
      }
    }
    __syncthreads();
    uint32_t run = s_prefix + pre;
#pragma unroll
    for (int j = 0; j < K4_ITEMS; ++j) {
      const uint32_t s = s0 + j;
      if (s < S) {
        const uint32_t split = w[j] != NONE ? 1u : 0u;
        if (s == Slo) c->Slo_next = Slo + run;
        const uint32_t ns = s + run;
        const uint32_t sb = s + 1 == S ? 0u : s + 1;
        Route r;
        r.ax = Tx[s];
        r.ay = Ty[s];
        r.bx = Tx[sb];
        r.by = Ty[sb];
        r.ns = ns;
        r.flags = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
        r.pad = 0;
        if (split) {
          r.cx = __ldcg(sx + w[j]);
          r.cy = __ldcg(sy + w[j]);
          r.cid = sid ? __ldcg(sid + w[j]) : w[j];
        } else {
          r.cx = 0.0;
          r.cy = 0.0;
          r.cid = NONE;
        }
        B.route[s] = r;
        if (ns + split >= B.s_cap) {
          c->status = ST_OVERFLOW;
        } else {
          Nx[ns] = r.ax;
          Ny[ns] = r.ay;
          Ni[ns] = Ti[s];
          Ndn[ns] = 0ull;
          Nwn[ns] = NONE;
          if (split) {
            Nx[ns + 1] = r.cx;
            Ny[ns + 1] = r.cy;
            Ni[ns + 1] = r.cid;
            Ndn[ns + 1] = 0ull;
            Nwn[ns + 1] = NONE;
          }
        }
        run += split;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    c->ticket = 0;
    c->tile_ctr = 0;
    *B.epoch = epoch + 1;
    c->table_ready = 1;
    __threadfence();
  }
}

// ===========================================================================
// K3: one refinement round -- route, keep, stable compaction, and the fused
// farthest-point search of the NEXT round.
// ===========================================================================

struct K3Smem {
  double st_x[TILE];
  double st_y[TILE];
  double st_d[TILE];
  uint32_t st_id[TILE];
  uint32_t st_seg[TILE];
  unsigned long long s_db[NSLOT];
  Cand s_rec[NSLOT];
  int s_owner[NSLOT];
};

SH_DEV Route load_route(const Route* R, uint32_t s) {
  const double2* p = reinterpret_cast<const double2*>(R + s);
  const double2 a = __ldg(p), b = __ldg(p + 1), cc = __ldg(p + 2);
  const uint4 t = __ldg(reinterpret_cast<const uint4*>(p + 3));
  Route r;
  r.ax = a.x; r.ay = a.y; r.cx = b.x; r.cy = b.y; r.bx = cc.x; r.by = cc.y;
  r.cid = t.x; r.ns = t.y; r.flags = t.z; r.pad = t.w;
  return r;
}

template <bool FIRST>
__global__ void __launch_bounds__(TPB, 2) k3_route(Bufs B) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K3Smem& sm = *reinterpret_cast<K3Smem*>(smem_raw);
  __shared__ uint32_t s_cnt[ITEMS * WARPS];
  __shared__ uint32_t s_tile, s_prefix, s_agg;
  __shared__ int s_last;

  Ctl* c = B.ctl;
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t par = c->parity;
  const uint32_t epoch = *(volatile uint32_t*)B.epoch;
  const uint32_t count = FIRST ? B.n : c->m_cur;
  const uint32_t ntiles = (count + TILE - 1) / TILE;
  const uint32_t Snext = c->S_next, Slo_next = c->Slo_next;
  const bool smem_slots = Snext <= (uint32_t)NSLOT;

  const double* __restrict__ Ix = FIRST ? B.in_x : B.Lx[par];
  const double* __restrict__ Iy = FIRST ? B.in_y : B.Ly[par];
  const uint32_t* __restrict__ Iid = FIRST ? B.in_id : B.Lid[par];
  const uint32_t* __restrict__ Iseg = B.Lseg[par];
  double* Ox = B.Lx[par ^ 1];
  double* Oy = B.Ly[par ^ 1];
  uint32_t* Oid = B.Lid[par ^ 1];
  uint32_t* Oseg = B.Lseg[par ^ 1];
  unsigned long long* Sdn = B.Sd[par ^ 1];
  uint32_t* Swn = B.Sw[par ^ 1];
  const Route* __restrict__ R = B.route;

  if (smem_slots) {
    for (uint32_t t = threadIdx.x; t < Snext; t += TPB) {
      sm.s_db[t] = 0ull;
      sm.s_rec[t] = empty_cand();
      sm.s_owner[t] = -1;
    }
  }
  Route rlo, rup;  // round 1: the two chains' route entries
  if (FIRST) {
    rlo = load_route(R, 0);
    rup = load_route(R, 1);
  }

  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t base = tile * TILE;

    double px[ITEMS], py[ITEMS], pd[ITEMS];
    uint32_t pid[ITEMS], pns[ITEMS], pold[ITEMS];
    uint32_t keepm = 0, leftm = 0;

    // ---- load ----
    uint32_t memb = 0;
    if (FIRST) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t e = base + j * TPB + threadIdx.x;
        const bool valid = e < count;
        uint32_t lo = 0, up = 0;
        if (valid) {
          lo = __ldg(B.bits_lo + (e >> 5));
          up = __ldg(B.bits_up + (e >> 5));
          px[j] = __ldg(Ix + e);
          py[j] = __ldg(Iy + e);
        }
        const bool lw = (lo >> lane) & 1u, uw = (up >> lane) & 1u;
        if (lw || uw) memb |= 1u << j;
        pold[j] = lw ? 0u : 1u;
        pid[j] = e;
      }
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t e = base + j * TPB + threadIdx.x;
        if (e < count) {
          px[j] = __ldcs(Ix + e);
          py[j] = __ldcs(Iy + e);
          pid[j] = __ldcs(Iid + e);
          pold[j] = __ldcs(Iseg + e);
          memb |= 1u << j;
        }
      }
    }

    // ---- route ----
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      pd[j] = 0.0;
      pns[j] = 0;
      if (memb & (1u << j)) {
        const Route r = FIRST ? (pold[j] == 0 ? rlo : rup) : load_route(R, pold[j]);
        if (FIRST) pid[j] = Iid ? __ldg(Iid + pid[j]) : pid[j];
        if ((r.flags & RT_SPLIT) && pid[j] != r.cid) {
          const bool lower = r.flags & RT_LOWER;
          const bool left = lower ? lex_less(px[j], py[j], r.cx, r.cy)
                                  : lex_less(r.cx, r.cy, px[j], py[j]);
          const Edge e = left ? make_edge(r.ax, r.ay, r.cx, r.cy)
                              : make_edge(r.cx, r.cy, r.bx, r.by);
          const double d = outward_e(e, px[j], py[j]);
          pd[j] = d;
          pns[j] = r.ns + (left ? 0u : 1u);
          if (d > 0.0) keepm |= 1u << j;  // hull.cpp:199 keep iff d > 0
          if (left) leftm |= 1u << j;
        }
      }
    }

    // ---- tile-local ranks (index order = (j, warp, lane)) ----
    uint32_t rank[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const unsigned bal = __ballot_sync(FULL, (keepm >> j) & 1u);
      if (lane == 0) s_cnt[j * WARPS + warp] = __popc(bal);
      rank[j] = __popc(bal & lanemask_lt());
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t v0 = s_cnt[2 * lane], v1 = s_cnt[2 * lane + 1];
      uint32_t incl = v0 + v1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - v0 - v1;
      s_cnt[2 * lane] = excl;
      s_cnt[2 * lane + 1] = excl + v0;
      const uint32_t agg = __shfl_sync(FULL, incl, 31);
      const uint32_t prefix = lookback_warp(B.tile_status, tile, agg, epoch);
      if (lane == 0) {
        s_prefix = prefix;
        s_agg = agg;
        if (tile == ntiles - 1) c->m_next = prefix + agg;
      }
    }
    __syncthreads();
    const uint32_t prefix = s_prefix, agg = s_agg;

    // ---- stage survivors in order; phase 1 of the shared-memory argmax ----
    uint32_t candm = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if ((keepm >> j) & 1u) {
        const uint32_t rk = s_cnt[j * WARPS + warp] + rank[j];
        rank[j] = rk;
        sm.st_x[rk] = px[j];
        sm.st_y[rk] = py[j];
        sm.st_d[rk] = pd[j];
        sm.st_id[rk] = pid[j];
        sm.st_seg[rk] = pns[j];
        if (smem_slots) {
          const unsigned long long db = (unsigned long long)__double_as_longlong(pd[j]);
          if (db >= *(volatile unsigned long long*)&sm.s_db[pns[j]]) {
            const unsigned long long old = atomicMax(&sm.s_db[pns[j]], db);
            if (db >= old) candm |= 1u << j;
          }
        }
      }
    }
    __syncthreads();

    // ---- coalesced write-out of the compacted tile ----
    for (uint32_t k = threadIdx.x; k < agg; k += TPB) {
      const uint32_t o = prefix + k;
      Ox[o] = sm.st_x[k];
      Oy[o] = sm.st_y[k];
      Oid[o] = sm.st_id[k];
      Oseg[o] = sm.st_seg[k];
    }
    __threadfence();

    if (smem_slots) {
      // phase 2: ties at the block maximum resolved with the full comparator
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if ((candm >> j) & 1u) {
          const uint32_t t = pns[j];
          const unsigned long long db = (unsigned long long)__double_as_longlong(pd[j]);
          if (db == *(volatile unsigned long long*)&sm.s_db[t]) {
            Cand me;
            me.d = pd[j]; me.x = px[j]; me.y = py[j]; me.id = pid[j]; me.pos = rank[j];
            const bool lower = t < Slo_next;
            int cur = *(volatile int*)&sm.s_owner[t];
            while (true) {
              Cand o;
              if (cur < 0) {
                o = sm.s_rec[t];
              } else {
                o.d = sm.st_d[cur]; o.x = sm.st_x[cur]; o.y = sm.st_y[cur]; o.id = sm.st_id[cur];
              }
              if (!(cur < 0 && o.id == NONE) && !cand_better(me, o, lower)) break;
              const int prev = atomicCAS(&sm.s_owner[t], cur, (int)rank[j]);
              if (prev == cur) break;
              cur = prev;
            }
          } else {
            candm &= ~(1u << j);
          }
        }
      }
    }
    __syncthreads();
    if (smem_slots) {
      // phase 3: the tile's winner of each slot becomes the block's record
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if ((candm >> j) & 1u) {
          const uint32_t t = pns[j];
          if (sm.s_owner[t] == (int)rank[j]) {
            Cand me;
            me.d = pd[j]; me.x = px[j]; me.y = py[j]; me.id = pid[j]; me.pos = prefix + rank[j];
            sm.s_rec[t] = me;
            sm.s_owner[t] = -1;
          }
        }
      }
    } else {
      // many segments: offer every survivor to its global slot directly
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if ((keepm >> j) & 1u) {
          const Route r = FIRST ? (pold[j] == 0 ? rlo : rup) : load_route(R, pold[j]);
          const bool left = (leftm >> j) & 1u;
          const Edge e = left ? make_edge(r.ax, r.ay, r.cx, r.cy)
                              : make_edge(r.cx, r.cy, r.bx, r.by);
          Cand me;
          me.d = pd[j]; me.x = px[j]; me.y = py[j]; me.id = pid[j]; me.pos = prefix + rank[j];
          slot_offer(Sdn + pns[j], Swn + pns[j], me, (r.flags & RT_LOWER) != 0, e, Ox, Oy, Oid);
        }
      }
    }
  }

  // ---- flush the block's shared-memory slots to the global slots ----
  if (smem_slots) {
    const double* Nx = B.Tx[par ^ 1];
    const double* Ny = B.Ty[par ^ 1];
    for (uint32_t t = threadIdx.x; t < Snext; t += TPB) {
      const Cand me = sm.s_rec[t];
      if (me.id != NONE) {
        const uint32_t t1 = t + 1 == Snext ? 0u : t + 1;
        const Edge e = make_edge(Nx[t], Ny[t], Nx[t1], Ny[t1]);
        slot_offer(Sdn + t, Swn + t, me, t < Slo_next, e, Ox, Oy, Oid);
      }
    }
  }

  // ---- last block: close the round ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    c->ticket = 0;
    c->tile_ctr = 0;
    *B.epoch = epoch + 1;
    const uint32_t r = c->round + 1;
    const uint32_t Sn = *(volatile uint32_t*)&c->S_next;
    const uint32_t mn = ntiles ? *(volatile uint32_t*)&c->m_next : 0u;
    const uint32_t before = c->S_cur + c->m_cur;
    const uint32_t after = Sn + mn;
    if (r <= (uint32_t)STATS_CAP) {
      StatRec st;
      st.segments = Sn;
      st.points_remaining = after;
      st.points_removed = before - after;
      st.pad = 0;
      B.stats[r - 1] = st;
    }
    c->round = r;
    c->S_cur = Sn;
    c->Slo_cur = c->Slo_next;
    c->m_cur = mn;
    c->parity = par ^ 1;
    c->table_ready = 0;
    if (mn == 0) {
      c->status = ST_DONE;
    } else if ((unsigned long long)r + 1 > (unsigned long long)B.n) {
      c->status = ST_INTERNAL;  // hull.cpp:265-267
    }
    __threadfence();
  }
  __syncthreads();
  if (*(volatile uint32_t*)&c->status == ST_RUNNING && *(volatile uint32_t*)&c->S_cur <= SMALL_S)
    build_table_block(B);
}

// ===========================================================================
// Device generators (dataio.hpp:44-58; SURVEY.md section 0 finding 3)
// ===========================================================================

SH_DEV unsigned long long sm64_mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// k-th draw (k >= 1) of SplitMix64(seed) as a double in [0,1)
SH_DEV double sm64_draw(unsigned long long seed, unsigned long long k) {
  return (double)(sm64_mix(seed + k * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
}

__global__ void k_gen_uniform(double* x, double* y, unsigned long long first,
                              unsigned long long count, unsigned long long seed) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       t < count; t += stride) {
    const unsigned long long i = first + t;
    x[t] = sm64_draw(seed, 2 * i + 1);
    y[t] = sm64_draw(seed, 2 * i + 2);
  }
}

// candidate pairs [cand0, cand0 + ncand): accept iff x*x + y*y < 1, compacted
// stably after `out_base` already-accepted points; writes only below n.
__global__ void __launch_bounds__(TPB) k_gen_disk(double* x, double* y, unsigned long long n,
                                                  unsigned long long seed,
                                                  unsigned long long cand0, uint32_t ncand,
                                                  unsigned long long out_base, Ctl* c,
                                                  unsigned long long* status, uint32_t* epoch_p) {
  __shared__ uint32_t s_cnt[ITEMS * WARPS];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t epoch = *(volatile uint32_t*)epoch_p;
  const uint32_t ntiles = (ncand + TILE - 1) / TILE;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    double px[ITEMS], py[ITEMS];
    uint32_t acc = 0, rank[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t e = tile * TILE + j * TPB + threadIdx.x;
      if (e < ncand) {
        const unsigned long long cj = cand0 + e;
        const double u = sm64_draw(seed, 2 * cj + 1), v = sm64_draw(seed, 2 * cj + 2);
        px[j] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
        py[j] = __dsub_rn(__dmul_rn(2.0, v), 1.0);
        if (__dadd_rn(__dmul_rn(px[j], px[j]), __dmul_rn(py[j], py[j])) < 1.0) acc |= 1u << j;
      }
      const unsigned bal = __ballot_sync(FULL, (acc >> j) & 1u);
      if (lane == 0) s_cnt[j * WARPS + warp] = __popc(bal);
      rank[j] = __popc(bal & lanemask_lt());
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t v0 = s_cnt[2 * lane], v1 = s_cnt[2 * lane + 1];
      uint32_t incl = v0 + v1;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t excl = incl - v0 - v1;
      s_cnt[2 * lane] = excl;
      s_cnt[2 * lane + 1] = excl + v0;
      const uint32_t agg = __shfl_sync(FULL, incl, 31);
      const uint32_t p = lookback_warp(status, tile, agg, epoch);
      if (lane == 0) {
        s_prefix = p;
        if (tile == ntiles - 1) c->m_next = p + agg;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if ((acc >> j) & 1u) {
        const unsigned long long o = out_base + s_prefix + s_cnt[j * WARPS + warp] + rank[j];
        if (o < n) {
          x[o] = px[j];
          y[o] = py[j];
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
    *epoch_p = epoch + 1;
    __threadfence();
  }
}

// ===========================================================================
// K5: emit the hull (segment heads in table order) into caller device memory
// ===========================================================================

__global__ void k5_emit(const double* __restrict__ Tx, const double* __restrict__ Ty,
                        const uint32_t* __restrict__ Tid, uint32_t h, double* ox, double* oy,
                        long long* oidx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h; i += gridDim.x * blockDim.x) {
    if (ox) ox[i] = Tx[i];
    if (oy) oy[i] = Ty[i];
    if (oidx) oidx[i] = (long long)Tid[i];
  }
}

// ===========================================================================
// host-side launch wrappers
// ===========================================================================

size_t k3_smem_bytes() { return sizeof(K3Smem); }

cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(k3_route<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(K3Smem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k3_route<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(K3Smem));
}

int k3_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_route<false>, TPB, sizeof(K3Smem));
  return b < 1 ? 1 : b;
}

void launch_k1(const Bufs& B, int grid, cudaStream_t s) { k1_extremes<<<grid, TPB, 0, s>>>(B); }

void launch_k2(const Bufs& B, bool filter, int grid, int reverse, cudaStream_t s) {
  if (filter)
    k2_classify<true><<<grid, TPB, 0, s>>>(B, reverse);
  else
    k2_classify<false><<<grid, TPB, 0, s>>>(B, reverse);
}

void launch_k3(const Bufs& B, bool first, int grid, cudaStream_t s) {
  if (first)
    k3_route<true><<<grid, TPB, sizeof(K3Smem), s>>>(B);
  else
    k3_route<false><<<grid, TPB, sizeof(K3Smem), s>>>(B);
}

void launch_k4(const Bufs& B, int grid, cudaStream_t s) { k4_table<<<grid, TPB, 0, s>>>(B); }

void launch_k5(const double* Tx, const double* Ty, const uint32_t* Tid, uint32_t h, double* ox,
               double* oy, long long* oidx, cudaStream_t s) {
  const int grid = (int)((h + 255) / 256 < 1024 ? (h + 255) / 256 : 1024);
  k5_emit<<<grid < 1 ? 1 : grid, 256, 0, s>>>(Tx, Ty, Tid, h, ox, oy, oidx);
}

void launch_gen_uniform(double* x, double* y, unsigned long long first, unsigned long long count,
                        unsigned long long seed, int grid, cudaStream_t s) {
  k_gen_uniform<<<grid, 256, 0, s>>>(x, y, first, count, seed);
}

void launch_gen_disk(double* x, double* y, unsigned long long n, unsigned long long seed,
                     unsigned long long cand0, uint32_t ncand, unsigned long long out_base, Ctl* c,
                     unsigned long long* status, uint32_t* epoch, int grid, cudaStream_t s) {
  k_gen_disk<<<grid, TPB, 0, s>>>(x, y, n, seed, cand0, ncand, out_base, c, status, epoch);
}

}  // namespace shb
