// k_rounds.cu -- the refinement rounds of the sm_100a QuickHull
// (hull.cpp:264-282; SURVEY.md section 7.3 "lex routing").
//
//   K3 k3_round1  round 1 straight from the input + K2's class bits: route
//                 every member of the two chains to the A->C or C->B edge of
//                 its chain's farthest point C, keep iff strictly outside
//                 (hull.cpp:196-201), append the survivors to the CTA's run
//                 of the live set and find round 2's farthest points
//   KR k_rounds   every later round in ONE persistent cooperative launch:
//                 per round a segment-table phase (rebuilt in each CTA's
//                 shared memory for small tables, a grid-wide scan for large
//                 ones), a point phase (route, keep, append, contend) and grid
//                 barriers; once a lone CTA holds a small table and a live set
//                 that fits on chip, it finishes in shared memory (solo tail)
//   K5 k5_emit    copy the final heads (the hull, CCW from P0) to the caller
//
// Compaction is order-free: the hull and the per-round stats depend only on
// segment membership and on the total order of the farthest-point
// comparator, never on where a survivor lands.  Each CTA appends to its own
// run with one shared-memory atomicAdd per warp; the next round reads the
// runs as one virtual range.  Farthest points between CTAs: per-CTA record
// rows or contender lists plus atomicMax on the distance bits, winners
// claimed by compare-and-swap after the barrier -- no global locks.
#include <cuda_runtime.h>

#include <type_traits>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

// ===========================================================================
// shared pieces
// ===========================================================================

// Route one member (x, y, id) of old segment s whose Route row is at rp
// (shared or, with GLOBAL, global memory), SURVEY.md section 7.3:
//   left = lower ? lex(p) < lex(C) : lex(C) < lex(p)
//   d    = outward_distance(left ? (A, C) : (C, B), p)   (geometry.hpp:25-27)
//   keep iff the segment splits, p is not C itself and d > 0 (hull.cpp:199)
// The row stores A | C | B | meta as consecutive 16-byte words.  In shared
// memory the edge endpoints are fetched by computed offset; from global
// memory the whole row is loaded at once (one L2 round trip, not two).
template <bool GLOBAL>
SH_DEV bool route_point(const Route* rp, double x, double y, uint32_t id, double& d,
                        uint32_t& nseg, bool& lower) {
  const double2* row = reinterpret_cast<const double2*>(rp);
  double2 A, C, Bv;
  uint4 meta;
  if (GLOBAL) {  // two 256-bit L2 loads (LDG.E.ENL2.256): A|C and B|meta
    unsigned long long m0, m1;
    asm("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(A.x), "=d"(A.y), "=d"(C.x), "=d"(C.y) : "l"(row));
    asm("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(Bv.x), "=d"(Bv.y), "=l"(m0), "=l"(m1) : "l"(row + 2));
    meta = make_uint4((uint32_t)m0, (uint32_t)(m0 >> 32), (uint32_t)m1, (uint32_t)(m1 >> 32));
  } else {
    C = row[1];
    meta = *reinterpret_cast<const uint4*>(row + 3);
  }
  lower = meta.z & RT_LOWER;
  const bool xeq = x == C.x;
  const bool lt = x < C.x || (xeq && y < C.y);
  const bool eq = xeq && y == C.y;
  const bool left = lower ? lt : !(lt || eq);
  double2 S, E;
  if (GLOBAL) {
    S = left ? A : C;
    E = left ? C : Bv;
  } else {
    const int o = left ? 0 : 1;
    S = row[o];
    E = row[o + 1];
  }
  d = outward_e(make_edge(S.x, S.y, E.x, E.y), x, y);
  nseg = meta.y + (left ? 0u : 1u);
  return (meta.z & RT_SPLIT) && id != meta.x && d > 0.0;
}

// Dense append of this thread's survivors to the CTA's run of the next live
// set: one shared-memory atomicAdd per warp, no global atomics, no barrier.
// With Oc, the survivors flagged in candm are also listed (distance,
// position, segment) at Oc[cbase + ...] through the counter s_coff.
// CAPPED (K3, whose runs are sized by the workspace's live capacity, not by
// its input share): a warp whose survivors would pass `lim` writes nothing
// and sets *ovf = ST_OVERFLOW; the host then regrows the live sets and reruns.
template <int NP, bool CAPPED = false>
SH_DEV void run_append(uint32_t keepm, const double (&px)[NP], const double (&py)[NP],
                       const uint32_t (&pid)[NP], const uint32_t (&pseg)[NP], uint32_t* s_off,
                       double2* Oxy, uint2* Ois, uint32_t base, const double (&pd)[NP] = {},
                       uint32_t candm = 0, uint32_t* s_coff = nullptr, LiveCand* Oc = nullptr,
                       uint32_t lim = 0, uint32_t* ovf = nullptr, uint32_t* eo = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t bal[NP];
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    bal[j] = __ballot_sync(FULL, (keepm >> j) & 1u);
    tot += __popc(bal[j]);
  }
  if (tot == 0) return;  // warp-uniform
  uint32_t off = 0;
  if (lane == 0) off = atom_add_shared(s_off, tot);
  off = base + __shfl_sync(FULL, off, 0);
  if (CAPPED && off + tot > lim) {  // warp-uniform
    if (lane == 0) *(volatile uint32_t*)ovf = ST_OVERFLOW;
    return;
  }
  const uint32_t lt = lanemask_lt();
  uint32_t e[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    e[j] = off + __popc(bal[j] & lt);
    if (eo != nullptr) eo[j] = e[j];
    if ((keepm >> j) & 1u) {
      Oxy[e[j]] = make_double2(px[j], py[j]);
      Ois[e[j]] = make_uint2(pid[j], pseg[j]);
    }
    off += __popc(bal[j]);
  }
  if (Oc != nullptr && __any_sync(FULL, candm)) {
    uint32_t cb[NP], ctot = 0;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      cb[j] = __ballot_sync(FULL, (candm >> j) & 1u);
      ctot += __popc(cb[j]);
    }
    uint32_t co = 0;
    if (lane == 0) co = atom_add_shared(s_coff, ctot);
    co = base + __shfl_sync(FULL, co, 0);
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if ((candm >> j) & 1u) {
        LiveCand lc;
        lc.d = pd[j];
        lc.pos = e[j];
        lc.seg = pseg[j];
        Oc[co + __popc(cb[j] & lt)] = lc;
      }
      co += __popc(cb[j]);
    }
  }
}

// Contender list of a large-table tile whose atomicMax results arrived: the
// survivors that reached the running maximum (db >= old) are listed
// (distance, live position, segment) at Oc[base + ...] through s_coff.
template <int NP>
SH_DEV void list_cands(uint32_t m, const unsigned long long (&db)[NP],
                       const unsigned long long (&old)[NP], const uint32_t (&pos)[NP],
                       const uint32_t (&seg)[NP], uint32_t* s_coff, LiveCand* Oc, uint32_t base) {
  uint32_t candm = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j)
    if (((m >> j) & 1u) && db[j] >= old[j]) candm |= 1u << j;
  if (!__any_sync(FULL, candm)) return;
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  uint32_t cb[NP], ctot = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    cb[j] = __ballot_sync(FULL, (candm >> j) & 1u);
    ctot += __popc(cb[j]);
  }
  uint32_t co = 0;
  if (lane == 0) co = atom_add_shared(s_coff, ctot);
  co = base + __shfl_sync(FULL, co, 0);
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if ((candm >> j) & 1u) {
      LiveCand lc;
      lc.d = __longlong_as_double((long long)db[j]);
      lc.pos = pos[j];
      lc.seg = seg[j];
      Oc[co + __popc(cb[j] & lt)] = lc;
    }
    co += __popc(cb[j]);
  }
}

// Farthest-point contenders of a CTA with shared-memory slots (small tables):
// a point that reaches the slot's running maximum of the distance's high word
// (native 32-bit shared atomicMax) settles the full comparator under the
// record's lock.  After a CTA's first tile almost no point passes the filter,
// so the lock is rare.
template <int NP>
SH_DEV void contend_tile(uint32_t* s_dh, SlotRec* s_rec, uint32_t keepm,
                         const double (&px)[NP], const double (&py)[NP],
                         const double (&pd)[NP], const uint32_t (&pid)[NP],
                         const uint32_t (&pseg)[NP], uint32_t lowm) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if ((keepm >> j) & 1u) {
      const uint32_t dh = (uint32_t)((unsigned long long)__double_as_longlong(pd[j]) >> 32);
      if (dh >= *(volatile uint32_t*)&s_dh[pseg[j]]) {
        const uint32_t old = atomicMax(&s_dh[pseg[j]], dh);
        if (dh >= old) {
          Cand me;
          me.d = pd[j]; me.x = px[j]; me.y = py[j]; me.id = pid[j]; me.pos = 0;
          rec_update<true>(&s_rec[pseg[j]], me, (lowm >> j) & 1u);
        }
      }
    }
  }
}

// Lock-free flush of a multi-CTA round's small-table records: the CTA's
// records go to its own row (plain stores), their distance bits to the
// global running maxima (fire-and-forget atomicMax).  After the grid barrier,
// claim_slots lets the rows that reached a slot's final maximum claim it.
SH_DEV void flush_rows(const SlotRec* s_rec, uint32_t Sn,
                       unsigned long long* Sd, SlotRec* row) {
  for (uint32_t t = threadIdx.x; t < Sn; t += blockDim.x) {
    const volatile SlotRec* r = s_rec + t;
    SlotRec o;
    o.d = r->d;
    o.x = r->x;
    o.y = r->y;
    o.id = r->id;
    o.lock = 0u;
    row[t] = o;
    if (o.id != NONE) atomicMax(Sd + t, (unsigned long long)__double_as_longlong(o.d));
  }
}

// The CTA's records whose distance equals the slot's final maximum claim the
// slot's winner word (this CTA's row index); exact ties run the full
// comparator (hull.cpp:171-179) in a compare-and-swap loop over rows.
SH_DEV void claim_slots(const SlotRec* s_rec, uint32_t Sn, uint32_t Slon,
                        const unsigned long long* Sd, uint32_t* Wn, const SlotRec* rows) {
  for (uint32_t t = threadIdx.x; t < Sn; t += blockDim.x) {
    const volatile SlotRec* r = s_rec + t;
    if (r->id == NONE) continue;
    Cand me;
    me.d = r->d; me.x = r->x; me.y = r->y; me.id = r->id; me.pos = 0;
    if ((unsigned long long)__double_as_longlong(me.d) != __ldcg(Sd + t)) continue;
    uint32_t cur = atomicCAS(Wn + t, NONE, blockIdx.x);
    while (cur != NONE) {
      const SlotRec* q = rows + (size_t)cur * NSLOT + t;
      Cand o;
      o.d = __ldcg(&q->d); o.x = __ldcg(&q->x); o.y = __ldcg(&q->y); o.id = __ldcg(&q->id); o.pos = 0;
      if (!cand_better(me, o, t < Slon)) break;
      const uint32_t prev = atomicCAS(Wn + t, cur, blockIdx.x);
      if (prev == cur) break;
      cur = prev;
    }
  }
}

// sum of nruns run counts, computed by the whole CTA (contains barriers)
SH_DEV uint32_t sum_runs(const uint32_t* cnt, uint32_t nruns, uint32_t* s_ws) {
  uint32_t v = 0;
  for (uint32_t j = threadIdx.x; j < nruns; j += blockDim.x) v += __ldcg(cnt + j);
  uint32_t tot;
  block_exclusive_scan(v, s_ws, &tot);
  return tot;
}

// ===========================================================================
// K3: round 1 straight from the input
// ===========================================================================

constexpr int K3_NP = 2 * Cfg3::CH;   // points per consumer thread per tile

template <bool IDS>
struct K3Layout {
#ifndef SHB_K3_NS_IDS
#define SHB_K3_NS_IDS SHB_K3_NS
#endif
  // with caller ids each point carries 4 more bytes: the ring may need fewer stages
  using Ring = TileRing<Cfg3::T, IDS ? SHB_K3_NS_IDS : Cfg3::NS, IDS, 16, Cfg3::CW>;
  static constexpr size_t kRing = (Ring::kBytes + 127) / 128 * 128;
  static constexpr size_t kBytes = kRing;
};

// CAPPED: the live set is lean (runs shorter than a CTA's input share), so
// every append is checked against the run (ST_OVERFLOW -> regrow, rerun); ~2%
// of K3, paid only where the workspace is lean (n > 2^24)
template <bool IDS, bool CAPPED>
__global__ void __launch_bounds__(Cfg3::TPB, 1) k3_round1(Bufs B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using L = K3Layout<IDS>;
  typename L::Ring R;
  R.carve(smem_raw);
  __shared__ Route s_rt[2];
  __shared__ uint32_t s_db[4];  // high words of the slots' running maxima
  __shared__ SlotRec s_rec[4];
  __shared__ uint32_t s_off, s_Sn, s_Slon;
  __shared__ int s_last;
  Ctl* c = B.ctl;
  if (threadIdx.x == 0) R.init();
  __syncthreads();
  // the points do not depend on K2 (their class bits do): start the ring on
  // them before waiting; the bits follow once K2 is complete
  const uint32_t pre = stream_prefetch(R, B.n, B.in_x, B.in_y, B.in_id, false, false);
  SHB_PROBE(const bool probe = blockIdx.x == 0 && threadIdx.x == 0 && c->tl_round == 255u);
  SHB_PROBE(if (probe) B.dbg[1602] = globaltimer_ns());
  pdl_wait();               // K2's classes and partials are complete and visible
  SHB_PROBE(if (probe) B.dbg[1603] = globaltimer_ns());
  pdl_launch_dependents();  // the round kernel may be scheduled on SMs this kernel frees
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) {
    stream_drain_points(R, pre, B.n, reinterpret_cast<const unsigned char*>(B.bits));
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n = B.n;
  const double* __restrict__ X = B.in_x;
  const double* __restrict__ Y = B.in_y;
  const uint32_t* __restrict__ I = B.in_id;

  // ---- every CTA combines K2's per-CTA partials (hull.cpp:101-158): the
  // farthest point of each chain, the kept count and collinearity ----
  __shared__ Cand s_cand[2];
  __shared__ unsigned long long s_best2[2][4];
  __shared__ unsigned long long s_kept;
  __shared__ uint32_t s_nc, s_status;
  {
    Cand a[2] = {empty_cand(), empty_cand()};
    unsigned long long kb = 0;
    uint32_t nc = 0;
    if (threadIdx.x < B.k2_grid) {
      const K2Partial* qp = B.k2part + threadIdx.x;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        a[ch].d = __ldcg(&qp->a[ch].d);
        a[ch].x = __ldcg(&qp->a[ch].x);
        a[ch].y = __ldcg(&qp->a[ch].y);
        a[ch].id = __ldcg(&qp->a[ch].id);
        a[ch].pos = __ldcg(&qp->a[ch].pos);
      }
      kb = __ldcg(&qp->kept);
      nc = __ldcg(&qp->noncol);
    }
    unsigned long long key[2][4];
    bool valid[2], win[2];
    cand_keys(a[0], true, key[0]);
    cand_keys(a[1], false, key[1]);
    valid[0] = a[0].d > 0.0;
    valid[1] = a[1].d > 0.0;
    if (threadIdx.x == 0) {
      s_kept = 0;
      s_nc = 0;
    }
    SHB_PROBE(if (probe) B.dbg[1606] = globaltimer_ns() + ((key[0][0] ^ kb) == 1ull ? 1ull : 0ull));
    cta_lexmin<2, 4>(key, valid, s_best2, win);  // starts with a barrier
    SHB_PROBE(if (probe) B.dbg[1607] = globaltimer_ns());
    {  // one shared atomic per warp (threads past the grid hold zeros)
      unsigned long long wk = kb;
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) wk += __shfl_xor_sync(FULL, wk, m);
      const bool wnc = __any_sync(FULL, nc != 0);
      if (lane == 0 && wk) atomicAdd(&s_kept, wk);
      if (lane == 0 && wnc) s_nc = 1u;
    }
    if (win[0]) s_cand[0] = a[0];
    if (win[1]) s_cand[1] = a[1];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int ch = 0; ch < 2; ++ch)
        if (s_best2[ch][0] == ~0ull) s_cand[ch] = empty_cand();
      const unsigned long long kept_all = s_kept;
      const uint32_t st = !s_nc ? ST_COLLINEAR : kept_all == 2 ? ST_DONE : ST_RUNNING;
      s_status = st;
      if (blockIdx.x == 0) {
        const unsigned long long now = globaltimer_ns() - c->t0_ns;
        c->mark[2] = now;
        c->mark[3] = now;
        c->kept = kept_all;
        c->noncollinear = s_nc;
        if (st == ST_COLLINEAR) {
          c->status = ST_COLLINEAR;  // hull.cpp:238-248
        } else {
          // first split (hull.cpp:101-158): P0 heads the lower chain, Pr the upper
          B.Tx[0][0] = c->ext_x[0];
          B.Ty[0][0] = c->ext_y[0];
          B.Tid[0][0] = c->ext_id[0];
          B.Tx[0][1] = c->ext_x[2];
          B.Ty[0][1] = c->ext_y[2];
          B.Tid[0][1] = c->ext_id[2];
          c->S_cur = 2;
          c->Slo_cur = 1;
          c->m_cur = (uint32_t)(kept_all - 2);
          c->round = 0;
          if (st == ST_DONE) c->status = ST_DONE;
        }
      }
    }
    __syncthreads();
    if (s_status != ST_RUNNING) {
      stream_drain_points(R, pre, B.n, reinterpret_cast<const unsigned char*>(B.bits));
      return;
    }
  }

  // ---- table phase (S = 2: the lower chain P0->Pr and the upper chain Pr->P0) ----
  if (threadIdx.x == 0) {
    uint32_t ns = 0, Slon = 1;
    const double hx[2] = {__ldcg(&c->ext_x[0]), __ldcg(&c->ext_x[2])};
    const double hy[2] = {__ldcg(&c->ext_y[0]), __ldcg(&c->ext_y[2])};
    const uint32_t hid[2] = {__ldcg(&c->ext_id[0]), __ldcg(&c->ext_id[2])};
    for (int s = 0; s < 2; ++s) {
      const Cand& cr = s_cand[s];
      const bool split = cr.d > 0.0;
      Route r;
      r.ax = hx[s];
      r.ay = hy[s];
      r.bx = hx[s ^ 1];
      r.by = hy[s ^ 1];
      r.cx = split ? cr.x : 0.0;
      r.cy = split ? cr.y : 0.0;
      r.cid = split ? cr.id : NONE;
      r.ns = ns;
      r.flags = (split ? RT_SPLIT : 0u) | (s == 0 ? RT_LOWER : 0u);
      r.pad = 0;
      s_rt[s] = r;
      if (blockIdx.x == 0) {
        B.Tx[1][ns] = r.ax;
        B.Ty[1][ns] = r.ay;
        B.Tid[1][ns] = hid[s];
        if (split) {
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
    s_off = 0;
    for (int t = 0; t < 4; ++t) rec_clear(&s_db[t], &s_rec[t]);
    if (blockIdx.x == 0)  // clear round 2's slots
      for (int t = 0; t < 8; ++t) {
        rec_clear(&B.Sd[2][t], &B.Srec[2][t]);
        B.Wn[2][t] = NONE;
      }
  }
  __syncthreads();
  const uint32_t Sn = s_Sn, Slon = s_Slon;
  const uint32_t run_base = blockIdx.x * B.run_q;
  double2* Oxy = B.Lxy[1];
  uint2* Ois = B.Lis[1];

  // ---- point phase: forward over the input (K2 left the head in L2) ----
  // FULLT: a full tile (no bounds checks); branch-free routing of every point
  // (non-members are masked), one warp-uniform branch for the rare contenders.
  auto tile = [&](auto fullt, int s, uint32_t first, uint32_t cnt) {
    constexpr bool FULLT = decltype(fullt)::value;
    const double* xs = R.xs + s * Cfg3::T;
    const double* ys = R.ys + s * Cfg3::T;
    const uint32_t* is = R.is + s * Cfg3::T;
    const uint4* bs = reinterpret_cast<const uint4*>(R.aux + s * L::Ring::kAuxBytes);
    const uint32_t c4 = cnt & ~3u;
    double px[K3_NP], py[K3_NP], pd[K3_NP];
    uint32_t pid[K3_NP], pseg[K3_NP];
    uint32_t keepm = 0, lowm = 0;
#pragma unroll
    for (int kk = 0; kk < K3_NP / 2; ++kk) {
      const uint32_t cc = kk * Cfg3::CW + warp;  // chunk of 64 points within the tile
      const uint32_t j = cc * 64 + 2 * lane;
      uint4 bits = make_uint4(0u, 0u, 0u, 0u);
      double2 xv = make_double2(0.0, 0.0), yv = xv;
      uint2 iv = make_uint2(0u, 0u);
      if (FULLT) {
        bits = bs[cc];
        xv = reinterpret_cast<const double2*>(xs)[j >> 1];
        yv = reinterpret_cast<const double2*>(ys)[j >> 1];
        if (IDS) iv = reinterpret_cast<const uint2*>(is)[j >> 1];
      } else if (cc * 64 < cnt) {
        bits = bs[cc];
        if (j + 1 < c4) {
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
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = 2 * kk + h;
        px[q] = h ? xv.y : xv.x;
        py[q] = h ? yv.y : yv.x;
        pid[q] = IDS ? (h ? iv.y : iv.x) : first + j + h;
        const uint32_t lw = ((h ? bits.y : bits.x) >> lane) & 1u;
        const uint32_t uw = ((h ? bits.w : bits.z) >> lane) & 1u;
        bool lower = false;
        const bool keep =
            route_point<false>(s_rt + opaque_u32(lw ^ 1u), px[q], py[q], pid[q], pd[q], pseg[q], lower);
        keepm |= (uint32_t)((lw | uw) & keep) << q;
        lowm |= lw << q;
      }
    }
    // contenders: kept points reaching the CTA slot's running maximum
    uint32_t candm = 0;
#pragma unroll
    for (int q = 0; q < K3_NP; ++q) {
      const uint32_t dh = (uint32_t)((unsigned long long)__double_as_longlong(pd[q]) >> 32);
      candm |= (uint32_t)(((keepm >> q) & 1u) & (dh >= *(volatile uint32_t*)&s_db[pseg[q] & 3u])) << q;
    }
    if (__any_sync(FULL, candm)) contend_tile<K3_NP>(s_db, s_rec, candm, px, py, pd, pid, pseg, lowm);
    if (CAPPED)
      run_append<K3_NP, true>(keepm, px, py, pid, pseg, &s_off, Oxy, Ois, run_base, pd, 0u, nullptr,
                              nullptr, run_base + B.run_q, &c->status);
    else
      run_append<K3_NP>(keepm, px, py, pid, pseg, &s_off, Oxy, Ois, run_base);
  };
  stream_input(R, n, X, Y, I, reinterpret_cast<const unsigned char*>(B.bits), false,
               [&](int s, uint32_t first, uint32_t cnt) {
    if (cnt == (uint32_t)Cfg3::T)
      tile(std::true_type{}, s, first, cnt);
    else
      tile(std::false_type{}, s, first, cnt);
  }, pre, true);
  if (threadIdx.x == 0 && c->tl_round == 255u) B.dbg[512 + blockIdx.x] = globaltimer_ns() - c->t0_ns;

  // ---- flush the CTA's records to the global slots of round 2's argmax ----
  __syncthreads();
  SHB_PROBE(if (threadIdx.x == 0 && c->tl_round == 255u) B.dbg[1400 + blockIdx.x] = globaltimer_ns());
  if (threadIdx.x == 0 && (s_off & 1u) && s_off < B.run_q) {  // pad the run to an even length
    Oxy[run_base + s_off] = make_double2(0.0, 0.0);
    Ois[run_base + s_off] = make_uint2(NONE, NONE);
  }
  if (threadIdx.x < 4) {  // this CTA's records -> its row (no contention)
    SlotRec o = s_rec[threadIdx.x];
    if (threadIdx.x >= Sn) o.id = NONE;
    o.lock = 0u;
    B.Rc[1][(size_t)blockIdx.x * NSLOT + threadIdx.x] = o;
  }
  if (threadIdx.x == 0) B.run_cnt[1][blockIdx.x] = s_off;

  // ---- last CTA closes round 1 ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  // the last CTA combines the CTAs' rows: one thread per row, every field
  // loaded in one round trip, run counts summed per warp
  if (!s_last) return;
  SHB_PROBE(const bool probe_c = threadIdx.x == 0 && c->tl_round == 255u);
  SHB_PROBE(if (probe_c) B.dbg[1611] = globaltimer_ns());
  __threadfence();
  __shared__ uint32_t s_mn;
  {  // the farthest record of each segment over the CTAs' rows -> Srec[1]
    __shared__ unsigned long long s_best4[4][4];
    Cand a[4];
    unsigned long long key[4][4];
    bool valid[4], win[4];
    const bool row = threadIdx.x < gridDim.x;
    const uint32_t rc = row ? __ldcg(B.run_cnt[1] + threadIdx.x) : 0u;
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // every field in one round trip
      a[t] = empty_cand();
      if (row) {
        const SlotRec* q = B.Rc[1] + (size_t)threadIdx.x * NSLOT + t;
        a[t].id = __ldcg(&q->id);
        a[t].d = __ldcg(&q->d);
        a[t].x = __ldcg(&q->x);
        a[t].y = __ldcg(&q->y);
      }
    }
    if (threadIdx.x == 0) s_mn = 0;
    const uint32_t wsum = __reduce_add_sync(FULL, rc);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      a[t].pos = 0;
      cand_keys(a[t], (uint32_t)t < Slon, key[t]);
      valid[t] = a[t].id != NONE;
    }
    __syncthreads();
    if (lane == 0 && wsum) atomicAdd(&s_mn, wsum);
    SHB_PROBE(if (probe_c) B.dbg[1612] = globaltimer_ns());
    cta_lexmin<4, 4>(key, valid, s_best4, win);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (win[t]) {
        SlotRec o;
        o.d = a[t].d; o.x = a[t].x; o.y = a[t].y; o.id = a[t].id; o.lock = 0u;
        B.Srec[1][t] = o;
        B.Sd[1][t] = (unsigned long long)__double_as_longlong(a[t].d);
      }
    }
  }
  if (threadIdx.x != 0) return;
  const uint32_t mn = s_mn;
  SHB_PROBE(if (probe_c) B.dbg[1613] = globaltimer_ns());
  c->ticket = 0;
  const uint32_t before = c->S_cur + c->m_cur;
  StatRec st;
  st.segments = Sn;
  st.points_remaining = Sn + mn;
  st.points_removed = before - (Sn + mn);
  st.pad = 0;
  st.end_ns = globaltimer_ns() - *(volatile unsigned long long*)&c->t0_ns;
  st.table_ns = 0;
  st.points_ns = 0;
  B.stats[0] = st;
  c->round = 1;
  c->S_cur = Sn;
  c->Slo_cur = Slon;
  c->m_cur = mn;
  c->nruns = gridDim.x;
  if (mn == 0) c->status = ST_DONE;
  c->mark[4] = globaltimer_ns() - c->t0_ns;
  __threadfence();
}

// ===========================================================================
// KR: rounds >= 2, one persistent cooperative launch
// ===========================================================================

constexpr int RW = RTPB / 32;          // warps per CTA
constexpr int KR_U = LIVE_T / RCTHREADS;  // live points per consumer thread per tile

#ifndef SHB_DEFER
#define SHB_DEFER 1  // large tables: consume a tile's atomicMax results one tile later
#endif
#ifndef SHB_MED
#define SHB_MED 1
#endif
struct RoundSmem {
  double2 lxy[LIVE_NS][LIVE_T];    // TMA ring of live points: xy          90 KB
  uint2 lis[LIVE_NS][LIVE_T];      //                          (id, seg)   45 KB
  Route rt[SMALL_S];               // route entries of a small table       32 KB
  uint32_t db[2 * NSLOT];          // CTA farthest slots: distance high words (first NSLOT) 8 KB
  SlotRec rec[NSLOT];              //                     records          32 KB
  unsigned long long lbar[LIVE_NS];   // full   (after everything the solo tail overlays)
  unsigned long long lebar[LIVE_NS];  // empty (one arrival per warp)
};

// medium tables reuse rt | db | rec (idle in large rounds) as one u64 array
[[maybe_unused]] constexpr int MED_S = (int)((sizeof(Route) * SMALL_S + 8 * NSLOT + sizeof(SlotRec) * NSLOT) / 8);
static_assert(offsetof(RoundSmem, db) == offsetof(RoundSmem, rt) + sizeof(Route) * SMALL_S &&
              offsetof(RoundSmem, rec) == offsetof(RoundSmem, db) + 8 * NSLOT,
              "rt, db, rec must be contiguous");

// Barrier over the CTAs still working on the rounds.
#ifndef SHB_BAR_CTR
#define SHB_BAR_CTR 1
#endif
// `bar` is this CTA's running arrival target (the same on every participant)
SH_DEV void rounds_barrier(Ctl* c, uint32_t P, unsigned long long& bar) {
#if SHB_BAR_CTR
  if (P > 1) {
    bar += P;
    grid_barrier_ctr(&c->bar_ctr, bar);
    return;
  }
#else
  if (P > 1) grid_barrier(&c->bar_count, &c->bar_gen, P);
#endif
  else __syncthreads();
}

// Route entry of old segment s from head table `pin` and farthest record `cr`.
SH_DEV Route make_route(const Bufs& B, uint32_t pin, const SlotRec* cr, uint32_t s, uint32_t S,
                        uint32_t Slo, uint32_t ns) {
  const bool shared = __isShared(cr);
  const uint32_t cid = shared ? cr->id : __ldcg(&cr->id);
  const bool split = cid != NONE;
  const uint32_t sb = s + 1 == S ? 0u : s + 1;
  Route r;
  r.ax = __ldcg(B.Tx[pin] + s);
  r.ay = __ldcg(B.Ty[pin] + s);
  r.bx = __ldcg(B.Tx[pin] + sb);
  r.by = __ldcg(B.Ty[pin] + sb);
  r.cx = split ? (shared ? cr->x : __ldcg(&cr->x)) : 0.0;
  r.cy = split ? (shared ? cr->y : __ldcg(&cr->y)) : 0.0;
  r.cid = cid;
  r.ns = ns;
  r.flags = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
  r.pad = 0;
  return r;
}

SH_DEV void write_heads(const Bufs& B, uint32_t pin, uint32_t pout, const Route& r, uint32_t s) {
  B.Tx[pout][r.ns] = r.ax;
  B.Ty[pout][r.ns] = r.ay;
  B.Tid[pout][r.ns] = __ldcg(B.Tid[pin] + s);
  if (r.flags & RT_SPLIT) {
    B.Tx[pout][r.ns + 1] = r.cx;
    B.Ty[pout][r.ns + 1] = r.cy;
    B.Tid[pout][r.ns + 1] = r.cid;
  }
}

// Where the farthest records of the current segments are: this CTA's shared
// slots (a lone CTA kept them), the global records Srec (written by K3, the
// small-input kernel or the solo tail), or the CTA rows of a multi-CTA round,
// resolved through the winner words Wn.
enum : uint32_t { RS_SMEM = 0, RS_SREC = 1, RS_ROWS = 2, RS_WIN = 3 };  // RS_WIN: solo import only
struct RecSrc {
  uint32_t kind;
  const SlotRec* base;  // sm.rec, Srec[sin] or Rc[parity of the previous round]
  const uint32_t* wn;   // RS_ROWS: Wn[sin]
};

// record of segment s, or nullptr when it has none (RS_ROWS without winner)
SH_DEV const SlotRec* rec_at(const RecSrc& rs, uint32_t s) {
  if (rs.kind != RS_ROWS) return rs.base + s;
  const uint32_t w = __ldcg(rs.wn + s);
  return w == NONE ? nullptr : rs.base + (size_t)w * NSLOT + s;
}
SH_DEV uint32_t rec_id(const SlotRec* r) {
  return r == nullptr ? NONE : (__isShared(r) ? r->id : __ldcg(&r->id));
}

// Small table (S <= SMALL_S), rebuilt by every participating CTA in smem.
// CTA 0 also writes the next head table.  The farthest records of the
// current segments come from the global slots, or -- when the previous round
// ran on this single CTA -- straight from its shared-memory slots.
// Returns S', S'lo.
SH_DEV void table_small(const Bufs& B, RoundSmem& sm, uint32_t S, uint32_t Slo, uint32_t pin,
                        uint32_t pout, const RecSrc& rs, uint32_t* s_ws,
                        uint32_t& Sn, uint32_t& Slon) {
  __shared__ SlotRec s_none;  // stands for "no record" in make_route
  if (threadIdx.x == 0) {
    s_none.d = s_none.x = s_none.y = 0.0;
    s_none.id = NONE;
    s_none.lock = 0u;
  }
  __syncthreads();
  const bool heads = blockIdx.x == 0;
  uint32_t running = 0, lower_splits = 0;
  for (uint32_t s0 = 0; s0 < S; s0 += RTPB) {
    const uint32_t s = s0 + threadIdx.x;
    const SlotRec* cr = s < S ? rec_at(rs, s) : nullptr;
    const uint32_t split = rec_id(cr) != NONE ? 1u : 0u;
    uint32_t total;
    const uint32_t pre = block_exclusive_scan(split, s_ws, &total);
    lower_splits += (uint32_t)__syncthreads_count(split && s < Slo);
    if (s < S) {
      const Route r = make_route(B, pin, cr ? cr : &s_none, s, S, Slo, s + running + pre);
      sm.rt[s] = r;
      if (heads) write_heads(B, pin, pout, r, s);
    }
    running += total;
  }
  Sn = S + running;
  Slon = Slo + lower_splits;
  __syncthreads();  // every route is built before the records are recycled
  for (uint32_t t = threadIdx.x; t < Sn; t += RTPB) rec_clear(&sm.db[t], &sm.rec[t]);
  __syncthreads();
}

// Large table (S > SMALL_S): a grid-wide two-step scan over the P
// participating CTAs.  Segment s splits iff it has a farthest point: its
// winner slot Wn[sin][s] holds C's position in the input live set -- or,
// right after a small round (from_rec), its flushed record Srec[sin][s].
// Each warp owns 32 x TS consecutive segments per step, lane-contiguous so
// every load and store is coalesced.  Finished segments (no split) cost one
// head copy; only split ones build a route row and prepare the two winner
// slots / distance maxima of their children.  Returns false on segment-table
// overflow (every CTA returns consistently).
#ifndef SHB_TS
#define SHB_TS 2
#endif
#ifndef SHB_T1_U
#define SHB_T1_U 8  // split-count pass: loads in flight per thread
#endif
#ifndef SHB_TL_PREF
#define SHB_TL_PREF 1  // heads of the next scatter step loaded one step ahead
#endif
constexpr int TS = SHB_TS;

SH_DEV bool table_large(const Bufs& B, uint32_t S, uint32_t Slo, uint32_t pin, uint32_t pout,
                        uint32_t sin, uint32_t sout, uint32_t P, bool from_rec, const RecSrc& rs,
                        uint32_t* s_ws, uint32_t& Sn, uint32_t& Slon, unsigned long long& bar) {
  Ctl* c = B.ctl;
  constexpr uint32_t STEP = RTPB * TS;
  // CTA ranges are whole warp chunks (32 * TS), so that the lane mapping is
  // identical in both passes
  const uint32_t chunks = (S + 32 * TS - 1) / (32 * TS);
  const uint32_t per = (chunks + P - 1) / P * (32 * TS);
  const uint32_t lo = min(S, blockIdx.x * per), hi = min(S, lo + per);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t* Win = B.Wn[sin];
  auto split_of = [&](uint32_t s) -> uint32_t {  // C's live position / record index, or NONE
    if (s >= hi) return NONE;
    if (from_rec) return rec_id(rec_at(rs, s)) != NONE ? s : NONE;
    return __ldcg(Win + s);
  };
  // T1: split counts of this CTA's range (total and lower chain)
  uint32_t cnt = 0, cnt_lo = 0;
#if SHB_T1_U
  // only the totals matter here: any mapping of [lo, hi), T1_U loads in flight
  constexpr int U1 = SHB_T1_U;
  for (uint32_t g0 = lo + threadIdx.x; g0 < hi; g0 += RTPB * U1) {
    uint32_t w[U1];
#pragma unroll
    for (int i = 0; i < U1; ++i) w[i] = split_of(g0 + i * RTPB);
#pragma unroll
    for (int i = 0; i < U1; ++i) {
      cnt += w[i] != NONE;
      cnt_lo += w[i] != NONE && g0 + i * RTPB < Slo;
    }
  }
#else
  for (uint32_t g0 = lo + wid * 32 * TS; g0 < hi; g0 += STEP) {
    uint32_t w[TS];
#pragma unroll
    for (int i = 0; i < TS; ++i) w[i] = split_of(g0 + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      const uint32_t s = g0 + i * 32 + lane;
      cnt += w[i] != NONE;
      cnt_lo += w[i] != NONE && s < Slo;
    }
  }
#endif
  {
    uint32_t t1, t2;
    block_exclusive_scan(cnt, s_ws, &t1);
    block_exclusive_scan(cnt_lo, s_ws, &t2);
    if (threadIdx.x == 0) {
      B.blk_cnt[blockIdx.x] = t1;
      B.blk_cnt[MAX_ROUND_BLOCKS + blockIdx.x] = t2;
    }
  }
  rounds_barrier(c, P, bar);
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
  const double* Tx = B.Tx[pin];
  const double* Ty = B.Ty[pin];
  const uint32_t* Tid = B.Tid[pin];
  double* Ox = B.Tx[pout];
  double* Oy = B.Ty[pout];
  uint32_t* Oid = B.Tid[pout];
  uint32_t* Wout = B.Wn[sout];
  unsigned long long* Sdo = B.Sd[sout];
  const uint32_t lt = lanemask_lt();
  uint32_t running = pre_all;
  // every step covers [lo + k*STEP, lo + (k+1)*STEP): warps in order.  All
  // loads of a step -- the heads, and for split segments the next head and C
  // -- are issued before the step's block scan, so one memory round trip
  // overlaps the scan; the end point B of segment s is the head of s + 1,
  // taken from the neighbouring lane.
  // The split words of the next step are loaded one step ahead.
  uint32_t wn[TS];
#pragma unroll
  for (int i = 0; i < TS; ++i) wn[i] = split_of(lo + wid * 32 * TS + i * 32 + lane);
#if SHB_TL_PREF
  // the heads of the next step are loaded one step ahead too
  double axn[TS], ayn[TS];
  uint32_t aidn[TS];
#pragma unroll
  for (int i = 0; i < TS; ++i) {
    const uint32_t s = min(lo + wid * 32 * TS + i * 32 + lane, S - 1);
    axn[i] = __ldcg(Tx + s);
    ayn[i] = __ldcg(Ty + s);
    aidn[i] = __ldcg(Tid + s);
  }
#endif
  for (uint32_t b0 = lo; b0 < hi; b0 += STEP) {
    const uint32_t g0 = b0 + wid * 32 * TS;
    uint32_t w[TS];
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      w[i] = wn[i];
      wn[i] = split_of(g0 + STEP + i * 32 + lane);
    }
    double ax[TS], ay[TS], cx[TS], cy[TS];
    uint32_t aid[TS], cid[TS];
#if SHB_TL_PREF
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      ax[i] = axn[i];
      ay[i] = ayn[i];
      aid[i] = aidn[i];
      const uint32_t s = min(g0 + STEP + i * 32 + lane, S - 1);
      axn[i] = __ldcg(Tx + s);
      ayn[i] = __ldcg(Ty + s);
      aidn[i] = __ldcg(Tid + s);
    }
#else
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      const uint32_t s = min(g0 + i * 32 + lane, S - 1);
      ax[i] = __ldcg(Tx + s);
      ay[i] = __ldcg(Ty + s);
      aid[i] = __ldcg(Tid + s);
    }
#endif
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      cx[i] = cy[i] = 0.0;
      cid[i] = NONE;
      if (w[i] != NONE) {  // implies s < hi
        if (from_rec) {
          const SlotRec* cr = rec_at(rs, g0 + i * 32 + lane);  // global, a winner exists
          cx[i] = __ldcg(&cr->x);
          cy[i] = __ldcg(&cr->y);
          cid[i] = __ldcg(&cr->id);
        } else {
          const double2 cv = __ldcg(B.Lxy[pin] + w[i]);
          cx[i] = cv.x;
          cy[i] = cv.y;
          cid[i] = __ldcg(&B.Lis[pin][w[i]].x);
        }
      }
    }
    uint32_t wpre[TS], wtot = 0;
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      const uint32_t bal = __ballot_sync(FULL, w[i] != NONE);
      wpre[i] = wtot + __popc(bal & lt);
      wtot += __popc(bal);
    }
    uint32_t total;
    const uint32_t wx = block_exclusive_scan(lane == 0 ? wtot : 0u, s_ws, &total);
    const uint32_t wbase = running + __shfl_sync(FULL, wx, 0);
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      const uint32_t s = g0 + i * 32 + lane;
      // B = head of s + 1: lane + 1 of this row, lane 0 of the next row, or
      // (last lane of the last row, the table's last segment) a load
      double bx = __shfl_down_sync(FULL, ax[i], 1);
      double by = __shfl_down_sync(FULL, ay[i], 1);
      if (i + 1 < TS) {
        const double nx = __shfl_sync(FULL, ax[i + 1 < TS ? i + 1 : i], 0);
        const double ny = __shfl_sync(FULL, ay[i + 1 < TS ? i + 1 : i], 0);
        if (lane == 31) bx = nx, by = ny;
      }
      if (s < hi) {
        const uint32_t ns = s + wbase + wpre[i];
        Ox[ns] = ax[i];
        Oy[ns] = ay[i];
        Oid[ns] = aid[i];
        Wout[ns] = NONE;
        if (w[i] != NONE) {
          if ((lane == 31 && i + 1 == TS) || s + 1 == S) {
            const uint32_t sb = s + 1 == S ? 0u : s + 1;
            bx = __ldcg(Tx + sb);
            by = __ldcg(Ty + sb);
          }
          Route r;
          r.ax = ax[i];
          r.ay = ay[i];
          r.cx = cx[i];
          r.cy = cy[i];
          r.bx = bx;
          r.by = by;
          r.cid = cid[i];
          r.ns = ns;
          r.flags = RT_SPLIT | (s < Slo ? RT_LOWER : 0u);
          r.pad = 0;
          B.route[s] = r;
          Ox[ns + 1] = r.cx;
          Oy[ns + 1] = r.cy;
          Oid[ns + 1] = r.cid;
          Wout[ns + 1] = NONE;
          Sdo[ns] = 0ull;
          Sdo[ns + 1] = 0ull;
        }
      }
    }
    running += total;
  }
  rounds_barrier(c, P, bar);
  return true;
}

// ---------------------------------------------------------------------------
// Solo tail: once a single CTA is left with a table of at most SOLO_S
// segments and a live set that fits its shared memory, it runs the remaining
// rounds with everything in shared memory -- live points (ping-pong), head
// table, routes and farthest records -- touching global memory only for the
// round stats and, at the end, the final head table.  It overlays the ring
// and the small-table storage (everything in RoundSmem before the mbarriers).
// Routes are compact: a point reads A, C and B from the new head table (A at
// the segment's new index ns, C at ns + 1, B at ns + 2), which the table step
// rewrites in place before the point step.
constexpr uint32_t SOLO_S = 2 * RTPB;  // segments before a solo round (disk 20M: h = 933)
constexpr uint32_t SOLO_NS = 2 * SOLO_S;
constexpr uint32_t SOLO_CAP = 1512;    // live points per ping-pong buffer
struct SoloSmem {
  double2 pxy[2][SOLO_CAP];
  uint2 pis[2][SOLO_CAP];          // (id, old segment)
  double2 hxy[SOLO_NS];            // head table
  uint32_t hid[SOLO_NS];
  uint4 rt[SOLO_S];                // (new index ns, C's id, flags, -)
  uint32_t db[SOLO_NS];            // farthest records of the next round's segments (high words)
  SlotRec rec[SOLO_NS];
};
static_assert(sizeof(SoloSmem) <= offsetof(RoundSmem, lbar), "solo tail does not fit");
static_assert(offsetof(SoloSmem, rec) % 16 == 0 && offsetof(SoloSmem, hxy) % 16 == 0, "alignment");

struct SoloState {
  uint32_t r, S, Slo, m, nruns;
};

// route_point for the solo tail's compact routes (the same rule)
SH_DEV bool route_solo(const SoloSmem& so, uint32_t Sn, uint32_t seg, double x, double y, uint32_t id,
                       double& d, uint32_t& nseg, bool& lower) {
  const uint4 r = so.rt[seg];
  lower = r.z & RT_LOWER;
  nseg = r.x;
  d = 0.0;
  if (!(r.z & RT_SPLIT)) return false;
  const uint32_t nb = r.x + 2 == Sn ? 0u : r.x + 2;
  const double2 A = so.hxy[r.x], C = so.hxy[r.x + 1], Bv = so.hxy[nb];
  const bool xeq = x == C.x;
  const bool lt = x < C.x || (xeq && y < C.y);
  const bool eq = xeq && y == C.y;
  const bool left = lower ? lt : !(lt || eq);
  const double2 S = left ? A : C, E = left ? C : Bv;
  d = outward_e(make_edge(S.x, S.y, E.x, E.y), x, y);
  nseg = r.x + (left ? 0u : 1u);
  return id != r.y && d > 0.0;
}

// Returns true when the call is finished (control block written), false when
// the table outgrew SOLO_S: the state is then exported to global memory (one
// run, records in Srec) and the caller continues with the grid-wide rounds.
// `rs` RS_WIN: the previous round used a large table (winner positions in Wn).
SH_DEV bool solo_rounds(const Bufs& B, RoundSmem& sm, SoloState& st, const RecSrc& rs,
                        uint32_t* s_ws, uint32_t* s_pref, uint32_t* s_off) {
  Ctl* c = B.ctl;
  SoloSmem& so = *reinterpret_cast<SoloSmem*>(&sm.lxy[0][0]);
  const uint32_t tid = threadIdx.x, q = B.run_q, n = B.n;
  uint32_t r = st.r, S = st.S, Slo = st.Slo, m = st.m;
  const unsigned long long t0 = *(volatile unsigned long long*)&c->t0_ns;
  {  // ---- import: heads, records, live set ----
    const uint32_t pin = (r - 1) & 1u;
    // the records first, into registers: with RS_SMEM they sit in sm.rec,
    // which the solo layout overlays
    SlotRec g[SOLO_S / RTPB];
#pragma unroll
    for (int h = 0; h < (int)(SOLO_S / RTPB); ++h) {
      const uint32_t s = tid + h * RTPB;
      g[h].id = NONE;
      g[h].d = g[h].x = g[h].y = 0.0;
      g[h].lock = 0u;
      if (s >= S) continue;
      if (rs.kind == RS_SMEM) {
        g[h] = sm.rec[s];
      } else if (rs.kind == RS_WIN) {  // winner's live position (large table)
        const uint32_t w = __ldcg(rs.wn + s);
        if (w != NONE) {
          const double2 v = __ldcg(B.Lxy[pin] + w);
          g[h].x = v.x;
          g[h].y = v.y;
          g[h].id = __ldcg(&B.Lis[pin][w].x);
          g[h].d = __longlong_as_double((long long)__ldcg(B.Sd[(r - 1) % 3u] + s));
        }
      } else {
        const SlotRec* p = rec_at(rs, s);
        if (rec_id(p) != NONE) {
          g[h].d = __ldcg(&p->d);
          g[h].x = __ldcg(&p->x);
          g[h].y = __ldcg(&p->y);
          g[h].id = __ldcg(&p->id);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < (int)(SOLO_S / RTPB); ++h) {
      const uint32_t s = tid + h * RTPB;
      if (s >= S) continue;
      so.rec[s] = g[h];
      so.db[s] = g[h].id == NONE ? 0u : (uint32_t)((unsigned long long)__double_as_longlong(g[h].d) >> 32);
      so.hxy[s] = make_double2(__ldcg(B.Tx[pin] + s), __ldcg(B.Ty[pin] + s));
      so.hid[s] = __ldcg(B.Tid[pin] + s);
    }
    const uint32_t nruns = st.nruns;
    uint32_t tot;
    for (uint32_t j0 = 0; j0 < nruns; j0 += RTPB) {
      const uint32_t j = j0 + tid;
      uint32_t v = j < nruns ? (nruns == 1 ? m : __ldcg(B.run_cnt[pin] + j)) : 0u;
      v += v & 1u;
      const uint32_t base0 = j0 ? s_pref[j0] : 0u;
      const uint32_t ex = block_exclusive_scan(v, s_ws, &tot);
      if (j < nruns) s_pref[j] = base0 + ex;
      if (tid == 0) s_pref[min(j0 + RTPB, nruns)] = base0 + tot;
      __syncthreads();
    }
    const uint32_t Mp = s_pref[nruns];
    for (uint32_t v = tid; v < Mp; v += RTPB) {
      uint32_t a0 = 0, a1 = nruns;
      while (a1 - a0 > 1) {
        const uint32_t mid = (a0 + a1) >> 1;
        if (s_pref[mid] <= v) a0 = mid; else a1 = mid;
      }
      const uint32_t phys = a0 * q + (v - s_pref[a0]);
      so.pxy[0][v] = __ldcg(B.Lxy[pin] + phys);
      so.pis[0][v] = __ldcg(B.Lis[pin] + phys);
    }
    m = Mp;  // entries of buffer 0, pads (segment NONE) included
    __syncthreads();
  }
  uint32_t cur = 0;
  while (true) {
    const uint32_t pout = r & 1u;
    // ---- table: new indices and heads (in place), then the compact routes ----
    uint32_t Sn, Slon;
    {
      constexpr int H = SOLO_S / RTPB;
      uint32_t ns[H], cid[H], fl[H];
      double ax[H], ay[H], cx[H], cy[H];
      uint32_t aid[H];
      uint32_t running = 0, lower_splits = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const uint32_t s = tid + h * RTPB;
        ns[h] = s;
        fl[h] = 0u;
        if (h > 0 && S <= (uint32_t)(h * RTPB)) continue;  // CTA-uniform: no segments here
        const bool split = s < S && so.rec[s].id != NONE;
        uint32_t total;
        const uint32_t pre = block_exclusive_scan(split ? 1u : 0u, s_ws, &total);
        lower_splits += (uint32_t)__syncthreads_count(split && s < Slo);
        ns[h] = s + running + pre;
        cid[h] = split ? so.rec[s].id : NONE;
        fl[h] = (split ? RT_SPLIT : 0u) | (s < Slo ? RT_LOWER : 0u);
        cx[h] = split ? so.rec[s].x : 0.0;
        cy[h] = split ? so.rec[s].y : 0.0;
        const double2 a = s < S ? so.hxy[s] : make_double2(0.0, 0.0);
        ax[h] = a.x;
        ay[h] = a.y;
        aid[h] = s < S ? so.hid[s] : NONE;
        running += total;
      }
      Sn = S + running;
      Slon = Slo + lower_splits;
      __syncthreads();  // every old head and record is read
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const uint32_t s = tid + h * RTPB;
        if (s >= S) continue;
        so.rt[s] = make_uint4(ns[h], cid[h], fl[h], 0u);
        so.hxy[ns[h]] = make_double2(ax[h], ay[h]);
        so.hid[ns[h]] = aid[h];
        if (fl[h] & RT_SPLIT) {
          so.hxy[ns[h] + 1] = make_double2(cx[h], cy[h]);
          so.hid[ns[h] + 1] = cid[h];
        }
      }
      for (uint32_t t = tid; t < Sn; t += RTPB) rec_clear(&so.db[t], &so.rec[t]);
      if (tid == 0) *s_off = 0;
      __syncthreads();
    }
    const unsigned long long t_table = globaltimer_ns();
    // ---- points: route, keep, contend, append to the other buffer ----
    const double2* ixy = so.pxy[cur];
    const uint2* iis = so.pis[cur];
    double2* oxy = so.pxy[cur ^ 1u];
    uint2* ois = so.pis[cur ^ 1u];
    for (uint32_t i0 = 0; i0 < m; i0 += 2 * RTPB) {
      double px[2], py[2], pd[2];
      uint32_t pid[2], pseg[2];
      uint32_t keepm = 0, lowm = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t i = i0 + u * RTPB + tid;
        px[u] = py[u] = pd[u] = 0.0;
        pid[u] = 0;
        pseg[u] = 0;
        if (i < m) {
          const double2 v = ixy[i];
          const uint2 is = iis[i];
          if (is.y != NONE) {
            bool lower = false;
            px[u] = v.x;
            py[u] = v.y;
            pid[u] = is.x;
            if (route_solo(so, Sn, is.y, v.x, v.y, is.x, pd[u], pseg[u], lower)) keepm |= 1u << u;
            if (lower) lowm |= 1u << u;
          }
        }
      }
      contend_tile<2>(so.db, so.rec, keepm, px, py, pd, pid, pseg, lowm);
      run_append<2>(keepm, px, py, pid, pseg, s_off, oxy, ois, 0u);
    }
    __syncthreads();
    const uint32_t mn = *(volatile uint32_t*)s_off;
    if (tid == 0 && r <= (uint32_t)STATS_CAP) {
      StatRec sr;
      sr.segments = Sn;
      sr.points_remaining = Sn + mn;
      sr.points_removed = (S + st.m) - (Sn + mn);
      sr.pad = 0;
      const unsigned long long now = globaltimer_ns();
      sr.end_ns = now - t0;
      sr.table_ns = t_table - t0;
      sr.points_ns = now - t0;
      B.stats[r - 1] = sr;
    }
    const bool done = mn == 0 || r + 1 > n;
    if (done || Sn > SOLO_S) {
      // ---- export: the head table (+ records and live set to continue) ----
      for (uint32_t t = tid; t < Sn; t += RTPB) {
        const double2 h = so.hxy[t];
        B.Tx[pout][t] = h.x;
        B.Ty[pout][t] = h.y;
        B.Tid[pout][t] = so.hid[t];
      }
      if (done) {
        if (tid == 0) {
          c->round = r;
          c->S_cur = Sn;
          c->Slo_cur = Slon;
          c->m_cur = mn;
          c->nruns = 1;
          c->status = mn == 0 ? ST_DONE : ST_INTERNAL;  // hull.cpp:265-267
          c->mark[6] = globaltimer_ns() - t0;
          __threadfence();
        }
        return true;
      }
      const uint32_t sout = r % 3u;
      for (uint32_t t = tid; t < Sn; t += RTPB) {
        B.Sd[sout][t] = so.rec[t].id == NONE ? 0ull : (unsigned long long)__double_as_longlong(so.rec[t].d);
        SlotRec* g = B.Srec[sout] + t;
        g->d = so.rec[t].d;
        g->x = so.rec[t].x;
        g->y = so.rec[t].y;
        g->id = so.rec[t].id;
        g->lock = 0u;
      }
      for (uint32_t t = tid; t < mn + (mn & 1u); t += RTPB) {
        B.Lxy[pout][t] = t < mn ? oxy[t] : make_double2(0.0, 0.0);
        B.Lis[pout][t] = t < mn ? ois[t] : make_uint2(NONE, NONE);
      }
      if (tid == 0) B.run_cnt[pout][0] = mn;
      __syncthreads();
      st.r = r + 1;
      st.S = Sn;
      st.Slo = Slon;
      st.m = mn;
      st.nruns = 1;
      return false;
    }
    S = Sn;
    Slo = Slon;
    st.m = mn;  // real points of the next round (for points_removed)
    m = mn;
    cur ^= 1u;
    ++r;
  }
}

#ifndef SHB_ROUND_TARGET
#define SHB_ROUND_TARGET 640
#endif
constexpr uint32_t ROUND_TARGET = SHB_ROUND_TARGET;  // live points per active CTA before CTAs retire
#ifndef SHB_KR_REVERSE
#define SHB_KR_REVERSE 1
#endif
#ifndef SHB_ONE_CTA_WORK
#define SHB_ONE_CTA_WORK 0
#endif
constexpr uint32_t ONE_CTA_WORK = SHB_ONE_CTA_WORK;

__global__ void __launch_bounds__(RTPB, 1) k_rounds(Bufs B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RoundSmem& sm = *reinterpret_cast<RoundSmem*>(smem_raw);
  __shared__ uint32_t s_ws[RW + 1];
  __shared__ uint32_t s_off, s_coff;
  __shared__ uint32_t s_pref[MAX_RUNS + 1];
  Ctl* c = B.ctl;
  SHB_PROBE(const bool probe = blockIdx.x == 0 && threadIdx.x == 0 && c->tl_round == 255u);
  SHB_PROBE(if (probe) B.dbg[1604] = globaltimer_ns());
  pdl_wait();  // round 1 (K3) is complete and visible
  SHB_PROBE(if (probe) B.dbg[1605] = globaltimer_ns());
  if (*(volatile uint32_t*)&c->status != ST_RUNNING) return;
  uint32_t r = *(volatile uint32_t*)&c->round + 1;
  const uint32_t trace_r = c->tl_round;  // debug timeline of CTA 0 in this round (0: off)
#define KR_MARK()                                                               \
  if (trace_r == r && blockIdx.x == 0 && threadIdx.x == 0 && c->tl_n < 32u)     \
    c->tl[c->tl_n++] = globaltimer_ns() - c->t0_ns;
  uint32_t S = *(volatile uint32_t*)&c->S_cur;
  uint32_t Slo = *(volatile uint32_t*)&c->Slo_cur;
  uint32_t m = *(volatile uint32_t*)&c->m_cur;
  uint32_t nruns = *(volatile uint32_t*)&c->nruns;
  const uint32_t n = B.n, q = B.run_q;
  const uint32_t target = min(ROUND_TARGET, q);
  uint32_t P = gridDim.x;
  uint32_t rec_kind = RS_SREC;  // where this round's input records are (RecSrc)
  unsigned long long bar = 0;   // grid-barrier arrival target (rounds_barrier)
  auto rec_src = [&](uint32_t kind, uint32_t rr) {
    RecSrc rs;
    rs.kind = kind;
    rs.wn = B.Wn[(rr - 1) % 3u];
    rs.base = kind == RS_SMEM ? sm.rec : kind == RS_SREC ? B.Srec[(rr - 1) % 3u] : B.Rc[(rr - 1) & 1u];
    return rs;
  };
  bool prev_small = true;  // the previous round used a small table
  uint32_t kbase = 0;      // live tiles this CTA consumed in earlier rounds
  if (blockIdx.x == 0 && threadIdx.x == 0) c->mark[5] = globaltimer_ns() - c->t0_ns;
  unsigned long long t_table = 0, t_points = 0;  // CTA 0 phase timestamps
  if (threadIdx.x == 0) {
    for (int i = 0; i < LIVE_NS; ++i) {
      mbar_init(&sm.lbar[i], 1);
      mbar_init(&sm.lebar[i], RCWARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  while (true) {
    // active CTAs for this round: ~ROUND_TARGET live points each (m only
    // shrinks, so retired CTAs never need to come back); every CTA sees the
    // same m, so the decision is consistent
    {
      const uint32_t work = max(m, S);  // live points, or segments of a large table
      // below ONE_CTA_WORK a lone CTA beats a grid: no slot flush, no barrier
      const uint32_t want =
          work <= ONE_CTA_WORK ? 1u : max(1u, min(P, (work + target - 1) / target));
      if (blockIdx.x >= want) return;
      P = want;
    }
    KR_MARK();  // round start
    if (P == 1 && S <= SOLO_S && m + nruns <= SOLO_CAP) {
      SoloState ss{r, S, Slo, m, nruns};
      const RecSrc rs0 = rec_src(rec_kind, r);
      if (solo_rounds(B, sm, ss, rs0, s_ws, s_pref, &s_off)) return;
      r = ss.r;
      S = ss.S;
      Slo = ss.Slo;
      m = ss.m;
      nruns = ss.nruns;
      rec_kind = RS_SREC;  // the solo tail exported its records to Srec
      prev_small = true;
      continue;
    }
    const uint32_t pin = (r - 1) & 1u, pout = r & 1u;
    const uint32_t sin = (r - 1) % 3u, sout = r % 3u, sres = (r + 1) % 3u;
    const bool small = S <= (uint32_t)SMALL_S;
    uint32_t Sn, Slon;
    if (small) {
      table_small(B, sm, S, Slo, pin, pout, rec_src(rec_kind, r), s_ws, Sn, Slon);
    } else if (!table_large(B, S, Slo, pin, pout, sin, sout, P, prev_small, rec_src(rec_kind, r),
                            s_ws, Sn, Slon, bar)) {
      return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) t_table = globaltimer_ns();
    KR_MARK();  // table done
    // clear round r+1's global farthest slots (at most 2 Sn segments) when
    // round r+1 will use a small table; a large table clears its own slots
    if (Sn <= (uint32_t)SMALL_S) {
      const uint32_t lim = min(2 * Sn, B.s_cap);
      for (uint32_t t = blockIdx.x * RTPB + threadIdx.x; t < lim; t += P * RTPB) {
        rec_clear(B.Sd[sres] + t, B.Srec[sres] + t);
        B.Wn[sres][t] = NONE;
      }
    }
    // prefix of the input run counts: the live set as one virtual range
    {
      uint32_t tot;
      for (uint32_t j0 = 0; j0 < nruns; j0 += RTPB) {
        const uint32_t j = j0 + threadIdx.x;
        uint32_t v = j < nruns ? (nruns == 1 ? m : __ldcg(B.run_cnt[pin] + j)) : 0u;
        v += v & 1u;  // runs are padded to even lengths
        const uint32_t base0 = j0 ? s_pref[j0] : 0u;
        const uint32_t ex = block_exclusive_scan(v, s_ws, &tot);
        if (j < nruns) s_pref[j] = base0 + ex;
        if (threadIdx.x == 0) s_pref[min(j0 + RTPB, nruns)] = base0 + tot;
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) s_off = s_coff = 0;
#if SHB_MED
    // medium tables (the next table fits the idle small-table smem) with
    // several points per segment per CTA: a CTA-local running maximum per
    // segment screens the global atomics
    unsigned long long* mdb = reinterpret_cast<unsigned long long*>(sm.rt);
    const bool med = !small && Sn <= (uint32_t)MED_S && (uint64_t)m >= 2ull * P * Sn;
    if (med)
      for (uint32_t t = threadIdx.x; t < Sn; t += RTPB) mdb[t] = 0ull;
#endif
    __syncthreads();
    KR_MARK();  // slots cleared, run prefix built

    // ---- point phase: virtual range [lo, hi) of the live set -> run j ----
    // The runs are read as one virtual range (padded counts, all even); each
    // tile of LIVE_T positions is fetched by bulk copies, one per run piece.
    const double2* Ixy = B.Lxy[pin];
    const uint2* Iis = B.Lis[pin];
    double2* Oxy = B.Lxy[pout];
    uint2* Ois = B.Lis[pout];
    unsigned long long* Sd = B.Sd[sout];
    const uint32_t obase = blockIdx.x * q;
    const uint32_t Mp = s_pref[nruns];
    const uint32_t lo = 2u * (uint32_t)((unsigned long long)(Mp / 2) * blockIdx.x / P);
    const uint32_t hi = 2u * (uint32_t)((unsigned long long)(Mp / 2) * (blockIdx.x + 1) / P);
    const uint32_t ntl = (hi - lo + LIVE_T - 1) / LIVE_T;
    // tiles newest-first: the tail of each run was written last (by this
    // round's predecessor) and is the part most likely still in L2
    auto tile_at = [&](uint32_t k) { return SHB_KR_REVERSE ? ntl - 1 - k : k; };
    // ring stages/phases continue across rounds: tile kk of this round is
    // the CTA's (kbase + kk)-th tile overall.  Fragmented live sets (short
    // runs: many tiny bulk copies, each ~70 ns to issue) are read with plain
    // loads by the consumers instead.
    const bool use_tma = Mp >= 256u * nruns;
    auto issue = [&](uint32_t kk) {  // producer lane
      const int st = (int)((kbase + kk) % LIVE_NS);
      const uint32_t t0 = lo + tile_at(kk) * LIVE_T, t1 = min(hi, t0 + LIVE_T);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&sm.lbar[st], (t1 - t0) * 24u);
      uint32_t a0 = 0, a1 = nruns;
      while (a1 - a0 > 1) {
        const uint32_t mid = (a0 + a1) >> 1;
        if (s_pref[mid] <= t0) a0 = mid; else a1 = mid;
      }
      for (uint32_t pos = t0, rb = a0; pos < t1; ++rb) {
        const uint32_t end = min(t1, s_pref[rb + 1]);
        if (end <= pos) continue;
        const uint32_t ph = rb * q + (pos - s_pref[rb]);
        tma_load_1d(&sm.lxy[st][pos - t0], Ixy + ph, (end - pos) * 16u, &sm.lbar[st]);
        tma_load_1d(&sm.lis[st][pos - t0], Iis + ph, (end - pos) * 8u, &sm.lbar[st]);
        pos = end;
      }
    };
    const int wid = threadIdx.x >> 5;
    if (wid == RCWARPS) {  // producer warp
      if (use_tma && (threadIdx.x & 31) == 0) {
        for (uint32_t kk = 0; kk < ntl; ++kk) {
          const uint32_t g = kbase + kk;
          // the stage's previous use (this round or an earlier one) was released;
          // across rounds this wait returns at once (the grid barrier ordered it)
          if (g >= (uint32_t)LIVE_NS) mbar_wait(&sm.lebar[g % LIVE_NS], ((g / LIVE_NS) - 1) & 1u);
          issue(kk);
        }
      }
    } else {
#if SHB_DEFER
      unsigned long long q_db[KR_U], q_old[KR_U];  // the pending tile (large tables)
      uint32_t q_pos[KR_U], q_seg[KR_U], q_m = 0;
#endif
      for (uint32_t k = 0; k < ntl; ++k) {
        const int st = (int)((kbase + k) % LIVE_NS);
        const uint32_t ph = ((kbase + k) / LIVE_NS) & 1u;
        const uint32_t t0 = lo + tile_at(k) * LIVE_T, tc = min(hi, t0 + LIVE_T) - t0;
        double px[KR_U], py[KR_U], pd[KR_U];
        uint32_t pid[KR_U], pseg[KR_U], oseg[KR_U];
        uint32_t keepm = 0, lowm = 0;
        if (use_tma) {
          mbar_wait(&sm.lbar[st], ph);
#pragma unroll
          for (int u = 0; u < KR_U; ++u) {
            const uint32_t e = u * RCTHREADS + threadIdx.x;
            px[u] = py[u] = 0.0;
            pid[u] = 0;
            oseg[u] = NONE;
            if (e < tc) {
              const double2 v = sm.lxy[st][e];
              const uint2 is = sm.lis[st][e];
              px[u] = v.x;
              py[u] = v.y;
              pid[u] = is.x;
              oseg[u] = is.y;  // NONE for the pad entry of an odd run
            }
          }
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.lebar[st]);  // stage read
        } else {
          // each point finds its run by binary search over the run prefix
          // (the positions of a tile can span dozens of short runs)
          uint32_t phys[KR_U];
#pragma unroll
          for (int u = 0; u < KR_U; ++u) {
            const uint32_t v0 = t0 + u * RCTHREADS + threadIdx.x;
            uint32_t a0 = 0, a1 = nruns;
            while (a1 - a0 > 1) {
              const uint32_t mid = (a0 + a1) >> 1;
              if (s_pref[mid] <= v0) a0 = mid; else a1 = mid;
            }
            phys[u] = a0 * q + (v0 - s_pref[a0]);
          }
#pragma unroll
          for (int u = 0; u < KR_U; ++u) {
            const uint32_t e = u * RCTHREADS + threadIdx.x;
            px[u] = py[u] = 0.0;
            pid[u] = 0;
            oseg[u] = NONE;
            if (e < tc) {
              const double2 v = __ldcg(Ixy + phys[u]);
              const uint2 is = __ldcg(Iis + phys[u]);
              px[u] = v.x;
              py[u] = v.y;
              pid[u] = is.x;
              oseg[u] = is.y;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < KR_U; ++u) {
          pd[u] = 0.0;
          pseg[u] = 0;
          if (oseg[u] != NONE) {
            bool lower = false;
            const bool keep = small ? route_point<false>(sm.rt + oseg[u], px[u], py[u], pid[u], pd[u], pseg[u], lower)
                                    : route_point<true>(B.route + oseg[u], px[u], py[u], pid[u], pd[u], pseg[u], lower);
            if (keep) keepm |= 1u << u;
            if (lower) lowm |= 1u << u;
          }
        }
#if !SHB_DEFER
        uint32_t candm = 0;
#endif
        if (small) {
          contend_tile<KR_U>(sm.db, sm.rec, keepm, px, py, pd, pid, pseg, lowm);
        } else {
          // large table: max of the distance bits in the global slot; a
          // survivor that reached the running maximum is listed for the
          // winner pass after the barrier
#if SHB_DEFER
          // the previous tile's atomicMax results are consumed only now, so
          // their L2 round trip overlapped this tile's route-row loads
          list_cands<KR_U>(q_m, q_db, q_old, q_pos, q_seg, &s_coff, B.Lc, obase);
          q_m = 0;
#endif
#pragma unroll
          for (int u = 0; u < KR_U; ++u) {
            if ((keepm >> u) & 1u) {
              const unsigned long long db = (unsigned long long)__double_as_longlong(pd[u]);
#if SHB_MED
              // below this CTA's running maximum: below the final one too
              if (med && db < atomicMax(mdb + pseg[u], db)) continue;
#endif
#if SHB_DEFER
              q_db[u] = db;
              q_seg[u] = pseg[u];
              q_old[u] = atomicMax(Sd + pseg[u], db);
              q_m |= 1u << u;
#else
              if (db >= atomicMax(Sd + pseg[u], db)) candm |= 1u << u;
#endif
            }
          }
        }
#if SHB_DEFER
        run_append<KR_U>(keepm, px, py, pid, pseg, &s_off, Oxy, Ois, obase, pd, 0u, nullptr,
                         nullptr, 0u, nullptr, q_pos);
#else
        run_append<KR_U>(keepm, px, py, pid, pseg, &s_off, Oxy, Ois, obase, pd, candm, &s_coff,
                         small ? nullptr : B.Lc);
#endif
      }
#if SHB_DEFER
      if (!small) list_cands<KR_U>(q_m, q_db, q_old, q_pos, q_seg, &s_coff, B.Lc, obase);
#endif
    }
    __syncthreads();
    KR_MARK();  // point loop done
    if (use_tma) kbase += ntl;  // stage uses so far (phase parity of the ring)
    if (threadIdx.x == 0 && (s_off & 1u) && s_off < B.run_q) {  // pad the run to an even length
      Oxy[obase + s_off] = make_double2(0.0, 0.0);
      Ois[obase + s_off] = make_uint2(NONE, NONE);
    }
    // a lone CTA whose next table is small keeps its records in smem
    const bool keep_smem = small && P == 1 && Sn <= (uint32_t)SMALL_S;
    if (small && !keep_smem) flush_rows(sm.rec, Sn, Sd, B.Rc[r & 1u] + (size_t)blockIdx.x * NSLOT);
    if (threadIdx.x == 0) B.run_cnt[pout][blockIdx.x] = s_off;
    if (blockIdx.x == 0 && threadIdx.x == 0) t_points = globaltimer_ns();
    if (threadIdx.x == 0 && r == trace_r) B.dbg[blockIdx.x] = globaltimer_ns() - c->t0_ns;
    KR_MARK();  // slots flushed
    rounds_barrier(c, P, bar);
    KR_MARK();  // barrier passed
    if (small && !keep_smem) {  // rows at the final maxima claim their slots
      claim_slots(sm.rec, Sn, Slon, Sd, B.Wn[sout], B.Rc[r & 1u]);
      rounds_barrier(c, P, bar);
    }
    if (!small) {
      // winner pass over this CTA's contenders (listed in its run's slice of
      // Lc, still hot in L2): the ones whose distance equals their segment's
      // final maximum claim its winner slot; exact ties settle the full
      // comparator with a compare-and-swap loop over live-set positions
      constexpr int WU = 4;
      uint32_t* Wout = B.Wn[sout];
      const LiveCand* Oc = B.Lc + obase;
      const uint32_t cnt = *(volatile uint32_t*)&s_coff;
      for (uint32_t e0 = threadIdx.x; e0 < cnt; e0 += RTPB * WU) {
        LiveCand cv[WU];
        unsigned long long mx[WU];
#pragma unroll
        for (int u = 0; u < WU; ++u) {
          const uint32_t e = e0 + u * RTPB;
          cv[u].seg = NONE;
          if (e < cnt) {
            const uint4 raw = __ldcg(reinterpret_cast<const uint4*>(Oc + e));
            cv[u].d = __hiloint2double((int)raw.y, (int)raw.x);
            cv[u].pos = raw.z;
            cv[u].seg = raw.w;
          }
        }
#pragma unroll
        for (int u = 0; u < WU; ++u) mx[u] = cv[u].seg != NONE ? __ldcg(Sd + cv[u].seg) : 0ull;
#pragma unroll
        for (int u = 0; u < WU; ++u) {
          if (cv[u].seg == NONE || (unsigned long long)__double_as_longlong(cv[u].d) != mx[u]) continue;
          uint32_t cur = atomicCAS(Wout + cv[u].seg, NONE, cv[u].pos);
          if (cur == NONE) continue;
          // a tie on the distance: the full comparator (hull.cpp:171-179)
          Cand me;
          const double2 mv = __ldcg(Oxy + cv[u].pos);
          me.d = cv[u].d; me.x = mv.x; me.y = mv.y; me.id = __ldcg(&Ois[cv[u].pos].x); me.pos = 0;
          const bool lower = cv[u].seg < Slon;
          while (cur != NONE) {
            Cand o;
            const double2 ov = __ldcg(Oxy + cur);
            o.d = me.d; o.x = ov.x; o.y = ov.y; o.id = __ldcg(&Ois[cur].x); o.pos = 0;
            if (!cand_better(me, o, lower)) break;
            const uint32_t prev = atomicCAS(Wout + cv[u].seg, cur, cv[u].pos);
            if (prev == cur) break;
            cur = prev;
          }
        }
      }
      rounds_barrier(c, P, bar);
    }

    KR_MARK();  // winner pass done
    // ---- close round r (every participating CTA computes the same) ----
    const uint32_t mn = P == 1 ? *(volatile uint32_t*)&s_off : sum_runs(B.run_cnt[pout], P, s_ws);
    if (blockIdx.x == 0 && threadIdx.x == 0 && r <= (uint32_t)STATS_CAP) {
      StatRec st;
      st.segments = Sn;
      st.points_remaining = Sn + mn;
      st.points_removed = (S + m) - (Sn + mn);
      st.pad = 0;
      const unsigned long long t0 = *(volatile unsigned long long*)&c->t0_ns;
      st.end_ns = globaltimer_ns() - t0;
      st.table_ns = t_table - t0;
      st.points_ns = t_points - t0;
      B.stats[r - 1] = st;
    }
    S = Sn;
    Slo = Slon;
    m = mn;
    nruns = P;
    rec_kind = small ? (keep_smem ? RS_SMEM : RS_ROWS) : RS_WIN;
    prev_small = small;
    if (mn == 0 || r + 1 > n) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->round = r;
        c->S_cur = S;
        c->Slo_cur = Slo;
        c->m_cur = m;
        c->nruns = nruns;
        c->status = mn == 0 ? ST_DONE : ST_INTERNAL;  // hull.cpp:265-267
        c->mark[6] = globaltimer_ns() - c->t0_ns;
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

__global__ void k5_emit(Bufs B, double* ox, double* oy, long long* oidx, uint64_t cap,
                        unsigned long long id_base) {
  const Ctl* c = B.ctl;
  pdl_wait();  // launched early (programmatic serialisation): the rounds are done
  if (c->status != ST_DONE) return;
  const uint32_t par = c->round & 1u;
  const uint32_t h = c->S_cur;
  const uint32_t lim = h < cap ? h : (uint32_t)cap;
  const double* Tx = B.Tx[par];
  const double* Ty = B.Ty[par];
  const uint32_t* Tid = B.Tid[par];
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  // one CTA per SM, four independent elements per thread in flight: a hull
  // of millions of vertices (the circle) streams at HBM rate
  constexpr int U = 4;
  for (; i + (U - 1) * stride < lim; i += U * stride) {
    double vx[U], vy[U];
    uint32_t vi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vx[u] = __ldcs(Tx + i + u * stride);
      vy[u] = __ldcs(Ty + i + u * stride);
      vi[u] = __ldcs(Tid + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (ox) ox[i + u * stride] = vx[u];
      if (oy) oy[i + u * stride] = vy[u];
      if (oidx) oidx[i + u * stride] = (long long)(vi[u] + id_base);
    }
  }
  for (; i < lim; i += stride) {
    if (ox) ox[i] = Tx[i];
    if (oy) oy[i] = Ty[i];
    if (oidx) oidx[i] = (long long)(Tid[i] + id_base);
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

cudaError_t configure_stream_kernels_k3() {
  cudaError_t e = cudaFuncSetAttribute(k3_round1<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)K3Layout<false>::kBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k3_round1<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)K3Layout<false>::kBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k3_round1<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)K3Layout<true>::kBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k3_round1<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)K3Layout<true>::kBytes);
  return e;
}

template <class K>
static cudaError_t launch_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t s,
                              const Bufs& B, bool cooperative) {
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

void launch_k3(const Bufs& B, bool ids, bool capped, int grid, cudaStream_t s) {
  const size_t sm = ids ? K3Layout<true>::kBytes : K3Layout<false>::kBytes;
  if (ids)
    launch_pdl(capped ? k3_round1<true, true> : k3_round1<true, false>, grid, Cfg3::TPB, sm, s, B, false);
  else
    launch_pdl(capped ? k3_round1<false, true> : k3_round1<false, false>, grid, Cfg3::TPB, sm, s, B,
               false);
}

cudaError_t launch_rounds(const Bufs& B, int grid, cudaStream_t s) {
  return launch_pdl(k_rounds, grid, RTPB, sizeof(RoundSmem), s, B, true);
}

#ifndef SHB_K5_GRID
#define SHB_K5_GRID 148
#endif
constexpr int K5_GRID = SHB_K5_GRID, K5_TPB = 512;

void launch_k5(const Bufs& B, double* ox, double* oy, long long* oidx, uint64_t cap,
               unsigned long long id_base, cudaStream_t s) {
#ifdef SHB_K5_PLAIN
  k5_emit<<<K5_GRID, K5_TPB, 0, s>>>(B, ox, oy, oidx, cap, id_base);
  return;
#endif
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(K5_GRID);
  cfg.blockDim = dim3(K5_TPB);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k5_emit, B, ox, oy, oidx, cap, id_base);
}

}  // namespace shb
