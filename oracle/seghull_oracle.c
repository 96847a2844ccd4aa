/*
 * oracle/seghull_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference's 2D QuickHull path
 * (`seghull::hull::run`, /root/reference/proj/core/src/hull.cpp:219-290) and
 * of its two generators and its monotone-chain oracle.  It exists to CHECK the
 * sm_100a implementation in paper_1501_04706_b200/: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path never calls it (there is no CPU fallback).
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - the reference's own known-answer tests (tests/test_hull.cpp:79 "47769",
 *     the first-split layouts at :88-121, the degenerate cases at :340-374),
 *   - bit-for-bit comparison with the reference itself, compiled from
 *     /root/reference sources by oracle/Makefile into oracle/_ref/, and golden
 *     fixtures generated from it (tests/golden/, tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference's own
 * CMake flags produce none, SURVEY.md section 0 finding 4).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "seghull_oracle.h"

typedef struct {
  double x, y;
} opt;

/* geometry.hpp:17-19 -- operand order and rounding exactly as written. */
static double cross(opt a, opt b, opt c) {
  return (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
}

/* geometry.hpp:25-27 */
static double outward(opt first, opt last, opt p) { return -cross(first, last, p); }

static int pt_eq(opt a, opt b) { return a.x == b.x && a.y == b.y; }

/* hull.cpp:47-49 (double comparisons: -0.0 == +0.0) */
static int lex_less(opt a, opt b) { return a.x != b.x ? a.x < b.x : a.y < b.y; }

/* ------------------------------------------------------------------------ */
/* generators: dataio.hpp:44-59, dataio.cpp:291-312                          */

static uint64_t sm64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double sm64_double(uint64_t* state) {
  return (double)(sm64_next(state) >> 11) * 0x1.0p-53;
}

void or_gen_uniform(uint64_t n, uint64_t seed, double* x, double* y) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) {
    x[i] = sm64_double(&s); /* x then y per point, dataio.cpp:295-298 */
    y[i] = sm64_double(&s);
  }
}

void or_gen_circle(uint64_t n, uint64_t seed, double* x, double* y) {
  uint64_t s = seed;
  const double two_pi = 2.0 * 3.141592653589793; /* std::numbers::pi, exact x2 */
  for (uint64_t i = 0; i < n; ++i) {
    const double angle = two_pi * sm64_double(&s); /* dataio.cpp:308 */
    x[i] = cos(angle);
    y[i] = sin(angle);
  }
}

/* Not in the reference (SURVEY.md section 8d defines it for config 3): one
 * SplitMix64 stream, candidate (2u-1, 2v-1), accepted iff x*x + y*y < 1.0
 * evaluated without contraction.  Returns the number of draws consumed. */
uint64_t or_gen_disk(uint64_t n, uint64_t seed, double* x, double* y) {
  uint64_t s = seed, draws = 0;
  for (uint64_t i = 0; i < n;) {
    const double u = sm64_double(&s);
    const double v = sm64_double(&s);
    draws += 2;
    const double px = 2.0 * u - 1.0, py = 2.0 * v - 1.0;
    const double r2 = px * px + py * py;
    if (r2 < 1.0) {
      x[i] = px;
      y[i] = py;
      ++i;
    }
  }
  return draws;
}

/* ------------------------------------------------------------------------ */
/* hull.cpp:25-45 find_extremes, directional ties, strict compares so exact
 * duplicates resolve to the lowest index.                                   */

typedef struct {
  uint64_t left, bottom, right, top;
} extremes;

static extremes find_extremes(const double* X, const double* Y, uint64_t n) {
  extremes e = {0, 0, 0, 0};
  for (uint64_t i = 1; i < n; ++i) {
    const double x = X[i], y = Y[i];
    if (x < X[e.left] || (x == X[e.left] && y < Y[e.left])) e.left = i;
    if (x > X[e.right] || (x == X[e.right] && y > Y[e.right])) e.right = i;
    if (y < Y[e.bottom] || (y == Y[e.bottom] && x > X[e.bottom])) e.bottom = i;
    if (y > Y[e.top] || (y == Y[e.top] && x < X[e.top])) e.top = i;
  }
  return e;
}

void or_find_extremes(const double* X, const double* Y, uint64_t n, uint64_t out[4]) {
  extremes e = find_extremes(X, Y, n);
  out[0] = e.left;
  out[1] = e.bottom;
  out[2] = e.right;
  out[3] = e.top;
}

/* ------------------------------------------------------------------------ */
/* hull.cpp:53-99 preprocess: strict quadrilateral interior filter followed by
 * a stable keep-left compaction.  Writes the kept points in input order and
 * (optionally) their input indices; returns the discard count.              */

uint64_t or_preprocess(const double* X, const double* Y, uint64_t n, double* out_x,
                       double* out_y, uint64_t* out_idx, uint64_t* out_kept) {
  if (n == 0) {
    *out_kept = 0;
    return 0;
  }
  const extremes e = find_extremes(X, Y, n);
  const opt corners[4] = {{X[e.left], Y[e.left]},
                          {X[e.bottom], Y[e.bottom]},
                          {X[e.right], Y[e.right]},
                          {X[e.top], Y[e.top]}};
  int distinct = 0;
  for (int i = 0; i < 4; ++i) {
    int seen = 0;
    for (int j = 0; j < i; ++j) seen |= pt_eq(corners[i], corners[j]);
    if (!seen) ++distinct;
  }
  opt ea[4], eb[4];
  int ne = 0;
  for (int i = 0; i < 4; ++i) {
    const opt a = corners[i], b = corners[(i + 1) % 4];
    if (!pt_eq(a, b)) {
      ea[ne] = a;
      eb[ne] = b;
      ++ne;
    }
  }
  uint64_t kept = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const opt p = {X[i], Y[i]};
    int inside = distinct >= 3;
    for (int k = 0; inside && k < ne; ++k) {
      if (cross(ea[k], eb[k], p) <= 0.0) inside = 0;
    }
    if (!inside) {
      if (out_x) out_x[kept] = p.x;
      if (out_y) out_y[kept] = p.y;
      if (out_idx) out_idx[kept] = i;
      ++kept;
    }
  }
  *out_kept = kept;
  return n - kept;
}

/* ------------------------------------------------------------------------ */
/* HullState (hull.hpp:19-33) restated as C arrays.                          */

typedef struct {
  uint64_t n;
  opt* p;
  uint64_t* src;   /* input index of each row (not in the reference; used only
                      to report which copy of a duplicate survived)           */
  double* dist;
  uint8_t* head;
  int64_t* keys;
  int64_t* first;
  uint8_t* flag;
} hstate;

static void hstate_free(hstate* s) {
  free(s->p);
  free(s->src);
  free(s->dist);
  free(s->head);
  free(s->keys);
  free(s->first);
  free(s->flag);
  memset(s, 0, sizeof(*s));
}

typedef struct {
  opt p;
  uint64_t src;
} row;

static int cmp_lex_asc(const void* a, const void* b) {
  const opt pa = ((const row*)a)->p, pb = ((const row*)b)->p;
  if (lex_less(pa, pb)) return -1;
  if (lex_less(pb, pa)) return 1;
  return 0;
}

static int cmp_lex_desc(const void* a, const void* b) { return cmp_lex_asc(b, a); }

static void rebuild_keys_first(hstate* s) {
  /* primitives.cpp:102-106 keys_from_heads, primitives.cpp:175-217
   * propagate_first_index (sequential walk). */
  int64_t key = -1, cur = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    if (s->head[i]) {
      ++key;
      cur = (int64_t)i;
    }
    s->keys[i] = key;
    s->first[i] = cur;
  }
}

/* hull.cpp:101-158 first_split: classify against P0->Pr (strictly below goes
 * lower, P0 forced lower), stable partition, sort lower ascending and upper
 * descending in (x, y), heads at 0 and lower_count.                         */
static int first_split(const double* X, const double* Y, const uint64_t* SRC, uint64_t n,
                       hstate* s) {
  const extremes e = find_extremes(X, Y, n);
  const opt p0 = {X[e.left], Y[e.left]};
  const opt pr = {X[e.right], Y[e.right]};
  if (pt_eq(p0, pr)) return OR_DEGENERATE_INPUT;
  row* rows = (row*)malloc(sizeof(row) * (n ? n : 1));
  uint8_t* in_lower = (uint8_t*)malloc(n ? n : 1);
  uint64_t lower_count = 0;
  for (uint64_t i = 0; i < n; ++i) { /* hull.cpp:113-118 */
    const opt p = {X[i], Y[i]};
    in_lower[i] = (i == e.left) || cross(p0, pr, p) < 0.0;
    lower_count += in_lower[i];
  }
  uint64_t w = 0; /* stable keep-left partition, hull.cpp:120-124 */
  for (uint64_t pass = 0; pass < 2; ++pass)
    for (uint64_t i = 0; i < n; ++i)
      if ((pass == 0) == (in_lower[i] != 0)) {
        rows[w].p.x = X[i];
        rows[w].p.y = Y[i];
        rows[w].src = SRC ? SRC[i] : i;
        ++w;
      }
  free(in_lower);
  qsort(rows, lower_count, sizeof(row), cmp_lex_asc);
  qsort(rows + lower_count, n - lower_count, sizeof(row), cmp_lex_desc);

  s->n = n;
  s->p = (opt*)malloc(sizeof(opt) * n);
  s->src = (uint64_t*)malloc(sizeof(uint64_t) * n);
  s->dist = (double*)calloc(n, sizeof(double));
  s->head = (uint8_t*)calloc(n, 1);
  s->keys = (int64_t*)malloc(sizeof(int64_t) * n);
  s->first = (int64_t*)malloc(sizeof(int64_t) * n);
  s->flag = (uint8_t*)malloc(n);
  for (uint64_t i = 0; i < n; ++i) {
    s->p[i] = rows[i].p;
    s->src[i] = rows[i].src;
    s->flag[i] = 1;
  }
  s->head[0] = 1;
  s->head[lower_count] = 1;
  rebuild_keys_first(s);
  free(rows);
  return OR_OK;
}

static uint64_t segments(const hstate* s) { return s->n ? (uint64_t)s->keys[s->n - 1] + 1 : 0; }

/* hull.cpp:160-180 compute_distances: line from the segment head to the next
 * segment's head; the last segment wraps to element 0.                      */
static void compute_distances(hstate* s, uint64_t* head_of) {
  const uint64_t nseg = segments(s);
  for (uint64_t i = 0; i < s->n; ++i)
    if (s->head[i]) head_of[s->keys[i]] = i;
  for (uint64_t i = 0; i < s->n; ++i) {
    const uint64_t k = (uint64_t)s->keys[i];
    const uint64_t last = k + 1 < nseg ? head_of[k + 1] : 0;
    s->dist[i] = outward(s->p[s->first[i]], s->p[last], s->p[i]);
  }
}

/* primitives.cpp:30-45,108-136 segmented_argmax: strictly greater replaces,
 * so the smallest index attaining the maximum wins.                          */
typedef struct {
  double value;
  uint64_t index;
} segmax;

static void segmented_argmax(const hstate* s, segmax* out) {
  int64_t cur = -1;
  for (uint64_t i = 0; i < s->n; ++i) {
    if (s->keys[i] != cur) {
      cur = s->keys[i];
      out[cur].value = s->dist[i];
      out[cur].index = i;
    } else if (s->dist[i] > out[cur].value) {
      out[cur].value = s->dist[i];
      out[cur].index = i;
    }
  }
}

/* hull.cpp:203-217 compact: stable removal of flag==0 rows. */
static uint64_t compact(hstate* s) {
  uint64_t w = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    if (s->flag[i]) {
      s->p[w] = s->p[i];
      s->src[w] = s->src[i];
      s->dist[w] = s->dist[i];
      s->head[w] = s->head[i];
      s->flag[w] = 1;
      ++w;
    }
  }
  const uint64_t removed = s->n - w;
  s->n = w;
  rebuild_keys_first(s);
  return removed;
}

int or_hull_run(const double* X, const double* Y, uint64_t n, int mode, double* out_x,
                double* out_y, uint64_t* out_src, uint64_t* out_h, or_segment_stats* stats,
                uint64_t stats_cap, uint64_t* out_rounds, uint64_t* out_kept,
                uint64_t* bad_index) {
  *out_h = 0;
  if (out_rounds) *out_rounds = 0;
  if (out_kept) *out_kept = n;
  if (n == 0) return OR_EMPTY_INPUT; /* hull.cpp:221 */
  for (uint64_t i = 0; i < n; ++i) { /* hull.cpp:222-227 */
    if (!isfinite(X[i]) || !isfinite(Y[i])) {
      if (bad_index) *bad_index = i;
      return OR_NON_FINITE_INPUT;
    }
  }
  const extremes e = find_extremes(X, Y, n); /* hull.cpp:231 */
  const opt lo = {X[e.left], Y[e.left]};
  const opt hi = {X[e.right], Y[e.right]};
  if (pt_eq(lo, hi)) { /* hull.cpp:234-237 */
    out_x[0] = lo.x;
    out_y[0] = lo.y;
    if (out_src) out_src[0] = e.left;
    *out_h = 1;
    return OR_OK;
  }
  int collinear = 1; /* hull.cpp:238-248 */
  for (uint64_t i = 0; i < n; ++i) {
    const opt p = {X[i], Y[i]};
    if (cross(lo, hi, p) != 0.0) {
      collinear = 0;
      break;
    }
  }
  if (collinear) {
    out_x[0] = lo.x;
    out_y[0] = lo.y;
    out_x[1] = hi.x;
    out_y[1] = hi.y;
    if (out_src) {
      out_src[0] = e.left;
      out_src[1] = e.right;
    }
    *out_h = 2;
    return OR_OK;
  }

  const double* SX = X;
  const double* SY = Y;
  double *fx = NULL, *fy = NULL;
  uint64_t* fsrc = NULL;
  uint64_t m = n;
  if (mode == 1) { /* hull.cpp:253-255 */
    fx = (double*)malloc(sizeof(double) * n);
    fy = (double*)malloc(sizeof(double) * n);
    fsrc = (uint64_t*)malloc(sizeof(uint64_t) * n);
    or_preprocess(X, Y, n, fx, fy, fsrc, &m);
    SX = fx;
    SY = fy;
  }
  if (out_kept) *out_kept = m;

  hstate s;
  memset(&s, 0, sizeof(s));
  int rc = first_split(SX, SY, fsrc, m, &s); /* hull.cpp:260 */
  free(fx);
  free(fy);
  free(fsrc);
  if (rc != OR_OK) return rc;

  uint64_t* head_of = (uint64_t*)malloc(sizeof(uint64_t) * (s.n + 1));
  segmax* far = (segmax*)malloc(sizeof(segmax) * (s.n + 1));
  uint64_t rounds = 0;
  for (uint64_t iteration = 1;; ++iteration) { /* hull.cpp:264-282 */
    if (iteration > n) {
      rc = OR_INTERNAL_ERROR;
      break;
    }
    compute_distances(&s, head_of);
    segmented_argmax(&s, far);
    const uint64_t nseg = segments(&s);
    int splittable = 0;
    for (uint64_t k = 0; k < nseg; ++k)
      if (far[k].value > 0.0) splittable = 1;
    if (!splittable && s.n == nseg) break;
    /* hull.cpp:186-194 split_segments */
    for (uint64_t k = 0; k < nseg; ++k)
      if (far[k].value > 0.0) s.head[far[k].index] = 1;
    rebuild_keys_first(&s);
    /* hull.cpp:196-201 mark_interior */
    compute_distances(&s, head_of);
    for (uint64_t i = 0; i < s.n; ++i) s.flag[i] = (s.head[i] || s.dist[i] > 0.0) ? 1 : 0;
    const uint64_t removed = compact(&s);
    if (stats && rounds < stats_cap) {
      stats[rounds].iteration = iteration;
      stats[rounds].segments = segments(&s);
      stats[rounds].points_remaining = s.n;
      stats[rounds].points_removed = removed;
    }
    ++rounds;
  }
  if (out_rounds) *out_rounds = rounds;
  if (rc == OR_OK) {
    for (uint64_t i = 0; i < s.n; ++i) { /* hull.cpp:285-288 */
      out_x[i] = s.p[i].x;
      out_y[i] = s.p[i].y;
      if (out_src) out_src[i] = s.src[i];
    }
    *out_h = s.n;
  }
  free(head_of);
  free(far);
  hstate_free(&s);
  return rc;
}

/* First-split layout for the per-phase known-answer tests
 * (tests/test_hull.cpp:88-121): rows, head flags and lower-chain size. */
int or_first_split(const double* X, const double* Y, uint64_t n, double* out_x, double* out_y,
                   uint8_t* out_head) {
  if (n == 0) return OR_EMPTY_INPUT;
  hstate s;
  memset(&s, 0, sizeof(s));
  const int rc = first_split(X, Y, NULL, n, &s);
  if (rc != OR_OK) return rc;
  for (uint64_t i = 0; i < n; ++i) {
    out_x[i] = s.p[i].x;
    out_y[i] = s.p[i].y;
    out_head[i] = s.head[i];
  }
  hstate_free(&s);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* oracle.cpp:17-58 monotone_chain: sorted-unique then Andrew's chain with
 * `cross <= 0` pops (collinear boundary points excluded).                    */

static int cmp_opt(const void* a, const void* b) {
  const opt pa = *(const opt*)a, pb = *(const opt*)b;
  if (lex_less(pa, pb)) return -1;
  if (lex_less(pb, pa)) return 1;
  return 0;
}

int or_monotone_chain(const double* X, const double* Y, uint64_t n, double* out_x,
                      double* out_y, uint64_t* out_h) {
  *out_h = 0;
  if (n == 0) return OR_EMPTY_INPUT;
  opt* p = (opt*)malloc(sizeof(opt) * n);
  for (uint64_t i = 0; i < n; ++i) {
    p[i].x = X[i];
    p[i].y = Y[i];
  }
  qsort(p, n, sizeof(opt), cmp_opt);
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (m == 0 || !pt_eq(p[m - 1], p[i])) p[m++] = p[i];
  if (m == 1) {
    out_x[0] = p[0].x;
    out_y[0] = p[0].y;
    *out_h = 1;
    free(p);
    return OR_OK;
  }
  opt* h = (opt*)malloc(sizeof(opt) * (2 * m + 1));
  uint64_t hs = 0;
  for (uint64_t i = 0; i < m; ++i) {
    while (hs >= 2 && cross(h[hs - 2], h[hs - 1], p[i]) <= 0.0) --hs;
    h[hs++] = p[i];
  }
  const uint64_t lower = hs;
  for (uint64_t i = m - 1; i-- > 0;) {
    while (hs > lower && cross(h[hs - 2], h[hs - 1], p[i]) <= 0.0) --hs;
    h[hs++] = p[i];
  }
  --hs; /* closing vertex repeats the start */
  for (uint64_t i = 0; i < hs; ++i) {
    out_x[i] = h[i].x;
    out_y[i] = h[i].y;
  }
  *out_h = hs;
  free(h);
  free(p);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Canonical index of each hull vertex: the lowest input index whose (x, y)
 * bit patterns equal the vertex's.  Sort-based.      */

typedef struct {
  uint64_t xb, yb, idx;
} keyrow;

static int cmp_keyrow(const void* a, const void* b) {
  const keyrow *ka = (const keyrow*)a, *kb = (const keyrow*)b;
  if (ka->xb != kb->xb) return ka->xb < kb->xb ? -1 : 1;
  if (ka->yb != kb->yb) return ka->yb < kb->yb ? -1 : 1;
  if (ka->idx != kb->idx) return ka->idx < kb->idx ? -1 : 1;
  return 0;
}

int or_canonical_index(const double* X, const double* Y, uint64_t n, const double* vx,
                       const double* vy, uint64_t h, int64_t* out_idx) {
  keyrow* k = (keyrow*)malloc(sizeof(keyrow) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    memcpy(&k[i].xb, &X[i], 8);
    memcpy(&k[i].yb, &Y[i], 8);
    k[i].idx = i;
  }
  qsort(k, n, sizeof(keyrow), cmp_keyrow);
  int missing = 0;
  for (uint64_t j = 0; j < h; ++j) {
    keyrow q;
    memcpy(&q.xb, &vx[j], 8);
    memcpy(&q.yb, &vy[j], 8);
    q.idx = 0;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (cmp_keyrow(&k[mid], &q) < 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo < n && k[lo].xb == q.xb && k[lo].yb == q.yb) {
      out_idx[j] = (int64_t)k[lo].idx;
    } else {
      out_idx[j] = -1;
      missing = 1;
    }
  }
  free(k);
  return missing ? OR_INTERNAL_ERROR : OR_OK;
}

/* FNV-1a-64 over the output vertex bits, x then y per vertex, little-endian
 * bytes. */
uint64_t or_fnv1a_vertices(const double* vx, const double* vy, uint64_t h) {
  uint64_t hash = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < h; ++i) {
    uint64_t w[2];
    memcpy(&w[0], &vx[i], 8);
    memcpy(&w[1], &vy[i], 8);
    for (int k = 0; k < 2; ++k)
      for (int b = 0; b < 8; ++b) {
        hash ^= (w[k] >> (8 * b)) & 0xffu;
        hash *= 0x100000001b3ull;
      }
  }
  return hash;
}
