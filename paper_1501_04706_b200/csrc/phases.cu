// phases.cu -- the reference's per-phase pipeline (hull.hpp:61-91) as device
// APIs over a device HullState in the REFERENCE's own layout (hull.hpp:19-33):
// SoA columns x, y, dist (f64) and head, keys, first_pts, flag (i32), rows
// sorted chain by chain exactly as first_split lays them out.
// section 8f row 4: these exist so the reference's per-stage tests
// (tests/test_hull.cpp:88-314) and any caller that drives the stages itself
// run against the device.  The fused hot path (sh_b200_hull) does not use
// them: it never sorts and never materialises this layout.
//
// Building blocks, all hand-written for sm_100a (no CUB/Thrust):
//   * tile scans: reduce tiles -> one-CTA scan of the tile totals -> re-scan
//     each tile with its prefix (u32 add for counts and keys, u32 max for
//     propagate_first_index);
//   * stable partition = exclusive count of the flags + scatter of every
//     column (primitives.hpp:100-115, primitives.cpp:238-285);
//   * a stable LSD radix sort of (x, y) under the reference's lex order
//     (8-bit digits over two order-preserving 64-bit keys; passes whose digit
//     is constant over the range are skipped), ranks within a tile by warp
//     match_any, so equal keys keep their order;
//   * segmented argmax with the reference's tie rule (primitives.cpp:31-46):
//     per-segment atomicMax of the order-preserving distance key, then
//     atomicMin of the index among elements equal to it.
// Every floating-point predicate is the reference's expression with explicit
// round-to-nearest operations in the reference's operand order (-fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/seghull_b200.h"
#include "device_common.cuh"

namespace shb {
namespace ph {

constexpr int PT = 256;         // threads per CTA
constexpr int PI = 8;           // items per thread of a scan tile
constexpr int TILE = PT * PI;   // scan tile (2048)
constexpr int RI = 16;          // items per thread of a sort tile
constexpr int RTILE = PT * RI;  // sort tile (4096)

struct AddOp {
  static __device__ __forceinline__ uint32_t id() { return 0u; }
  static __device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) { return a + b; }
};
struct MaxOp {
  static __device__ __forceinline__ uint32_t id() { return 0u; }
  static __device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b) { return a > b ? a : b; }
};

// Block-wide exclusive scan under Op (blockDim.x == PT).  Returns the
// exclusive prefix of v; *total receives the block aggregate.
template <class Op>
__device__ uint32_t block_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t s_w[PT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x = Op::op(y, x);
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < PT / 32 ? s_w[lane] : Op::id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w = Op::op(y, w);
    }
    if (lane < PT / 32) s_w[lane] = w;
    if (lane == PT / 32 - 1) s_w[PT / 32] = w;
  }
  __syncthreads();
  const uint32_t before = warp == 0 ? Op::id() : s_w[warp - 1];
  const uint32_t excl_in_warp = __shfl_up_sync(FULL, x, 1);
  const uint32_t r = lane == 0 ? before : Op::op(before, excl_in_warp);
  *total = s_w[PT / 32];
  __syncthreads();
  return r;
}

// ---- inputs and outputs of the scans ---------------------------------------

struct InFlag {  // 1 where flag != 0
  const int32_t* f;
  __device__ uint32_t operator()(uint64_t i) const { return f[i] != 0 ? 1u : 0u; }
};
struct InU32 {
  const uint32_t* f;
  __device__ uint32_t operator()(uint64_t i) const { return f[i]; }
};
struct InHeadRaw {  // inclusive_scan adds the raw head values (primitives.cpp:59-66)
  const int32_t* h;
  __device__ uint32_t operator()(uint64_t i) const { return (uint32_t)h[i]; }
};
struct InHeadPos {  // propagate_first_index: the largest head position so far
  const int32_t* h;
  __device__ uint32_t operator()(uint64_t i) const { return h[i] ? (uint32_t)i : 0u; }
};

struct OutKeys {  // keys_from_heads: inclusive - 1
  int32_t* keys;
  __device__ void operator()(uint64_t i, uint32_t incl, uint32_t) const {
    keys[i] = (int32_t)incl - 1;
  }
};
struct OutExcl {  // exclusive prefix in place
  uint32_t* o;
  __device__ void operator()(uint64_t i, uint32_t incl, uint32_t v) const { o[i] = incl - v; }
};
struct OutI32 {
  int32_t* o;
  __device__ void operator()(uint64_t i, uint32_t incl, uint32_t) const { o[i] = (int32_t)incl; }
};
// stable keep-left partition destination (partition_destinations): kept rows
// go to [0, ones) in order, the others to [ones, n) in order
struct OutDest {
  uint32_t* dest;
  const uint32_t* total;  // ones (written by the tile-total scan)
  __device__ void operator()(uint64_t i, uint32_t incl, uint32_t v) const {
    const uint32_t excl = incl - v;
    dest[i] = v ? excl : *total + (uint32_t)i - excl;
  }
};

template <class Op, class In>
__global__ void k_tile_reduce(In in, uint64_t n, uint32_t* sums) {
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  uint32_t acc = Op::id();
#pragma unroll
  for (int k = 0; k < PI; ++k) {
    const uint64_t i = base + (uint64_t)k * PT + threadIdx.x;
    if (i < n) acc = Op::op(acc, in(i));
  }
  uint32_t tot;
  block_scan<Op>(acc, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the tile totals in place; sums[ntiles] = total
template <class Op>
__global__ void k_scan_totals(uint32_t* sums, uint32_t ntiles) {
  uint32_t carry = Op::id();
  for (uint32_t b0 = 0; b0 < ntiles; b0 += PT) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < ntiles ? sums[b] : Op::id();
    uint32_t tot;
    const uint32_t ex = block_scan<Op>(v, &tot);
    if (b < ntiles) sums[b] = Op::op(carry, ex);
    carry = Op::op(carry, tot);
  }
  if (threadIdx.x == 0) sums[ntiles] = carry;
}

template <class Op, class In, class Out>
__global__ void k_tile_scan(In in, Out out, uint64_t n, const uint32_t* prefix) {
  const uint64_t base = (uint64_t)blockIdx.x * TILE + (uint64_t)threadIdx.x * PI;
  uint32_t v[PI];
  uint32_t acc = Op::id();
#pragma unroll
  for (int k = 0; k < PI; ++k) {
    v[k] = base + k < n ? in(base + k) : Op::id();
    acc = Op::op(acc, v[k]);
  }
  uint32_t tot;
  uint32_t run = Op::op(prefix[blockIdx.x], block_scan<Op>(acc, &tot));
#pragma unroll
  for (int k = 0; k < PI; ++k) {
    run = Op::op(run, v[k]);
    if (base + k < n) out(base + k, run, v[k]);
  }
}

// scratch = ceil(n / TILE) + 1 words
template <class Op, class In, class Out>
void scan(In in, Out out, uint64_t n, uint32_t* scratch, cudaStream_t s) {
  if (n == 0) return;
  const uint32_t nt = (uint32_t)((n + TILE - 1) / TILE);
  k_tile_reduce<Op><<<nt, PT, 0, s>>>(in, n, scratch);
  k_scan_totals<Op><<<1, PT, 0, s>>>(scratch, nt);
  k_tile_scan<Op><<<nt, PT, 0, s>>>(in, out, n, scratch);
}

// ---- extremes (hull.cpp:25-45): left = min x, tie min y; right = max x,
// tie max y; exact ties -> the lowest index (the reference's first hit) ----

struct Key3 {
  unsigned long long a, b;
  uint32_t i;
};
__device__ __forceinline__ bool key3_less(const Key3& p, const Key3& q) {
  return p.a != q.a ? p.a < q.a : p.b != q.b ? p.b < q.b : p.i < q.i;
}
__device__ __forceinline__ Key3 shfl_key3(const Key3& k, int m) {
  Key3 o;
  o.a = __shfl_xor_sync(FULL, k.a, m);
  o.b = __shfl_xor_sync(FULL, k.b, m);
  o.i = __shfl_xor_sync(FULL, k.i, m);
  return o;
}

__global__ void k_lr_partial(const double* x, const double* y, uint64_t n, Key3* part) {
  Key3 lo{~0ull, ~0ull, NONE}, hi{~0ull, ~0ull, NONE};
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT) {
    const unsigned long long kx = fkey(x[i]), ky = fkey(y[i]);
    const Key3 l{kx, ky, (uint32_t)i}, r{~kx, ~ky, (uint32_t)i};
    if (key3_less(l, lo)) lo = l;
    if (key3_less(r, hi)) hi = r;
  }
#pragma unroll
  for (int m = 16; m; m >>= 1) {
    const Key3 a = shfl_key3(lo, m), b = shfl_key3(hi, m);
    if (key3_less(a, lo)) lo = a;
    if (key3_less(b, hi)) hi = b;
  }
  __shared__ Key3 s_lo[PT / 32], s_hi[PT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PT / 32; ++w) {
      if (key3_less(s_lo[w], lo)) lo = s_lo[w];
      if (key3_less(s_hi[w], hi)) hi = s_hi[w];
    }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}

__global__ void k_lr_final(const Key3* part, int nparts, uint32_t* out_lr) {
  if (threadIdx.x != 0) return;
  Key3 lo = part[0], hi = part[1];
  for (int b = 1; b < nparts; ++b) {
    if (key3_less(part[2 * b], lo)) lo = part[2 * b];
    if (key3_less(part[2 * b + 1], hi)) hi = part[2 * b + 1];
  }
  out_lr[0] = lo.i;
  out_lr[1] = hi.i;
}

// ---- first_split (hull.cpp:101-158) ----

// in_lower[i] = cross(P0, Pr, p_i) < 0, and P0 itself leads the lower chain
__global__ void k_classify(const double* x, const double* y, uint64_t n, const uint32_t* lr,
                           int32_t* lower) {
  const uint32_t l = lr[0], r = lr[1];
  const Edge e = make_edge(x[l], y[l], x[r], y[r]);
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT)
    lower[i] = (cross_e(e, x[i], y[i]) < 0.0 || i == l) ? 1 : 0;
}

// rows in chain order: sort keys (lower ascending lex, upper inverted so an
// ascending sort reads descending lex), payload = input row
__global__ void k_chain_rows(const double* x, const double* y, uint64_t n, const uint32_t* dest,
                             const uint32_t* lower_count, unsigned long long* kx,
                             unsigned long long* ky, uint32_t* row) {
  const uint32_t lc = *lower_count;
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT) {
    const uint32_t d = dest[i];
    unsigned long long a = fkey(x[i]), b = fkey(y[i]);
    if (d >= lc) {
      a = ~a;
      b = ~b;
    }
    kx[d] = a;
    ky[d] = b;
    row[d] = (uint32_t)i;
  }
}

__global__ void k_state_init(const double* x, const double* y, uint64_t n, const uint32_t* row,
                             const uint32_t* lower_count, double* sx, double* sy, double* dist,
                             int32_t* head, int32_t* keys, int32_t* first, int32_t* flag) {
  const uint32_t lc = *lower_count;
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT) {
    const uint32_t r = row[i];
    sx[i] = x[r];
    sy[i] = y[r];
    dist[i] = 0.0;
    const bool up = i >= lc;
    head[i] = (i == 0 || i == lc) ? 1 : 0;
    keys[i] = up ? 1 : 0;
    first[i] = up ? (int32_t)lc : 0;
    flag[i] = 1;
  }
}

// ---- stable LSD radix sort of (kx, ky) + row payload ----

__device__ __forceinline__ uint32_t digit_of(unsigned long long kx, unsigned long long ky, int d) {
  return d < 8 ? (uint32_t)(ky >> (8 * d)) & 0xFFu : (uint32_t)(kx >> (8 * (d - 8))) & 0xFFu;
}

// histograms of all 16 digits over the range (to skip constant digits)
__global__ void k_hist_all(const unsigned long long* kx, const unsigned long long* ky, uint64_t m,
                           uint32_t* hist /* [16][256] */) {
  __shared__ uint32_t s[16 * 256];
  for (int t = threadIdx.x; t < 16 * 256; t += PT) s[t] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < m; i += (uint64_t)gridDim.x * PT) {
    const unsigned long long a = kx[i], b = ky[i];
#pragma unroll
    for (int d = 0; d < 16; ++d) atomicAdd(&s[d * 256 + digit_of(a, b, d)], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 16 * 256; t += PT)
    if (s[t]) atomicAdd(&hist[t], s[t]);
}

// per-tile histogram of digit d, digit-major: th[dig * ntiles + tile]
__global__ void k_tile_hist(const unsigned long long* kx, const unsigned long long* ky, uint64_t m,
                            int d, uint32_t ntiles, uint32_t* th) {
  __shared__ uint32_t s[256];
  s[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * RTILE;
#pragma unroll 4
  for (int k = 0; k < RI; ++k) {
    const uint64_t i = base + (uint64_t)k * PT + threadIdx.x;
    if (i < m) atomicAdd(&s[digit_of(kx[i], ky[i], d)], 1u);
  }
  __syncthreads();
  th[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s[threadIdx.x];
}

// stable scatter of one tile by digit d: items in index order (round k,
// thread t -> item k*PT + t); rank among equal digits = earlier rounds
// (s_run) + earlier warps of this round + earlier lanes (match_any)
__global__ void k_scatter_digit(const unsigned long long* kx, const unsigned long long* ky,
                                const uint32_t* row, uint64_t m, int d, uint32_t ntiles,
                                const uint32_t* off /* exclusive, digit-major */,
                                unsigned long long* ox, unsigned long long* oy, uint32_t* orow) {
  __shared__ uint32_t s_run[256];
  __shared__ uint32_t s_wc[PT / 32][256];
  const int warp = threadIdx.x >> 5;
  s_run[threadIdx.x] = off[(uint64_t)threadIdx.x * ntiles + blockIdx.x];
  for (int w = 0; w < PT / 32; ++w) s_wc[w][threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * RTILE;
  const uint32_t lt = lanemask_lt();
  for (int k = 0; k < RI; ++k) {
    const uint64_t i = base + (uint64_t)k * PT + threadIdx.x;
    const bool valid = i < m;
    unsigned long long a = 0, b = 0;
    uint32_t r = 0, dg = 0xFFFFu;  // invalid items get a digit of their own
    if (valid) {
      a = kx[i];
      b = ky[i];
      r = row[i];
      dg = digit_of(a, b, d);
    }
    const uint32_t peers = __match_any_sync(FULL, dg);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) s_wc[warp][dg] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pos = s_run[dg] + rank;
      for (int w = 0; w < warp; ++w) pos += s_wc[w][dg];
      ox[pos] = a;
      oy[pos] = b;
      orow[pos] = r;
    }
    __syncthreads();
    uint32_t add = 0;
    for (int w = 0; w < PT / 32; ++w) {
      add += s_wc[w][threadIdx.x];
      s_wc[w][threadIdx.x] = 0;
    }
    s_run[threadIdx.x] += add;
    __syncthreads();
  }
}

// ---- compute_distances / mark_interior (hull.cpp:160-180, 196-201) ----

__global__ void k_head_of_segment(const int32_t* head, const int32_t* keys, uint64_t n,
                                  uint32_t* hos) {
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT)
    if (head[i]) hos[keys[i]] = (uint32_t)i;
}

template <bool MARK>
__global__ void k_distances(const double* x, const double* y, const int32_t* head,
                            const int32_t* keys, const int32_t* first, uint64_t n,
                            const uint32_t* hos, double* dist, int32_t* flag) {
  const uint32_t nseg = (uint32_t)keys[n - 1] + 1u;
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT) {
    const uint32_t f = (uint32_t)first[i];
    const uint32_t k = (uint32_t)keys[i];
    const uint32_t last = k + 1 < nseg ? hos[k + 1] : 0u;
    const Edge e = make_edge(x[f], y[f], x[last], y[last]);
    const double d = outward_e(e, x[i], y[i]);  // -cross(first, last, p), geometry.hpp:25-27
    dist[i] = d;
    if (MARK) flag[i] = (head[i] != 0 || d > 0.0) ? 1 : 0;
  }
}

// ---- find_farthest (segmented_argmax, primitives.cpp:108-136) ----

__global__ void k_seg_max(const double* dist, const int32_t* keys, uint64_t n,
                          unsigned long long* smax) {
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT)
    atomicMax(smax + keys[i], fkey(dist[i]));
}

__global__ void k_seg_arg(const double* dist, const int32_t* keys, uint64_t n,
                          const unsigned long long* smax, uint32_t* sarg) {
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT) {
    const int32_t k = keys[i];
    if (fkey(dist[i]) == smax[k]) atomicMin(sarg + k, (uint32_t)i);
  }
}

__global__ void k_seg_out(const double* dist, const uint32_t* sarg, uint64_t nseg,
                          sh_segment_max* out) {
  for (uint64_t k = blockIdx.x * (uint64_t)PT + threadIdx.x; k < nseg; k += (uint64_t)gridDim.x * PT) {
    const uint32_t i = sarg[k];
    sh_segment_max e;
    e.key = (int32_t)k;
    e.pad = 0;
    e.value = dist[i];
    e.index = i;
    out[k] = e;
  }
}

// ---- split_segments (hull.cpp:186-194) / compact (203-217) ----

__global__ void k_promote(const sh_segment_max* far, uint64_t m, int32_t* head) {
  for (uint64_t j = blockIdx.x * (uint64_t)PT + threadIdx.x; j < m; j += (uint64_t)gridDim.x * PT) {
    const sh_segment_max e = far[j];
    if (e.value > 0.0) head[e.index] = 1;
  }
}

template <class T>
__global__ void k_scatter_col(const T* in, const uint32_t* dest, uint64_t n, T* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)PT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * PT)
    out[dest[i]] = in[i];
}

}  // namespace ph
}  // namespace shb

// ===========================================================================
// host side
// ===========================================================================

using namespace shb;
using namespace shb::ph;

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define PCK(call)                                                                     \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw Fail{SH_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                    " at " #call};                                    \
  } while (0)

int grid_for(uint64_t n) {
  const uint64_t g = (n + PT - 1) / PT;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, 148ull * 8));
}

// stream-ordered scratch, freed at scope exit on the same stream
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T>
  T* get(uint64_t count) {
    void* p = nullptr;
    PCK(cudaMallocAsync(&p, std::max<uint64_t>(count, 1) * sizeof(T), s));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int d) {
    cudaGetDevice(&prev);
    if (cudaSetDevice(d) != cudaSuccess) throw Fail{SH_CUDA_ERROR, "cudaSetDevice failed"};
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return SH_OK;
  } catch (const Fail& e) {
    cudaGetLastError();
    if (err && errlen) std::snprintf(err, errlen, "%s", e.msg.c_str());
    return e.code;
  }
}

bool valid_state(const sh_hull_state* st) {
  return st && st->x && st->y && st->dist && st->head && st->keys && st->first_pts && st->flag &&
         st->n <= st->cap && st->n < 0x7FFFFFFFull;
}

// stable LSD radix sort of [0, m) of (kx, ky, row); the result is in the
// first buffer set on return
void radix_sort(unsigned long long* kx, unsigned long long* ky, uint32_t* row, uint64_t m,
                Scratch& sc, cudaStream_t s) {
  if (m < 2) return;
  uint32_t* hist = sc.get<uint32_t>(16 * 256);
  PCK(cudaMemsetAsync(hist, 0, 16 * 256 * sizeof(uint32_t), s));
  k_hist_all<<<grid_for(m), PT, 0, s>>>(kx, ky, m, hist);
  std::vector<uint32_t> h(16 * 256);
  PCK(cudaMemcpyAsync(h.data(), hist, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  std::vector<int> passes;
  for (int d = 0; d < 16; ++d) {
    bool constant = false;
    for (int v = 0; v < 256; ++v) constant |= h[d * 256 + v] == m;
    if (!constant) passes.push_back(d);
  }
  if (passes.empty()) return;
  const uint32_t nt = (uint32_t)((m + RTILE - 1) / RTILE);
  unsigned long long* bx = sc.get<unsigned long long>(m);
  unsigned long long* by = sc.get<unsigned long long>(m);
  uint32_t* br = sc.get<uint32_t>(m);
  uint32_t* th = sc.get<uint32_t>((uint64_t)256 * nt + 1);
  uint32_t* tmp = sc.get<uint32_t>(((uint64_t)256 * nt + TILE - 1) / TILE + 1);
  unsigned long long *ix = kx, *iy = ky, *ox = bx, *oy = by;
  uint32_t *ir = row, *orw = br;
  for (int d : passes) {
    k_tile_hist<<<nt, PT, 0, s>>>(ix, iy, m, d, nt, th);
    // exclusive prefix over (digit, tile) in digit-major order
    scan<AddOp>(InU32{th}, OutExcl{th}, (uint64_t)256 * nt, tmp, s);
    k_scatter_digit<<<nt, PT, 0, s>>>(ix, iy, ir, m, d, nt, th, ox, oy, orw);
    std::swap(ix, ox);
    std::swap(iy, oy);
    std::swap(ir, orw);
  }
  if (ix != kx) {  // odd number of passes: back into the caller's buffers
    PCK(cudaMemcpyAsync(kx, ix, m * 8, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(ky, iy, m * 8, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(row, ir, m * 4, cudaMemcpyDeviceToDevice, s));
  }
}

void propagate_first(const sh_hull_state* st, uint64_t n, Scratch& sc, cudaStream_t s) {
  uint32_t* tmp = sc.get<uint32_t>((n + TILE - 1) / TILE + 1);
  scan<MaxOp>(InHeadPos{st->head}, OutI32{st->first_pts}, n, tmp, s);
}

void distances(const sh_hull_state* st, bool mark, Scratch& sc, cudaStream_t s) {
  const uint64_t n = st->n;
  if (n == 0) return;
  uint32_t* hos = sc.get<uint32_t>(n);
  k_head_of_segment<<<grid_for(n), PT, 0, s>>>(st->head, st->keys, n, hos);
  if (mark)
    k_distances<true><<<grid_for(n), PT, 0, s>>>(st->x, st->y, st->head, st->keys, st->first_pts,
                                                  n, hos, st->dist, st->flag);
  else
    k_distances<false><<<grid_for(n), PT, 0, s>>>(st->x, st->y, st->head, st->keys,
                                                   st->first_pts, n, hos, st->dist, st->flag);
  PCK(cudaGetLastError());
}

}  // namespace

extern "C" {

int sh_b200_first_split(const double* x, const double* y, uint64_t n, sh_hull_state* st,
                        int device, void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (n == 0) throw Fail{SH_EMPTY_INPUT, "first_split: empty point set"};  // hull.cpp:103
    if (!x || !y || !valid_state(st) || st->cap < n || n >= 0x7FFFFFFFull)
      throw Fail{SH_INVALID_ARGUMENT, "first_split: invalid state or capacity"};
    DeviceScope ds(device);
    cudaStream_t s = (cudaStream_t)stream;
    Scratch sc(s);
    // extremes
    const int g = std::min(grid_for(n), 296);
    Key3* part = sc.get<Key3>(2 * g);
    uint32_t* lr = sc.get<uint32_t>(2);
    k_lr_partial<<<g, PT, 0, s>>>(x, y, n, part);
    k_lr_final<<<1, 32, 0, s>>>(part, g, lr);
    uint32_t h_lr[2];
    PCK(cudaMemcpyAsync(h_lr, lr, sizeof(h_lr), cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    double p[4];
    PCK(cudaMemcpy(&p[0], x + h_lr[0], 8, cudaMemcpyDeviceToHost));
    PCK(cudaMemcpy(&p[1], y + h_lr[0], 8, cudaMemcpyDeviceToHost));
    PCK(cudaMemcpy(&p[2], x + h_lr[1], 8, cudaMemcpyDeviceToHost));
    PCK(cudaMemcpy(&p[3], y + h_lr[1], 8, cudaMemcpyDeviceToHost));
    if (p[0] == p[2] && p[1] == p[3])  // hull.cpp:108-110
      throw Fail{SH_DEGENERATE_INPUT, "first_split: fewer than 2 distinct points"};
    // chains: classify, stable partition (lower first), sort each chain
    int32_t* lower = sc.get<int32_t>(n);
    k_classify<<<grid_for(n), PT, 0, s>>>(x, y, n, lr, lower);
    uint32_t* dest = sc.get<uint32_t>(n);
    uint32_t* tmp = sc.get<uint32_t>((n + TILE - 1) / TILE + 1);
    const uint32_t nt = (uint32_t)((n + TILE - 1) / TILE);
    scan<AddOp>(InFlag{lower}, OutDest{dest, tmp + nt}, n, tmp, s);
    unsigned long long* kx = sc.get<unsigned long long>(n);
    unsigned long long* ky = sc.get<unsigned long long>(n);
    uint32_t* row = sc.get<uint32_t>(n);
    k_chain_rows<<<grid_for(n), PT, 0, s>>>(x, y, n, dest, tmp + nt, kx, ky, row);
    PCK(cudaGetLastError());
    uint32_t lc = 0;
    PCK(cudaMemcpyAsync(&lc, tmp + nt, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    radix_sort(kx, ky, row, lc, sc, s);
    radix_sort(kx + lc, ky + lc, row + lc, n - lc, sc, s);
    k_state_init<<<grid_for(n), PT, 0, s>>>(x, y, n, row, tmp + nt, st->x, st->y, st->dist,
                                             st->head, st->keys, st->first_pts, st->flag);
    PCK(cudaGetLastError());
    st->n = n;
    PCK(cudaStreamSynchronize(s));
  });
}

int sh_b200_compute_distances(const sh_hull_state* st, int device, void* stream) {
  return guarded(nullptr, 0, [&] {
    if (!valid_state(st)) throw Fail{SH_INVALID_ARGUMENT, ""};
    DeviceScope ds(device);
    Scratch sc((cudaStream_t)stream);
    distances(st, false, sc, (cudaStream_t)stream);
  });
}

int sh_b200_find_farthest(const sh_hull_state* st, sh_segment_max* out, uint64_t cap,
                          uint64_t* nseg, int device, void* stream) {
  return guarded(nullptr, 0, [&] {
    if (!valid_state(st) || !nseg) throw Fail{SH_INVALID_ARGUMENT, ""};
    *nseg = 0;
    const uint64_t n = st->n;
    if (n == 0) return;
    DeviceScope ds(device);
    cudaStream_t s = (cudaStream_t)stream;
    int32_t last = 0;
    PCK(cudaMemcpyAsync(&last, st->keys + n - 1, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    const uint64_t m = (uint64_t)last + 1;
    *nseg = m;
    if (m > cap || !out) throw Fail{SH_CAP_TOO_SMALL, ""};
    Scratch sc(s);
    unsigned long long* smax = sc.get<unsigned long long>(m);
    uint32_t* sarg = sc.get<uint32_t>(m);
    PCK(cudaMemsetAsync(smax, 0, m * 8, s));
    PCK(cudaMemsetAsync(sarg, 0xFF, m * 4, s));
    k_seg_max<<<grid_for(n), PT, 0, s>>>(st->dist, st->keys, n, smax);
    k_seg_arg<<<grid_for(n), PT, 0, s>>>(st->dist, st->keys, n, smax, sarg);
    k_seg_out<<<grid_for(m), PT, 0, s>>>(st->dist, sarg, m, out);
    PCK(cudaGetLastError());
  });
}

int sh_b200_split_segments(const sh_hull_state* st, const sh_segment_max* farthest, uint64_t m,
                           int device, void* stream) {
  return guarded(nullptr, 0, [&] {
    if (!valid_state(st) || (m && !farthest)) throw Fail{SH_INVALID_ARGUMENT, ""};
    const uint64_t n = st->n;
    if (n == 0) return;
    DeviceScope ds(device);
    cudaStream_t s = (cudaStream_t)stream;
    Scratch sc(s);
    if (m) k_promote<<<grid_for(m), PT, 0, s>>>(farthest, m, st->head);
    uint32_t* tmp = sc.get<uint32_t>((n + TILE - 1) / TILE + 1);
    scan<AddOp>(InHeadRaw{st->head}, OutKeys{st->keys}, n, tmp, s);  // keys_from_heads
    propagate_first(st, n, sc, s);
    PCK(cudaGetLastError());
  });
}

int sh_b200_mark_interior(const sh_hull_state* st, int device, void* stream) {
  return guarded(nullptr, 0, [&] {
    if (!valid_state(st)) throw Fail{SH_INVALID_ARGUMENT, ""};
    DeviceScope ds(device);
    Scratch sc((cudaStream_t)stream);
    distances(st, true, sc, (cudaStream_t)stream);
  });
}

int sh_b200_compact(sh_hull_state* st, uint64_t* removed, int device, void* stream) {
  return guarded(nullptr, 0, [&] {
    if (!valid_state(st)) throw Fail{SH_INVALID_ARGUMENT, ""};
    if (removed) *removed = 0;
    const uint64_t n = st->n;
    if (n == 0) return;
    DeviceScope ds(device);
    cudaStream_t s = (cudaStream_t)stream;
    Scratch sc(s);
    uint32_t* dest = sc.get<uint32_t>(n);
    uint32_t* tmp = sc.get<uint32_t>((n + TILE - 1) / TILE + 1);
    const uint32_t nt = (uint32_t)((n + TILE - 1) / TILE);
    scan<AddOp>(InFlag{st->flag}, OutDest{dest, tmp + nt}, n, tmp, s);
    // first_pts is rebuilt below, so it does not ride through the partition
    double* c8 = sc.get<double>(3 * n);
    int32_t* c4 = sc.get<int32_t>(3 * n);
    const int g = grid_for(n);
    k_scatter_col<double><<<g, PT, 0, s>>>(st->x, dest, n, c8);
    k_scatter_col<double><<<g, PT, 0, s>>>(st->y, dest, n, c8 + n);
    k_scatter_col<double><<<g, PT, 0, s>>>(st->dist, dest, n, c8 + 2 * n);
    k_scatter_col<int32_t><<<g, PT, 0, s>>>(st->head, dest, n, c4);
    k_scatter_col<int32_t><<<g, PT, 0, s>>>(st->keys, dest, n, c4 + n);
    k_scatter_col<int32_t><<<g, PT, 0, s>>>(st->flag, dest, n, c4 + 2 * n);
    PCK(cudaGetLastError());
    uint32_t kept = 0;
    PCK(cudaMemcpyAsync(&kept, tmp + nt, 4, cudaMemcpyDeviceToHost, s));
    PCK(cudaStreamSynchronize(s));
    PCK(cudaMemcpyAsync(st->x, c8, 8 * kept, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->y, c8 + n, 8 * kept, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->dist, c8 + 2 * n, 8 * kept, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->head, c4, 4 * kept, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->keys, c4 + n, 4 * kept, cudaMemcpyDeviceToDevice, s));
    PCK(cudaMemcpyAsync(st->flag, c4 + 2 * n, 4 * kept, cudaMemcpyDeviceToDevice, s));
    st->n = kept;
    propagate_first(st, kept, sc, s);
    PCK(cudaGetLastError());
    if (removed) *removed = n - kept;
  });
}

}  // extern "C"
