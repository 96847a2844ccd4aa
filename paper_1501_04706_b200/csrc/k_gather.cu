// k_gather.cu -- the multi-GPU exchange step on the
// device: no host packing, no torch.
//
//   k5_pack    a shard's hull -> one fixed-size payload block
//              {x f64[cap] | y f64[cap] | global index i64[cap]}, vertices
//              [0, h) then copies of vertex 0 (a duplicate carries the same
//              coordinates and index, so it changes neither the merged hull
//              nor its canonical indices).  The block may live in a PEER
//              GPU's memory: with P2P enabled over NVLink/NVSwitch the shard
//              GPU stores its hull straight into the root's gather buffer.
//              A hull with h > cap writes NaN x and h into index[0]: the merge
//              then reports SH_CAP_TOO_SMALL with the capacity it needs.
//              Pad entries carry index -1, so the merge can drop them: thousands
//              of exact copies of one vertex would all tie for the farthest
//              point and serialise on its record (8 x 2048 padded vertices took
//              1.75 ms to merge, the ~450 real ones take ~40 us).
//   k_count /  R gathered blocks -> the merge hull's SoA input x[], y[] and
//   k_unpack   u32 ids of the REAL vertices only (global input indices; they
//              break ties and become the output indices, so the merged hull
//              carries canonical GLOBAL indices exactly as the whole-input run
//              would).  An overflow block (NaN x) is copied whole, so the merge
//              reports it.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

__global__ void k5_pack(Bufs B, double* blk, uint64_t cap, unsigned long long id_base) {
  const Ctl* c = B.ctl;
  pdl_wait();
  double* ox = blk;
  double* oy = blk + cap;
  long long* oi = reinterpret_cast<long long*>(blk + 2 * cap);
  const uint32_t st = c->status;
  uint32_t h = 0;
  const double* Tx = nullptr;
  const double* Ty = nullptr;
  const uint32_t* Tid = nullptr;
  if (st == ST_DONE) {
    const uint32_t par = c->round & 1u;
    h = c->S_cur;
    Tx = B.Tx[par];
    Ty = B.Ty[par];
    Tid = B.Tid[par];
  } else if (st == ST_SINGLE) {
    h = 1;  // {lo} (hull.cpp:234-237)
  } else if (st == ST_COLLINEAR) {
    h = 2;  // {lo, hi} (hull.cpp:238-248)
  }
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (h == 0 || h > cap) {  // error status or overflow: the NaN marker
    for (uint64_t i = tid; i < cap; i += stride) {
      ox[i] = __longlong_as_double(0x7FF8000000000000ll);
      oy[i] = 0.0;
      oi[i] = i == 0 ? (long long)h : 0;
    }
    return;
  }
  auto vert = [&](uint32_t k, double& x, double& y, uint32_t& id) {
    if (Tx) {
      x = Tx[k];
      y = Ty[k];
      id = Tid[k];
    } else {
      const int w = k == 0 ? 0 : 2;  // extremes: left, bottom, RIGHT, top
      x = c->ext_x[w];
      y = c->ext_y[w];
      id = c->ext_id[w];
    }
  };
  double x0, y0;
  uint32_t id0;
  vert(0, x0, y0, id0);
  for (uint64_t i = tid; i < cap; i += stride) {
    double x = x0, y = y0;
    uint32_t id = id0;
    if (i < h) vert((uint32_t)i, x, y, id);
    ox[i] = x;
    oy[i] = y;
    oi[i] = i < h ? (long long)(id_base + id) : -1ll;  // -1: padding
  }
}

// per block: its entries to keep (the real vertices, or every entry of an
// overflow block) -> cnt[b]; one CTA per block
__global__ void k_count(const double* __restrict__ pay, uint64_t cap, uint32_t* cnt) {
  const double* blk = pay + (uint64_t)blockIdx.x * 3 * cap;
  const long long* idx = reinterpret_cast<const long long*>(blk + 2 * cap);
  const bool overflow = blk[0] != blk[0];  // NaN marker
  uint32_t c = 0;
  for (uint64_t k = threadIdx.x; k < cap; k += blockDim.x) c += (overflow || idx[k] >= 0) ? 1u : 0u;
  c = __reduce_add_sync(FULL, c);
  __shared__ uint32_t s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_c, c);
  __syncthreads();
  if (threadIdx.x == 0) cnt[blockIdx.x] = s_c;
}

// kept entries of block b -> [sum of cnt[< b], ...): x, y, u32 ids; the total
// goes to cnt[R] (block 0)
__global__ void k_unpack(const double* __restrict__ pay, uint32_t R, uint64_t cap,
                         uint32_t* __restrict__ cnt, double* __restrict__ x,
                         double* __restrict__ y, uint32_t* __restrict__ ids) {
  __shared__ uint32_t s_base, s_tot;
  if (threadIdx.x == 0) s_base = s_tot = 0;
  __syncthreads();
  uint32_t base = 0, tot = 0;
  for (uint32_t b = threadIdx.x; b < R; b += blockDim.x) {
    const uint32_t v = cnt[b];
    tot += v;
    if (b < blockIdx.x) base += v;
  }
  base = __reduce_add_sync(FULL, base);
  tot = __reduce_add_sync(FULL, tot);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_base, base);
    atomicAdd(&s_tot, tot);
  }
  __syncthreads();
  const double* blk = pay + (uint64_t)blockIdx.x * 3 * cap;
  const long long* idx = reinterpret_cast<const long long*>(blk + 2 * cap);
  const uint32_t keep = cnt[blockIdx.x];  // real vertices are the block's prefix
  for (uint32_t k = threadIdx.x; k < keep; k += blockDim.x) {
    const uint32_t o = s_base + k;
    x[o] = blk[k];
    y[o] = blk[cap + k];
    ids[o] = (uint32_t)idx[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[R] = s_tot;
}

void launch_k5_pack(const Bufs& B, double* blk, uint64_t cap, unsigned long long id_base,
                    cudaStream_t s) {
  const int grid = (int)(cap / 512 + 1 < 148 ? cap / 512 + 1 : 148);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k5_pack, B, blk, cap, id_base);
}

// cnt: R + 1 words of device scratch; cnt[R] = points of the merge input
void launch_unpack(const double* pay, uint32_t R, uint64_t cap, uint32_t* cnt, double* x,
                   double* y, uint32_t* ids, cudaStream_t s) {
  k_count<<<R, 256, 0, s>>>(pay, cap, cnt);
  k_unpack<<<R, 256, 0, s>>>(pay, R, cap, cnt, x, y, ids);
}

}  // namespace shb
