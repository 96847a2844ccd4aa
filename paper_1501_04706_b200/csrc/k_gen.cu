// k_gen.cu -- device twins of the reference's point generators
// (dataio.hpp:44-58, dataio.cpp:291-301; SURVEY.md section 0 finding 3 and
// section 8d).  Not on the hull path: they produce the synthetic inputs of
// the configs directly in HBM (the 1B-point config cannot afford 16 GB of H2D).
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "hull_kernels.cuh"

namespace shb {

constexpr int GEN_ITEMS = 8;
constexpr int GEN_TILE = TPB * GEN_ITEMS;

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
  __shared__ uint32_t s_cnt[GEN_ITEMS * WARPS];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t epoch = *(volatile uint32_t*)epoch_p;
  const uint32_t ntiles = (ncand + GEN_TILE - 1) / GEN_TILE;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    double px[GEN_ITEMS], py[GEN_ITEMS];
    uint32_t acc = 0, rank[GEN_ITEMS];
#pragma unroll
    for (int j = 0; j < GEN_ITEMS; ++j) {
      const uint32_t e = tile * GEN_TILE + j * TPB + threadIdx.x;
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
    for (int j = 0; j < GEN_ITEMS; ++j) {
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

void launch_gen_uniform(double* x, double* y, unsigned long long first, unsigned long long count,
                        unsigned long long seed, int grid, cudaStream_t s) {
  k_gen_uniform<<<grid, 256, 0, s>>>(x, y, first, count, seed);
}

void launch_gen_disk(double* x, double* y, unsigned long long n, unsigned long long seed,
                     unsigned long long cand0, uint32_t ncand, unsigned long long out_base, Ctl* c,
                     unsigned long long* status, uint32_t* epoch, int grid, cudaStream_t s) {
  k_gen_disk<<<grid, TPB, 0, s>>>(x, y, n, seed, cand0, ncand, out_base, c, status, epoch);
}

int gen_tile_points() { return GEN_TILE; }

}  // namespace shb
