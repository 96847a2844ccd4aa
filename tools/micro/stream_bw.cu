// Micro-benchmark: how fast can one pass over 2 x 160 MB SoA f64 arrays be
// consumed on this B200?  (a) plain vectorised loads, (b) the TMA bulk ring
// of K1-K3 with T points per tile and NS stages.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1501_04706_b200/csrc/device_common.cuh"
using namespace shb;

__global__ void plain(const double2* X, const double2* Y, uint32_t npairs, double* out) {
  double acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  for (; q + 3 * stride < npairs; q += 4 * stride) {
    double2 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { a[u] = __ldcs(X + q + u * stride); b[u] = __ldcs(Y + q + u * stride); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += a[u].x + a[u].y + b[u].x + b[u].y;
  }
  for (; q < npairs; q += stride) { double2 a = X[q], b = Y[q]; acc += a.x + a.y + b.x + b.y; }
  if (acc == 12345.0) *out = acc;
}

template <int T, int NS>
__global__ void __launch_bounds__(512, 1) ring(const double* X, const double* Y, uint32_t n, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileRing<T, NS, false> R;
  R.carve(smem_raw);
  if (threadIdx.x == 0) R.init();
  __syncthreads();
  double acc = 0;
  stream_input(R, n, X, Y, (const uint32_t*)nullptr, (const unsigned char*)nullptr, false,
               [&](int s, uint32_t first, uint32_t cnt) {
    const double2* xs = reinterpret_cast<const double2*>(R.xs + s * T);
    const double2* ys = reinterpret_cast<const double2*>(R.ys + s * T);
    for (uint32_t p = threadIdx.x; p < cnt / 2; p += blockDim.x) { double2 a = xs[p], b = ys[p]; acc += a.x + a.y + b.x + b.y; }
  });
  if (acc == 12345.0) *out = acc;
}

// AoS live-set style: xy double2 + is uint2 per point, CTA b streams either its
// own contiguous region (REGION) or tiles b, b+G, ... (interleaved)
template <int T, int NS, bool REGION>
__global__ void __launch_bounds__(512, 1) live(const double2* XY, const uint2* IS, uint32_t n, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sxy = reinterpret_cast<double2*>(smem_raw);
  uint2* sis = reinterpret_cast<uint2*>(sxy + NS * T);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sis + NS * T);
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1); mbar_fence_init(); }
  __syncthreads();
  const uint32_t ntiles = n / T, G = gridDim.x, b = blockIdx.x;
  const uint32_t per = (ntiles + G - 1) / G;
  const uint32_t mine = REGION ? min(per, ntiles - min(ntiles, b * per)) : (b < ntiles ? (ntiles - 1 - b) / G + 1 : 0);
  auto tile_of = [&](uint32_t k) { return REGION ? b * per + k : b + k * G; };
  auto issue = [&](uint32_t k) {
    const int s = k % NS; const uint32_t t = tile_of(k);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar + s, T * 24);
    tma_load_1d(sxy + s * T, XY + (size_t)t * T, T * 16, bar + s);
    tma_load_1d(sis + s * T, IS + (size_t)t * T, T * 8, bar + s);
  };
  if (threadIdx.x == 0) for (uint32_t k = 0; k < mine && k < NS; ++k) issue(k);
  double acc = 0;
  for (uint32_t k = 0; k < mine; ++k) {
    const int s = k % NS;
    mbar_wait(bar + s, (k / NS) & 1);
    for (uint32_t p = threadIdx.x; p < T; p += blockDim.x) { double2 a = sxy[s * T + p]; acc += a.x + a.y + sis[s * T + p].x; }
    __syncthreads();
    if (threadIdx.x == 0 && k + NS < mine) issue(k + NS);
  }
  if (acc == 12345.0) *out = acc;
}

template <int T, int NS, bool REGION>
void run_live(const double2* XY, const uint2* IS, uint32_t n, double* out, int sms, cudaEvent_t a, cudaEvent_t b) {
  const size_t sm = (size_t)NS * T * 24 + NS * 8;
  cudaFuncSetAttribute(live<T, NS, REGION>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(a);
    live<T, NS, REGION><<<sms, 512, sm>>>(XY, IS, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("live T=%5d NS=%d %s: %8.1f us  %7.1f GB/s  (%s)\n", T, NS, REGION ? "region     " : "interleaved", best * 1e3, 24.0 * n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int T, int NS>
void run_ring(const double* X, const double* Y, uint32_t n, double* out, int sms, int bps, cudaEvent_t a, cudaEvent_t b) {
  const size_t sm = TileRing<T, NS, false>::kBytes;
  if (cudaFuncSetAttribute(ring<T, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) { printf("ring T=%d NS=%d: smem too big\n", T, NS); cudaGetLastError(); return; }
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(a);
    ring<T, NS><<<sms * bps, 512, sm>>>(X, Y, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("ring T=%5d NS=%d ctas/sm=%d smem=%6zu: %8.1f us  %7.1f GB/s  (%s)\n", T, NS, bps, sm, best * 1e3, 16.0 * n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint32_t n = 20000000;
  double *X, *Y, *out, *flush;
  cudaMalloc(&X, 8ull * n); cudaMalloc(&Y, 8ull * n); cudaMalloc(&out, 8); cudaMalloc(&flush, 256 << 20);
  cudaMemset(X, 0, 8ull * n); cudaMemset(Y, 0, 8ull * n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int g : {1, 2, 4, 8, 16}) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256 << 20);
      cudaEventRecord(a);
      plain<<<sms * g, 256>>>((const double2*)X, (const double2*)Y, n / 2, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("plain grid=%4d x 256: %8.1f us  %7.1f GB/s\n", sms * g, best * 1e3, 16.0 * n / best / 1e6);
  }
  {
    const uint32_t m = 5200000 / 1024 * 1024;
    double2* XY; uint2* IS;
    cudaMalloc(&XY, 16ull * m); cudaMalloc(&IS, 8ull * m);
    cudaMemset(XY, 0, 16ull * m); cudaMemset(IS, 0, 8ull * m);
    run_live<1024, 6, true>(XY, IS, m, out, sms, a, b);
    run_live<1024, 6, false>(XY, IS, m, out, sms, a, b);
    run_live<1024, 4, true>(XY, IS, m, out, sms, a, b);
    run_live<1024, 4, false>(XY, IS, m, out, sms, a, b);
    run_live<2048, 3, true>(XY, IS, m, out, sms, a, b);
    run_live<2048, 3, false>(XY, IS, m, out, sms, a, b);
  }
  run_ring<2048, 3>(X, Y, n, out, sms, 1, a, b);
  run_ring<2048, 4>(X, Y, n, out, sms, 1, a, b);
  run_ring<2048, 6>(X, Y, n, out, sms, 1, a, b);
  run_ring<1024, 6>(X, Y, n, out, sms, 1, a, b);
  run_ring<1024, 12>(X, Y, n, out, sms, 1, a, b);
  run_ring<4096, 3>(X, Y, n, out, sms, 1, a, b);
  run_ring<1024, 4>(X, Y, n, out, sms, 2, a, b);
  run_ring<1024, 6>(X, Y, n, out, sms, 2, a, b);
  run_ring<512, 8>(X, Y, n, out, sms, 2, a, b);
  run_ring<512, 12>(X, Y, n, out, sms, 2, a, b);
  return 0;
}
