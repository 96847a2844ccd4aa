// l2_atomics.cu -- throughput of random-address L2 operations on B200, the
// access pattern of the round kernel's large-table point phase: N operations,
// each on a uniformly random slot of an S-entry table.
//   atom : 64-bit atomicMax whose result is used   (ATOMG.E.MAX.64)
//   red  : 64-bit atomicMax, result unused          (REDG.E.MAX.64)
//   ld8  : 8-byte load                              (LDG.E.64)
//   row64: two 32-byte loads of a 64-byte row       (the Route row)
//   ldred: 8-byte load, then red only if larger     (screened atomics)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_atomics l2_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(512) kern(unsigned long long* tab, const double4* rows, uint32_t S,
                                            uint32_t N, unsigned long long* sink) {
  unsigned long long acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride * 3) {
    uint32_t s[3];
    unsigned long long v[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const uint32_t h = hash32(i + u * stride);
      s[u] = h % S;
      v[u] = hash32(h) ;
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (i + u * stride >= N) continue;
      if (MODE == 0) acc ^= atomicMax(tab + s[u], v[u]);
      if (MODE == 1) atomicMax(tab + s[u], v[u]);
      if (MODE == 2) acc ^= __ldcg(tab + s[u]);
      if (MODE == 3) {
        double a0, a1, a2, a3, b0, b1, b2, b3;
        asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(rows + 2 * s[u]));
        asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(b0), "=d"(b1), "=d"(b2), "=d"(b3) : "l"(rows + 2 * s[u] + 1));
        acc ^= (unsigned long long)__double_as_longlong(a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3);
      }
      if (MODE == 4) {
        if (v[u] > __ldcg(tab + s[u])) atomicMax(tab + s[u], v[u]);
      }
    }
  }
  if (acc == 0x1234567ull) *sink = acc;
}

int main() {
  const uint32_t N = 4u << 20;
  const uint32_t Ss[] = {2048, 32768, 262144, 1u << 20, 4u << 20};
  unsigned long long *tab, *sink;
  double4* rows;
  cudaMalloc(&tab, 8ull * (4u << 20));
  cudaMalloc(&rows, 64ull * (4u << 20));
  cudaMalloc(&sink, 8);
  cudaMemset(rows, 0, 64ull * (4u << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"atom", "red", "ld8", "row64", "ldred"};
  for (uint32_t S : Ss) {
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(tab, 0, 8ull * S);
        cudaEventRecord(e0);
        switch (mode) {
          case 0: kern<0><<<148, 512>>>(tab, rows, S, N, sink); break;
          case 1: kern<1><<<148, 512>>>(tab, rows, S, N, sink); break;
          case 2: kern<2><<<148, 512>>>(tab, rows, S, N, sink); break;
          case 3: kern<3><<<148, 512>>>(tab, rows, S, N, sink); break;
          case 4: kern<4><<<148, 512>>>(tab, rows, S, N, sink); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("S %8u %-6s %8.1f us  %6.1f Gops/s\n", S, names[mode], best * 1e3, N / (best * 1e6));
    }
  }
  return 0;
}
