// Does a lone warp run at the SM clock?  CTA 0 / warp 0 times a chain of
// dependent integer ops and FP64 compares with clock64 and %globaltimer,
// (a) while the other CTAs have exited, (b) while they spin.
#include <cstdio>
#include <cstdint>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(unsigned long long* out, int iters, int others_spin, volatile int* flag) {
  if (blockIdx.x != 0) {
    if (others_spin) while (*flag == 0) {}
    return;
  }
  if (threadIdx.x >= 32) return;
  unsigned long long a = threadIdx.x + 1, b = 7;
  double x = threadIdx.x * 0.5, y = 1.0;
  const long long c0 = clock64(); const unsigned long long g0 = gt();
  for (int i = 0; i < iters; ++i) { a = a * 3 + (b ^ (a >> 7)); b += (a < b) ? 1 : 2; }
  const long long c1 = clock64(); const unsigned long long g1 = gt();
  for (int i = 0; i < iters; ++i) { x = (x < y) ? x + 1.0 : x - 0.5; y = (y <= x) ? y * 1.5 : y; }
  const long long c2 = clock64(); const unsigned long long g2 = gt();
  for (int i = 0; i < iters; ++i) { a += __shfl_xor_sync(0xffffffffu, a, 1 + (i & 15)); }
  const long long c3 = clock64(); const unsigned long long g3 = gt();
  if (threadIdx.x == 0) {
    out[0] = c1 - c0; out[1] = g1 - g0; out[2] = c2 - c1; out[3] = g2 - g1; out[4] = c3 - c2; out[5] = g3 - g2;
    out[6] = a + (unsigned long long)x + b + (unsigned long long)y;
    *flag = 1;
  }
}
int main() {
  unsigned long long* out; int* flag;
  cudaMalloc(&out, 64); cudaMalloc(&flag, 4);
  unsigned long long h[8];
  for (int spin = 0; spin < 2; ++spin) for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(flag, 0, 4);
    k<<<148, 512>>>(out, 10000, spin, flag);
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("others %s: int chain %llu cyc / %llu ns (%.2f GHz) | fp64 cmp chain %llu cyc / %llu ns (%.2f GHz) | shfl %llu cyc / %llu ns (%.2f GHz)\n",
           spin ? "spin " : "exit ", h[0], h[1], (double)h[0] / h[1], h[2], h[3], (double)h[2] / h[3], h[4], h[5], (double)h[4] / h[5]);
  }
  return 0;
}
