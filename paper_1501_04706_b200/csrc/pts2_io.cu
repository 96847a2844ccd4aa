// pts2_io.cu -- PTS2 binary point files straight to HBM (SURVEY.md section
// 8f row 3; replaces seghull::read_points_binary, dataio.cpp:114-153).
//
// Layout (dataio.cpp:22, 319-345): "PTS2", u64 LE count, then count x
// {f64 LE x, f64 LE y} -- an array of structures.  The hull kernels take
// structure-of-arrays input, so the loader streams the file through pinned
// host buffers (double-buffered: the next chunk is read from the file while
// the previous one is copied and split), and a split kernel writes x[] and
// y[] and records the first non-finite point (the reference rejects the
// file there, naming the point).
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <sys/stat.h>

#include "../../include/seghull_b200.h"

namespace {

constexpr uint64_t CHUNK = 1ull << 21;  // points per chunk (32 MB)

__global__ void k_split_pts2(const double2* __restrict__ aos, uint64_t cnt, uint64_t first,
                             double* __restrict__ x, double* __restrict__ y,
                             unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 p = aos[i];
    x[first + i] = p.x;
    y[first + i] = p.y;
    const uint32_t M = 0x7ff00000u;
    if (((uint32_t)__double2hiint(p.x) & M) == M || ((uint32_t)__double2hiint(p.y) & M) == M)
      atomicMin(bad, (unsigned long long)(first + i));
  }
}

struct Pool {  // per-process staging, grown on demand (pinned allocation is slow)
  std::mutex mu;
  double2* host[2] = {nullptr, nullptr};
  int dev = -1;
  double2* dbuf[2] = {nullptr, nullptr};
  unsigned long long* dbad = nullptr;
  unsigned long long* hbad = nullptr;
};
Pool g_pool;

void put(char* err, size_t len, const std::string& s) {
  if (err && len) std::snprintf(err, len, "%s", s.c_str());
}

uint64_t load_u64_le(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}

}  // namespace

extern "C" int sh_b200_read_pts2(const char* path, int device, void* stream, double* x, double* y,
                                 uint64_t cap, uint64_t* n, char* err, size_t errlen) {
  if (!path || !n) {
    put(err, errlen, "null argument");
    return SH_INVALID_ARGUMENT;
  }
  const std::string ps(path);
  FILE* f = std::fopen(path, "rb");
  if (!f) {  // open_input (dataio.cpp:81-91)
    struct stat st;
    if (stat(path, &st) != 0) {
      put(err, errlen, "no such file: " + ps);
      return SH_FILE_NOT_FOUND;
    }
    put(err, errlen, "cannot open " + ps);
    return SH_IO_ERROR;
  }
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  unsigned char hdr[12];
  if (std::fread(hdr, 1, 4, f) != 4) {
    put(err, errlen, ps + ": truncated header");
    return SH_PARSE_ERROR;
  }
  if (std::memcmp(hdr, "PTS2", 4) != 0) {
    put(err, errlen, ps + ": bad magic, expected PTS2");
    return SH_PARSE_ERROR;
  }
  if (std::fread(hdr + 4, 1, 8, f) != 8) {
    put(err, errlen, ps + ": truncated count");
    return SH_PARSE_ERROR;
  }
  const uint64_t count = load_u64_le(hdr + 4);
  struct stat st;
  if (stat(path, &st) == 0 && (uint64_t)st.st_size != 12 + 16 * count) {
    put(err, errlen, ps + ": size does not match declared point count");
    return SH_PARSE_ERROR;
  }
  *n = count;
  if (!x || !y) return SH_OK;
  if (cap < count) {
    put(err, errlen, "capacity " + std::to_string(cap) + " < " + std::to_string(count) + " points");
    return SH_CAP_TOO_SMALL;
  }
  if (count == 0) return SH_OK;

  std::lock_guard<std::mutex> lk(g_pool.mu);
  int prev = 0;
  cudaGetDevice(&prev);
  auto fail = [&](cudaError_t e, const char* what) {
    put(err, errlen, std::string(what) + ": " + cudaGetErrorString(e));
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(e, "cudaSetDevice");
  if (!g_pool.host[0]) {
    for (int b = 0; b < 2; ++b)
      if ((e = cudaMallocHost((void**)&g_pool.host[b], CHUNK * sizeof(double2))) != cudaSuccess)
        return fail(e, "cudaMallocHost");
    if ((e = cudaMallocHost((void**)&g_pool.hbad, sizeof(unsigned long long))) != cudaSuccess)
      return fail(e, "cudaMallocHost");
  }
  if (g_pool.dev != device) {
    for (int b = 0; b < 2; ++b) {
      if (g_pool.dbuf[b]) cudaFree(g_pool.dbuf[b]);
      if ((e = cudaMalloc((void**)&g_pool.dbuf[b], CHUNK * sizeof(double2))) != cudaSuccess)
        return fail(e, "cudaMalloc");
    }
    if (g_pool.dbad) cudaFree(g_pool.dbad);
    if ((e = cudaMalloc((void**)&g_pool.dbad, sizeof(unsigned long long))) != cudaSuccess)
      return fail(e, "cudaMalloc");
    g_pool.dev = device;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t done[2];
  for (int b = 0; b < 2; ++b) cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  struct EvCloser {
    cudaEvent_t* d;
    ~EvCloser() {
      cudaEventDestroy(d[0]);
      cudaEventDestroy(d[1]);
    }
  } evc{done};
  cudaMemsetAsync(g_pool.dbad, 0xFF, sizeof(unsigned long long), s);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  for (uint64_t first = 0, k = 0; first < count; first += CHUNK, ++k) {
    const int b = (int)(k & 1);
    const uint64_t cnt = count - first < CHUNK ? count - first : CHUNK;
    if (k >= 2) cudaEventSynchronize(done[b]);  // the copy out of host[b] is complete
    if (std::fread(g_pool.host[b], sizeof(double2), cnt, f) != cnt) {
      cudaStreamSynchronize(s);
      put(err, errlen, ps + ": truncated at point " + std::to_string(first));
      cudaSetDevice(prev);
      return SH_PARSE_ERROR;
    }
    cudaMemcpyAsync(g_pool.dbuf[b], g_pool.host[b], cnt * sizeof(double2), cudaMemcpyHostToDevice, s);
    const int grid = (int)std::min<uint64_t>((cnt + 255) / 256, (uint64_t)sms * 8);
    k_split_pts2<<<grid, 256, 0, s>>>(g_pool.dbuf[b], cnt, first, x, y, g_pool.dbad);
    cudaEventRecord(done[b], s);
  }
  cudaMemcpyAsync(g_pool.hbad, g_pool.dbad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e, "read_pts2");
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "read_pts2");
  cudaSetDevice(prev);
  if (*g_pool.hbad != ~0ull) {  // dataio.cpp:143-148
    put(err, errlen, ps + ": non-finite coordinate at point " + std::to_string(*g_pool.hbad));
    return SH_NON_FINITE_INPUT;
  }
  return SH_OK;
}
