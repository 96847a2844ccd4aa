// seghull_b200.cu -- host orchestration and the C-ABI (include/seghull_b200.h).
//
// One call = one device-resident pipeline on one stream:
//   [H2D] -> K1 -> K2 -> K3<first> -> { K4 -> K3 }* -> D2H(result)
// Round bookkeeping lives in the device control block; the host only polls
// the status word between batches of rounds (no per-round host logic).
// Workspaces (all device buffers + pinned staging + events) are pooled per
// device under a mutex, so repeated calls allocate nothing.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <chrono>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/seghull_b200.h"
#include "hull_kernels.cuh"

namespace shb {
void launch_k1(const Bufs& B, bool ids, int grid, cudaStream_t s);
void launch_small(const Bufs& B, bool filter, bool ids, cudaStream_t s);
void launch_k2(const Bufs& B, bool filter, bool ids, int grid, cudaStream_t s);
void launch_k3(const Bufs& B, bool ids, bool capped, int grid, cudaStream_t s);
cudaError_t configure_stream_kernels_pre();
cudaError_t configure_stream_kernels_k3();
size_t rounds_smem_bytes();
cudaError_t configure_round_kernels();
int rounds_blocks_per_sm();
cudaError_t launch_rounds(const Bufs& B, int grid, cudaStream_t s);
void launch_k5(const Bufs& B, double* ox, double* oy, long long* oidx, uint64_t cap,
               unsigned long long id_base, cudaStream_t s);
void launch_gen_uniform(double* x, double* y, unsigned long long first, unsigned long long count,
                        unsigned long long seed, int grid, cudaStream_t s);
void launch_gen_disk(double* x, double* y, unsigned long long n, unsigned long long seed,
                     unsigned long long cand0, uint32_t ncand, unsigned long long out_base,
                     Ctl* c, unsigned long long* status, uint32_t* epoch, int grid,
                     cudaStream_t s);
int gen_tile_points();
void launch_preprocess(const Bufs& B, double* ox, double* oy, unsigned long long cap, int grid,
                       cudaStream_t s);
void launch_k5_pack(const Bufs& B, double* blk, uint64_t cap, unsigned long long id_base,
                    cudaStream_t s);
void launch_unpack(const double* pay, uint32_t R, uint64_t cap, uint32_t* cnt, double* x,
                   double* y, uint32_t* ids, cudaStream_t s);
}  // namespace shb

using namespace shb;

namespace {

struct CudaFail {
  cudaError_t err;
  const char* what;
};

#define CK(call)                                      \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) throw CudaFail{e_, #call}; \
  } while (0)

struct DeviceInfo {
  int sm_count = 0;
  bool configured = false;
  int rounds_bps = 1;  // co-resident CTAs of the cooperative round kernel per SM
};

std::mutex g_mutex;
int g_trace_round = 0;                          // debug: trace CTA 0's tiles of this round
thread_local unsigned long long g_last_tl[33];  // debug: [0] = count, then timestamps
thread_local std::vector<unsigned long long> g_last_ctas;  // debug: per-CTA point-phase ends
// One entry per CUDA device, sized once (never reallocated afterwards) and
// only read or written under g_mutex; callers get a copy.
std::vector<DeviceInfo> g_dev;
std::vector<size_t> g_dev_mem;  // HBM bytes per device (same lifetime and lock as g_dev)

// Host->device staging ring for pageable inputs (and the reverse for large
// hulls): pinned chunks + one event each.  Owned by a workspace, so every
// call -- and every host thread of a multi-GPU call -- has its own ring on
// its own device: no shared host state, no lock held across a copy.
constexpr size_t H2D_CHUNK = 8u << 20;  // default chunk (SHB_H2D_CHUNK_MB)
constexpr int H2D_NBUF = 4;             // default chunks in flight (SHB_H2D_NBUF)
constexpr int H2D_MAXBUF = 8;
struct PinnedRing {
  char* buf[H2D_MAXBUF] = {};
  cudaEvent_t done[H2D_MAXBUF] = {};
  size_t chunk = H2D_CHUNK;
  int nbuf = 0;      // 0: not allocated yet
  int threads = 10;  // host threads packing / unpacking a chunk
};

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = std::getenv(name);
  if (!e) return dflt;
  const int v = std::atoi(e);
  return v < lo ? lo : v > hi ? hi : v;
}

struct Workspace {
  int device = 0;
  uint64_t n_cap = 0, s_cap = 0, live_n = 0;  // points, segments, live-set entries
  size_t bytes = 0;                            // device bytes (arena + staging)
  bool has_stage = false, has_stage_ids = false;
  cudaStream_t stream = nullptr;
  void* arena = nullptr;
  void* stage = nullptr;
  Bufs B{};
  uint32_t* epoch = nullptr;
  unsigned char* h_res = nullptr;  // pinned: {Ctl; StatRec[STATS_EAGER]}, one copy per call
  Ctl* h_ctl = nullptr;            // = h_res
  StatRec* h_stats = nullptr;      // pinned, all rounds
  cudaEvent_t ev[8] = {};
  size_t tiles_cap = 0;
  int stream_grid = 0, rounds_grid = 0;
  PinnedRing ring;

  ~Workspace() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);  // nothing of ours may still be in flight
    for (int b = 0; b < H2D_MAXBUF; ++b) {
      if (ring.done[b]) cudaEventSynchronize(ring.done[b]);
      if (ring.done[b]) cudaEventDestroy(ring.done[b]);
      if (ring.buf[b]) cudaFreeHost(ring.buf[b]);
    }
    if (arena) cudaFree(arena);
    if (stage) cudaFree(stage);
    if (h_res) cudaFreeHost(h_res);
    if (h_stats) cudaFreeHost(h_stats);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    cudaSetDevice(cur);
  }
};

std::vector<std::vector<std::unique_ptr<Workspace>>> g_pool;  // free workspaces per device

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Caller holds g_mutex.  The device's kernels are configured on first use.
DeviceInfo device_info_locked(int device) {
  if (g_dev.empty()) {
    int nd = 0;
    CK(cudaGetDeviceCount(&nd));
    g_dev.resize(std::max(nd, 1));
    g_dev_mem.assign(g_dev.size(), (size_t)48 << 30);
    for (int d = 0; d < nd; ++d) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, d) == cudaSuccess) g_dev_mem[d] = p.totalGlobalMem;
    }
    cudaGetLastError();
  }
  if (device < 0 || device >= (int)g_dev.size()) throw CudaFail{cudaErrorInvalidDevice, "device"};
  DeviceInfo& d = g_dev[device];
  if (!d.configured) {
    CK(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(configure_round_kernels());
    d.rounds_bps = rounds_blocks_per_sm();
    CK(configure_stream_kernels_pre());
    CK(configure_stream_kernels_k3());
    d.configured = true;
  }
  return d;
}

DeviceInfo device_info(int device) {
  std::lock_guard<std::mutex> lk(g_mutex);
  return device_info_locked(device);
}

// Segment-table and live-set capacities of a fresh workspace.  Up to 2^24
// points every point may become a head, up to 2^27 every point may survive
// round 1.  Beyond, the tables start at n/16 segments (140 B each) and the
// live sets at 3n/8 points (64 B each: two 24-B ping-pong sets + the 16-B
// contender list):
// uniform 1B needs 55 heads and 0.23 n round-1 survivors.  An input that
// outgrows either ends the call with ST_OVERFLOW; the call then regrows the
// workspace to n + 2 segments and n live points and reruns (the grown
// workspace stays in the pool for the next call).
// SHB_SEG_CAP / SHB_LIVE_CAP (tests) cap them to force that path on small inputs.
#ifndef SHB_LEAN_LOG2
#define SHB_LEAN_LOG2 24
#endif
constexpr uint64_t LEAN_N = 1ull << SHB_LEAN_LOG2;  // above this, tables and live sets start lean

uint64_t seg_capacity(uint64_t n) {
  uint64_t cap = n <= LEAN_N ? n + 2 : std::max<uint64_t>(LEAN_N, n / 16);
  if (const char* e = std::getenv("SHB_SEG_CAP")) {
    const uint64_t v = std::strtoull(e, nullptr, 10);
    if (v >= 4096) cap = std::min(cap, v);  // >= 2 NSLOT: small tables never check
  }
  return cap;
}

constexpr uint64_t LEAN_LIVE_N = 1ull << 27;  // live sets start lean above this

uint64_t live_capacity(uint64_t n) {
  // full up to 2^27 points (8.6 GB): K3 then needs no per-append check
  uint64_t cap = n <= LEAN_LIVE_N ? n : std::max<uint64_t>(LEAN_N, (3 * n / 8 + 63) & ~63ull);
  if (const char* e = std::getenv("SHB_LIVE_CAP")) {  // tests: force K3's overflow check
    const uint64_t v = std::strtoull(e, nullptr, 10);
    if (v >= 4096) cap = std::min(cap, v);
  }
  return cap;
}

std::unique_ptr<Workspace> make_workspace(int device, uint64_t n_cap, uint64_t s_cap,
                                          uint64_t live_cap) {
  auto ws = std::make_unique<Workspace>();
  ws->device = device;
  ws->n_cap = n_cap;
  ws->s_cap = s_cap;
  const DeviceInfo di = device_info(device);
  CK(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking));
  for (auto& e : ws->ev) CK(cudaEventCreate(&e));
  CK(cudaMallocHost((void**)&ws->h_res, HOST_RES_BYTES));
  ws->h_ctl = reinterpret_cast<Ctl*>(ws->h_res);
  CK(cudaMallocHost((void**)&ws->h_stats, sizeof(StatRec) * STATS_CAP));

  const uint64_t N = std::max<uint64_t>(n_cap, 64), S = std::max<uint64_t>(s_cap, 64);
  // streaming kernels: 4 CTAs of 256 threads per SM; the round kernel: every
  // co-resident CTA (cooperative launch)
  ws->stream_grid = di.sm_count;  // K1/K2/K3: one TMA-fed CTA per SM
  ws->rounds_grid = std::min(di.sm_count * di.rounds_bps, MAX_ROUND_BLOCKS);
  ws->tiles_cap = (N + gen_tile_points() - 1) / gen_tile_points() + 64;

  // carve one arena
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_ctl = take(HOST_RES_STATS + sizeof(StatRec) * STATS_CAP);  // Ctl, then the stats
  const size_t o_epoch = take(sizeof(uint32_t));
  const size_t o_k1 = take(sizeof(K1Partial) * ws->stream_grid);
  const size_t o_k2 = take(sizeof(K2Partial) * ws->stream_grid);
  const size_t o_blk = take(sizeof(uint32_t) * 2 * MAX_ROUND_BLOCKS);
  const size_t o_dbg = take(sizeof(unsigned long long) * DBG_SLOTS);
  const size_t o_tiles = take(sizeof(unsigned long long) * ws->tiles_cap);
  const size_t o_bits = take(sizeof(uint4) * ((N + 63) / 64));
  size_t o_lxy[2], o_lis[2], o_rc[2], o_tx[2], o_ty[2], o_tid[2], o_sd[3], o_sw[3];
  // live set runs: K3's CTA j owns [j*run_q, (j+1)*run_q); the rounding of
  // run_q to whole tiles costs at most one tile per CTA
  const uint64_t LN = std::max<uint64_t>(std::min(live_cap, N), 64) +
                     2ull * (uint64_t)di.sm_count * Cfg3::T;
  ws->live_n = LN;
  for (int p = 0; p < 2; ++p) {
    o_lxy[p] = take(16 * LN);
    o_lis[p] = take(8 * LN);
    o_rc[p] = take(4 * MAX_RUNS);
  }
  for (int p = 0; p < 2; ++p) {
    o_tx[p] = take(8 * S);
    o_ty[p] = take(8 * S);
    o_tid[p] = take(4 * S);
  }
  size_t o_wn[3];
  for (int p = 0; p < 3; ++p) {
    o_sd[p] = take(8 * S);
    o_sw[p] = take(sizeof(SlotRec) * NSLOT);  // records exist for small tables only
    o_wn[p] = take(4 * S);
  }
  const size_t o_lc = take(sizeof(LiveCand) * LN);
  const size_t rows = (size_t)std::max(ws->rounds_grid, ws->stream_grid);
  const size_t o_rc0 = take(sizeof(SlotRec) * NSLOT * rows);
  const size_t o_rc1 = take(sizeof(SlotRec) * NSLOT * rows);
  const size_t o_route = take(sizeof(Route) * S);
  CK(cudaMalloc(&ws->arena, off));
  ws->bytes = off;
  char* a = (char*)ws->arena;
  CK(cudaMemset(a, 0, o_bits));
  Bufs& B = ws->B;
  B.ctl = (Ctl*)(a + o_ctl);
  ws->epoch = B.epoch = (uint32_t*)(a + o_epoch);
  const uint32_t one = 1;
  CK(cudaMemcpy(ws->epoch, &one, sizeof(one), cudaMemcpyHostToDevice));
  B.k1part = (K1Partial*)(a + o_k1);
  B.k2part = (K2Partial*)(a + o_k2);
  B.stats = (StatRec*)(a + o_ctl + HOST_RES_STATS);
  B.blk_cnt = (uint32_t*)(a + o_blk);
  B.dbg = (unsigned long long*)(a + o_dbg);
  B.tile_status = (unsigned long long*)(a + o_tiles);
  B.bits = (uint4*)(a + o_bits);
  for (int p = 0; p < 2; ++p) {
    B.Lxy[p] = (double2*)(a + o_lxy[p]);
    B.Lis[p] = (uint2*)(a + o_lis[p]);
    B.run_cnt[p] = (uint32_t*)(a + o_rc[p]);
    B.Tx[p] = (double*)(a + o_tx[p]);
    B.Ty[p] = (double*)(a + o_ty[p]);
    B.Tid[p] = (uint32_t*)(a + o_tid[p]);
  }
  for (int p = 0; p < 3; ++p) {
    B.Sd[p] = (unsigned long long*)(a + o_sd[p]);
    B.Srec[p] = (SlotRec*)(a + o_sw[p]);
    B.Wn[p] = (uint32_t*)(a + o_wn[p]);
  }
  B.Lc = (LiveCand*)(a + o_lc);
  B.Rc[0] = (SlotRec*)(a + o_rc0);
  B.Rc[1] = (SlotRec*)(a + o_rc1);
  B.route = (Route*)(a + o_route);
  B.s_cap = (uint32_t)std::min<uint64_t>(s_cap, 0xFFFFFFF0ull);
  return ws;
}

void ensure_stage(Workspace& ws, bool ids) {
  if (ws.has_stage && (!ids || ws.has_stage_ids)) return;
  if (ws.stage) CK(cudaFree(ws.stage));
  ws.stage = nullptr;
  const size_t bytes = 2 * align_up(8 * ws.n_cap, 256) + (ids ? align_up(4 * ws.n_cap, 256) : 0);
  CK(cudaMalloc(&ws.stage, bytes));
  ws.bytes += bytes;
  ws.has_stage = true;
  ws.has_stage_ids = ids;
}

// make_workspace; on failure (out of memory) drop every pooled workspace on
// the device and retry once.
std::unique_ptr<Workspace> make_workspace_retry(int device, uint64_t n_cap, uint64_t s_cap,
                                                uint64_t live_cap) {
  try {
    return make_workspace(device, n_cap, s_cap, live_cap);
  } catch (const CudaFail&) {
    cudaGetLastError();
    std::vector<std::unique_ptr<Workspace>> drop;
    {
      std::lock_guard<std::mutex> lk(g_mutex);
      if ((int)g_pool.size() > device) drop.swap(g_pool[device]);
    }
    drop.clear();  // destructors run outside the lock
    return make_workspace(device, n_cap, s_cap, live_cap);
  }
}

std::unique_ptr<Workspace> acquire(int device, uint64_t n) {
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    device_info_locked(device);
    if ((int)g_pool.size() <= device) g_pool.resize(device + 1);
    auto& v = g_pool[device];
    int best = -1;
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i]->n_cap >= n && (best < 0 || v[i]->n_cap < v[best]->n_cap)) best = (int)i;
    if (best >= 0) {
      auto ws = std::move(v[best]);
      v.erase(v.begin() + best);
      return ws;
    }
  }
  const uint64_t cap = std::max<uint64_t>(n, 1u << 12);
  return make_workspace_retry(device, cap, seg_capacity(cap), live_capacity(cap));
}

void release(std::unique_ptr<Workspace> ws) {
  std::vector<std::unique_ptr<Workspace>> drop_list;  // destroyed after the lock
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    if ((int)g_pool.size() <= ws->device) g_pool.resize(ws->device + 1);
    auto& v = g_pool[ws->device];
    v.push_back(std::move(ws));
    // bounded by bytes (at most 3/8 of the device's HBM parked in the pool)
    // and by count: drop the smallest workspaces first
    size_t total = 0;
    for (auto& w : v) total += w->bytes;
    const size_t budget = g_dev_mem.size() > (size_t)v.back()->device
                              ? g_dev_mem[v.back()->device] / 8 * 3 : (size_t)48 << 30;
    while (v.size() > 1 && (v.size() > 8 || total > budget)) {
      size_t small = 0;
      for (size_t i = 1; i < v.size(); ++i)
        if (v[i]->bytes < v[small]->bytes) small = i;
      total -= v[small]->bytes;
      drop_list.push_back(std::move(v[small]));
      v.erase(v.begin() + small);
    }
  }
}

void put_err(char* err, size_t len, const std::string& s) {
  if (!err || !len) return;
  std::snprintf(err, len, "%s", s.c_str());
}

struct RunOut {
  int code = SH_OK;
  uint64_t h = 0, rounds = 0, kept = 0, bad = 0;
  uint32_t launches = 0;
  std::string msg;
};

void ensure_ring(Workspace& ws) {
  PinnedRing& R = ws.ring;
  if (R.nbuf) return;
  R.chunk = (size_t)env_int("SHB_H2D_CHUNK_MB", (int)(H2D_CHUNK >> 20), 1, 64) << 20;
  const int nb = env_int("SHB_H2D_NBUF", H2D_NBUF, 2, H2D_MAXBUF);
  // 10 packing threads: on the 16-core B200 host, 8 fell into a slow mode in 2 of
  // 6 processes (7.45 vs 6.7 ms per 320 MB); 10 stayed at 6.72-6.82 ms in all six
  R.threads = env_int("SHB_H2D_THREADS", 10, 1, 64);
  for (int b = 0; b < nb; ++b) {
    CK(cudaMallocHost((void**)&R.buf[b], R.chunk));
    CK(cudaEventCreateWithFlags(&R.done[b], cudaEventDisableTiming));
  }
  R.nbuf = nb;
}

// Host -> device copy of a caller's buffer.  Pinned (or registered) memory
// goes straight to the copy engine.  Pageable memory would be staged by the
// driver through one bounce buffer at ~11 GB/s; instead it is packed into the
// workspace's pinned chunks by the host cores (OpenMP) and each chunk is
// copied while the next ones are packed (nbuf chunks in flight).
void h2d_or_copy(Workspace& ws, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                 bool host, cudaStream_t st) {
  if (!host || bytes < (H2D_CHUNK >> 2)) {
    CK(cudaMemcpyAsync(dst, src, bytes, kind, st));
    return;
  }
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
    CK(cudaMemcpyAsync(dst, src, bytes, kind, st));  // already pinned
    return;
  }
  cudaGetLastError();  // pageable pointers may leave an error on older drivers
  ensure_ring(ws);
  PinnedRing& R = ws.ring;
  const char* s = (const char*)src;
  char* d = (char*)dst;
  const int nt = R.threads;
  (void)nt;  // (used by the OpenMP clause below)
  const size_t nchunks = (bytes + R.chunk - 1) / R.chunk;
  // ONE parallel region for the whole transfer: a team forked per chunk lets
  // its idle workers fall asleep while the master waits on a chunk's event,
  // and every wake-up then delays the next chunk (a bimodal 6.7 / 7.5 ms per
  // 320 MB on a 16-core VM).  Here the workers only cross spinning barriers;
  // the master alone calls CUDA (event waits, copies, records).
  cudaError_t err = cudaSuccess;
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
    for (size_t k = 0; k < nchunks; ++k) {
      const int b = (int)(k % R.nbuf);
      const size_t off = k * R.chunk, len = std::min(R.chunk, bytes - off);
#pragma omp master
      {
        const cudaError_t e = cudaEventSynchronize(R.done[b]);  // buf[b]'s earlier copy finished
        if (e != cudaSuccess && err == cudaSuccess) err = e;
      }
#pragma omp barrier
      const size_t a = len * t / T, e = len * (t + 1) / T;
      std::memcpy(R.buf[b] + a, s + off + a, e - a);
#pragma omp barrier
#pragma omp master
      {
        cudaError_t e2 = cudaMemcpyAsync(d + off, R.buf[b], len, cudaMemcpyHostToDevice, st);
        if (e2 == cudaSuccess) e2 = cudaEventRecord(R.done[b], st);
        if (e2 != cudaSuccess && err == cudaSuccess) err = e2;
      }
    }
  }
  CK(err);
}

// The reverse direction for a large hull (the circle: millions of vertices)
// into pageable host memory: device chunks are copied into the pinned ring
// and unpacked by the host cores into the caller's array while the next
// chunks are in flight; `widen` turns the u32 vertex ids into int64 (plus
// id_base).  Synchronous: the caller's array is complete on return.
void d2h_ring(Workspace& ws, void* dst, const void* src, size_t n, bool widen, uint64_t id_base,
              cudaStream_t st) {
  ensure_ring(ws);
  PinnedRing& R = ws.ring;
  const size_t esz = widen ? 4 : 8;  // source element size
  const size_t per = R.chunk / esz;  // elements per chunk
  const size_t nchunks = (n + per - 1) / per;
  const int nt = R.threads;
  const char* s = (const char*)src;
  auto issue = [&](size_t k) {
    const int b = (int)(k % R.nbuf);
    const size_t len = std::min(per, n - k * per) * esz;
    CK(cudaEventSynchronize(R.done[b]));  // an earlier H2D out of buf[b] may still run
    CK(cudaMemcpyAsync(R.buf[b], s + k * per * esz, len, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(R.done[b], st));
  };
  for (size_t k = 0; k < nchunks && k < (size_t)R.nbuf; ++k) issue(k);
  for (size_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k % R.nbuf);
    CK(cudaEventSynchronize(R.done[b]));
    const size_t e0 = k * per, cnt = std::min(per, n - e0);
    const long parts = 2 * nt;
    if (widen) {
      const uint32_t* pb = (const uint32_t*)R.buf[b];
      int64_t* d = (int64_t*)dst + e0;
#pragma omp parallel for num_threads(nt) schedule(static)
      for (long t = 0; t < parts; ++t) {
        const size_t a = cnt * t / parts, e = cnt * (t + 1) / parts;
        for (size_t i = a; i < e; ++i) d[i] = (int64_t)(pb[i] + id_base);
      }
    } else {
      const char* pb = R.buf[b];
      char* d = (char*)dst + e0 * 8;
#pragma omp parallel for num_threads(nt) schedule(static)
      for (long t = 0; t < parts; ++t) {
        const size_t a = cnt * 8 * t / parts, e = cnt * 8 * (t + 1) / parts;
        std::memcpy(d + a, pb + a, e - a);
      }
    }
    if (k + R.nbuf < nchunks) issue(k + R.nbuf);
  }
}

// Runs the whole pipeline with ONE host synchronisation: H2D (host inputs),
// K1, K2, K3, the cooperative round kernel, K5 (device outputs), and the
// read-back of the control block + the first STATS_EAGER round stats.
// SHB_HOST_TIMING=1: host-side wall clock of one call's steps on stderr (debug)
const bool g_host_timing = std::getenv("SHB_HOST_TIMING") != nullptr;
struct HostClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  char buf[512];
  int len = 0;
  void mark(const char* what) {
    if (!g_host_timing) return;
    const auto now = std::chrono::steady_clock::now();
    len += std::snprintf(buf + len, sizeof(buf) - len, " %s %.1f",
                         what, std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
  }
  void print() {
    if (g_host_timing) std::fprintf(stderr, "[host us]%s\n", buf);
  }
};

RunOut parse_ctl(Workspace& ws, const sh_hull_request& rq, const sh_hull_result& res);

// Enqueues the whole pipeline; with `wait` it synchronises and parses the
// control block, otherwise it returns code -2 (pending): ws.ev[7] marks the
// end of the call's device work, parse_ctl() finishes it later.
RunOut run_pipeline(Workspace& ws, const sh_hull_request& rq, sh_hull_result& res,
                    cudaStream_t st, bool timings, const uint32_t* n_dev = nullptr,
                    bool wait = true) {
  HostClock hc;
  RunOut out;
  Bufs B = ws.B;
  const uint64_t n = rq.n;
  const bool host = !(rq.flags & SH_DEVICE_PTRS);
  if (timings) CK(cudaEventRecord(ws.ev[0], st));
  // The TMA bulk copies of K1-K3 need 16-byte aligned x/y/ids: host inputs and
  // unaligned device inputs go through the workspace's aligned staging copy.
  const bool aligned = ((uintptr_t)rq.x % 16 == 0) && ((uintptr_t)rq.y % 16 == 0) &&
                       (!rq.ids || (uintptr_t)rq.ids % 16 == 0);
  if (host || !aligned) {
    ensure_stage(ws, rq.ids != nullptr);
    B = ws.B;
    double* sx = (double*)ws.stage;
    double* sy = (double*)((char*)ws.stage + align_up(8 * ws.n_cap, 256));
    uint32_t* sid = (uint32_t*)((char*)ws.stage + 2 * align_up(8 * ws.n_cap, 256));
    const cudaMemcpyKind k = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    h2d_or_copy(ws, sx, rq.x, 8 * n, k, host, st);
    h2d_or_copy(ws, sy, rq.y, 8 * n, k, host, st);
    if (rq.ids) h2d_or_copy(ws, sid, rq.ids, 4 * n, k, host, st);
    B.in_x = sx;
    B.in_y = sy;
    B.in_id = rq.ids ? sid : nullptr;
  } else {
    B.in_x = rq.x;
    B.in_y = rq.y;
    B.in_id = rq.ids;
  }
  if (timings) CK(cudaEventRecord(ws.ev[1], st));
  B.n = (uint32_t)n;
  B.n_dev = n <= SMALL_N ? n_dev : nullptr;
  const bool ids = B.in_id != nullptr;

  hc.mark("stage");
  // a zeroed control block is the initial state (ST_RUNNING == 0)
  CK(cudaMemsetAsync(B.ctl, 0, sizeof(Ctl), st));
  hc.mark("memset");
  if (g_trace_round) {
    const uint32_t tr = (uint32_t)g_trace_round;
    CK(cudaMemcpyAsync(&B.ctl->tl_round, &tr, sizeof(tr), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }

  if (n <= SMALL_N) {
    // one CTA does K1 + K2 + the round-0 compaction, the round kernel takes
    // over at round 1 with as many CTAs as the live set can use
    const int gr = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 1919) / 1920, ws.rounds_grid));
    B.run_q = (uint32_t)(((n + gr - 1) / gr + 2 + 1) & ~1ull);
    launch_small(B, rq.mode == SH_MODE_WITH_PREPROCESS, ids, st);
    CK(cudaGetLastError());
    CK(launch_rounds(B, gr, st));
    out.launches = 2;
  } else {
  // per-kernel grids: one CTA per SM, at most one per tile
  auto grid_of = [&](int T) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + T - 1) / T, (uint64_t)ws.stream_grid));
  };
  const int g1 = grid_of(Cfg1::T), g2 = grid_of(Cfg2::T), gs = grid_of(Cfg3::T);
  B.k1_grid = (uint32_t)g1;
  B.k2_grid = (uint32_t)g2;
  // K3's CTA j owns run j of the live set: its tiles j, j + gs, ...
  const uint64_t ntiles3 = (n + Cfg3::T - 1) / Cfg3::T;
  // a run holds the CTA's whole input share, or (lean live sets) an even
  // 1/gs of the live capacity -- K3 then checks every append against it
  const uint64_t share = (ntiles3 + gs - 1) / gs * Cfg3::T;  // a K3 CTA's input share
  B.run_q = (uint32_t)std::min<uint64_t>(share, (ws.live_n / gs) & ~1ull);
  const bool capped = B.run_q < share;  // lean live set: K3 checks its appends
  // K1 -> K2 -> K3 -> rounds with programmatic dependent launch: no events
  // between them (per-kernel times come from device %globaltimer marks)
  launch_k1(B, ids, g1, st);
  launch_k2(B, rq.mode == SH_MODE_WITH_PREPROCESS, ids, g2, st);
  launch_k3(B, ids, capped, gs, st);
  CK(cudaGetLastError());
  // the round kernel's CTA j owns run j of each live set: at most gs runs
  CK(launch_rounds(B, std::min(ws.rounds_grid, gs), st));
  out.launches = 4;
  }
  hc.mark("launch");
  if (timings) CK(cudaEventRecord(ws.ev[5], st));
  const bool out_dev = (rq.flags & SH_OUT_DEVICE) != 0;
  if (out_dev && (rq.flags & SH_OUT_PAD)) {
    launch_k5_pack(B, res.x, res.cap, rq.id_base, st);
    CK(cudaGetLastError());
    out.launches += 1;
  } else if (out_dev && (res.x || res.y || res.idx)) {
    launch_k5(B, res.x, res.y, (long long*)res.idx, res.cap, rq.id_base, st);
    CK(cudaGetLastError());
    out.launches += 1;
  }
  // ONE copy: the control block and the first round stats
  CK(cudaMemcpyAsync(ws.h_res, B.ctl, HOST_RES_BYTES, cudaMemcpyDeviceToHost, st));
  const bool want_stats = res.stats && res.stats_cap && !(rq.flags & SH_NO_STATS);
  if (timings) CK(cudaEventRecord(ws.ev[6], st));
  hc.mark("k5+d2h");
  if (!wait) {
    CK(cudaEventRecord(ws.ev[7], st));
    out.code = -2;
    return out;
  }
  CK(cudaStreamSynchronize(st));
  hc.mark("sync");
  hc.print();
  (void)want_stats;
  RunOut parsed = parse_ctl(ws, rq, res);
  parsed.launches = out.launches;
  return parsed;
}

// The control block of a finished call (in ws.h_res) -> RunOut.
RunOut parse_ctl(Workspace& ws, const sh_hull_request& rq, const sh_hull_result& res) {
  RunOut out;
  const uint64_t n = rq.n;
  const Bufs& B = ws.B;
  const bool want_stats = res.stats && res.stats_cap && !(rq.flags & SH_NO_STATS);
  if (want_stats)
    std::memcpy(ws.h_stats, ws.h_res + HOST_RES_STATS,
                sizeof(StatRec) * std::min<uint64_t>(ws.h_ctl->round, STATS_EAGER));

  const Ctl& c = *ws.h_ctl;
  g_last_tl[0] = c.tl_n;
  for (uint32_t i = 0; i < c.tl_n && i < 32; ++i) g_last_tl[i + 1] = c.tl[i];
  if (g_trace_round == 255) {  // debug: the kernel marks instead (t0 = K1 start)
    g_last_tl[0] = 8;
    for (int i = 0; i < 8; ++i) g_last_tl[i + 1] = c.mark[i];
  }
  if (g_trace_round) {
    g_last_ctas.resize(DBG_SLOTS);
    CK(cudaMemcpy(g_last_ctas.data(), B.dbg, sizeof(unsigned long long) * DBG_SLOTS,
                  cudaMemcpyDeviceToHost));
    for (int i = DBG_RAW; i < DBG_SLOTS; ++i)  // raw %globaltimer probes -> since K1 start
      if (g_last_ctas[i]) g_last_ctas[i] -= c.t0_ns;
  }
  out.rounds = c.round;
  out.kept = rq.mode == SH_MODE_WITH_PREPROCESS ? c.kept : n;
  out.bad = c.bad_index;
  switch (c.status) {
    case ST_DONE:
      out.h = c.S_cur;
      break;
    case ST_SINGLE:
      out.h = 1;
      out.kept = n;
      break;
    case ST_COLLINEAR:
      out.h = 2;
      break;
    case ST_NONFINITE:
      out.code = SH_NON_FINITE_INPUT;
      out.msg = "run: non-finite coordinate at index " + std::to_string(c.bad_index);
      break;
    case ST_INTERNAL:
      out.code = SH_INTERNAL_ERROR;
      out.msg = "run: refinement failed to terminate";
      break;
    case ST_OVERFLOW:
      out.code = -1;  // caller regrows the segment tables
      break;
    default:
      out.code = SH_INTERNAL_ERROR;
      out.msg = "run: unexpected device status " + std::to_string(c.status);
  }
  return out;
}

int hull_finish(std::unique_ptr<Workspace>& ws, const sh_hull_request& rqv, sh_hull_result* res,
                cudaStream_t st, bool timings, RunOut o, std::unique_ptr<Workspace>* keep,
                const uint32_t* n_dev, int prev_dev);

// An SH_ASYNC call between sh_b200_hull_ex and sh_b200_hull_wait: its request,
// output description, stream and the workspace it holds.
struct Pending {
  sh_hull_request rq;
  sh_hull_result res;
  cudaStream_t st = nullptr;
  uint32_t launches = 0;
  std::unique_ptr<Workspace> ws;
};
std::unordered_map<uint64_t, std::unique_ptr<Pending>> g_pending;  // under g_mutex
uint64_t g_ticket = 0;

// One hull on one device.  `keep`: on success the workspace is handed back to
// the caller instead of the pool (the multi-GPU path re-packs from its final
// head table when a shard hull outgrew the payload).
// n_dev (internal, the shard merge): the real point count lives on the device
// (<= rq->n, which bounds it and sizes the grids); small inputs only.
int hull_impl(const sh_hull_request* rq, sh_hull_result* res,
              std::unique_ptr<Workspace>* keep = nullptr, const uint32_t* n_dev = nullptr) {
  if (!rq || !res) return SH_INVALID_ARGUMENT;
  res->h = 0;
  res->rounds = 0;
  res->kept = 0;
  res->bad_index = 0;
  res->kernel_launches = 0;
  res->err[0] = 0;
  std::memset(&res->phases, 0, sizeof(res->phases));
  const uint64_t n = rq->n;
  if (n == 0) {
    put_err(res->err, sizeof(res->err), "run: empty point set");
    return SH_EMPTY_INPUT;  // hull.cpp:221
  }
  if (n >= 0xFFFFFFF0ull) {
    put_err(res->err, sizeof(res->err), "run: input too large for 32-bit point ids");
    return SH_INPUT_TOO_LARGE;
  }
  if (!rq->x || !rq->y) return SH_INVALID_ARGUMENT;
  if (rq->mode != SH_MODE_WITH_PREPROCESS && rq->mode != SH_MODE_WITHOUT_PREPROCESS)
    return SH_INVALID_ARGUMENT;
  const bool out_dev = (rq->flags & SH_OUT_DEVICE) != 0;
  const bool pad = (rq->flags & SH_OUT_PAD) != 0;
  if (pad && (!out_dev || !res->x || res->cap == 0)) return SH_INVALID_ARGUMENT;
  std::unique_ptr<Workspace> ws;
  int prev_dev = 0;
  cudaGetDevice(&prev_dev);
  try {
    CK(cudaSetDevice(rq->device));
    ws = acquire(rq->device, n);
    const bool timings = (rq->flags & SH_PHASE_TIMINGS) != 0;
    cudaStream_t st = rq->stream ? (cudaStream_t)rq->stream : ws->stream;
    if (rq->flags & SH_ASYNC) {  // enqueue only; sh_b200_hull_wait finishes
      RunOut o = run_pipeline(*ws, *rq, *res, st, timings, n_dev, false);
      auto pd = std::make_unique<Pending>();
      pd->launches = o.launches;
      pd->rq = *rq;
      pd->res = *res;
      pd->st = st;
      pd->ws = std::move(ws);
      {
        std::lock_guard<std::mutex> lk(g_mutex);
        res->ticket = ++g_ticket;
        g_pending[res->ticket] = std::move(pd);
      }
      cudaSetDevice(prev_dev);
      return SH_OK;
    }
    RunOut o = run_pipeline(*ws, *rq, *res, st, timings, n_dev);
    return hull_finish(ws, *rq, res, st, timings, o, keep, n_dev, prev_dev);
  } catch (const CudaFail& f) {
    put_err(res->err, sizeof(res->err),
            std::string("CUDA error: ") + cudaGetErrorString(f.err) + " at " + f.what);
    cudaGetLastError();
    ws.reset();  // a failed workspace is not returned to the pool
    cudaSetDevice(prev_dev);
    return SH_CUDA_ERROR;
  } catch (const std::bad_alloc&) {
    put_err(res->err, sizeof(res->err), "host allocation failed");
    cudaSetDevice(prev_dev);
    return SH_CUDA_ERROR;
  }
}

// Everything after the pipeline ran: overflow regrow + rerun, outputs, stats,
// timings, workspace back to the pool (or to *keep).
int hull_finish(std::unique_ptr<Workspace>& ws, const sh_hull_request& rqv, sh_hull_result* res,
                cudaStream_t st, bool timings, RunOut o, std::unique_ptr<Workspace>* keep,
                const uint32_t* n_dev, int prev_dev) {
  const sh_hull_request* rq = &rqv;
  const uint64_t n = rq->n;
  const bool out_dev = (rq->flags & SH_OUT_DEVICE) != 0;
  const bool pad = (rq->flags & SH_OUT_PAD) != 0;
  try {
    if (o.code == -1) {  // segment tables or live sets too small: regrow to the worst case, rerun
      const int dev = ws->device;
      const uint64_t cap = std::max<uint64_t>(n, 1u << 12);
      ws.reset();  // synchronises its stream before freeing anything
      ws = make_workspace_retry(dev, cap, cap + 2, cap);
      st = rq->stream ? (cudaStream_t)rq->stream : ws->stream;  // the old pool stream is gone
      o = run_pipeline(*ws, *rq, *res, st, timings, n_dev);
      if (o.code == -1) {
        o.code = SH_INTERNAL_ERROR;
        o.msg = "run: segment table overflow";
      }
    }
    res->rounds = o.rounds;
    res->kept = o.kept;
    res->bad_index = o.bad;
    res->kernel_launches = o.launches;
    std::memset(&res->kernels, 0, sizeof(res->kernels));
    res->h = o.h;
    if (o.code != SH_OK) {
      put_err(res->err, sizeof(res->err), o.msg);
      release(std::move(ws));
      cudaSetDevice(prev_dev);
      return o.code;
    }
    const Ctl& c = *ws->h_ctl;
    if (o.h > res->cap && (res->x || res->y || res->idx)) {
      // (pad mode: the payload already carries the NaN marker with h)
      put_err(res->err, sizeof(res->err), "output capacity too small");
      if (keep) *keep = std::move(ws);
      else release(std::move(ws));
      cudaSetDevice(prev_dev);
      return SH_CAP_TOO_SMALL;
    }
    const bool want_stats = res->stats && res->stats_cap && !(rq->flags & SH_NO_STATS);
    const uint64_t nst =
        want_stats ? std::min<uint64_t>({o.rounds, (uint64_t)STATS_CAP, res->stats_cap}) : 0;
    const uint64_t base = rq->id_base;
    bool sync2 = false;
    std::vector<uint32_t> ids;
    if (pad) {
      // K5-pack wrote the payload block (degenerate hulls included)
    } else if (c.status == ST_DONE) {
      // heads of the final table (CCW from P0); device outputs were written by K5
      const uint32_t par = c.round & 1u;
      if (!out_dev && o.h * 8 >= (H2D_CHUNK >> 2)) {  // a large hull: the pinned ring
        if (res->x) d2h_ring(*ws, res->x, ws->B.Tx[par], o.h, false, 0, st);
        if (res->y) d2h_ring(*ws, res->y, ws->B.Ty[par], o.h, false, 0, st);
        if (res->idx) d2h_ring(*ws, res->idx, ws->B.Tid[par], o.h, true, base, st);
      } else if (!out_dev && o.h) {
        if (res->x) CK(cudaMemcpyAsync(res->x, ws->B.Tx[par], 8 * o.h, cudaMemcpyDeviceToHost, st));
        if (res->y) CK(cudaMemcpyAsync(res->y, ws->B.Ty[par], 8 * o.h, cudaMemcpyDeviceToHost, st));
        if (res->idx) {
          ids.resize(o.h);
          CK(cudaMemcpyAsync(ids.data(), ws->B.Tid[par], 4 * o.h, cudaMemcpyDeviceToHost, st));
        }
        sync2 = true;
      }
    } else {
      // degenerate: {lo} or {lo, hi} (hull.cpp:234-248)
      const int which[2] = {0, 2};
      double vx[2] = {0, 0}, vy[2] = {0, 0};
      int64_t vi[2] = {0, 0};
      for (uint64_t i = 0; i < o.h; ++i) {
        vx[i] = c.ext_x[which[i]];
        vy[i] = c.ext_y[which[i]];
        vi[i] = (int64_t)(c.ext_id[which[i]] + base);
      }
      if (out_dev) {
        if (res->x) CK(cudaMemcpyAsync(res->x, vx, 8 * o.h, cudaMemcpyHostToDevice, st));
        if (res->y) CK(cudaMemcpyAsync(res->y, vy, 8 * o.h, cudaMemcpyHostToDevice, st));
        if (res->idx) CK(cudaMemcpyAsync(res->idx, vi, 8 * o.h, cudaMemcpyHostToDevice, st));
        sync2 = true;
      } else {
        for (uint64_t i = 0; i < o.h; ++i) {
          if (res->x) res->x[i] = vx[i];
          if (res->y) res->y[i] = vy[i];
          if (res->idx) res->idx[i] = vi[i];
        }
      }
    }
    if (nst > (uint64_t)STATS_EAGER) {
      CK(cudaMemcpyAsync(ws->h_stats + STATS_EAGER, ws->B.stats + STATS_EAGER,
                         sizeof(StatRec) * (nst - STATS_EAGER), cudaMemcpyDeviceToHost, st));
      sync2 = true;
    }
    if (sync2) CK(cudaStreamSynchronize(st));
    for (uint64_t i = 0; !out_dev && res->idx && i < ids.size(); ++i)
      res->idx[i] = (int64_t)(ids[i] + base);
    for (uint64_t i = 0; i < nst; ++i) {
      res->stats[i].iteration = i + 1;
      res->stats[i].segments = ws->h_stats[i].segments;
      res->stats[i].points_remaining = ws->h_stats[i].points_remaining;
      res->stats[i].points_removed = ws->h_stats[i].points_removed;
      res->stats[i].end_ns = ws->h_stats[i].end_ns;
      res->stats[i].table_ns = ws->h_stats[i].table_ns;
      res->stats[i].points_ns = ws->h_stats[i].points_ns;
    }
    if (timings) {
      auto el = [&](int i, int j) {
        float v = 0.f;
        CK(cudaEventElapsedTime(&v, ws->ev[i], ws->ev[j]));
        return (double)v;
      };
      // kernel times from the device marks (ns since K1 started); each span
      // runs from the previous kernel's end, so launch gaps are included
      const unsigned long long* mk = c.mark;
      const double k1 = mk[0] * 1e-6, k2 = mk[2] * 1e-6, k3 = mk[4] * 1e-6, kr = mk[6] * 1e-6;
      res->kernels.h2d_ms = el(0, 1);
      res->kernels.extremes_ms = k1;
      res->kernels.filter_ms = k2 > k1 ? k2 - k1 : 0.0;
      res->kernels.first_round_ms = k3 > k2 ? k3 - k2 : 0.0;
      res->kernels.rounds_ms = kr > k3 ? kr - k3 : 0.0;
      res->kernels.d2h_ms = el(5, 6);
      res->phases.pre_ms = k2;
      res->phases.split_ms = res->kernels.first_round_ms;
      res->phases.recurse_ms = res->kernels.rounds_ms;
      res->phases.total_ms = el(0, 6);
    }
    if (keep) *keep = std::move(ws);
    else release(std::move(ws));
    cudaSetDevice(prev_dev);
    return SH_OK;
  } catch (const CudaFail& f) {
    put_err(res->err, sizeof(res->err),
            std::string("CUDA error: ") + cudaGetErrorString(f.err) + " at " + f.what);
    cudaGetLastError();
    ws.reset();  // a failed workspace is not returned to the pool
    cudaSetDevice(prev_dev);
    return SH_CUDA_ERROR;
  } catch (const std::bad_alloc&) {
    put_err(res->err, sizeof(res->err), "host allocation failed");
    cudaSetDevice(prev_dev);
    return SH_CUDA_ERROR;
  }
}

// ---------------------------------------------------------------------------
// Multi-GPU: per-shard hulls -> one payload block per
// shard in the root GPU's memory -> merge hull with global ids.

// Device scratch buffers for gathered payloads, pooled per device.
struct DevBuf {
  int device = 0;
  void* p = nullptr;
  size_t bytes = 0;
};
std::vector<DevBuf> g_bufs;  // free buffers (under g_mutex)

DevBuf take_buf(int device, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    for (size_t i = 0; i < g_bufs.size(); ++i)
      if (g_bufs[i].device == device && g_bufs[i].bytes >= bytes) {
        DevBuf b = g_bufs[i];
        g_bufs.erase(g_bufs.begin() + i);
        return b;
      }
  }
  DevBuf b;
  b.device = device;
  b.bytes = std::max<size_t>(bytes, 1u << 20);
  int cur = 0;
  cudaGetDevice(&cur);
  CK(cudaSetDevice(device));
  const cudaError_t e = cudaMalloc(&b.p, b.bytes);
  cudaSetDevice(cur);
  if (e != cudaSuccess) throw CudaFail{e, "cudaMalloc(gather buffer)"};
  return b;
}

void give_buf(DevBuf b) {
  if (!b.p) return;
  std::lock_guard<std::mutex> lk(g_mutex);
  g_bufs.push_back(b);
  if (g_bufs.size() > 16) {  // bounded: free the oldest
    DevBuf old = g_bufs.front();
    g_bufs.erase(g_bufs.begin());
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(old.device);
    cudaFree(old.p);
    cudaSetDevice(cur);
  }
}

// P2P over NVLink/NVSwitch between `dev` and `root` (both directions); false
// when the pair cannot map each other (the caller then stages + copies).
bool enable_peer(int dev, int root) {
  if (dev == root) return true;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, root) != cudaSuccess || !can) {
    cudaGetLastError();
    return false;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  cudaError_t e = cudaDeviceEnablePeerAccess(root, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
  cudaGetLastError();
  cudaSetDevice(cur);
  return e == cudaSuccess;
}

// The merge: R payload blocks (device memory on `device`) -> hull with
// global ids.  Returns SH_CAP_TOO_SMALL with res->h = the block capacity the
// largest shard hull needs when some block carries the overflow marker.
int gathered_impl(const double* pay, uint32_t R, uint64_t bcap, uint64_t n_total, int mode,
                  uint32_t flags, int device, void* stream, sh_hull_result* res) {
  res->h = 0;
  res->err[0] = 0;
  if (!pay || R == 0 || bcap == 0) return SH_INVALID_ARGUMENT;
  if (n_total >= 0xFFFFFFF0ull) {
    put_err(res->err, sizeof(res->err), "run: input too large for 32-bit point ids");
    return SH_INPUT_TOO_LARGE;
  }
  const uint64_t m = (uint64_t)R * bcap;
  int prev = 0;
  cudaGetDevice(&prev);
  std::unique_ptr<Workspace> ws;
  try {
    CK(cudaSetDevice(device));
    ws = acquire(device, m);
    ensure_stage(*ws, true);
    cudaStream_t st = stream ? (cudaStream_t)stream : ws->stream;
    double* sx = (double*)ws->stage;
    double* sy = (double*)((char*)ws->stage + align_up(8 * ws->n_cap, 256));
    uint32_t* sid = (uint32_t*)((char*)ws->stage + 2 * align_up(8 * ws->n_cap, 256));
    // per-block counts in the workspace's scan scratch (2 MAX_ROUND_BLOCKS words)
    if (R + 1 > 2u * MAX_ROUND_BLOCKS) throw CudaFail{cudaErrorInvalidValue, "more than 2047 blocks"};
    uint32_t* cnt = ws->B.blk_cnt;
    launch_unpack(pay, R, bcap, cnt, sx, sy, sid, st);
    CK(cudaGetLastError());
    // the merge input is the real vertices only; their count stays on the
    // device for the one-CTA small path (no read-back), else it is read back
    uint32_t mreal = (uint32_t)m;
    const uint32_t* n_dev = nullptr;
    if (m <= SMALL_N) {
      n_dev = cnt + R;
    } else {
      CK(cudaMemcpyAsync(ws->h_res, cnt + R, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::memcpy(&mreal, ws->h_res, sizeof(mreal));
    }
    sh_hull_request rq;
    std::memset(&rq, 0, sizeof(rq));
    rq.x = sx;
    rq.y = sy;
    rq.ids = sid;
    rq.n = mreal;
    rq.mode = mode;
    rq.flags = SH_DEVICE_PTRS | (flags & (SH_OUT_DEVICE | SH_NO_STATS | SH_PHASE_TIMINGS));
    rq.device = device;
    rq.stream = st;
    // the staging arrays stay ours until the merge has read them
    std::unique_ptr<Workspace> hold = std::move(ws);
    int rc = hull_impl(&rq, res, nullptr, n_dev);
    if (rc == SH_NON_FINITE_INPUT) {  // a NaN marker: which block, what it needs
      uint64_t need = 0;
      for (uint32_t b = 0; b < R; ++b) {
        double x0 = 0;
        long long h = 0;
        CK(cudaMemcpy(&x0, pay + (uint64_t)b * 3 * bcap, 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&h, pay + (uint64_t)b * 3 * bcap + 2 * bcap, 8, cudaMemcpyDeviceToHost));
        if (std::isnan(x0) && h > 0) need = std::max<uint64_t>(need, (uint64_t)h);
      }
      if (need) {
        res->h = need;
        put_err(res->err, sizeof(res->err), "shard hull exceeds the payload block capacity");
        rc = SH_CAP_TOO_SMALL;
      }
    }
    release(std::move(hold));
    cudaSetDevice(prev);
    return rc;
  } catch (const CudaFail& f) {
    put_err(res->err, sizeof(res->err),
            std::string("CUDA error: ") + cudaGetErrorString(f.err) + " at " + f.what);
    cudaGetLastError();
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  }
}

constexpr uint64_t PAYLOAD_CAP = 2048;  // shard-hull vertices per block in the first pass

int shards_impl(const sh_shard* sh, int nsh, int mode, uint32_t flags, int root, int64_t* out_idx,
                double* out_x, double* out_y, uint64_t cap, uint64_t* out_h, sh_multi_ms* tm,
                char* err, size_t errlen) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (out_h) *out_h = 0;
  if (tm) std::memset(tm, 0, sizeof(*tm));
  if (!sh || nsh <= 0) return SH_INVALID_ARGUMENT;
  if (mode != SH_MODE_WITH_PREPROCESS && mode != SH_MODE_WITHOUT_PREPROCESS)
    return SH_INVALID_ARGUMENT;
  uint64_t n_total = 0;
  std::vector<int> live;  // non-empty shards, in order
  for (int g = 0; g < nsh; ++g) {
    if (sh[g].n == 0) continue;
    if (!sh[g].x || !sh[g].y) return SH_INVALID_ARGUMENT;
    live.push_back(g);
    n_total = std::max<uint64_t>(n_total, sh[g].first + sh[g].n);
  }
  if (live.empty()) {
    put_err(err, errlen, "run: empty point set");
    return SH_EMPTY_INPUT;  // hull.cpp:221
  }
  if (n_total >= 0xFFFFFFF0ull) {
    put_err(err, errlen, "run: input too large for 32-bit point ids");
    return SH_INPUT_TOO_LARGE;
  }
  const uint32_t R = (uint32_t)live.size();
  int prev = 0;
  cudaGetDevice(&prev);
  DevBuf pay;
  std::vector<std::unique_ptr<Workspace>> kept(R);
  try {
    uint64_t bcap = PAYLOAD_CAP;
    pay = take_buf(root, 24 * bcap * R);
    std::vector<int> code(R, SH_OK);
    std::vector<sh_hull_result> rs(R);
    std::vector<DevBuf> local(R);  // staging blocks of shards without P2P to the root
    std::vector<char> p2p(R, 0);
    for (uint32_t r = 0; r < R; ++r) p2p[r] = enable_peer(sh[live[r]].device, root);
    auto block = [&](uint32_t r) { return (double*)pay.p + (uint64_t)r * 3 * bcap; };
    auto run_shard = [&](uint32_t r) {
      const sh_shard& s = sh[live[r]];
      sh_hull_request rq;
      std::memset(&rq, 0, sizeof(rq));
      rq.x = s.x;
      rq.y = s.y;
      rq.n = s.n;
      rq.mode = mode;
      rq.flags = (flags & SH_DEVICE_PTRS) | SH_OUT_DEVICE | SH_OUT_PAD | SH_NO_STATS;
      rq.device = s.device;
      rq.id_base = s.first;
      sh_hull_result& res = rs[r];
      std::memset(&res, 0, sizeof(res));
      try {
        if (!p2p[r]) local[r] = take_buf(s.device, 24 * bcap);
      } catch (const CudaFail&) {
        code[r] = SH_CUDA_ERROR;
        return;
      }
      res.x = p2p[r] ? block(r) : (double*)local[r].p;
      res.cap = bcap;
      code[r] = hull_impl(&rq, &res, &kept[r]);
    };
    {
      std::vector<std::thread> th;
      for (uint32_t r = 1; r < R; ++r) th.emplace_back(run_shard, r);
      run_shard(0);
      for (auto& t : th) t.join();
    }
    const auto t1 = clk::now();
    // errors in shard order: the first non-finite shard holds the global first index
    for (uint32_t r = 0; r < R; ++r) {
      if (code[r] == SH_OK || code[r] == SH_CAP_TOO_SMALL) continue;
      std::string m = rs[r].err;
      if (code[r] == SH_NON_FINITE_INPUT)
        m = "run: non-finite coordinate at index " + std::to_string(rs[r].bad_index + sh[live[r]].first);
      put_err(err, errlen, m);
      for (auto& w : kept)
        if (w) release(std::move(w));
      for (auto& b : local) give_buf(b);
      give_buf(pay);
      cudaSetDevice(prev);
      return code[r];
    }
    uint64_t need = 0;
    for (uint32_t r = 0; r < R; ++r)
      if (code[r] == SH_CAP_TOO_SMALL) need = std::max<uint64_t>(need, rs[r].h);
    if (need) {  // second pass: re-pack every shard from its retained head table
      give_buf(pay);
      bcap = need;
      pay = take_buf(root, 24 * bcap * R);
      for (uint32_t r = 0; r < R; ++r) {
        give_buf(local[r]);
        local[r] = DevBuf{};
        CK(cudaSetDevice(kept[r]->device));
        if (!p2p[r]) local[r] = take_buf(kept[r]->device, 24 * bcap);
        launch_k5_pack(kept[r]->B, p2p[r] ? block(r) : (double*)local[r].p, bcap, sh[live[r]].first,
                       kept[r]->stream);
        CK(cudaGetLastError());
      }
    }
    for (uint32_t r = 0; r < R; ++r) {  // shards without P2P: one peer copy each
      if (p2p[r]) continue;
      CK(cudaSetDevice(kept[r]->device));
      CK(cudaMemcpyPeerAsync(block(r), root, local[r].p, kept[r]->device, 24 * bcap,
                             kept[r]->stream));
    }
    for (uint32_t r = 0; r < R; ++r) {
      CK(cudaSetDevice(kept[r]->device));
      CK(cudaStreamSynchronize(kept[r]->stream));
    }
    for (auto& w : kept) release(std::move(w));
    for (auto& b : local) give_buf(b);
    const auto t2 = clk::now();
    sh_hull_result res;
    std::memset(&res, 0, sizeof(res));
    res.x = out_x;
    res.y = out_y;
    res.idx = out_idx;
    res.cap = cap;
    const int rc = gathered_impl((const double*)pay.p, R, bcap, n_total, mode,
                                 (flags & SH_OUT_DEVICE) | SH_NO_STATS, root, nullptr, &res);
    give_buf(pay);
    const auto t3 = clk::now();
    if (out_h) *out_h = res.h;
    put_err(err, errlen, res.err);
    if (tm) {
      auto ms = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
      };
      tm->shards_ms = ms(t0, t1);
      tm->gather_ms = ms(t1, t2);
      tm->merge_ms = ms(t2, t3);
      tm->total_ms = ms(t0, t3);
      tm->shards = R;
      tm->block_cap = bcap;
    }
    cudaSetDevice(prev);
    return rc;
  } catch (const CudaFail& f) {
    put_err(err, errlen, std::string("CUDA error: ") + cudaGetErrorString(f.err) + " at " + f.what);
    cudaGetLastError();
    for (auto& w : kept) w.reset();
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  }
}

}  // namespace

extern "C" {

int sh_b200_abi_version(void) { return SH_B200_ABI_VERSION; }

// Debug aid (not part of include/seghull_b200.h): trace CTA 0's tile waits
// in round `r` of subsequent calls; read them back after a call.
void sh_b200_debug_trace_round(int r) { g_trace_round = r; }
int sh_b200_debug_last_ctas(unsigned long long* out, int cap) {
  const int n = (int)g_last_ctas.size();
  for (int i = 0; i < n && i < cap; ++i) out[i] = g_last_ctas[i];
  return n;
}
int sh_b200_debug_last_timeline(unsigned long long* out, int cap) {
  const int n = (int)g_last_tl[0];
  for (int i = 0; i < n && i < cap; ++i) out[i] = g_last_tl[i + 1];
  return n;
}

int sh_b200_hull_ex(const sh_hull_request* req, sh_hull_result* res) {
  if (req && (req->flags & SH_ASYNC) && !(req->flags & SH_DEVICE_PTRS)) return SH_INVALID_ARGUMENT;
  if (res) res->ticket = 0;
  return hull_impl(req, res);
}

int sh_b200_hull_wait(uint64_t ticket, sh_hull_result* res) {
  if (!res) return SH_INVALID_ARGUMENT;
  std::unique_ptr<Pending> pd;
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    auto it = g_pending.find(ticket);
    if (it == g_pending.end()) return SH_INVALID_ARGUMENT;
    pd = std::move(it->second);
    g_pending.erase(it);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  // the caller's stats buffer may be given here (the ticket keeps its outputs)
  sh_hull_result r = pd->res;
  r.stats = res->stats ? res->stats : r.stats;
  r.stats_cap = res->stats ? res->stats_cap : r.stats_cap;
  r.err[0] = 0;
  try {
    CK(cudaSetDevice(pd->rq.device));
    CK(cudaEventSynchronize(pd->ws->ev[7]));
    const bool timings = (pd->rq.flags & SH_PHASE_TIMINGS) != 0;
    RunOut o = parse_ctl(*pd->ws, pd->rq, r);
    o.launches = pd->launches;
    const int rc = hull_finish(pd->ws, pd->rq, &r, pd->st, timings, o, nullptr, nullptr, prev);
    r.ticket = ticket;
    *res = r;
    return rc;
  } catch (const CudaFail& f) {
    put_err(res->err, sizeof(res->err),
            std::string("CUDA error: ") + cudaGetErrorString(f.err) + " at " + f.what);
    cudaGetLastError();
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  }
}

int sh_b200_hull_shards(const sh_shard* shards, int nshards, int mode, uint32_t flags,
                        int root_device, int64_t* out_idx, double* out_x, double* out_y,
                        uint64_t cap, uint64_t* out_h, sh_multi_ms* times, char* err,
                        size_t errlen) {
  return shards_impl(shards, nshards, mode, flags, root_device, out_idx, out_x, out_y, cap, out_h,
                     times, err, errlen);
}

int sh_b200_hull_multi(const double* x, const double* y, uint64_t n, int mode, uint32_t flags,
                       const int* devices, int ndev, int64_t* out_idx, double* out_x,
                       double* out_y, uint64_t cap, uint64_t* out_h, sh_multi_ms* times,
                       char* err, size_t errlen) {
  if (out_h) *out_h = 0;
  if (n == 0) {
    put_err(err, errlen, "run: empty point set");
    return SH_EMPTY_INPUT;
  }
  if (!x || !y || !devices || ndev <= 0 || (flags & SH_DEVICE_PTRS)) return SH_INVALID_ARGUMENT;
  std::vector<sh_shard> sh(ndev);
  for (int g = 0; g < ndev; ++g) {  // contiguous shards [g n / ndev, (g + 1) n / ndev)
    const uint64_t b = n * g / ndev, e = n * (g + 1) / ndev;
    sh[g].device = devices[g];
    sh[g].x = x + b;
    sh[g].y = y + b;
    sh[g].n = e - b;
    sh[g].first = b;
  }
  return shards_impl(sh.data(), ndev, mode, flags & ~(uint32_t)SH_DEVICE_PTRS, devices[0], out_idx,
                     out_x, out_y, cap, out_h, times, err, errlen);
}

int sh_b200_hull_gathered(const double* payload, uint32_t nblocks, uint64_t block_cap,
                          uint64_t n_total, int mode, uint32_t flags, int device, void* stream,
                          int64_t* out_idx, double* out_x, double* out_y, uint64_t cap,
                          uint64_t* out_h, char* err, size_t errlen) {
  sh_hull_result res;
  std::memset(&res, 0, sizeof(res));
  res.x = out_x;
  res.y = out_y;
  res.idx = out_idx;
  res.cap = cap;
  const int rc = gathered_impl(payload, nblocks, block_cap, n_total, mode, flags | SH_NO_STATS,
                               device, stream, &res);
  if (out_h) *out_h = res.h;
  put_err(err, errlen, res.err);
  return rc;
}

int sh_b200_hull(const double* x, const double* y, uint64_t n, int mode, uint32_t flags,
                 int device, int64_t* out_idx, double* out_x, double* out_y, uint64_t cap,
                 uint64_t* out_h, sh_round_stat* stats, uint64_t stats_cap,
                 uint64_t* out_rounds, sh_phase_ms* phases, char* err, size_t errlen) {
  sh_hull_request rq;
  std::memset(&rq, 0, sizeof(rq));
  rq.x = x;
  rq.y = y;
  rq.n = n;
  rq.mode = mode;
  rq.flags = flags;
  rq.device = device;
  sh_hull_result res;
  std::memset(&res, 0, sizeof(res));
  res.idx = out_idx;
  res.x = out_x;
  res.y = out_y;
  res.cap = cap;
  res.stats = stats;
  res.stats_cap = stats_cap;
  const int rc = hull_impl(&rq, &res);
  if (out_h) *out_h = res.h;
  if (out_rounds) *out_rounds = res.rounds;
  if (phases) *phases = res.phases;
  put_err(err, errlen, res.err);
  return rc;
}

int sh_b200_gen_uniform(double* x, double* y, uint64_t first, uint64_t count, uint64_t seed,
                        int device, void* stream) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return SH_CUDA_ERROR;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((count + 255) / 256, (uint64_t)sms * 16));
  launch_gen_uniform(x, y, first, count, seed, grid, (cudaStream_t)stream);
  const cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  return e == cudaSuccess ? SH_OK : SH_CUDA_ERROR;
}

int sh_b200_gen_disk(double* x, double* y, uint64_t n, uint64_t seed, int device, void* stream) {
  if (n == 0) return SH_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  std::unique_ptr<Workspace> ws;
  try {
    CK(cudaSetDevice(device));
    ws = acquire(device, n);
    cudaStream_t st = stream ? (cudaStream_t)stream : ws->stream;
    Ctl init;
    std::memset(&init, 0, sizeof(init));
    *ws->h_ctl = init;
    CK(cudaMemcpyAsync(ws->B.ctl, ws->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    uint64_t accepted = 0, cand0 = 0;
    const uint64_t max_batch = (uint64_t)(ws->tiles_cap - 64) * gen_tile_points();
    while (accepted < n) {
      const uint64_t need = n - accepted;
      uint64_t batch = need + need / 4 + 4096;
      batch = std::min<uint64_t>(batch, max_batch);
      launch_gen_disk(x, y, n, seed, cand0, (uint32_t)batch, accepted, ws->B.ctl,
                      ws->B.tile_status, ws->epoch, ws->stream_grid, st);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(ws->h_ctl, ws->B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      accepted += ws->h_ctl->m_next;
      cand0 += batch;
    }
    release(std::move(ws));
    cudaSetDevice(prev);
    return SH_OK;
  } catch (const CudaFail&) {
    cudaGetLastError();
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  }
}

int sh_b200_preprocess(const double* x, const double* y, uint64_t n, int device, void* stream,
                       double* out_x, double* out_y, uint64_t cap, uint64_t* kept,
                       uint64_t* discarded, char* err, size_t errlen) {
  if (kept) *kept = 0;
  if (discarded) *discarded = 0;
  if (n == 0) {  // hull.cpp:55
    put_err(err, errlen, "preprocess: empty point set");
    return SH_EMPTY_INPUT;
  }
  if (!x || !y || !kept) {
    put_err(err, errlen, "null argument");
    return SH_INVALID_ARGUMENT;
  }
  if (n >= (1ull << 32) - (1ull << 20)) {
    put_err(err, errlen, "preprocess: more than 2^32 - 2^20 points");
    return SH_INPUT_TOO_LARGE;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  std::unique_ptr<Workspace> ws;
  try {
    CK(cudaSetDevice(device));
    ws = acquire(device, n);
    cudaStream_t st = stream ? (cudaStream_t)stream : ws->stream;
    Bufs B = ws->B;
    // K1's bulk copies need 16-byte aligned inputs: stage unaligned ones
    if ((uintptr_t)x % 16 || (uintptr_t)y % 16) {
      ensure_stage(*ws, false);
      B = ws->B;
      double* sx = (double*)ws->stage;
      double* sy = (double*)((char*)ws->stage + align_up(8 * ws->n_cap, 256));
      CK(cudaMemcpyAsync(sx, x, 8 * n, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(sy, y, 8 * n, cudaMemcpyDeviceToDevice, st));
      B.in_x = sx;
      B.in_y = sy;
    } else {
      B.in_x = x;
      B.in_y = y;
    }
    B.in_id = nullptr;
    B.n = (uint32_t)n;
    const int g1 = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + Cfg1::T - 1) / Cfg1::T,
                                                                 (uint64_t)ws->stream_grid));
    B.k1_grid = (uint32_t)g1;
    CK(cudaMemsetAsync(B.ctl, 0, sizeof(Ctl), st));
    launch_k1(B, false, g1, st);
    launch_preprocess(B, out_x, out_y, out_x && out_y ? cap : 0, ws->stream_grid * 8, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ws->h_ctl, B.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const Ctl& c = *ws->h_ctl;
    int rc = SH_OK;
    if (c.status == ST_NONFINITE) {
      put_err(err, errlen, "preprocess: non-finite coordinate at index " + std::to_string(c.bad_index));
      rc = SH_NON_FINITE_INPUT;
    } else {
      *kept = c.m_next;
      if (discarded) *discarded = n - c.m_next;
      if ((out_x || out_y) && c.m_next > cap) {
        put_err(err, errlen, "output capacity too small");
        rc = SH_CAP_TOO_SMALL;
      }
    }
    release(std::move(ws));
    cudaSetDevice(prev);
    return rc;
  } catch (const CudaFail& f) {
    put_err(err, errlen, std::string(f.what) + ": " + cudaGetErrorString(f.err));
    cudaGetLastError();
    cudaSetDevice(prev);
    return SH_CUDA_ERROR;
  }
}

int sh_b200_gen_circle_host(double* x, double* y, uint64_t n, uint64_t seed) {
  uint64_t state = seed;
  const double two_pi = 2.0 * 3.141592653589793;  // std::numbers::pi
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double angle = two_pi * ((double)(z >> 11) * 0x1.0p-53);
    x[i] = std::cos(angle);
    y[i] = std::sin(angle);
  }
  return SH_OK;
}

int sh_b200_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                        uint64_t* hbm_bytes, char* name, size_t namelen) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) {
    cudaGetLastError();
    return SH_CUDA_ERROR;
  }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (hbm_bytes) *hbm_bytes = p.totalGlobalMem;
  if (name && namelen) std::snprintf(name, namelen, "%s", p.name);
  return SH_OK;
}

void sh_b200_release_pool(void) {
  std::lock_guard<std::mutex> lk(g_mutex);
  g_pool.clear();
}

}  // extern "C"
