// hull_kernels.cuh -- data layout shared by the host orchestration and the
// sm_100a kernels of the segment-based QuickHull.
//
// HBM layout (SoA everywhere, per workspace):
//   input        x[n], y[n] f64 (+ optional ids[n] u32)
//   chain bits   lo[ceil(n/32)], up[ceil(n/32)] u32: K2's per-point class
//   live set L   ping-pong {x f64, y f64, id u32, seg u32}[n]   24 B/point
//   segment tbl  ping-pong heads {x f64, y f64, id u32}[S]        20 B/segment
//   farthest     ping-pong slots {dbits u64, win u32}[S]         12 B/segment
//   route tbl    Route[S] 64 B: the (A, C, B) triangle of each old segment
//   tile status  u64[tiles] for the decoupled look-back scans
#pragma once

#include <cstdint>

namespace shb {

constexpr int TPB = 256;           // threads per block of the streaming kernels
constexpr int WARPS = TPB / 32;
constexpr int ITEMS = 8;           // points per thread per tile
constexpr int TILE = TPB * ITEMS;  // 2048 points per tile
constexpr int NSLOT = 1024;        // per-block shared-memory farthest slots
constexpr uint32_t SMALL_S = 4096; // segment tables up to this size are built by one block
constexpr int STATS_CAP = 1 << 16;

enum Status : uint32_t {
  ST_RUNNING = 0,
  ST_DONE = 1,
  ST_SINGLE = 2,      // lo == hi  (hull.cpp:234-237)
  ST_COLLINEAR = 3,   // all cross(lo,hi,p) == 0 (hull.cpp:238-248)
  ST_NONFINITE = 4,   // hull.cpp:222-227
  ST_INTERNAL = 5,    // refinement failed to terminate (hull.cpp:265-267)
  ST_OVERFLOW = 6     // segment table capacity exceeded (host regrows, reruns)
};

struct ExtRec {
  double x, y;
  uint32_t id, pos;
};

struct K1Partial {
  ExtRec e[4];  // left, bottom, right, top
  unsigned long long bad;
};

// 64-byte route entry of an old segment s: head A, next head B, farthest C.
struct __align__(16) Route {
  double ax, ay, cx, cy, bx, by;
  uint32_t cid;    // id of C (it becomes a head and leaves the member set)
  uint32_t ns;     // index of s in the next segment table
  uint32_t flags;  // RT_SPLIT | RT_LOWER
  uint32_t pad;
};
constexpr uint32_t RT_SPLIT = 1u, RT_LOWER = 2u;

struct StatRec {
  uint32_t segments, points_remaining, points_removed, pad;
};

// Device-resident control block: all round bookkeeping lives here so the
// host never has to read anything between rounds.
struct Ctl {
  uint32_t status;
  uint32_t parity;      // which ping-pong half is current
  uint32_t round;       // refinement rounds completed
  uint32_t table_ready; // route table for the next round already built
  unsigned long long bad_index;
  // extremes: left, bottom, right, top (K1)
  double ext_x[4], ext_y[4];
  uint32_t ext_id[4], ext_pos[4];
  int distinct, nedges;
  double edges[4][4];   // hoisted (ax, ay, ex, ey) of the quadrilateral edges
  // K2
  unsigned long long kept;
  uint32_t noncollinear;
  // rounds
  uint32_t S_cur, Slo_cur, m_cur;
  uint32_t S_next, Slo_next, m_next;
  // tickets
  uint32_t ticket, tile_ctr;
  uint32_t n;
  uint32_t s_cap;
  uint32_t mode;
  uint32_t pad0;
};

struct Bufs {
  // input
  const double* in_x;
  const double* in_y;
  const uint32_t* in_id;  // may be null: id == position
  uint32_t n;
  uint32_t s_cap;
  // control
  Ctl* ctl;
  uint32_t* epoch;        // persistent launch-epoch counter (never reset)
  K1Partial* k1part;
  StatRec* stats;
  unsigned long long* tile_status;
  // classification bits
  uint32_t* bits_lo;
  uint32_t* bits_up;
  // live set
  double* Lx[2];
  double* Ly[2];
  uint32_t* Lid[2];
  uint32_t* Lseg[2];
  // segment tables
  double* Tx[2];
  double* Ty[2];
  uint32_t* Tid[2];
  unsigned long long* Sd[2];
  uint32_t* Sw[2];
  Route* route;
  // output
  double* out_x;
  double* out_y;
  uint32_t* out_id;
};

}  // namespace shb
