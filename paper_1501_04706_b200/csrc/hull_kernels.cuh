// hull_kernels.cuh -- data layout shared by the host orchestration and the
// sm_100a kernels of the segment-based QuickHull.
//
// HBM layout (per workspace):
//   input        x[n], y[n] f64 SoA (caller's, or the H2D staging copy)
//                (+ optional ids[n] u32 -- global ids of a shard-merge input)
//   chain bits   uint4[ceil(n/64)]: K2's per-point class for one 64-point
//                chunk {lower even, lower odd, upper even, upper odd}; bit l of
//                word "even" is point 64c+2l, of "odd" point 64c+2l+1
//   live set     ping-pong {xy double2, (id, seg) uint2}[cap]    24 B/point,
//                organised as RUNS: run j occupies [j*run_q, j*run_q + cnt_j);
//                CTA j of a round writes its survivors densely into run j
//                (CTA-local offsets, no global atomics), run_cnt[par][j] = cnt_j;
//                an odd run is padded with one dead entry (seg = NONE) so
//                every run can be fetched with 16-byte bulk copies
//   head table   ping-pong {x f64, y f64, id u32}[S]              20 B/segment
//   farthest     3-way rotating slots {dbits u64, SlotRec 32 B}[S] 40 B/segment
//   route table  Route[S] 64 B (large tables only; small ones live in smem)
//
// Round numbering follows hull.cpp:264-282: round r >= 1 splits the
// segments of round r-1 at their farthest points, routes every member to
// the A->C or C->B edge and drops the interior ones.  "Round 0" is K2 (the
// first split + the round-1 farthest points).
//   round r reads  heads Tab[(r-1)&1], farthest slots Slot[(r-1)%3],
//                  live set Live[(r-1)&1] (round 1: the input)
//   round r writes heads Tab[r&1], slots Slot[r%3] (next round's farthest
//                  points), live set Live[r&1] + its run counts
//   round r clears Slot[(r+1)%3] for round r+1
// so no buffer is ever cleared while another CTA may still read it.
#pragma once

#include <cstdint>

namespace shb {

constexpr int TPB = 256;             // K1 / K2 / K3 (streaming kernels)
constexpr int WARPS = TPB / 32;
#ifndef SHB_RTPB
#define SHB_RTPB 512
#endif
constexpr int RTPB = SHB_RTPB;       // persistent round kernel
// TMA-fed streaming kernels K1/K2/K3: one CTA per SM, warp CW is the TMA
// producer, warps 0..CW-1 consume CH 64-point chunks each per tile.
template <int TPB_, int CH_, int NS_>
struct StreamCfg {
  static constexpr int TPB = TPB_;
  static constexpr int WARPS = TPB / 32;
  static constexpr int CW = WARPS - 1;     // consumer warps
  static constexpr int CT = 32 * CW;       // consumer threads
  static constexpr int CH = CH_;           // chunks per consumer warp per tile
  static constexpr int T = 64 * CW * CH;   // points per tile
  static constexpr int NS = NS_;           // ring stages
};
#ifndef SHB_K1_TPB
#define SHB_K1_TPB 512
#endif
#ifndef SHB_K1_CH
#define SHB_K1_CH 2
#endif
#ifndef SHB_K1_NS
#define SHB_K1_NS 4
#endif
#ifndef SHB_K2_TPB
#define SHB_K2_TPB 768
#endif
#ifndef SHB_K2_CH
#define SHB_K2_CH 2
#endif
#ifndef SHB_K2_NS
#define SHB_K2_NS 3
#endif
#ifndef SHB_K3_TPB
#define SHB_K3_TPB 1024
#endif
#ifndef SHB_K3_CH
#define SHB_K3_CH 1
#endif
#ifndef SHB_K3_NS
#define SHB_K3_NS 4
#endif
using Cfg1 = StreamCfg<SHB_K1_TPB, SHB_K1_CH, SHB_K1_NS>;  // K1 extremes: memory-bound, light consumer
using Cfg2 = StreamCfg<SHB_K2_TPB, SHB_K2_CH, SHB_K2_NS>;  // K2 filter: FP64-heavy consumer
using Cfg3 = StreamCfg<SHB_K3_TPB, SHB_K3_CH, SHB_K3_NS>;  // K3 round 1: <= 64 registers at 1024 threads
constexpr int SMALL_S = 512;         // tables up to this size are rebuilt per CTA in smem
constexpr int NSLOT = 2 * SMALL_S;   // next-round segments of a small table
constexpr uint32_t TAIL_M = 4096;    // live sets up to this size finish in one CTA
constexpr int STATS_CAP = 1 << 16;
constexpr int STATS_EAGER = 64;      // stats read back together with the control block
constexpr int MAX_ROUND_BLOCKS = 1024;
// debug probes (Ctl::tl_round == 255): Bufs::dbg[DBG_SLOTS]; [0, 1024) relative
// times written by the kernels, [DBG_RAW, DBG_SLOTS) raw %globaltimer values:
//   1024 + b K1 CTA end | 1200 + b K2 CTA end | 1400 + b K3 CTA stream end (all warps)
//   1600/1601 K2 CTA 0 entry / past griddepcontrol.wait, 1602/1603 K3, 1604/1605 KR
constexpr int DBG_SLOTS = 2048, DBG_RAW = 1024;
constexpr int MAX_RUNS = MAX_ROUND_BLOCKS;
constexpr int RCWARPS = RTPB / 32 - 1;  // round kernel: consumer warps (+ 1 producer warp)
constexpr int RCTHREADS = 32 * RCWARPS;
#ifndef SHB_LIVE_U
#define SHB_LIVE_U 3
#endif
#ifndef SHB_LIVE_NS
#define SHB_LIVE_NS 4
#endif
constexpr int LIVE_T = SHB_LIVE_U * RCTHREADS;  // live points per TMA tile of the round kernel (1440)
constexpr int LIVE_NS = SHB_LIVE_NS;            // its ring stages
constexpr int MAXW = 32;             // warps per CTA upper bound (shared scratch arrays)
constexpr uint32_t SMALL_N = 16384;  // inputs up to this size take the one-CTA path (k_small_pre)

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

// farthest-point candidate (distance d of point (x, y), id, input index)
struct Cand {
  double d, x, y;
  uint32_t id, pos;
};

// K2's per-CTA result, combined by every CTA of K3
struct K2Partial {
  Cand a[2];                // farthest candidate of the lower / upper chain
  unsigned long long kept;  // points surviving the quadrilateral filter
  uint32_t noncol, pad;     // some point off the line P0 -> Pr
};

// 64-byte route entry of an old segment s: head A, farthest point C, next
// head B (hull.cpp:186-201 restated per segment).
struct __align__(16) Route {
  double ax, ay, cx, cy, bx, by;
  uint32_t cid;    // id of C (it becomes a head and leaves the member set)
  uint32_t ns;     // index of s in the next head table
  uint32_t flags;  // RT_SPLIT | RT_LOWER
  uint32_t pad;
};
constexpr uint32_t RT_SPLIT = 1u, RT_LOWER = 2u;

// Farthest-point record of one segment slot: the best candidate so far
// under the full comparator (d, then chain-lex, then id).  Updated under
// `lock` by the rare contenders that reach the slot's running maximum
// distance (dbits); C's coordinates are read straight from here by the next
// round's table phase.
struct __align__(16) SlotRec {
  double d, x, y;
  uint32_t id;    // NONE: no candidate (segment not splittable)
  uint32_t lock;
};

// Farthest-point contender of a large-table round: a survivor whose
// atomicMax on its new segment's distance bits returned a value <= its own.
struct __align__(16) LiveCand {
  double d;
  uint32_t pos;  // position in the live set just written
  uint32_t seg;  // new segment
};

struct StatRec {
  uint32_t segments, points_remaining, points_removed, pad;
  unsigned long long end_ns;     // %globaltimer at the end of the round (minus Ctl::t0_ns)
  unsigned long long table_ns;   // ... when CTA 0 finished the segment-table phase
  unsigned long long points_ns;  // ... when CTA 0 finished its point phase
};

// Device-resident control block.  The host writes it once per call and
// reads it once at the end; all round bookkeeping stays on the device.
struct __align__(16) Ctl {
  uint32_t status;
  uint32_t round;       // refinement rounds completed
  uint32_t S_cur;       // segments after `round`
  uint32_t Slo_cur;     // of which lower-chain segments
  uint32_t m_cur;       // live members after `round`
  uint32_t n;
  unsigned long long bad_index;
  // extremes: left, bottom, right, top (K1)
  double ext_x[4], ext_y[4];
  uint32_t ext_id[4], ext_pos[4];
  int distinct, nedges;
  double edges[4][4];   // hoisted (ax, ay, ex, ey) of the quadrilateral edges
  unsigned long long kept;
  uint32_t noncollinear;
  uint32_t ticket;      // last-CTA ticket of K1 / K2 / K3
  uint32_t nruns;       // runs of the live set after `round`
  uint32_t bar_count;   // grid barrier of the round kernel
  uint32_t bar_gen;
  uint32_t mode;
  uint32_t tile_ctr;    // generator scratch
  uint32_t m_next;      // generator scratch
  unsigned long long t0_ns;  // %globaltimer when K1 started (per-round timestamps)
  unsigned long long mark[8]; // device times (ns since t0): K1 end, K2 start/end, K3 start/end, KR start/end
  unsigned long long tl[32]; // debug timeline of CTA 0 (sh_b200_last_timeline)
  unsigned long long bar_ctr; // round kernel: arrivals at its grid barriers (never reset in a call)
  uint32_t tl_round;         // round whose tiles are traced (0: none)
  uint32_t tl_n;
};

struct Bufs {
  // input
  const double* in_x;
  const double* in_y;
  const uint32_t* in_id;  // may be null: id == position
  uint32_t n;
  const uint32_t* n_dev;  // small path only, may be null: the real point count is
                          // *n_dev <= n, written on the device by an earlier kernel
  uint32_t s_cap;
  // control
  Ctl* ctl;
  uint32_t* epoch;        // launch-epoch counter of the generator's look-back scan
  K1Partial* k1part;
  K2Partial* k2part;
  uint32_t k1_grid, k2_grid;  // CTAs of K1 / K2 (partials to combine)
  StatRec* stats;
  unsigned long long* tile_status;
  uint32_t* blk_cnt;      // [2 * MAX_ROUND_BLOCKS] per-CTA counts of a large table scan
  unsigned long long* dbg;  // [DBG_SLOTS] debug probes (see DBG_SLOTS)
  // classification bits
  uint4* bits;
  // live set (runs)
  double2* Lxy[2];
  uint2* Lis[2];          // (id, segment)
  uint32_t* run_cnt[2];   // [MAX_RUNS] survivors per run
  uint32_t run_q;         // run stride in points
  // head tables
  double* Tx[2];
  double* Ty[2];
  uint32_t* Tid[2];
  // farthest-point slots: running maximum of the distance bits per segment
  // (S entries); records of small tables (NSLOT entries, small rounds only)
  unsigned long long* Sd[3];
  SlotRec* Srec[3];
  // large tables: winner slot per segment = position of its farthest point
  // in the live set the round wrote (NONE: no kept member); Lc lists, per
  // CTA run, the survivors that reached their segment's running maximum
  uint32_t* Wn[3];
  LiveCand* Lc;
  // small tables, multi-CTA rounds: each CTA's farthest records, one row of
  // NSLOT per CTA (ping-pong by round parity); Wn then names the winning row
  SlotRec* Rc[2];
  Route* route;
};
// The control block and the round stats are contiguous in the arena, so ONE
// device-to-host copy of {Ctl; StatRec[STATS_EAGER]} ends a call.
constexpr size_t HOST_RES_STATS = (sizeof(Ctl) + 15) / 16 * 16;
constexpr size_t HOST_RES_BYTES = HOST_RES_STATS + sizeof(StatRec) * STATS_EAGER;

}  // namespace shb
