/*
 * seghull_b200.h -- C-ABI of the B200-native 2D QuickHull (sm_100a).
 *
 * Drop-in boundary for the reference's hot path
 *     seghull::hull::HullResult seghull::hull::run(const PointSet&, Mode, Backend)
 *     (/root/reference/proj/core/include/seghull/hull.hpp:95,
 *      /root/reference/proj/core/src/hull.cpp:219-290)
 * The reference has no FFI of its own; this header is what its C++ `run`
 * binds when a maintainer adds `Backend::B200` (INTEGRATION.md shows the
 * patch).  Plain pointers and sizes only -- no C++ or torch types.
 *
 * Semantics (bit-exact with the reference):
 *   - the output is the hull CCW from the leftmost vertex (ties: lowest y),
 *     no repeated vertex, no collinear boundary point (hull.hpp:53-59);
 *   - coordinates are returned bit-for-bit, plus the canonical input index of
 *     each vertex: the lowest index among inputs with those coordinates;
 *   - per-round SegmentStats equal the reference's (hull.hpp:35-40);
 *   - orientation predicates are FP64 without contraction (-fmad=false).
 *
 * Errors mirror seghull::Errc (error.hpp:8-19): the return value is 0 or
 * 1 + Errc; SH_CAP_TOO_SMALL sets *out_h to the required capacity;
 * SH_CUDA_ERROR reports a CUDA runtime failure (message in `err`).
 * Thread safety: re-entrant; every call uses a workspace taken from a
 * per-device pool under a mutex ("independent run() calls may
 * proceed in parallel").
 */
#ifndef SEGHULL_B200_H
#define SEGHULL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SH_B200_ABI_VERSION 4

/* return codes: 0 or 1 + seghull::Errc (error.hpp:8-19) */
enum sh_status {
  SH_OK = 0,
  SH_EMPTY_INPUT = 1,         /* Errc::EmptyInput      hull.cpp:221      */
  SH_NON_FINITE_INPUT = 2,    /* Errc::NonFiniteInput  hull.cpp:222-227  */
  SH_DEGENERATE_INPUT = 3,    /* Errc::DegenerateInput hull.cpp:108-110  */
  SH_INPUT_TOO_LARGE = 4,     /* Errc::InputTooLarge   (n >= 2^32 here)  */
  SH_INTERNAL_ERROR = 5,      /* Errc::InternalError   hull.cpp:265-267  */
  SH_FILE_NOT_FOUND = 6,      /* Errc::FileNotFound    dataio.cpp:84-86  */
  SH_PARSE_ERROR = 7,         /* Errc::ParseError      dataio.cpp:117-134 */
  SH_IO_ERROR = 9,            /* Errc::IoError         dataio.cpp:88      */
  SH_CAP_TOO_SMALL = 100,     /* out buffers too small; *out_h = needed  */
  SH_CUDA_ERROR = 101,        /* CUDA runtime error (no device, OOM, ...) */
  SH_INVALID_ARGUMENT = 102
};

/* hull.hpp:48-51 Mode */
enum sh_mode { SH_MODE_WITH_PREPROCESS = 1, SH_MODE_WITHOUT_PREPROCESS = 2 };

/* flags */
enum sh_flags {
  SH_HOST_PTRS = 0u,      /* x, y (and idx) are host memory: H2D inside the call   */
  SH_DEVICE_PTRS = 1u,    /* x, y (and idx) are device memory on `device`          */
  SH_PHASE_TIMINGS = 2u,  /* record CUDA events per phase into sh_phase_ms         */
  SH_NO_STATS = 4u,       /* skip the per-round stats read-back                    */
  SH_OUT_DEVICE = 8u,     /* out_idx/out_x/out_y are device memory on `device`:      */
                          /* the vertices never leave HBM (shard hulls -> gather)    */
  SH_OUT_PAD = 16u,       /* with SH_OUT_DEVICE: write ONE fixed-size payload block  */
                          /* at out_x: {x f64[cap] | y f64[cap] | index i64[cap]},   */
                          /* the h vertices, then padding (copies of vertex 0 with   */
                          /* index -1); h > cap writes NaN x and h into index[0]     */
                          /* (see sh_b200_hull_gathered)                             */
  SH_ASYNC = 32u          /* with SH_DEVICE_PTRS: sh_b200_hull_ex only enqueues the  */
                          /* call on its stream and returns a ticket in res->ticket; */
                          /* sh_b200_hull_wait(ticket, res) completes it.  The call  */
                          /* keeps its workspace until then, so a caller can issue   */
                          /* hull i+1 while hull i runs (host work off the GPU's     */
                          /* critical path)                                          */
};

/* hull.hpp:35-40 SegmentStats, plus the device time at which the round ended */
typedef struct {
  uint64_t iteration;
  uint64_t segments;
  uint64_t points_remaining;
  uint64_t points_removed;
  uint64_t end_ns;     /* %globaltimer at the end of the round, relative to the start of K1 */
  uint64_t table_ns;   /* ... when the segment-table phase ended (CTA 0; 0 for round 1)   */
  uint64_t points_ns;  /* ... when the point phase ended (CTA 0; 0 for round 1)           */
} sh_round_stat;

/* hull.hpp:42-46 PhaseTimings (device time from CUDA events) */
typedef struct {
  double pre_ms;      /* extremes + quadrilateral filter + chain classification */
  double split_ms;    /* first split: round-1 routing of the filtered set         */
  double recurse_ms;  /* remaining rounds until only hull vertices remain         */
  double total_ms;    /* whole call on the device, H2D/D2H included when HOST_PTRS */
} sh_phase_ms;

/* Per-kernel device times of one call (CUDA events on the call's stream;
 * filled with SH_PHASE_TIMINGS).  Used for the roofline fractions. */
typedef struct {
  double h2d_ms;         /* input host->device copy (HOST_PTRS only)            */
  double extremes_ms;    /* K1: extremes + finite check                         */
  double filter_ms;      /* K2: quad filter + chain classes + round-0 farthest  */
  double first_round_ms; /* K3<first>: round 1 straight from the input          */
  double rounds_ms;      /* K4/K3 rounds >= 2, including the status polls       */
  double d2h_ms;         /* result read-back                                    */
} sh_kernel_ms;

/*
 * Convex hull of (x[i], y[i]), i < n.  Equivalent of
 * seghull::hull::run(points, Mode(mode), Backend::B200).
 *   out_idx/out_x/out_y : caller-owned, capacity `cap` vertices (any may be NULL)
 *   out_h               : number of hull vertices
 *   stats/stats_cap     : per-round SegmentStats (may be NULL)
 *   out_rounds          : number of refinement rounds executed (may be NULL)
 *   phases              : per-phase device times (may be NULL; needs SH_PHASE_TIMINGS)
 *   err/errlen          : message buffer (may be NULL)
 */
int sh_b200_hull(const double* x, const double* y, uint64_t n, int mode, uint32_t flags,
                 int device, int64_t* out_idx, double* out_x, double* out_y, uint64_t cap,
                 uint64_t* out_h, sh_round_stat* stats, uint64_t stats_cap,
                 uint64_t* out_rounds, sh_phase_ms* phases, char* err, size_t errlen);

/* Extended request: caller stream and caller-supplied point ids. */
typedef struct {
  const double* x;
  const double* y;
  uint64_t n;
  const uint32_t* ids;  /* optional: id of each point (tie-break + output index);
                           NULL means ids are 0..n-1.  Used by the shard merge,
                           where ids are global input indices.                  */
  int mode;
  uint32_t flags;
  int device;
  void* stream;         /* cudaStream_t on `device`, or NULL for a pool stream   */
  uint64_t id_base;     /* added to every output index (a shard's first global
                           index); 0 for a whole input                          */
} sh_hull_request;

typedef struct {
  int64_t* idx;
  double* x;
  double* y;
  uint64_t cap;
  uint64_t h;
  sh_round_stat* stats;
  uint64_t stats_cap;
  uint64_t rounds;
  uint64_t kept;        /* points surviving the Mode-1 filter (n in Mode 2)      */
  uint64_t bad_index;   /* first non-finite index when SH_NON_FINITE_INPUT       */
  sh_phase_ms phases;
  sh_kernel_ms kernels;
  uint32_t kernel_launches; /* kernels this call launched (evidence of GPU work) */
  char err[256];
  uint64_t ticket;      /* SH_ASYNC: the handle for sh_b200_hull_wait              */
} sh_hull_result;

int sh_b200_hull_ex(const sh_hull_request* req, sh_hull_result* res);

/* Completes an SH_ASYNC call: waits for its device work, then fills `res` like
 * a synchronous call (outputs in the buffers given at submission; `res->stats`
 * may name a stats buffer now).  Each ticket is waited for exactly once. */
int sh_b200_hull_wait(uint64_t ticket, sh_hull_result* res);

/*
 * Multi-GPU hull (SURVEY.md section 8b "sh_b200_hull_multi", 8e; hull.hpp:95
 * with the input split over several B200s of one node).
 * hull(union of S_g) == hull(union of hull(S_g)): every shard is hulled on
 * its own GPU by its own host thread (own workspace, stream and pinned ring),
 * each shard GPU writes its hull as one fixed-size payload block straight
 * into the root GPU's gather buffer (P2P stores over NVLink/NVSwitch; a
 * cudaMemcpyPeerAsync when the pair has no peer mapping), and the root hulls
 * the gathered vertices with their GLOBAL input indices as ids.  Output: the
 * same vertices and canonical (lowest) global indices as sh_b200_hull on the
 * whole input.  Per-round stats are not returned: a sharded run has no
 * whole-input rounds.  A shard hull larger than the first-pass block (2048
 * vertices) is re-packed from its retained head table, not recomputed.
 */
typedef struct {
  int device;        /* CUDA device that hulls this shard                      */
  const double* x;   /* shard points: host memory, or device memory on `device` */
  const double* y;   /*   (SH_DEVICE_PTRS)                                      */
  uint64_t n;        /* shard size (0: skipped)                                */
  uint64_t first;    /* global index of the shard's first point                */
} sh_shard;

typedef struct {
  double shards_ms;  /* host wall time: all shard hulls (parallel threads)     */
  double gather_ms;  /* ... payload blocks complete on the root                */
  double merge_ms;   /* ... merge hull on the root, results in caller buffers  */
  double total_ms;
  uint32_t shards;   /* non-empty shards                                       */
  uint64_t block_cap;/* payload block capacity used                            */
} sh_multi_ms;

/* Contiguous split of host arrays x, y over `ndev` devices (shard g =
 * [g n/ndev, (g+1) n/ndev) on devices[g]); the merge runs on devices[0].
 * devices may repeat (several shards on one GPU).  flags: SH_OUT_DEVICE puts
 * the outputs in devices[0]'s memory; SH_DEVICE_PTRS is invalid here.       */
int sh_b200_hull_multi(const double* x, const double* y, uint64_t n, int mode, uint32_t flags,
                       const int* devices, int ndev, int64_t* out_idx, double* out_x,
                       double* out_y, uint64_t cap, uint64_t* out_h, sh_multi_ms* times,
                       char* err, size_t errlen);

/* Explicit shard layout (e.g. shards generated on their own devices). */
int sh_b200_hull_shards(const sh_shard* shards, int nshards, int mode, uint32_t flags,
                        int root_device, int64_t* out_idx, double* out_x, double* out_y,
                        uint64_t cap, uint64_t* out_h, sh_multi_ms* times, char* err,
                        size_t errlen);

/* The merge step alone, for one-process-per-GPU callers (torch.distributed):
 * `payload` = nblocks gathered SH_OUT_PAD blocks of block_cap vertices each
 * (device memory on `device`, e.g. the output of one all-gather); n_total =
 * points in the whole input.  Padding (index -1) is dropped on the device
 * before the merge hull, whose input is the real vertices only.  Returns SH_CAP_TOO_SMALL with *out_h = the
 * block capacity needed when a block carries the overflow marker.           */
int sh_b200_hull_gathered(const double* payload, uint32_t nblocks, uint64_t block_cap,
                          uint64_t n_total, int mode, uint32_t flags, int device, void* stream,
                          int64_t* out_idx, double* out_x, double* out_y, uint64_t cap,
                          uint64_t* out_h, char* err, size_t errlen);

/*
 * Device generators, bit-identical to the
 * reference's host generators: SplitMix64 is counter-based, so point i of
 * gen_uniform(n_total, seed) is x = draw(2i+1), y = draw(2i+2)
 * (dataio.hpp:44-58, dataio.cpp:291-301).  Writes points
 * [first, first + count) of the stream into device arrays x, y.
 */
int sh_b200_gen_uniform(double* x, double* y, uint64_t first, uint64_t count, uint64_t seed,
                        int device, void* stream);

/* Device twin of the disk generator defined in SURVEY.md section 8d
 * (one stream, candidates (2u-1, 2v-1), accept iff x*x + y*y < 1 without FMA).
 * Produces the first n accepted points; returns SH_OK. */
int sh_b200_gen_disk(double* x, double* y, uint64_t n, uint64_t seed, int device, void* stream);

/* Host twin of gen_circle (dataio.cpp:303-312): angle = 2*pi*u, (cos, sin)
 * from the host libm, because device cos/sin are not bit-identical to glibc.
 * Circle inputs are therefore generated on the host and uploaded. */
int sh_b200_gen_circle_host(double* x, double* y, uint64_t n, uint64_t seed);

/*
 * PTS2 binary point file straight to HBM,
 * replacing seghull::read_points_binary (dataio.cpp:114-153; layout: "PTS2",
 * u64 LE count, then count x {f64 LE x, f64 LE y}).  The file is read in
 * chunks into pinned host buffers, copied to the device and split into the
 * caller's device arrays x[count], y[count] on `stream`, overlapping the
 * file read with the transfer.  x == NULL or y == NULL: only *n = count.
 * Returns SH_OK, SH_CAP_TOO_SMALL (cap < count; *n = count),
 * SH_FILE_NOT_FOUND, SH_IO_ERROR, SH_PARSE_ERROR (truncated header, bad
 * magic, size != 12 + 16 count) or SH_NON_FINITE_INPUT ("non-finite
 * coordinate at point i", the first such i) with the reference's messages.
 */
int sh_b200_read_pts2(const char* path, int device, void* stream, double* x, double* y,
                      uint64_t cap, uint64_t* n, char* err, size_t errlen);

/*
 * hull::preprocess as a device API (hull.hpp:61-64,
 * hull.cpp:53-99): the points outside the strict interior of the quadrilateral
 * of the four extremes, in input order, written to out_x/out_y (device, cap
 * entries; NULL = count only).  *kept = survivors, *discarded = n - kept.
 * x, y are device arrays.  Returns SH_OK, SH_EMPTY_INPUT, SH_CAP_TOO_SMALL,
 * SH_NON_FINITE_INPUT (first bad index; the reference does not check here)
 * or SH_CUDA_ERROR.
 */
int sh_b200_preprocess(const double* x, const double* y, uint64_t n, int device, void* stream,
                       double* out_x, double* out_y, uint64_t cap, uint64_t* kept,
                       uint64_t* discarded, char* err, size_t errlen);

/*
 * Per-phase device APIs (hull.hpp:61-91): the
 * reference's stages over a device HullState in the REFERENCE's layout
 * (hull.hpp:19-33) -- rows laid out by first_split as the lower chain sorted
 * lex-ascending then the upper chain lex-descending, head/keys/first_pts/flag
 * as i32 -- so the reference's per-stage tests (tests/test_hull.cpp:88-314)
 * run against the device bit for bit.  The fused path (sh_b200_hull) does not
 * use them.  All columns are caller-owned device memory on `device` with
 * `cap` rows; calls are ordered on `stream` (NULL: the legacy default stream)
 * and return SH_OK, SH_INVALID_ARGUMENT, SH_CAP_TOO_SMALL or SH_CUDA_ERROR
 * (first_split also SH_EMPTY_INPUT / SH_DEGENERATE_INPUT, hull.cpp:103-110).
 * compute_distances / split_segments / mark_interior are asynchronous;
 * first_split, find_farthest and compact synchronise (they return counts).
 */
typedef struct {
  double* x;
  double* y;
  double* dist;        /* signed outward measure vs the segment's base line */
  int32_t* head;       /* 1 at segment starts                               */
  int32_t* keys;       /* segment id per row                                */
  int32_t* first_pts;  /* row of the row's segment head                     */
  int32_t* flag;       /* 1 = survives the next compaction                  */
  uint64_t n;          /* rows in use (set by first_split and compact)      */
  uint64_t cap;        /* rows every column can hold                        */
} sh_hull_state;

/* primitives::SegmentMax (primitives.hpp:24-30) */
typedef struct {
  int32_t key;
  int32_t pad;
  double value;
  uint64_t index;      /* smallest row attaining value within the segment   */
} sh_segment_max;

/* hull::first_split (hull.cpp:101-158): x, y device arrays of n points */
int sh_b200_first_split(const double* x, const double* y, uint64_t n, sh_hull_state* st,
                        int device, void* stream, char* err, size_t errlen);
/* hull::compute_distances (hull.cpp:160-180) */
int sh_b200_compute_distances(const sh_hull_state* st, int device, void* stream);
/* hull::find_farthest (hull.cpp:182-184, primitives.cpp:108-136): one entry
 * per segment into device array out[cap]; *nseg = segments */
int sh_b200_find_farthest(const sh_hull_state* st, sh_segment_max* out, uint64_t cap,
                          uint64_t* nseg, int device, void* stream);
/* hull::split_segments (hull.cpp:186-194): farthest = device array of m */
int sh_b200_split_segments(const sh_hull_state* st, const sh_segment_max* farthest, uint64_t m,
                           int device, void* stream);
/* hull::mark_interior (hull.cpp:196-201) */
int sh_b200_mark_interior(const sh_hull_state* st, int device, void* stream);
/* hull::compact (hull.cpp:203-217): st->n shrinks; *removed = rows dropped */
int sh_b200_compact(sh_hull_state* st, uint64_t* removed, int device, void* stream);

/* Library/device information; returns SH_OK or SH_CUDA_ERROR. */
int sh_b200_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                        uint64_t* hbm_bytes, char* name, size_t namelen);

/* Release every pooled workspace on every device. */
void sh_b200_release_pool(void);

/* ABI version (SH_B200_ABI_VERSION). */
int sh_b200_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SEGHULL_B200_H */
