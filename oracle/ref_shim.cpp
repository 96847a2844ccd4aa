// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the UNMODIFIED reference library, compiled from the reference's
// own sources (/root/reference/proj/core/src/*.cpp) by oracle/Makefile into
// oracle/_ref/libseghull_ref.so.  Used by tests (to pin the C restatement and
// the CUDA path against the real reference) and by bench.py's reference arm
// (`--impl reference`, which times seghull::hull::run with Backend::Multicore).
// Nothing here is shipped in the product library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "seghull/dataio.hpp"
#include "seghull/error.hpp"
#include "seghull/hull.hpp"
#include "seghull/oracle.hpp"

using namespace seghull;

namespace {

PointSet make_set(const double* x, const double* y, std::uint64_t n) {
  PointSet p;
  p.x.assign(x, x + n);
  p.y.assign(y, y + n);
  return p;
}

void put_err(char* err, std::size_t errlen, const char* what) {
  if (err && errlen) {
    std::strncpy(err, what, errlen - 1);
    err[errlen - 1] = 0;
  }
}

}  // namespace

extern "C" {

struct ref_segment_stats {
  std::uint64_t iteration, segments, points_remaining, points_removed;
};

struct ref_phase_timings {
  double pre_ms, split_ms, recurse_ms;
};

void ref_gen_uniform(std::uint64_t n, std::uint64_t seed, double* x, double* y) {
  const PointSet p = gen_uniform(n, seed);
  std::memcpy(x, p.x.data(), n * 8);
  std::memcpy(y, p.y.data(), n * 8);
}

void ref_gen_circle(std::uint64_t n, std::uint64_t seed, double* x, double* y) {
  const PointSet p = gen_circle(n, seed);
  std::memcpy(x, p.x.data(), n * 8);
  std::memcpy(y, p.y.data(), n * 8);
}

// seghull::hull::run (hull.hpp:95).  backend 0 = Sequential, 1 = Multicore.
// Returns 0, or 1 + Errc on a seghull::Error, or 100 on cap overflow.
int ref_hull_run(const double* x, const double* y, std::uint64_t n, int mode, int backend,
                 double* out_x, double* out_y, std::uint64_t cap, std::uint64_t* out_h,
                 ref_segment_stats* stats, std::uint64_t stats_cap, std::uint64_t* out_rounds,
                 ref_phase_timings* phases, char* err, std::size_t errlen) {
  try {
    const PointSet pts = make_set(x, y, n);
    const hull::HullResult r =
        hull::run(pts, mode == 1 ? hull::Mode::WithPreprocess : hull::Mode::WithoutPreprocess,
                  backend == 1 ? Backend::Multicore : Backend::Sequential);
    *out_h = r.vertices.size();
    if (out_rounds) *out_rounds = r.stats.size();
    if (phases) {
      phases->pre_ms = r.phase_timings.pre_ms;
      phases->split_ms = r.phase_timings.split_ms;
      phases->recurse_ms = r.phase_timings.recurse_ms;
    }
    for (std::size_t i = 0; stats && i < r.stats.size() && i < stats_cap; ++i) {
      stats[i] = {r.stats[i].iteration, r.stats[i].segments, r.stats[i].points_remaining,
                  r.stats[i].points_removed};
    }
    if (r.vertices.size() > cap) return 100;
    for (std::size_t i = 0; i < r.vertices.size(); ++i) {
      out_x[i] = r.vertices[i].x;
      out_y[i] = r.vertices[i].y;
    }
    return 0;
  } catch (const Error& e) {
    put_err(err, errlen, e.what());
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1 + static_cast<int>(Errc::InternalError);
  }
}

// Timing-only entry for the reference arm: runs hull::run on a prebuilt set
// (so the copy into std::vector stays outside the timed region).
void* ref_pointset_new(const double* x, const double* y, std::uint64_t n) {
  return new PointSet(make_set(x, y, n));
}

void ref_pointset_free(void* p) { delete static_cast<PointSet*>(p); }

int ref_hull_run_set(const void* set, int mode, int backend, std::uint64_t* out_h) {
  try {
    const auto& pts = *static_cast<const PointSet*>(set);
    const hull::HullResult r =
        hull::run(pts, mode == 1 ? hull::Mode::WithPreprocess : hull::Mode::WithoutPreprocess,
                  backend == 1 ? Backend::Multicore : Backend::Sequential);
    *out_h = r.vertices.size();
    return 0;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  }
}

// hull::preprocess (hull.hpp:64): returns the discard count.
std::uint64_t ref_preprocess_discards(const double* x, const double* y, std::uint64_t n) {
  return hull::preprocess(make_set(x, y, n), Backend::Sequential).second;
}

int ref_monotone_chain(const double* x, const double* y, std::uint64_t n, double* out_x,
                       double* out_y, std::uint64_t* out_h) {
  try {
    const auto v = oracle::monotone_chain(make_set(x, y, n));
    *out_h = v.size();
    for (std::size_t i = 0; i < v.size(); ++i) {
      out_x[i] = v[i].x;
      out_y[i] = v[i].y;
    }
    return 0;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  }
}

// hull::preprocess (hull.hpp:64): the filtered set in input order.
int ref_preprocess(const double* x, const double* y, std::uint64_t n, double* out_x,
                   double* out_y, std::uint64_t* kept, std::uint64_t* discarded) {
  try {
    const auto r = hull::preprocess(make_set(x, y, n), Backend::Sequential);
    *kept = r.first.size();
    *discarded = r.second;
    for (std::size_t i = 0; i < r.first.size(); ++i) {
      out_x[i] = r.first.x[i];
      out_y[i] = r.first.y[i];
    }
    return 0;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  }
}

// seghull::write_points(..., PointFormat::Binary) / read_points_binary
// (dataio.cpp:114-153, 319-345): the reference's own PTS2 writer and reader.
int ref_write_points_binary(const char* path, const double* x, const double* y, std::uint64_t n,
                            char* err, std::size_t errlen) {
  try {
    write_points(make_set(x, y, n), path, PointFormat::Binary);
    return 0;
  } catch (const Error& e) {
    put_err(err, errlen, e.what());
    return 1 + static_cast<int>(e.code());
  }
}

int ref_read_points_binary(const char* path, double* x, double* y, std::uint64_t cap,
                           std::uint64_t* n, char* err, std::size_t errlen) {
  try {
    const PointSet p = read_points(path, PointFormat::Binary);
    *n = p.size();
    if (p.size() > cap) return 100;
    for (std::size_t i = 0; i < p.size(); ++i) {
      x[i] = p.x[i];
      y[i] = p.y[i];
    }
    return 0;
  } catch (const Error& e) {
    put_err(err, errlen, e.what());
    return 1 + static_cast<int>(e.code());
  }
}

// --- the per-phase API of hull.hpp:61-91 on a reference HullState ---------
// (pins the device per-phase API, include/seghull_b200.h sh_b200_first_split..)

void* ref_state_first_split(const double* x, const double* y, std::uint64_t n, int* code) {
  try {
    *code = 0;
    return new hull::HullState(hull::first_split(make_set(x, y, n), Backend::Sequential));
  } catch (const Error& e) {
    *code = 1 + static_cast<int>(e.code());
    return nullptr;
  }
}

void* ref_state_new(std::uint64_t n, const double* x, const double* y, const double* dist,
                    const std::int32_t* head, const std::int32_t* keys, const std::int32_t* first,
                    const std::int32_t* flag) {
  auto* s = new hull::HullState;
  s->x.assign(x, x + n);
  s->y.assign(y, y + n);
  s->dist.assign(dist, dist + n);
  s->head.assign(head, head + n);
  s->keys.assign(keys, keys + n);
  s->first_pts.assign(first, first + n);
  s->flag.assign(flag, flag + n);
  return s;
}

void ref_state_free(void* s) { delete static_cast<hull::HullState*>(s); }

std::uint64_t ref_state_size(void* s) { return static_cast<hull::HullState*>(s)->size(); }

void ref_state_get(void* sp, double* x, double* y, double* dist, std::int32_t* head,
                   std::int32_t* keys, std::int32_t* first, std::int32_t* flag) {
  const auto& s = *static_cast<hull::HullState*>(sp);
  const std::size_t n = s.size();
  std::memcpy(x, s.x.data(), 8 * n);
  std::memcpy(y, s.y.data(), 8 * n);
  std::memcpy(dist, s.dist.data(), 8 * n);
  std::memcpy(head, s.head.data(), 4 * n);
  std::memcpy(keys, s.keys.data(), 4 * n);
  std::memcpy(first, s.first_pts.data(), 4 * n);
  std::memcpy(flag, s.flag.data(), 4 * n);
}

void ref_state_compute_distances(void* s) {
  hull::compute_distances(*static_cast<hull::HullState*>(s), Backend::Sequential);
}

std::uint64_t ref_state_find_farthest(void* s, std::int32_t* key, double* value,
                                      std::uint64_t* index, std::uint64_t cap) {
  const auto far = hull::find_farthest(*static_cast<hull::HullState*>(s), Backend::Sequential);
  for (std::size_t j = 0; j < far.size() && j < cap; ++j) {
    key[j] = far[j].key;
    value[j] = far[j].value;
    index[j] = far[j].index;
  }
  return far.size();
}

void ref_state_split_segments(void* s, const std::int32_t* key, const double* value,
                              const std::uint64_t* index, std::uint64_t m) {
  std::vector<primitives::SegmentMax> far(m);
  for (std::size_t j = 0; j < m; ++j) far[j] = {key[j], value[j], index[j]};
  hull::split_segments(*static_cast<hull::HullState*>(s), far, Backend::Sequential);
}

void ref_state_mark_interior(void* s) {
  hull::mark_interior(*static_cast<hull::HullState*>(s), Backend::Sequential);
}

std::uint64_t ref_state_compact(void* s) {
  return hull::compact(*static_cast<hull::HullState*>(s), Backend::Sequential);
}

}  // extern "C"
