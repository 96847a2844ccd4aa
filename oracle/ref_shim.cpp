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

}  // extern "C"
