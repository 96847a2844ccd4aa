// oracle/ref_1b.cpp -- TEST INFRASTRUCTURE ONLY: the golden generator for the
// 1B-point config (BASELINE.json configs[4]).
//
// Links the UNMODIFIED reference core (oracle/_ref/*.o, compiled from
// /root/reference/proj/core/src by oracle/Makefile) and prints one JSON object:
// the reference hull of gen_uniform(n, seed) -- vertices (hex), canonical input
// indices, per-round SegmentStats when the run is whole, and FNV-1a of the
// vertex bits in tests/golden/configs.json's convention.
//
//   ref_1b N SEED SHARDS
//
// SHARDS == 0: one monolithic seghull::hull::run(gen_uniform(N, SEED),
//   WithPreprocess, Multicore) (hull.cpp:219-290, dataio.cpp:291-301).  About
//   63 GB of RSS at N = 1e9, so it runs where host RAM allows.
// SHARDS == S > 0: the route SURVEY 8d prescribes when RAM is short.  Shard g
//   owns [g*N/S, (g+1)*N/S).  Its points are drawn from the reference's own
//   SplitMix64 (dataio.hpp:44-59) with the state advanced to the shard's first
//   draw (the generator is counter based: draw j uses state seed + (j+1)*gamma),
//   so the concatenated shards ARE gen_uniform(N, SEED).  Each shard is hulled
//   by hull::run; the union of the shard hulls is hulled by one more hull::run.
//   hull(union of S_g) == hull(union of hull(S_g)).  Per-round stats
//   of the whole run do not exist on this route and are not printed.
#include <omp.h>

#include <algorithm>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "seghull/dataio.hpp"
#include "seghull/hull.hpp"

using namespace seghull;

namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

std::uint64_t bits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}

// FNV-1a-64 over (x bits, y bits) per vertex, little-endian bytes
// (oracle/seghull_oracle.c or_fnv1a_vertices: the configs.json convention).
std::uint64_t fnv1a(const std::vector<Point>& v) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (const Point& p : v) {
    const std::uint64_t w[2] = {bits(p.x), bits(p.y)};
    for (std::uint64_t word : w)
      for (int b = 0; b < 8; ++b) {
        h ^= (word >> (8 * b)) & 0xffu;
        h *= 0x100000001b3ull;
      }
  }
  return h;
}

PointSet gen_range(std::uint64_t begin, std::uint64_t end, std::uint64_t seed) {
  PointSet p;
  const std::uint64_t n = end - begin;
  p.x.resize(n);
  p.y.resize(n);
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    SplitMix64 rng(seed);
    rng.state = seed + 2 * (begin + lo) * kGamma;  // x then y per point
    for (std::uint64_t i = lo; i < hi; ++i) {
      p.x[i] = rng.next_double();
      p.y[i] = rng.next_double();
    }
  }
  return p;
}

// Lowest index i in [0, n) with (x[i], y[i]) bit-equal to each vertex.
std::vector<std::int64_t> canonical(const PointSet& p, const std::vector<Point>& v,
                                    std::int64_t base) {
  std::vector<std::int64_t> out(v.size(), -1);
  std::vector<std::uint64_t> vx(v.size());
  for (std::size_t k = 0; k < v.size(); ++k) vx[k] = bits(v[k].x);
  std::vector<std::uint64_t> sorted = vx;
  std::sort(sorted.begin(), sorted.end());
  const std::int64_t n = static_cast<std::int64_t>(p.size());
#pragma omp parallel
  {
    std::vector<std::int64_t> mine(v.size(), -1);
#pragma omp for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) {
      const std::uint64_t xb = bits(p.x[i]);
      if (!std::binary_search(sorted.begin(), sorted.end(), xb)) continue;
      for (std::size_t k = 0; k < v.size(); ++k)
        if (vx[k] == xb && bits(v[k].y) == bits(p.y[i]) && mine[k] < 0) mine[k] = i;
    }
#pragma omp critical
    for (std::size_t k = 0; k < v.size(); ++k)
      if (mine[k] >= 0 && (out[k] < 0 || mine[k] < out[k])) out[k] = mine[k];
  }
  for (auto& o : out) o += base;
  return out;
}

void print_result(const char* route, std::uint64_t n, std::uint64_t seed, int shards,
                  const std::vector<Point>& v, const std::vector<std::int64_t>& idx,
                  const std::vector<hull::SegmentStats>* stats,
                  const std::vector<std::uint64_t>& shard_h, double secs) {
  std::printf("{\"generator\": \"uniform\", \"n\": %" PRIu64 ", \"seed\": %" PRIu64
              ", \"route\": \"%s\", \"shards\": %d, \"threads\": %d, \"seconds\": %.1f,\n",
              n, seed, route, shards, omp_get_max_threads(), secs);
  std::printf(" \"mode1\": {\"h\": %zu, \"fnv1a\": \"%016" PRIx64 "\",\n", v.size(), fnv1a(v));
  if (stats) {
    std::printf("  \"rounds\": %zu, \"stats\": [", stats->size());
    for (std::size_t i = 0; i < stats->size(); ++i) {
      const auto& s = (*stats)[i];
      std::printf("%s[%zu, %zu, %zu, %zu]", i ? ", " : "", s.iteration, s.segments,
                  s.points_remaining, s.points_removed);
    }
    std::printf("],\n");
  }
  if (!shard_h.empty()) {
    std::printf("  \"shard_h\": [");
    for (std::size_t g = 0; g < shard_h.size(); ++g)
      std::printf("%s%" PRIu64, g ? ", " : "", shard_h[g]);
    std::printf("],\n");
  }
  std::printf("  \"first\": [\"%a\", \"%a\"],\n  \"vx\": [", v[0].x, v[0].y);
  for (std::size_t k = 0; k < v.size(); ++k) std::printf("%s\"%a\"", k ? ", " : "", v[k].x);
  std::printf("],\n  \"vy\": [");
  for (std::size_t k = 0; k < v.size(); ++k) std::printf("%s\"%a\"", k ? ", " : "", v[k].y);
  std::printf("],\n  \"idx\": [");
  for (std::size_t k = 0; k < idx.size(); ++k)
    std::printf("%s%" PRId64, k ? ", " : "", idx[k]);
  std::printf("]}}\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: ref_1b N SEED SHARDS\n");
    return 2;
  }
  const std::uint64_t n = std::strtoull(argv[1], nullptr, 10);
  const std::uint64_t seed = std::strtoull(argv[2], nullptr, 10);
  const int shards = std::atoi(argv[3]);
  const double t0 = omp_get_wtime();
  if (shards == 0) {
    const PointSet p = gen_uniform(n, seed);
    const hull::HullResult r = hull::run(p, hull::Mode::WithPreprocess, Backend::Multicore);
    const auto idx = canonical(p, r.vertices, 0);
    print_result("whole", n, seed, 0, r.vertices, idx, &r.stats, {}, omp_get_wtime() - t0);
    return 0;
  }
  PointSet uni;
  std::vector<std::int64_t> uni_idx;
  std::vector<std::uint64_t> shard_h;
  for (int g = 0; g < shards; ++g) {
    const std::uint64_t b = n * g / shards, e = n * (g + 1) / shards;
    const PointSet p = gen_range(b, e, seed);
    const hull::HullResult r = hull::run(p, hull::Mode::WithPreprocess, Backend::Multicore);
    const auto idx = canonical(p, r.vertices, static_cast<std::int64_t>(b));
    for (std::size_t k = 0; k < r.vertices.size(); ++k) {
      uni.x.push_back(r.vertices[k].x);
      uni.y.push_back(r.vertices[k].y);
      uni_idx.push_back(idx[k]);
    }
    shard_h.push_back(r.vertices.size());
    std::fprintf(stderr, "shard %d: h=%zu (%.1f s)\n", g, r.vertices.size(), omp_get_wtime() - t0);
  }
  const hull::HullResult m = hull::run(uni, hull::Mode::WithPreprocess, Backend::Sequential);
  // Union rows are in shard order, and each row's index is its shard's lowest,
  // so the lowest union row with equal bits carries the global canonical index.
  const auto rows = canonical(uni, m.vertices, 0);
  std::vector<std::int64_t> idx(rows.size());
  for (std::size_t k = 0; k < rows.size(); ++k) idx[k] = uni_idx[rows[k]];
  print_result("shards+merge", n, seed, shards, m.vertices, idx, nullptr, shard_h,
               omp_get_wtime() - t0);
  return 0;
}
