// oracle/hullbench_b200.cpp -- INTEGRATION HARNESS (test infrastructure).
//
// the reference's OWN benchmark harness --
// seghull::bench::run_bench with its warm-up / median protocol, its
// monotone-chain baseline + verification and its CSV writer
// (core/src/bench.cpp:39-114) -- driving the B200 backend.  This is the
// INTEGRATION.md patch done at link time instead of in the reference's
// sources: `Backend::B200` is the enumerator value 2 the patch adds to
// primitives.hpp:14, and every call bench.o makes to seghull::hull::run is
// redirected (ld --wrap) to a dispatcher that sends Backend 2 to the C-ABI
// (sh_b200_hull) and everything else to the reference's own run.  The
// reference objects are compiled unmodified from /root/reference by
// oracle/Makefile; nothing of this file ships in the product library.
//
//   hullbench_b200 --gen uniform:N:SEED | --gen circle:N:SEED | --input FILE
//                  [--mode 1|2]... [--backend seq|par|b200] [--repeat K]
//                  [--csv PATH] [--verify] [--emit-hull PATH]
// Exit codes as the reference's hullbench: 0 ok, 1 verification failed, 2 error.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "seghull/bench.hpp"
#include "seghull/dataio.hpp"
#include "seghull/error.hpp"
#include "seghull/hull.hpp"
#include "seghull_b200.h"

using namespace seghull;

namespace {

constexpr Backend kB200 = static_cast<Backend>(2);  // enum class Backend {.., B200}

hull::HullResult run_b200(const PointSet& pts, hull::Mode mode) {
  const std::size_t n = pts.size();
  // uninitialised buffers: zero-filling n doubles would cost more than the hull
  const std::size_t cap = n > 2 ? n : 2;
  std::unique_ptr<double[]> vx(new double[cap]), vy(new double[cap]);
  constexpr std::size_t kStats = 1u << 12;
  std::unique_ptr<sh_round_stat[]> st(new sh_round_stat[kStats]);
  uint64_t h = 0, rounds = 0;
  sh_phase_ms ph{};
  char err[256] = {0};
  const int rc = sh_b200_hull(pts.x.data(), pts.y.data(), n,
                              mode == hull::Mode::WithPreprocess ? SH_MODE_WITH_PREPROCESS
                                                                 : SH_MODE_WITHOUT_PREPROCESS,
                              SH_HOST_PTRS | SH_PHASE_TIMINGS, 0, nullptr, vx.get(), vy.get(),
                              cap, &h, st.get(), kStats, &rounds, &ph, err, sizeof err);
  if (rc >= SH_EMPTY_INPUT && rc <= SH_IO_ERROR) throw Error(static_cast<Errc>(rc - 1), err);
  if (rc != SH_OK) throw Error(Errc::InternalError, err);
  hull::HullResult out;
  out.vertices.reserve(h);
  for (uint64_t i = 0; i < h; ++i) out.vertices.push_back({vx[i], vy[i]});
  for (uint64_t r = 0; r < rounds && r < kStats; ++r)
    out.stats.push_back({static_cast<std::size_t>(st[r].iteration),
                         static_cast<std::size_t>(st[r].segments),
                         static_cast<std::size_t>(st[r].points_remaining),
                         static_cast<std::size_t>(st[r].points_removed)});
  out.phase_timings.pre_ms = ph.pre_ms;
  out.phase_timings.split_ms = ph.split_ms;
  out.phase_timings.recurse_ms = ph.recurse_ms;
  return out;
}

bench::DatasetSpec gen_spec(const std::string& spec) {
  const auto a = spec.find(':'), b = spec.find(':', a + 1);
  if (a == std::string::npos || b == std::string::npos)
    throw Error(Errc::ParseError, "--gen expects KIND:N:SEED, got '" + spec + "'");
  const std::string kind = spec.substr(0, a);
  const std::size_t n = std::stoull(spec.substr(a + 1, b - a - 1));
  const std::uint64_t seed = std::stoull(spec.substr(b + 1));
  bench::DatasetSpec d;
  d.label = spec;
  if (kind == "uniform") d.points = gen_uniform(n, seed);
  else if (kind == "circle") d.points = gen_circle(n, seed);
  else throw Error(Errc::ParseError, "unknown generator '" + kind + "'");
  return d;
}

bench::DatasetSpec input_spec(const std::string& path) {
  char magic[4] = {};
  std::ifstream probe(path, std::ios::binary);
  probe.read(magic, 4);
  bench::DatasetSpec d;
  d.label = path;
  d.points = read_points(path, std::memcmp(magic, "PTS2", 4) == 0 ? PointFormat::Binary
                                                                   : PointFormat::Text);
  return d;
}

}  // namespace

// ld --wrap=<hull::run>: bench.o's calls land here
extern "C" hull::HullResult __real__ZN7seghull4hull3runERKNS_8PointSetENS0_4ModeENS_7BackendE(
    const PointSet&, hull::Mode, Backend);
extern "C" hull::HullResult __wrap__ZN7seghull4hull3runERKNS_8PointSetENS0_4ModeENS_7BackendE(
    const PointSet& p, hull::Mode m, Backend b) {
  if (b == kB200) return run_b200(p, m);
  return __real__ZN7seghull4hull3runERKNS_8PointSetENS0_4ModeENS_7BackendE(p, m, b);
}

int main(int argc, char** argv) {
  try {
    bench::BenchConfig cfg;
    std::vector<hull::Mode> modes;
    std::string csv;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto next = [&]() -> std::string {
        if (i + 1 >= argc) throw Error(Errc::ParseError, a + " needs a value");
        return argv[++i];
      };
      if (a == "--gen") cfg.datasets.push_back(gen_spec(next()));
      else if (a == "--input") cfg.datasets.push_back(input_spec(next()));
      else if (a == "--mode") modes.push_back(static_cast<hull::Mode>(std::stoi(next())));
      else if (a == "--backend") {
        const std::string b = next();
        cfg.backend = b == "par" ? Backend::Multicore : b == "b200" ? kB200 : Backend::Sequential;
      } else if (a == "--repeat") cfg.repeat = std::stoi(next());
      else if (a == "--csv") csv = next();
      else if (a == "--verify") cfg.verify = true;
      else if (a == "--emit-hull") cfg.emit_hull = next();
      else throw Error(Errc::ParseError, "unknown option " + a);
    }
    if (cfg.datasets.empty()) {
      std::cerr << "hullbench_b200: no datasets; pass --gen or --input\n";
      return 2;
    }
    if (!modes.empty()) cfg.modes = modes;
    const auto records = bench::run_bench(cfg);
    std::printf("%-24s %10s %4s %10s %9s %9s %11s %12s %8s %8s %8s\n", "dataset", "size", "mode",
                "total_ms", "pre_ms", "split_ms", "recurse_ms", "baseline_ms", "speedup", "hull",
                "verified");
    for (const auto& r : records)
      std::printf("%-24s %10zu %4d %10.3f %9.3f %9.3f %11.3f %12.3f %8.1f %8zu %8s\n",
                  r.dataset.c_str(), r.size, r.mode, r.total_ms, r.pre_ms, r.split_ms,
                  r.recurse_ms, r.baseline_ms, r.speedup, r.hull_size, r.verified ? "yes" : "NO");
    if (!csv.empty()) {
      std::ofstream out(csv, std::ios::trunc);
      bench::write_csv(records, out);
    }
  } catch (const Error& e) {
    std::cerr << "hullbench_b200: " << e.what() << '\n';
    return e.code() == Errc::VerificationFailed ? 1 : 2;
  } catch (const std::exception& e) {
    std::cerr << "hullbench_b200: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
