// TEST / BENCH INFRASTRUCTURE ONLY — the CPU "port" baseline and the
// full-batch parity checker (SURVEY.md §8(c) "count-only CPU restatement").
//
// Same workload file and sub-batch protocol as ref_bench.cpp, but runs the
// restatement in oracle.cpp.  Prints one JSON object per batch and a summary.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "oracle.hpp"
#include "workload.hpp"

using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: oracle_bench <workload.bin> [--threads N] [--prefix P] [--batches B] [--time-cap S]\n");
    return 2;
  }
  std::string path = argv[1];
  std::uint32_t threads = std::max(1u, std::thread::hardware_concurrency());
  std::uint64_t prefix = 0, max_batches = ~0ull;
  double time_cap = 0;
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i], v = argv[i + 1];
    if (k == "--threads") threads = std::uint32_t(std::stoul(v));
    else if (k == "--prefix") prefix = std::stoull(v);
    else if (k == "--batches") max_batches = std::stoull(v);
    else if (k == "--time-cap") time_cap = std::stod(v);
  }
  char err[512] = {0};
  auto t_build = Clock::now();
  wl::Workload w = wl::load(path);
  orc_engine* h = orc_create(std::uint32_t(w.nv), w.vlabels.data(), w.ne, w.eu.data(), w.ev.data(),
                             w.has_elab ? w.elab.data() : nullptr, 2, err, sizeof(err));
  if (!h) {
    std::printf("{\"error\": \"%s\"}\n", err);
    return 1;
  }
  double build_s = secs(t_build);
  auto t_init = Clock::now();
  if (orc_add_query(h, std::uint32_t(w.qn), w.qlabels.data(), std::uint32_t(w.qm), w.qa.data(),
                    w.qb.data(), w.qlab.data(), err, sizeof(err)) < 0) {
    std::printf("{\"error\": \"%s\"}\n", err);
    return 1;
  }
  double init_s = secs(t_init);
  std::uint64_t nb = std::min<std::uint64_t>(w.nbatches, max_batches);
  std::vector<double> times;
  std::uint64_t timed_updates = 0;
  double timed_total = 0;
  std::vector<std::uint8_t> ops(w.total);
  for (std::uint64_t i = 0; i < w.total; ++i) ops[i] = std::uint8_t(w.uop[i]);
  for (std::uint64_t b = 0; b < nb; ++b) {
    std::uint64_t lo = w.boffs[b], hi = w.boffs[b + 1];
    std::uint64_t cut = prefix ? std::min(hi, lo + prefix) : hi;
    std::uint64_t pos = 0, neg = 0, st[ORC_NSTATS] = {0};
    auto t0 = Clock::now();
    int rc = orc_apply_batch(h, cut - lo, &w.uu[lo], &w.uv[lo], &ops[lo], &w.ulab[lo], threads, 0, 1,
                             &pos, &neg, st, err, sizeof(err));
    double s = secs(t0);
    if (rc != 0) {
      std::printf("{\"error\": \"%s\", \"status\": %d}\n", err, rc);
      return 1;
    }
    times.push_back(s);
    timed_total += s;
    timed_updates += cut - lo;
    std::printf(
        "{\"batch\": %llu, \"updates\": %llu, \"positive\": %llu, \"negative\": %llu, \"ms\": %.3f, "
        "\"dfs_visits\": %llu, \"intersection_ops\": %llu, \"tasks\": %llu, \"calls\": %llu, "
        "\"b_phase\": %llu, \"b_upd\": %llu, \"dfs_visits_pruned\": %llu}\n",
        (unsigned long long)b, (unsigned long long)(cut - lo), (unsigned long long)pos,
        (unsigned long long)neg, s * 1e3, (unsigned long long)st[0], (unsigned long long)st[1],
        (unsigned long long)st[2], (unsigned long long)st[3], (unsigned long long)st[4],
        (unsigned long long)st[5], (unsigned long long)st[6]);
    std::fflush(stdout);
    if (cut < hi) {
      rc = orc_apply_batch(h, hi - cut, &w.uu[cut], &w.uv[cut], &ops[cut], &w.ulab[cut], threads, 0, 1,
                           nullptr, nullptr, nullptr, err, sizeof(err));
      if (rc != 0) {
        std::printf("{\"error\": \"%s\", \"status\": %d}\n", err, rc);
        return 1;
      }
    }
    if (time_cap > 0 && timed_total > time_cap) {
      nb = b + 1;
      break;
    }
  }
  std::sort(times.begin(), times.end());
  double median = times.empty() ? 0 : times[times.size() / 2];
  std::printf(
      "{\"summary\": true, \"batches\": %llu, \"threads\": %u, \"prefix\": %llu, \"median_ms\": %.3f, "
      "\"timed_s\": %.6f, \"timed_updates\": %llu, \"updates_per_s\": %.3f, \"build_s\": %.3f, "
      "\"init_s\": %.3f}\n",
      (unsigned long long)nb, threads, (unsigned long long)prefix, median * 1e3, timed_total,
      (unsigned long long)timed_updates, timed_total > 0 ? timed_updates / timed_total : 0.0, build_s,
      init_s);
  orc_destroy(h);
  return 0;
}
