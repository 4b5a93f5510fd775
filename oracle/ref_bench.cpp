// TEST / BENCH INFRASTRUCTURE ONLY — the CPU reference arm.
//
// Drives the UNMODIFIED reference library (oracle/_ref/libbdsm_ref.a, built
// from /root/reference/proj/src by oracle/Makefile) through its own public
// API: LabeledGraph::build_from_edges (src/graph.cpp:35-72),
// QueryEncodingState::initialize (src/matcher.cpp:10-18), a plan, then
// bdsm::match_batch (src/matcher.cpp:370-389) per batch with
// MatchOptions{coalesce=false, workers=W, stealing=active} (SURVEY.md F1,
// BASELINE.md §3).
//
// Sub-batch protocol: with --prefix P only the
// first P updates of each batch are timed through match_batch; the remaining
// updates are then applied untimed with the reference's own
// LabeledGraph::apply_batch + QueryEncodingState::refresh, so batch b+1 sees
// exactly the graph the full stream produces and stays valid.
//
// Output: one JSON object per batch on stdout, then a summary object.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "bdsm/graph.hpp"
#include "bdsm/matcher.hpp"
#include "bdsm/query_analysis.hpp"
#include "workload.hpp"

using namespace bdsm;
using Clock = std::chrono::steady_clock;

namespace {

constexpr std::uint32_t kNone = 0xffffffffu;

double secs(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

std::vector<EdgeUpdate> updates_of(const wl::Workload& w, std::uint64_t lo, std::uint64_t hi) {
  std::vector<EdgeUpdate> ups;
  ups.reserve(hi - lo);
  for (std::uint64_t i = lo; i < hi; ++i) {
    std::optional<LabelId> l;
    if (w.ulab[i] != kNone) l = w.ulab[i];
    ups.push_back({w.uop[i] ? EdgeUpdate::Op::kDelete : EdgeUpdate::Op::kInsert, w.uu[i], w.uv[i], l, 0});
  }
  return ups;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: ref_bench <workload.bin> [--workers N] [--prefix P] [--batches B] "
                 "[--plan 0|1] [--time-cap S]\n");
    return 2;
  }
  std::string path = argv[1];
  std::size_t workers = std::max(1u, std::thread::hardware_concurrency());
  std::uint64_t prefix = 0;  // 0 = full batch
  std::uint64_t max_batches = ~0ull;
  int plan_mode = 0;
  double time_cap = 0;  // stop after the batch that crosses it (0 = none)
  for (int i = 2; i + 1 < argc; i += 2) {
    std::string k = argv[i];
    std::string v = argv[i + 1];
    if (k == "--workers") workers = std::stoul(v);
    else if (k == "--prefix") prefix = std::stoull(v);
    else if (k == "--batches") max_batches = std::stoull(v);
    else if (k == "--plan") plan_mode = std::stoi(v);
    else if (k == "--time-cap") time_cap = std::stod(v);
  }
  try {
    auto t_load = Clock::now();
    wl::Workload w = wl::load(path);
    double load_s = secs(t_load);

    auto t_build = Clock::now();
    std::vector<VertexRecord> vs(w.nv);
    for (std::uint32_t i = 0; i < w.nv; ++i) vs[i] = {i, w.vlabels[i]};
    std::vector<EdgeRecord> es(w.ne);
    for (std::uint64_t i = 0; i < w.ne; ++i) {
      std::optional<LabelId> l;
      if (w.has_elab && w.elab[i] != kNone) l = w.elab[i];
      es[i] = {w.eu[i], w.ev[i], l};
    }
    LabeledGraph g = LabeledGraph::build_from_edges(vs, es);
    vs.clear();
    vs.shrink_to_fit();
    es.clear();
    es.shrink_to_fit();
    double build_s = secs(t_build);

    std::vector<LabelId> ql(w.qlabels.begin(), w.qlabels.end());
    std::vector<QueryEdge> qe(w.qm);
    for (std::uint64_t i = 0; i < w.qm; ++i) {
      std::optional<LabelId> l;
      if (w.qlab[i] != kNone) l = w.qlab[i];
      qe[i] = {w.qa[i], w.qb[i], l};
    }
    QueryGraph q(std::move(ql), std::move(qe));

    auto t_init = Clock::now();
    auto enc = QueryEncodingState::initialize(g, q, 2);
    QueryPlan plan;
    if (plan_mode == 1) {
      plan = build_query_plan(q, enc.table, PlanOptions{false, {}});
    } else {
      plan.coalescing = false;
      plan.edge_plans.resize(q.edge_count());
      for (std::size_t e = 0; e < q.edge_count(); ++e) {
        plan.edge_plans[e].order = generate_matching_order(q, e, enc.table);
      }
    }
    double init_s = secs(t_init);

    MatchOptions opts;
    opts.coalesce = false;
    opts.scheduler.workers = workers;
    opts.scheduler.stealing = workers > 1 ? StealMode::kActive : StealMode::kOff;

    std::uint64_t nb = std::min<std::uint64_t>(w.nbatches, max_batches);
    std::vector<double> times;
    std::uint64_t timed_updates = 0;
    double timed_total = 0;
    for (std::uint64_t b = 0; b < nb; ++b) {
      std::uint64_t lo = w.boffs[b], hi = w.boffs[b + 1];
      std::uint64_t cut = prefix ? std::min(hi, lo + prefix) : hi;
      UpdateBatch head(updates_of(w, lo, cut));
      MatchStats stats;
      auto t0 = Clock::now();
      IncrementalMatchSet r = match_batch(g, q, plan, enc, head, opts, &stats);
      double s = secs(t0);
      times.push_back(s);
      timed_total += s;
      timed_updates += cut - lo;
      std::printf(
          "{\"batch\": %llu, \"updates\": %llu, \"positive\": %zu, \"negative\": %zu, "
          "\"ms\": %.3f, \"dfs_visits\": %llu, \"intersection_ops\": %llu, \"tasks\": %llu}\n",
          (unsigned long long)b, (unsigned long long)(cut - lo), r.positive.size(),
          r.negative.size(), s * 1e3, (unsigned long long)stats.dfs_visits,
          (unsigned long long)stats.intersection_ops, (unsigned long long)stats.tasks_run);
      std::fflush(stdout);
      if (cut < hi) {  // untimed: keep the graph on the full stream's trajectory
        UpdateBatch rest(updates_of(w, cut, hi));
        g.apply_batch(rest);
        enc.refresh(g, rest);
      }
      if (time_cap > 0 && timed_total > time_cap) {
        nb = b + 1;
        break;
      }
    }
    std::vector<double> sorted = times;
    std::sort(sorted.begin(), sorted.end());
    double median = sorted.empty() ? 0 : sorted[sorted.size() / 2];
    std::printf(
        "{\"summary\": true, \"batches\": %llu, \"workers\": %zu, \"prefix\": %llu, "
        "\"median_ms\": %.3f, \"timed_s\": %.6f, \"timed_updates\": %llu, "
        "\"updates_per_s\": %.3f, \"load_s\": %.3f, \"build_s\": %.3f, \"init_s\": %.3f}\n",
        (unsigned long long)nb, workers, (unsigned long long)prefix, median * 1e3, timed_total,
        (unsigned long long)timed_updates, timed_total > 0 ? timed_updates / timed_total : 0.0,
        load_s, build_s, init_s);
    return 0;
  } catch (const BatchError& e) {
    std::printf("{\"error\": \"BatchError\", \"what\": \"%s\"}\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"exception\", \"what\": \"%s\"}\n", e.what());
    return 1;
  }
}
