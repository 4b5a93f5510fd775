// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// pytest suite and tests/golden/make_golden.py drive the reference's own
// `bdsm::match_batch` (src/matcher.cpp:370-389) and its brute-force oracle
// `bdsm::oracle::incremental_diff_oracle` (src/oracle.cpp:101-114) on plain
// arrays, so the CPU restatement in oracle/oracle.cpp and the CUDA engine can
// be pinned against the reference itself.
//
// Parity configuration: MatchOptions{coalesce=false}.  The plan
// is either the reference's build_query_plan (plan_mode 1,
// src/query_analysis.cpp:365-447) or one generate_matching_order per query
// edge (plan_mode 0, src/query_analysis.cpp:358-363) — the latter is the plan
// the restatement and the GPU engine use, which makes dfs_visits comparable.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <vector>

#include "bdsm/graph.hpp"
#include "bdsm/matcher.hpp"
#include "bdsm/oracle.hpp"
#include "bdsm/query_analysis.hpp"
#include "bdsm/query_graph.hpp"

using namespace bdsm;

namespace {

constexpr std::uint32_t kNone = 0xffffffffu;

void set_err(char* err, std::size_t cap, const std::string& msg) {
  if (!err || cap == 0) return;
  std::size_t n = std::min(cap - 1, msg.size());
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

LabeledGraph make_graph(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                        const std::uint32_t* eu, const std::uint32_t* ev,
                        const std::uint32_t* elab) {
  std::vector<VertexRecord> vs(nv);
  for (std::uint32_t i = 0; i < nv; ++i) vs[i] = {i, vlabels[i]};
  std::vector<EdgeRecord> es(ne);
  for (std::uint64_t i = 0; i < ne; ++i) {
    std::optional<LabelId> l;
    if (elab && elab[i] != kNone) l = elab[i];
    es[i] = {eu[i], ev[i], l};
  }
  return LabeledGraph::build_from_edges(vs, es);
}

QueryGraph make_query(std::uint32_t n, const std::uint32_t* qlabels, std::uint32_t m,
                      const std::uint32_t* qa, const std::uint32_t* qb,
                      const std::uint32_t* qlab) {
  std::vector<LabelId> labels(qlabels, qlabels + n);
  std::vector<QueryEdge> edges(m);
  for (std::uint32_t i = 0; i < m; ++i) {
    std::optional<LabelId> l;
    if (qlab && qlab[i] != kNone) l = qlab[i];
    edges[i] = {qa[i], qb[i], l};
  }
  return QueryGraph(std::move(labels), std::move(edges));
}

std::vector<EdgeUpdate> make_updates(std::uint64_t n, const std::uint32_t* uu,
                                     const std::uint32_t* uv, const std::uint8_t* uop,
                                     const std::uint32_t* ulab) {
  std::vector<EdgeUpdate> ups(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    std::optional<LabelId> l;
    if (ulab && ulab[i] != kNone) l = ulab[i];
    ups[i] = {uop[i] ? EdgeUpdate::Op::kDelete : EdgeUpdate::Op::kInsert, uu[i], uv[i], l, 0};
  }
  return ups;
}

QueryPlan make_plan(const QueryGraph& q, const CandidateTable& table, int plan_mode) {
  if (plan_mode == 1) return build_query_plan(q, table, PlanOptions{false, {}});
  if (!q.connected()) throw std::invalid_argument("disconnected query graph");
  QueryPlan plan;
  plan.coalescing = false;
  plan.edge_plans.resize(q.edge_count());
  for (std::size_t e = 0; e < q.edge_count(); ++e) {
    plan.edge_plans[e].order = generate_matching_order(q, e, table);
  }
  plan.column_sizes.resize(q.vertex_count());
  for (QueryVertexId u = 0; u < q.vertex_count(); ++u) {
    plan.column_sizes[u] = table.column(u).size();
  }
  return plan;
}

}  // namespace

extern "C" {

// The reference's per-edge matching orders, generate_matching_order
// (src/query_analysis.cpp:358-363) for every query edge (plan_mode 0 above:
// the plan the restatement and the GPU engine implement; build_query_plan
// additionally re-orders the edges of k-degenerated coalescing groups with a
// zone and join tail, :375-435, which only feeds the coalesced search, SURVEY
// F1): orders_out[e * 32 + i] and the candidate column sizes (colsizes_out[u]).
// Returns 0, or 2 / 3 on invalid_argument / other exceptions.
int ref_plan_orders(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne, const std::uint32_t* eu,
                    const std::uint32_t* ev, const std::uint32_t* elab, std::uint32_t qn,
                    const std::uint32_t* qlabels, std::uint32_t qm, const std::uint32_t* qa,
                    const std::uint32_t* qb, const std::uint32_t* qlab, std::uint32_t group_bits,
                    std::uint32_t* orders_out, std::uint64_t* colsizes_out, char* err, std::size_t errcap) {
  try {
    LabeledGraph g = make_graph(nv, vlabels, ne, eu, ev, elab);
    QueryGraph q = make_query(qn, qlabels, qm, qa, qb, qlab);
    auto enc = QueryEncodingState::initialize(g, q, group_bits);
    QueryPlan plan = make_plan(q, enc.table, 0);
    for (std::size_t e = 0; e < plan.edge_plans.size(); ++e)
      if (plan.edge_plans[e].order)
        for (std::size_t i = 0; i < plan.edge_plans[e].order->order.size(); ++i)
        orders_out[e * 32 + i] = plan.edge_plans[e].order->order[i];
    for (std::size_t u = 0; u < plan.column_sizes.size(); ++u) colsizes_out[u] = plan.column_sizes[u];
    return 0;
  } catch (const std::invalid_argument& e) {
    set_err(err, errcap, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 3;
  }
}

// Status: 0 ok, 1 BatchError (err_index = first failing update, in batch
// err_batch), 2 std::invalid_argument, 3 other exception.
//
// out_* arrays have nbatches entries.  stats_out (nullable) receives, summed
// over the stream: dfs_visits, intersection_ops, tasks_run, matches_emitted.
int ref_run_stream(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                   const std::uint32_t* eu, const std::uint32_t* ev, const std::uint32_t* elab,
                   std::uint32_t qn, const std::uint32_t* qlabels, std::uint32_t qm,
                   const std::uint32_t* qa, const std::uint32_t* qb, const std::uint32_t* qlab,
                   std::uint32_t nbatches, const std::uint64_t* batch_offsets,
                   const std::uint32_t* uu, const std::uint32_t* uv, const std::uint8_t* uop,
                   const std::uint32_t* ulab, std::uint32_t workers, int plan_mode,
                   std::uint32_t group_bits, std::uint64_t* out_pos, std::uint64_t* out_neg,
                   std::uint64_t* out_visits, double* out_ms, std::uint64_t* stats_out,
                   std::uint64_t* err_batch, std::uint64_t* err_index, char* err,
                   std::size_t errcap) {
  try {
    LabeledGraph g = make_graph(nv, vlabels, ne, eu, ev, elab);
    QueryGraph q = make_query(qn, qlabels, qm, qa, qb, qlab);
    auto enc = QueryEncodingState::initialize(g, q, group_bits);
    QueryPlan plan = make_plan(q, enc.table, plan_mode);
    MatchOptions opts;
    opts.coalesce = false;
    opts.scheduler.workers = workers == 0 ? 1 : workers;
    opts.scheduler.stealing = opts.scheduler.workers > 1 ? StealMode::kActive : StealMode::kOff;
    MatchStats total;
    for (std::uint32_t b = 0; b < nbatches; ++b) {
      std::uint64_t lo = batch_offsets[b], hi = batch_offsets[b + 1];
      if (err_batch) *err_batch = b;
      UpdateBatch batch(make_updates(hi - lo, uu + lo, uv + lo, uop + lo, ulab ? ulab + lo : nullptr));
      MatchStats stats;
      auto t0 = std::chrono::steady_clock::now();
      IncrementalMatchSet r;
      try {
        r = match_batch(g, q, plan, enc, batch, opts, &stats);
      } catch (const BatchError& e) {
        if (err_index) *err_index = e.failures.empty() ? 0 : e.failures.front().index;
        set_err(err, errcap, e.what());
        return 1;
      }
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      out_pos[b] = r.positive.size();
      out_neg[b] = r.negative.size();
      if (out_visits) out_visits[b] = stats.dfs_visits;
      if (out_ms) out_ms[b] = ms;
      total.merge(stats);
    }
    if (stats_out) {
      stats_out[0] = total.dfs_visits;
      stats_out[1] = total.intersection_ops;
      stats_out[2] = total.tasks_run;
      stats_out[3] = total.matches_emitted;
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    set_err(err, errcap, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 3;
  }
}

// Brute-force incremental diff (reference oracle, <= 60 vertices).
int ref_oracle_diff(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                    const std::uint32_t* eu, const std::uint32_t* ev, const std::uint32_t* elab,
                    std::uint32_t qn, const std::uint32_t* qlabels, std::uint32_t qm,
                    const std::uint32_t* qa, const std::uint32_t* qb, const std::uint32_t* qlab,
                    std::uint64_t nu, const std::uint32_t* uu, const std::uint32_t* uv,
                    const std::uint8_t* uop, const std::uint32_t* ulab, std::uint64_t* out_pos,
                    std::uint64_t* out_neg, char* err, std::size_t errcap) {
  try {
    LabeledGraph g = make_graph(nv, vlabels, ne, eu, ev, elab);
    QueryGraph q = make_query(qn, qlabels, qm, qa, qb, qlab);
    UpdateBatch batch(make_updates(nu, uu, uv, uop, ulab));
    auto d = oracle::incremental_diff_oracle(g, batch, q);
    *out_pos = d.positive.size();
    *out_neg = d.negative.size();
    return 0;
  } catch (const std::invalid_argument& e) {
    set_err(err, errcap, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 3;
  }
}

// Static match count (reference oracle enumerate_all_matches, <= 60 vertices).
int ref_oracle_count(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                     const std::uint32_t* eu, const std::uint32_t* ev, const std::uint32_t* elab,
                     std::uint32_t qn, const std::uint32_t* qlabels, std::uint32_t qm,
                     const std::uint32_t* qa, const std::uint32_t* qb, const std::uint32_t* qlab,
                     std::uint64_t* out_count, char* err, std::size_t errcap) {
  try {
    LabeledGraph g = make_graph(nv, vlabels, ne, eu, ev, elab);
    QueryGraph q = make_query(qn, qlabels, qm, qa, qb, qlab);
    *out_count = oracle::enumerate_all_matches(g, q).matches.size();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 3;
  }
}

}  // extern "C"
