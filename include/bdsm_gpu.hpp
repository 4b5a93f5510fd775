// bdsm_gpu.hpp — header-only C++ host API over the C ABI (bdsm_gpu.h), in the
// reference's call shape: an engine built from vertex/edge
// records (LabeledGraph::build_from_edges, include/bdsm/graph.hpp:69-70),
// queries registered per engine (QueryEncodingState::initialize +
// build_query_plan, include/bdsm/matcher.hpp:26-27,
// include/bdsm/query_analysis.hpp:93-94), and match_batch returning
// |positive| / |negative| per query (include/bdsm/matcher.hpp:106-108).
// Errors are rethrown as the reference's exception types: BatchError
// (include/bdsm/graph.hpp:42-52), std::invalid_argument, std::runtime_error,
// std::bad_alloc.
#ifndef BDSM_GPU_HPP_
#define BDSM_GPU_HPP_

#include <cstdint>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bdsm_gpu.h"

namespace bdsm::gpu {

struct VertexRecord {  // include/bdsm/graph.hpp VertexRecord
  std::uint32_t id;
  std::uint32_t label;
};

struct EdgeRecord {  // include/bdsm/graph.hpp EdgeRecord
  std::uint32_t u, v;
  std::optional<std::uint32_t> label;
};

struct QueryEdge {  // include/bdsm/query_graph.hpp QueryEdge
  std::uint32_t a, b;
  std::optional<std::uint32_t> label;
};

struct EdgeUpdate {  // include/bdsm/graph.hpp:14-22 (order = index in the batch)
  enum class Op { kInsert, kDelete };
  Op op;
  std::uint32_t u, v;
  std::optional<std::uint32_t> edge_label;
  bool is_insert() const { return op == Op::kInsert; }
};

struct UpdateError {  // include/bdsm/graph.hpp:36-39
  std::size_t index;
  std::string reason;
};

class BatchError : public std::runtime_error {  // include/bdsm/graph.hpp:42-52
 public:
  BatchError(const std::string& what, std::vector<UpdateError> failures)
      : std::runtime_error(what), failures(std::move(failures)) {}
  std::vector<UpdateError> failures;
};

struct Counts {
  std::uint64_t positive = 0, negative = 0;
};

inline const char* update_error_reason(std::uint32_t code) {
  switch (code) {
    case 1: return "unknown vertex";
    case 2: return "insert of existing edge";
    case 3: return "delete of missing edge";
    default: return "invalid update";
  }
}

class Engine {
 public:
  // LabeledGraph::build_from_edges semantics: vertex ids dense, 0-based, unique
  // (src/graph.cpp:38-46); edge errors are reported by the engine.
  // devices: more than one entry builds a multi-device group (bdsm_group_*,
  // a replica per device, work units split over them); the calls below keep
  // their meaning.
  Engine(const std::vector<VertexRecord>& vs, const std::vector<EdgeRecord>& es, bdsm_options opts = defaults(),
         const std::vector<std::int32_t>& devices = {}) {
    std::vector<std::uint32_t> labels(vs.size(), 0xffffffffu);
    std::vector<bool> seen(vs.size(), false);
    for (const auto& r : vs) {
      if (r.id >= vs.size() || seen[r.id])
        throw std::invalid_argument("vertex ids must be dense 0-based and unique (got " + std::to_string(r.id) +
                                    ")");
      seen[r.id] = true;
      labels[r.id] = r.label;
    }
    std::vector<std::uint32_t> src(es.size()), dst(es.size()), el(es.size());
    bool any_label = false;
    for (std::size_t i = 0; i < es.size(); ++i) {
      src[i] = es[i].u;
      dst[i] = es[i].v;
      el[i] = es[i].label ? *es[i].label : BDSM_NO_LABEL;
      any_label |= bool(es[i].label);
    }
    bdsm_graph_desc g{std::uint32_t(vs.size()), labels.data(), es.size(), src.data(), dst.data(),
                      any_label ? el.data() : nullptr};
    if (devices.size() > 1) {
      check(bdsm_group_create(&g, &opts, devices.data(), std::uint32_t(devices.size()), &g_));
      e_ = bdsm_group_engine(g_, 0);
    } else {
      if (devices.size() == 1) opts.device = devices[0];
      check(bdsm_engine_create(&g, &opts, &e_));
    }
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ~Engine() {
    if (g_) bdsm_group_destroy(g_);
    else bdsm_engine_destroy(e_);
  }

  static bdsm_options defaults() {
    bdsm_options o{};
    o.group_bits = 2;
    o.coalesce = 0;
    o.device = 0;
    return o;
  }

  // QueryGraph(labels, edges) + initialize + build_query_plan (coalesce off).
  int add_query(const std::vector<std::uint32_t>& labels, const std::vector<QueryEdge>& edges) {
    std::vector<std::uint32_t> a, b, l;
    bool any_label = false;
    for (const auto& e : edges) {
      a.push_back(e.a);
      b.push_back(e.b);
      l.push_back(e.label ? *e.label : BDSM_NO_LABEL);
      any_label |= bool(e.label);
    }
    bdsm_query_desc d{std::uint32_t(labels.size()), labels.data(), std::uint32_t(edges.size()), a.data(), b.data(),
                      any_label ? l.data() : nullptr};
    int r = g_ ? bdsm_group_add_query(g_, &d) : bdsm_engine_add_query(e_, &d);
    if (r < 0) check(bdsm_status(-r));
    ++nq_;
    return r;
  }

  // match_batch (src/matcher.cpp:370-389) for every registered query.
  std::vector<Counts> match_batch(const std::vector<EdgeUpdate>& batch, bdsm_batch_stats* stats = nullptr) {
    const std::vector<bdsm_update> ups = pack(batch);
    std::vector<std::uint64_t> pos(nq_), neg(nq_);
    check(g_ ? bdsm_group_apply_batch(g_, ups.data(), ups.size(), pos.data(), neg.data(), stats)
             : bdsm_engine_apply_batch(e_, ups.data(), ups.size(), pos.data(), neg.data(), stats));
    return counts(pos, neg);
  }

  // Pipelined match_batch (run_pipeline's stage overlap, src/bench.cpp:370-564):
  // submit returns once the batch is enqueued; wait returns its counts.
  void submit(const std::vector<EdgeUpdate>& batch) { submit_packed(pack(batch)); }
  // the same with a batch already packed (so the caller can pack batch i+1
  // while batch i runs)
  void submit_packed(const std::vector<bdsm_update>& ups) {
    check(g_ ? bdsm_group_submit_batch(g_, ups.data(), ups.size())
             : bdsm_engine_submit_batch(e_, ups.data(), ups.size()));
  }
  std::vector<Counts> wait(bdsm_batch_stats* stats = nullptr) {
    std::vector<std::uint64_t> pos(nq_), neg(nq_);
    check(g_ ? bdsm_group_wait(g_, pos.data(), neg.data(), stats) : bdsm_engine_wait(e_, pos.data(), neg.data(), stats));
    return counts(pos, neg);
  }

  void set_deadline(int query, double seconds_from_now) {
    check(g_ ? bdsm_group_set_deadline(g_, query, seconds_from_now)
             : bdsm_engine_set_deadline(e_, query, seconds_from_now));
  }
  // run_pipeline drops an unsolved query from later batches (src/bench.cpp:420-432)
  void set_query_active(int query, bool active) {
    check(g_ ? bdsm_group_set_query_active(g_, query, active ? 1 : 0)
             : bdsm_engine_set_query_active(e_, query, active ? 1 : 0));
  }
  // MatchStats::timed_out of `query` in the last batch (its counts were dropped)
  bool query_timed_out(int query) {
    const int r = g_ ? bdsm_group_query_timed_out(g_, query) : bdsm_engine_query_timed_out(e_, query);
    if (r < 0) check(bdsm_status(-r));
    return r != 0;
  }
  void replan(int query) { check(g_ ? bdsm_group_replan(g_, query) : bdsm_engine_replan(e_, query)); }
  std::vector<std::uint64_t> column_sizes(int query, std::uint32_t n) {
    std::vector<std::uint64_t> out(32);
    check(bdsm_engine_column_sizes(e_, query, out.data()));
    out.resize(n);
    return out;
  }
  // Bounded match materialisation for later batches (0: counts only).
  void collect_matches(std::uint64_t cap) {
    check(g_ ? bdsm_group_collect_matches(g_, cap) : bdsm_engine_collect_matches(e_, cap));
    collect_cap_ = cap;
  }
  // Matches of the last batch for (query, phase 0 negative / 1 positive),
  // flattened num_vertices words each, sorted; throws std::length_error when
  // more matches exist than the engine collected (raise the cap).
  std::vector<std::uint32_t> matches(int query, int phase, std::uint32_t num_vertices) {
    auto fetch = [&](std::uint32_t* out, std::size_t cap) {
      return g_ ? bdsm_group_matches(g_, query, phase, out, cap) : bdsm_engine_matches(e_, query, phase, out, cap);
    };
    std::int64_t total = fetch(nullptr, 0);
    if (total < 0) check(bdsm_status(-total));
    if (std::uint64_t(total) > collect_cap_)
      throw std::length_error(std::to_string(total) + " matches, only " + std::to_string(collect_cap_) +
                              " collected (raise the collect_matches cap)");
    std::vector<std::uint32_t> out(std::size_t(total) * num_vertices);
    std::int64_t again = fetch(out.data(), std::size_t(total));
    if (again < 0) check(bdsm_status(-again));
    return out;
  }
  std::uint32_t vertex_count() const { return bdsm_engine_num_vertices(e_); }
  std::uint64_t edge_count() const { return bdsm_engine_num_edges(e_); }
  std::size_t query_count() const { return nq_; }
  bdsm_engine* handle() { return e_; }

  static std::vector<bdsm_update> pack(const std::vector<EdgeUpdate>& batch) {
    std::vector<bdsm_update> ups;
    ups.reserve(batch.size());
    for (const auto& u : batch)
      ups.push_back({u.u, u.v, u.is_insert() ? 0u : 1u,
                     u.is_insert() && u.edge_label ? *u.edge_label : BDSM_NO_LABEL});
    return ups;
  }

 private:
  std::vector<Counts> counts(const std::vector<std::uint64_t>& pos, const std::vector<std::uint64_t>& neg) const {
    std::vector<Counts> out(nq_);
    for (std::size_t i = 0; i < nq_; ++i) out[i] = {pos[i], neg[i]};
    return out;
  }
  void check(bdsm_status s) {
    if (s == BDSM_OK) return;
    std::string msg = bdsm_last_error();
    if (s == BDSM_BATCH_ERROR) {
      std::vector<bdsm_update_error> f(bdsm_last_batch_errors(e_, nullptr, 0));
      bdsm_last_batch_errors(e_, f.data(), f.size());
      std::vector<UpdateError> fails;
      for (const auto& x : f) fails.push_back({std::size_t(x.index), update_error_reason(x.reason)});
      throw BatchError(msg, std::move(fails));
    }
    if (s == BDSM_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (s == BDSM_OUT_OF_MEMORY) throw std::bad_alloc();
    throw std::runtime_error(msg);
  }
  bdsm_engine* e_ = nullptr;  // the engine, or the group's engine 0 (introspection)
  bdsm_group* g_ = nullptr;
  std::size_t nq_ = 0;
  std::uint64_t collect_cap_ = 0;
};

}  // namespace bdsm::gpu

#endif  // BDSM_GPU_HPP_
