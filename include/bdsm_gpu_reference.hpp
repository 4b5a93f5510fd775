// bdsm_gpu_reference.hpp — the reference-side binding of libbdsm_b200.so.
//
// This is the header a maintainer of the reference (/root/reference/proj,
// namespace bdsm) adds next to include/bdsm/matcher.hpp: it takes the
// reference's OWN types (VertexRecord, EdgeRecord, LabeledGraph, QueryGraph,
// UpdateBatch) and throws the reference's OWN exceptions, so run_pipeline
// (src/bench.cpp:408-472) and the reference's tests swap
//
//     bdsm::match_batch(g, q, plan, enc, batch, opts, &stats)   // src/matcher.cpp:370-389
//
// for one DeviceMatcher::match_batch(batch) per batch (every registered query
// at once).  It needs only the reference's include/ and the C ABI
// (include/bdsm_gpu.h); tests/test_reference_binding.py compiles it against
// /root/reference/proj/include and links it with the unmodified reference
// library.
//
// Error mapping:
//   BDSM_BATCH_ERROR      -> bdsm::BatchError, UpdateError reasons formatted as
//                            LabeledGraph::validate_batch does (src/graph.cpp:116-135)
//   BDSM_INVALID_ARGUMENT -> std::invalid_argument (UpdateBatch ctor src/graph.cpp:8-23,
//                            build_from_edges :35-72, QueryGraph / planner)
//   BDSM_OUT_OF_MEMORY    -> std::bad_alloc
//   other                 -> std::runtime_error
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "bdsm/graph.hpp"
#include "bdsm/query_graph.hpp"
#include "bdsm_gpu.h"

namespace bdsm::gpu_ref {

// |IncrementalMatchSet::positive|, |negative| (include/bdsm/matcher.hpp:55-58).
struct DeltaCounts {
  std::uint64_t positive = 0;
  std::uint64_t negative = 0;
};

class DeviceMatcher {
 public:
  // LabeledGraph::build_from_edges(vertices, edges) (include/bdsm/graph.hpp:69-70):
  // the device copy of the graph.  Vertex ids are dense and 0-based.
  DeviceMatcher(const std::vector<VertexRecord>& vertices, const std::vector<EdgeRecord>& edges,
                std::uint32_t group_bits = 2, int device = 0) {
    std::vector<LabelId> labels(vertices.size(), kNoLabel);
    for (const VertexRecord& r : vertices) {
      if (r.id >= vertices.size() || labels[r.id] != kNoLabel)
        throw std::invalid_argument("vertex ids must be dense 0-based and unique (got " + std::to_string(r.id) +
                                    ")");
      labels[r.id] = r.label;
    }
    std::vector<std::uint32_t> src, dst, el;
    bool any_label = false;
    src.reserve(edges.size());
    dst.reserve(edges.size());
    el.reserve(edges.size());
    for (const EdgeRecord& e : edges) {
      src.push_back(e.u);
      dst.push_back(e.v);
      el.push_back(e.label ? *e.label : BDSM_NO_LABEL);
      any_label |= bool(e.label);
    }
    create(labels, src, dst, any_label ? &el : nullptr, group_bits, device);
  }

  // The device copy of an existing reference graph (its edges, u < v).
  explicit DeviceMatcher(const LabeledGraph& g, std::uint32_t group_bits = 2, int device = 0) {
    std::vector<LabelId> labels(g.vertex_count());
    std::vector<std::uint32_t> src, dst, el;
    bool any_label = false;
    for (VertexId v = 0; v < g.vertex_count(); ++v) {
      labels[v] = g.label(v);
      g.for_each_neighbor(v, [&](VertexId w) {
        if (w <= v) return;
        src.push_back(v);
        dst.push_back(w);
        const std::optional<LabelId> l = g.edge_label(v, w);
        el.push_back(l ? *l : BDSM_NO_LABEL);
        any_label |= bool(l);
      });
    }
    create(labels, src, dst, any_label ? &el : nullptr, group_bits, device);
  }

  DeviceMatcher(const DeviceMatcher&) = delete;
  DeviceMatcher& operator=(const DeviceMatcher&) = delete;
  ~DeviceMatcher() { bdsm_engine_destroy(e_); }

  // QueryGraph + QueryEncodingState::initialize + build_query_plan with
  // coalescing off (src/matcher.cpp:10-18, src/query_analysis.cpp:358-363).
  // Returns the query's index in every later match_batch result.
  int add_query(const QueryGraph& q) {
    std::vector<std::uint32_t> a, b, l;
    bool any_label = false;
    for (const QueryEdge& e : q.edges()) {
      a.push_back(e.a);
      b.push_back(e.b);
      l.push_back(e.label ? *e.label : BDSM_NO_LABEL);
      any_label |= bool(e.label);
    }
    const std::vector<LabelId>& labels = q.labels();
    bdsm_query_desc d{std::uint32_t(labels.size()), labels.data(), std::uint32_t(a.size()), a.data(), b.data(),
                      any_label ? l.data() : nullptr};
    const int r = bdsm_engine_add_query(e_, &d);
    if (r < 0) check(bdsm_status(-r), nullptr);
    ++nq_;
    return r;
  }

  // match_batch (src/matcher.cpp:370-389) for every registered query: the
  // graph is validated, matched on G, updated and matched on G' in place
  // (all-or-nothing).  Batch order is UpdateBatch's (src/graph.cpp:21).
  std::vector<DeltaCounts> match_batch(const UpdateBatch& batch, bdsm_batch_stats* stats = nullptr) {
    std::vector<bdsm_update> ups;
    ups.reserve(batch.size());
    for (const EdgeUpdate& u : batch.updates())
      ups.push_back({u.u, u.v, u.is_insert() ? 0u : 1u,
                     u.is_insert() && u.edge_label ? *u.edge_label : BDSM_NO_LABEL});
    std::vector<std::uint64_t> pos(nq_), neg(nq_);
    check(bdsm_engine_apply_batch(e_, ups.data(), ups.size(), pos.data(), neg.data(), stats), &batch);
    std::vector<DeltaCounts> out(nq_);
    for (std::size_t i = 0; i < nq_; ++i) out[i] = {pos[i], neg[i]};
    return out;
  }

  // run_pipeline's per-query deadline and unsolved-query drop (src/bench.cpp:418-432, :463-467).
  void set_deadline(int query, double seconds_from_now) {
    check(bdsm_engine_set_deadline(e_, query, seconds_from_now), nullptr);
  }
  void set_query_active(int query, bool active) {
    check(bdsm_engine_set_query_active(e_, query, active ? 1 : 0), nullptr);
  }
  bool timed_out(int query) {
    const int r = bdsm_engine_query_timed_out(e_, query);
    if (r < 0) check(bdsm_status(-r), nullptr);
    return r != 0;
  }

  std::size_t query_count() const { return nq_; }
  bdsm_engine* handle() { return e_; }

 private:
  void create(const std::vector<LabelId>& labels, const std::vector<std::uint32_t>& src,
              const std::vector<std::uint32_t>& dst, const std::vector<std::uint32_t>* el, std::uint32_t group_bits,
              int device) {
    bdsm_graph_desc g{std::uint32_t(labels.size()), labels.data(), src.size(), src.data(), dst.data(),
                      el ? el->data() : nullptr};
    bdsm_options o{};
    o.group_bits = group_bits;
    o.device = device;
    check(bdsm_engine_create(&g, &o, &e_), nullptr);
  }

  void check(bdsm_status s, const UpdateBatch* batch) {
    if (s == BDSM_OK) return;
    const std::string msg = bdsm_last_error();
    if (s == BDSM_BATCH_ERROR && e_) {
      std::vector<bdsm_update_error> f(bdsm_last_batch_errors(e_, nullptr, 0));
      bdsm_last_batch_errors(e_, f.data(), f.size());
      std::vector<UpdateError> fails;
      for (const bdsm_update_error& x : f) {
        const std::size_t i = std::size_t(x.index);
        std::string pair;
        if (batch && i < batch->size())
          pair = " (" + std::to_string(batch->updates()[i].u) + "," + std::to_string(batch->updates()[i].v) + ")";
        switch (x.reason) {
          case 1: fails.push_back({i, "unknown vertex"}); break;
          case 2: fails.push_back({i, "insert of existing edge" + pair}); break;
          case 3: fails.push_back({i, "delete of missing edge" + pair}); break;
          default: fails.push_back({i, "invalid update"}); break;
        }
      }
      throw BatchError(msg, std::move(fails));
    }
    if (s == BDSM_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (s == BDSM_OUT_OF_MEMORY) throw std::bad_alloc();
    throw std::runtime_error(msg);
  }

  bdsm_engine* e_ = nullptr;
  std::size_t nq_ = 0;
};

}  // namespace bdsm::gpu_ref
