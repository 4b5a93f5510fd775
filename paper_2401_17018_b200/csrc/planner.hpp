// Host-side query model and planner (north_star item 2): query validation,
// the NLF encoding of query vertices, matching orders and the per-level
// matching programs uploaded to the device.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace bdsm_b200 {

struct QEdge {
  uint32_t a, b, label;  // label kNone = unlabelled
};

// QueryGraph (reference include/bdsm/query_graph.hpp, src/query_graph.cpp:10-27).
struct HostQuery {
  uint32_t n = 0;
  std::vector<uint32_t> labels;
  std::vector<QEdge> edges;
  std::vector<uint32_t> adjmask;
  std::vector<uint32_t> degree;

  HostQuery() = default;
  HostQuery(std::vector<uint32_t> vertex_labels, std::vector<QEdge> qedges);

  bool adjacent(uint32_t u, uint32_t v) const { return (adjmask[u] >> v) & 1u; }
  uint32_t edge_label(uint32_t u, uint32_t v) const;
  bool connected() const;
};

// Encoding of a query for the candidate filter (src/encoding.cpp:17-24,
// :96-113): the sorted distinct query labels (one counter group each) and
// the saturated per-group neighbour counts of every query vertex.
struct QueryEncoding {
  std::vector<uint32_t> group_labels;  // sorted
  uint32_t cap = 3;                    // 2^group_bits - 1
  std::vector<uint8_t> qcnt;           // [n][G]
};

QueryEncoding encode_query(const HostQuery& q, uint32_t group_bits);

// Matching order anchored at query edge e: try_order with no zone and no
// tail (src/query_analysis.cpp:295-363): greedy minimum |C(u)|/max(deg,1),
// ties by higher query degree, then lower id; every prefix connected.
std::vector<uint32_t> matching_order(const HostQuery& q, uint32_t e,
                                     const std::vector<uint64_t>& column_sizes);

// Device program for one (query, edge) from its order.  label_range[u] is
// the internal-id range [lo, hi) holding query vertex u's label.
EdgeProg build_program(const HostQuery& q, uint32_t query_index, const std::vector<uint32_t>& order,
                       const std::vector<std::pair<uint32_t, uint32_t>>& label_range,
                       const std::vector<uint32_t>& label_class);

// Automorphisms of q (vertex permutations preserving labels, adjacency and
// edge labels), at most `limit` (the reference's KDegenOptions limit is
// 20,000, include/bdsm/query_analysis.hpp:42-45); false when truncated.
bool automorphisms(const HostQuery& q, size_t limit, std::vector<std::vector<uint32_t>>& out);

// Exact coalescing.  Directed query edge d = 2e + flip
// (flip 0: (a, b), 1: (b, a)) anchors the matches M with M(d) = the update's
// (u, v).  For an automorphism phi, M -> M o phi^-1 maps the matches anchored
// at d one-to-one onto those anchored at phi(d), with the same image edge set
// (so the same lowest-order decision, src/matcher.cpp:110-117).  Counting one
// representative per orbit of directed edges and multiplying by the orbit
// size therefore equals the coalesce-off count on every batch (unlike the
// reference's coalesced_expand).  Returns mult[d] = orbit size
// for the representative (lowest d) of each orbit, 0 for the others; all 1
// when the automorphisms exceed `limit`.
std::vector<uint32_t> directed_edge_orbits(const HostQuery& q, size_t limit = 20000);

// Canonical split of work units over ranks: owner = floor(world * prefix / total).
void shard_owners(const uint64_t* costs, size_t n, uint32_t world, uint32_t* owners);

}  // namespace bdsm_b200
