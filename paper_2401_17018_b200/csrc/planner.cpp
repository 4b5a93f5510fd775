// Host planner.  Follows the reference's coalesce-off plan: one greedy
// matching order per query edge (src/query_analysis.cpp:295-363, :437-441).
#include "planner.hpp"

#include <algorithm>

namespace bdsm_b200 {

HostQuery::HostQuery(std::vector<uint32_t> vertex_labels, std::vector<QEdge> qedges)
    : labels(std::move(vertex_labels)) {
  n = static_cast<uint32_t>(labels.size());
  if (n == 0) throw std::invalid_argument("empty query graph");
  if (n > 32) throw std::invalid_argument("query graph too large");
  adjmask.assign(n, 0);
  degree.assign(n, 0);
  for (const QEdge& e : qedges) {
    if (e.a >= n || e.b >= n) throw std::invalid_argument("query edge references unknown vertex");
    if (e.a == e.b) throw std::invalid_argument("query self-loop");
    if (adjacent(e.a, e.b)) throw std::invalid_argument("duplicate query edge");
    adjmask[e.a] |= 1u << e.b;
    adjmask[e.b] |= 1u << e.a;
    ++degree[e.a];
    ++degree[e.b];
    edges.push_back(e);
  }
}

uint32_t HostQuery::edge_label(uint32_t u, uint32_t v) const {
  for (const QEdge& e : edges) {
    if ((e.a == u && e.b == v) || (e.a == v && e.b == u)) return e.label;
  }
  return kNone;
}

bool HostQuery::connected() const {  // src/query_graph.cpp:43-55
  uint32_t seen = 1, frontier = 1;
  while (frontier) {
    uint32_t next = 0;
    for (uint32_t u = 0; u < n; ++u) {
      if ((frontier >> u) & 1u) next |= adjmask[u];
    }
    frontier = next & ~seen;
    seen |= next;
  }
  return seen == (n == 32 ? ~0u : (1u << n) - 1);
}

QueryEncoding encode_query(const HostQuery& q, uint32_t group_bits) {
  if (group_bits == 0 || group_bits > 8) throw std::invalid_argument("group_bits must be in 1..8");
  QueryEncoding enc;
  enc.group_labels = q.labels;
  std::sort(enc.group_labels.begin(), enc.group_labels.end());
  enc.group_labels.erase(std::unique(enc.group_labels.begin(), enc.group_labels.end()),
                         enc.group_labels.end());
  enc.cap = (1u << group_bits) - 1;
  size_t G = enc.group_labels.size();
  enc.qcnt.assign(size_t(q.n) * G, 0);
  for (uint32_t u = 0; u < q.n; ++u) {
    for (uint32_t w = 0; w < q.n; ++w) {
      if (!q.adjacent(u, w)) continue;
      size_t g = size_t(std::lower_bound(enc.group_labels.begin(), enc.group_labels.end(), q.labels[w]) -
                        enc.group_labels.begin());
      uint8_t& c = enc.qcnt[u * G + g];
      if (c < enc.cap) ++c;
    }
  }
  return enc;
}

std::vector<uint32_t> matching_order(const HostQuery& q, uint32_t e,
                                     const std::vector<uint64_t>& column_sizes) {
  const QEdge& anchor = q.edges.at(e);
  std::vector<uint32_t> order{anchor.a, anchor.b};
  uint32_t assigned = (1u << anchor.a) | (1u << anchor.b);
  uint32_t all = q.n == 32 ? ~0u : (1u << q.n) - 1;
  auto sel = [&](uint32_t u) {
    return double(column_sizes[u]) / double(std::max<uint32_t>(q.degree[u], 1));
  };
  while ((assigned & all) != all) {
    int best = -1;
    for (uint32_t u = 0; u < q.n; ++u) {
      if ((assigned >> u) & 1u) continue;
      if (!(q.adjmask[u] & assigned)) continue;  // prefix connectivity
      if (best < 0) {
        best = int(u);
        continue;
      }
      uint32_t bu = uint32_t(best);
      double su = sel(u), sb = sel(bu);
      if (su < sb || (su == sb && (q.degree[u] > q.degree[bu] ||
                                   (q.degree[u] == q.degree[bu] && u < bu)))) {
        best = int(u);
      }
    }
    if (best < 0) throw std::invalid_argument("disconnected query graph");
    order.push_back(uint32_t(best));
    assigned |= 1u << best;
  }
  return order;
}

EdgeProg build_program(const HostQuery& q, uint32_t query_index, const std::vector<uint32_t>& order,
                       const std::vector<std::pair<uint32_t, uint32_t>>& label_range,
                       const std::vector<uint32_t>& label_class) {
  EdgeProg p{};
  p.n = q.n;
  p.query = query_index;
  for (uint32_t i = 0; i < q.n; ++i) p.order[i] = order[i];
  for (uint32_t l = 0; l < q.n; ++l) {
    LevelProg& lp = p.lv[l];
    uint32_t u = order[l];
    lp.qbit = 1u << u;
    lp.vlo = label_range[u].first;
    lp.vhi = label_range[u].second;
    lp.lcls = label_class[u];
    lp.nback = 0;
    for (uint32_t j = 0; j < l; ++j) {
      if (q.adjacent(order[j], u)) {
        lp.backmask |= 1u << j;
        lp.back[lp.nback] = uint8_t(j);
        lp.elab[lp.nback] = q.edge_label(order[j], u);
        ++lp.nback;
      }
      if (q.labels[order[j]] == q.labels[u]) lp.eqmask |= 1u << j;
    }
  }
  // Counted tail.  T is the deepest level the kernel enumerates; every level
  // t > T is counted instead, and must be either
  //  * independent: all backward neighbours before T and no same-label
  //    position at or after T — its candidate set depends only on M[0..T),
  //    so its count is computed once per prefix (cached per warp) and
  //    multiplied; or
  //  * a leaf of T: T is its only backward neighbour and its only possible
  //    same-label position — its count is a function of M[T] alone, the
  //    per-vertex weight f(M[T]) memoised across the launch.
  // Tail levels are pairwise non-adjacent (by construction) and carry
  // pairwise distinct labels, so no injectivity couples them.
  auto counted = [&](uint32_t T) {
    for (uint32_t t = T + 1; t < q.n; ++t) {
      const LevelProg& lp = p.lv[t];
      const bool indep = (lp.backmask >> T) == 0 && (lp.eqmask >> T) == 0;
      const bool leaf = lp.backmask == (1u << T) && (lp.eqmask & ~(1u << T)) == 0;
      if (!indep && !leaf) return false;
      for (uint32_t s2 = T + 1; s2 < t; ++s2)
        if (q.labels[order[s2]] == q.labels[order[t]]) return false;
    }
    return true;
  };
  p.tail = q.n >= 3 ? q.n - 1 : 0;
  while (p.tail > 2 && counted(p.tail - 1)) --p.tail;
  p.leafmask = 0;
  p.natail = 0;
  for (uint32_t t = 0; t < uint32_t(kMaxQ); ++t) p.atail_slot[t] = 0xff;
  for (uint32_t t = p.tail + 1; t < q.n; ++t) {
    const LevelProg& lp = p.lv[t];
    if ((lp.backmask >> p.tail) != 0) {  // leaf of T: weight memoised per M[T]
      p.leafmask |= 1u << t;
      p.sig[t] = (order[p.tail] << 4) | order[t];
      continue;
    }
    const uint32_t dep = lp.backmask | lp.eqmask;  // what level t's candidate set depends on
    for (uint32_t j = 0; j < q.n; ++j)
      if ((dep >> j) & 1u) p.inval[j] |= 1u << t;
    // a single backward neighbour j (and no other same-label position): the
    // count is the memoised per-vertex weight of M[j], like a leaf of T
    if (lp.nback == 1 && (lp.eqmask & ~lp.backmask) == 0) {
      p.singlemask |= 1u << t;
      p.sig[t] = (order[lp.back[0]] << 4) | order[t];
    } else if ((dep & ~3u) == 0) {
      // depends on the anchor pair only: one count per task, shared by all of
      // the task's work items (EdgeProg::atail_slot)
      p.atail_slot[t] = uint8_t(p.natail++);
    }
  }
  return p;
}

namespace {

// Backtracking over label-, degree- and edge-label-preserving vertex
// permutations, adjacency checked against every vertex already mapped (the
// pruning of the reference's automorphism_backtrack, src/query_analysis.cpp:43-80).
void auto_backtrack(const HostQuery& q, std::vector<uint32_t>& image, uint32_t used, uint32_t depth,
                    std::vector<std::vector<uint32_t>>& out, size_t limit, bool& truncated) {
  if (truncated) return;
  if (depth == q.n) {
    if (out.size() >= limit) {
      truncated = true;
      return;
    }
    out.push_back(image);
    return;
  }
  for (uint32_t c = 0; c < q.n; ++c) {
    if ((used >> c) & 1u) continue;
    if (q.labels[c] != q.labels[depth] || q.degree[c] != q.degree[depth]) continue;
    bool ok = true;
    for (uint32_t j = 0; j < depth && ok; ++j) {
      const bool e0 = q.adjacent(depth, j), e1 = q.adjacent(c, image[j]);
      ok = e0 == e1 && (!e0 || q.edge_label(depth, j) == q.edge_label(c, image[j]));
    }
    if (!ok) continue;
    image[depth] = c;
    auto_backtrack(q, image, used | (1u << c), depth + 1, out, limit, truncated);
    if (truncated) return;
  }
}

}  // namespace

bool automorphisms(const HostQuery& q, size_t limit, std::vector<std::vector<uint32_t>>& out) {
  out.clear();
  std::vector<uint32_t> image(q.n, 0);
  bool truncated = false;
  auto_backtrack(q, image, 0, 0, out, limit, truncated);
  return !truncated;
}

std::vector<uint32_t> directed_edge_orbits(const HostQuery& q, size_t limit) {
  const size_t m = q.edges.size();
  std::vector<uint32_t> mult(2 * m, 1);
  std::vector<std::vector<uint32_t>> autos;
  if (!automorphisms(q, limit, autos)) return mult;  // too symmetric to enumerate: every edge its own orbit
  auto dir_index = [&](uint32_t x, uint32_t y) -> uint32_t {
    for (uint32_t e = 0; e < m; ++e) {
      if (q.edges[e].a == x && q.edges[e].b == y) return 2 * e;
      if (q.edges[e].a == y && q.edges[e].b == x) return 2 * e + 1;
    }
    throw std::logic_error("automorphism does not preserve the edge set");
  };
  // union-find over directed edges d = 2e + flip, flip 0 = (a, b), 1 = (b, a)
  std::vector<uint32_t> parent(2 * m);
  for (uint32_t d = 0; d < 2 * m; ++d) parent[d] = d;
  auto find = [&](uint32_t d) {
    while (parent[d] != d) d = parent[d] = parent[parent[d]];
    return d;
  };
  for (const auto& phi : autos) {
    for (uint32_t e = 0; e < m; ++e) {
      const uint32_t x = q.edges[e].a, y = q.edges[e].b;
      const uint32_t fwd = find(2 * e), f2 = find(dir_index(phi[x], phi[y]));
      const uint32_t rev = find(2 * e + 1), r2 = find(dir_index(phi[y], phi[x]));
      parent[std::max(fwd, f2)] = std::min(fwd, f2);
      const uint32_t rr = find(rev), rr2 = find(r2);
      parent[std::max(rr, rr2)] = std::min(rr, rr2);
    }
  }
  std::fill(mult.begin(), mult.end(), 0u);
  for (uint32_t d = 0; d < 2 * m; ++d) ++mult[find(d)];
  return mult;
}

void shard_owners(const uint64_t* costs, size_t n, uint32_t world, uint32_t* owners) {
  if (world <= 1) {
    std::fill(owners, owners + n, 0u);
    return;
  }
  unsigned __int128 total = 0;
  for (size_t k = 0; k < n; ++k) total += costs[k];
  unsigned __int128 prefix = 0;
  for (size_t k = 0; k < n; ++k) {
    owners[k] = total ? uint32_t((prefix * world) / total) : 0;
    prefix += costs[k];
  }
}

}  // namespace bdsm_b200
