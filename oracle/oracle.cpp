// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
// See oracle.hpp for the contract and the reference lines each part follows.

#include "oracle.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <omp.h>
#include <bit>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

constexpr std::uint32_t kNone = 0xffffffffu;

std::uint64_t pair_key(std::uint32_t u, std::uint32_t v) {  // types.hpp:16-23
  if (u > v) std::swap(u, v);
  return (static_cast<std::uint64_t>(u) << 32) | v;
}

void set_err(char* err, std::size_t cap, const std::string& msg) {
  if (!err || cap == 0) return;
  std::size_t n = std::min(cap - 1, msg.size());
  std::memcpy(err, msg.data(), n);
  err[n] = '\0';
}

struct Graph {
  std::vector<std::uint32_t> labels;
  std::vector<std::vector<std::uint32_t>> adj;  // sorted, both directions
  std::unordered_map<std::uint64_t, std::uint32_t> elab;

  bool has_edge(std::uint32_t u, std::uint32_t v) const {
    const auto& a = adj[u];
    return std::binary_search(a.begin(), a.end(), v);
  }
  std::uint32_t edge_label(std::uint32_t u, std::uint32_t v) const {
    auto it = elab.find(pair_key(u, v));
    return it == elab.end() ? kNone : it->second;
  }
};

struct QEdge {
  std::uint32_t a, b, label;
};

struct Query {
  std::uint32_t n = 0;
  std::vector<std::uint32_t> labels;
  std::vector<QEdge> edges;
  std::vector<std::uint32_t> adjmask;
  std::vector<std::uint32_t> degree;

  bool adjacent(std::uint32_t u, std::uint32_t v) const { return (adjmask[u] >> v) & 1u; }
  int edge_index(std::uint32_t u, std::uint32_t v) const {  // query_graph.cpp:29-35
    for (std::size_t i = 0; i < edges.size(); ++i) {
      if ((edges[i].a == u && edges[i].b == v) || (edges[i].a == v && edges[i].b == u)) return int(i);
    }
    return -1;
  }
  std::uint32_t edge_label(std::uint32_t u, std::uint32_t v) const {
    int i = edge_index(u, v);
    return i < 0 ? kNone : edges[std::size_t(i)].label;
  }
};

// Per-phase memo of column(u) ∩ N(x) for long lists: the graph and the
// candidate rows are fixed within a phase, so the filtered list is a function
// of (x, u).  Lists live until the memo is reset at the next phase.
struct ColListMemo {
  std::vector<std::atomic<const std::vector<std::uint32_t>*>> cell;  // [V * n]
  std::vector<std::unique_ptr<std::vector<std::uint32_t>>> owned;
  std::mutex m;
  std::uint32_t n = 0;
  void reset(std::size_t V, std::uint32_t qn) {
    if (n != qn || cell.size() != V * qn) {
      n = qn;
      cell = std::vector<std::atomic<const std::vector<std::uint32_t>*>>(V * qn);
    } else if (!owned.empty()) {
      for (auto& c : cell) c.store(nullptr, std::memory_order_relaxed);
    }
    owned.clear();
  }
};

// Per-query filter state: encoding.cpp's scheme + per-vertex saturated
// neighbour-label counters + CandidateTable rows and sorted columns.
struct QState {
  Query q;
  std::vector<std::uint32_t> group_labels;  // sorted distinct query labels
  std::uint32_t cap = 3;
  std::vector<std::uint8_t> qcnt;           // [n][G]
  std::vector<std::uint8_t> vcnt;           // [V][G]
  std::vector<std::uint32_t> rows;          // [V]
  std::vector<std::uint64_t> colsize;       // |column(u)| (columns = rows' bits, encoding.hpp:95-97)
  std::vector<std::vector<std::uint32_t>> orders;  // per query edge
  std::shared_ptr<ColListMemo> memo = std::make_shared<ColListMemo>();

  int group_index(std::uint32_t l) const {
    auto it = std::lower_bound(group_labels.begin(), group_labels.end(), l);
    if (it == group_labels.end() || *it != l) return -1;
    return int(it - group_labels.begin());
  }
  std::size_t G() const { return group_labels.size(); }

  void encode_vertex(const Graph& g, std::uint32_t v, std::uint8_t* out) const {  // encoding.cpp:70-87
    std::vector<std::uint32_t> c(G(), 0);
    for (std::uint32_t w : g.adj[v]) {
      int gi = group_index(g.labels[w]);
      if (gi >= 0) ++c[std::size_t(gi)];
    }
    for (std::size_t i = 0; i < G(); ++i) out[i] = std::uint8_t(std::min(c[i], cap));
  }
  std::uint32_t compute_row(const Graph& g, std::uint32_t v) const {  // encoding.cpp:115-122,145-153
    std::uint32_t row = 0;
    const std::uint8_t* dv = &vcnt[std::size_t(v) * G()];
    for (std::uint32_t u = 0; u < q.n; ++u) {
      if (g.labels[v] != q.labels[u]) continue;  // exact label compare (F5)
      bool ok = true;
      const std::uint8_t* du = &qcnt[std::size_t(u) * G()];
      for (std::size_t gi = 0; gi < G() && ok; ++gi) ok = dv[gi] >= du[gi];
      if (ok) row |= 1u << u;
    }
    return row;
  }
};

struct Update {
  std::uint32_t u, v, label, order;
  bool insert;
};

struct Stats {
  std::uint64_t visits = 0, iops = 0, tasks = 0, calls = 0, balg = 0, emitted = 0;
  // visits outside the subtrees of candidates whose edge to an earlier
  // position is hidden by dedupe_by_order: the tree the CUDA engine walks
  // (it applies the rule when it generates candidates, not when it emits)
  std::uint64_t vpruned = 0;
  void add(const Stats& o) {
    visits += o.visits;
    vpruned += o.vpruned;
    iops += o.iops;
    tasks += o.tasks;
    calls += o.calls;
    balg += o.balg;
    emitted += o.emitted;
  }
};

struct Task {
  std::uint32_t upd;
  std::uint32_t edge;
  bool flipped;
  std::uint32_t lo, hi;  // level-2 driver range owned by this shard (hi = ~0: all)
  bool whole;
};

}  // namespace

struct orc_engine {
  Graph g;
  std::uint32_t group_bits = 2;
  std::vector<QState> queries;
  std::vector<std::pair<std::uint64_t, std::uint32_t>> errors;
};

namespace {

// try_order with zone = 0 and no tail (query_analysis.cpp:295-354).
std::vector<std::uint32_t> matching_order(const QState& qs, std::uint32_t e) {
  const Query& q = qs.q;
  std::vector<std::uint32_t> order{q.edges[e].a, q.edges[e].b};
  std::uint32_t assigned = (1u << q.edges[e].a) | (1u << q.edges[e].b);
  std::uint32_t all = q.n == 32 ? ~0u : (1u << q.n) - 1;
  auto sel = [&](std::uint32_t u) {
    return double(qs.colsize[u]) / double(std::max<std::uint32_t>(q.degree[u], 1));
  };
  while ((assigned & all) != all) {
    int best = -1;
    for (std::uint32_t u = 0; u < q.n; ++u) {
      if ((assigned >> u) & 1u) continue;
      if (!(q.adjmask[u] & assigned)) continue;
      if (best < 0) {
        best = int(u);
        continue;
      }
      std::uint32_t bu = std::uint32_t(best);
      double su = sel(u), sb = sel(bu);
      if (su < sb || (su == sb && (q.degree[u] > q.degree[bu] ||
                                   (q.degree[u] == q.degree[bu] && u < bu)))) {
        best = int(u);
      }
    }
    if (best < 0) throw std::invalid_argument("disconnected query graph");
    order.push_back(std::uint32_t(best));
    assigned |= 1u << best;
  }
  return order;
}

// Reference intersect_sorted (matcher.cpp:59-73) charges
// size(small) * (1 + bit_width(size(large))) intersection_ops per call; the
// set it returns is small ∩ large in ascending order.  The restatement
// computes the same sets (the first, column-sided intersection by row-bit
// filtering, since column(u) = {v : row[v] bit u}, encoding.hpp:95-97; the
// rest by binary search) and charges the same ops from the operand sizes, so
// intersection_ops stays equal to the reference's.
inline std::uint64_t iops_of(std::uint64_t a, std::uint64_t b) {
  std::uint64_t small = std::min(a, b), large = std::max(a, b);
  return small * (1 + std::uint64_t(std::bit_width(large)));
}

// labeled_neighbors with oracle semantics (F4): unlabelled query edges accept
// only unlabelled data edges.
const std::vector<std::uint32_t>& labeled_neighbors(const Graph& g, std::uint32_t v,
                                                    std::uint32_t el,
                                                    std::vector<std::uint32_t>& scratch) {
  if (g.elab.empty() && el == kNone) return g.adj[v];
  scratch.clear();
  for (std::uint32_t w : g.adj[v]) {
    if (g.edge_label(v, w) == el) scratch.push_back(w);
  }
  return scratch;
}

// Same-kind updates of the phase incident to a vertex, for the visibility
// rule on counted last levels: sorted (vertex << 32 | other, order).
struct UpdAdj {
  std::vector<std::pair<std::uint64_t, std::uint32_t>> e;
  template <typename F>
  void for_each(std::uint32_t x, F&& f) const {
    auto it = std::lower_bound(e.begin(), e.end(), std::make_pair(std::uint64_t(x) << 32, 0u));
    for (; it != e.end() && (it->first >> 32) == x; ++it) f(std::uint32_t(it->first), it->second);
  }
};

struct Ctx {
  const Graph& g;
  const QState& qs;
  const std::vector<Update>& ups;
  const std::unordered_map<std::uint64_t, std::uint32_t>& order_by_pair;  // UpdateIndex
  const std::vector<std::uint8_t>& endpoint;  // v is an endpoint of a same-kind update
  const UpdAdj& upd_adj;
  ColListMemo& memo;
  bool fast;  // no edge labels anywhere: neighbour lists are the adjacency itself
};

// Lists at or above this length use the memoised column counts (first
// intersection) and the counted last level; 0 forces them everywhere (tests).
std::size_t memo_min() {
  static const std::size_t v = [] {
    const char* e = std::getenv("ORC_MEMO_MIN");
    return e ? std::size_t(std::strtoull(e, nullptr, 10)) : std::size_t(512);
  }();
  return v;
}

const std::vector<std::uint32_t>& col_list(const Ctx& c, std::uint32_t x, std::uint32_t u) {
  auto& cell = c.memo.cell[std::size_t(x) * c.memo.n + u];
  if (const auto* p = cell.load(std::memory_order_acquire)) return *p;
  const std::uint32_t ubit = 1u << u;
  auto fresh = std::make_unique<std::vector<std::uint32_t>>();
  for (std::uint32_t y : c.g.adj[x]) {
    if (c.qs.rows[y] & ubit) fresh->push_back(y);
  }
  const std::vector<std::uint32_t>* expect = nullptr;
  const std::vector<std::uint32_t>* mine = fresh.get();
  if (cell.compare_exchange_strong(expect, mine, std::memory_order_acq_rel)) {
    std::lock_guard<std::mutex> lk(c.memo.m);
    c.memo.owned.push_back(std::move(fresh));
    return *mine;
  }
  return *expect;
}

// Backward-neighbour lists of position `level` in ascending i.
struct BackLists {
  const std::vector<std::uint32_t>* l[32];
  std::uint32_t who[32];
  std::size_t m = 0;
};

void back_lists(const Ctx& c, const std::vector<std::uint32_t>& order, const std::uint32_t* assign,
                std::size_t level, BackLists& bl, Stats& st) {
  const Query& q = c.qs.q;
  const std::uint32_t u = order[level];
  bl.m = 0;
  for (std::size_t i = 0; i < level; ++i) {
    if (!q.adjacent(order[i], u)) continue;
    st.balg += 4ull * c.g.adj[assign[i]].size();
    bl.l[bl.m] = &c.g.adj[assign[i]];
    bl.who[bl.m++] = assign[i];
  }
}

void erase_assigned(std::vector<std::uint32_t>& res, const std::uint32_t* assign, std::size_t level) {
  if (res.empty()) return;
  std::erase_if(res, [&](std::uint32_t v) {
    for (std::size_t i = 0; i < level; ++i) {
      if (assign[i] == v) return true;
    }
    return false;
  });
}

// Sorted-set intersection small ∩ large (both ascending) by galloping from
// the previous match position: the result equals the reference's binary
// search of each element of the smaller list (matcher.cpp:59-73).
template <typename Keep>
void gallop_intersect(const std::vector<std::uint32_t>& small, const std::vector<std::uint32_t>& large,
                      std::vector<std::uint32_t>& out, Keep&& keep) {
  const std::uint32_t* lo = large.data();
  const std::uint32_t* const end = lo + large.size();
  for (std::uint32_t x : small) {
    if (lo == end) break;
    if (!keep(x)) continue;
    std::size_t step = 1;
    const std::uint32_t* hi = lo;
    while (hi < end && *hi < x) {
      lo = hi + 1;
      hi = lo + step - 1 < end ? lo + step - 1 : end;
      step <<= 1;
    }
    lo = std::lower_bound(lo, hi < end ? hi + 1 : end, x);
    if (lo != end && *lo == x) out.push_back(x);
  }
}

// gen_candidates (matcher.cpp:87-108), general form (edge labels): column(u)
// ∩ N(M(π[i])) over the backward neighbours i < level in ascending i,
// stopping once empty, then the already-assigned vertices removed.
void gen_candidates_labelled(const Ctx& c, const std::vector<std::uint32_t>& order,
                             const std::uint32_t* assign, std::size_t level,
                             std::vector<std::uint32_t>& res, Stats& st) {
  const Query& q = c.qs.q;
  const std::uint32_t u = order[level];
  const std::uint32_t ubit = 1u << u;
  for (std::size_t i = 0; i < level; ++i) {
    if (q.adjacent(order[i], u)) st.balg += 4ull * c.g.adj[assign[i]].size();
  }
  static thread_local std::vector<std::uint32_t> scratch, tmp;
  std::uint64_t cur = c.qs.colsize[u];
  bool own = false;
  res.clear();
  for (std::size_t i = 0; i < level && cur != 0; ++i) {
    std::uint32_t prev = order[i];
    if (!q.adjacent(prev, u)) continue;
    const auto& nbrs = labeled_neighbors(c.g, assign[i], q.edge_label(prev, u), scratch);
    st.iops += iops_of(cur, nbrs.size());
    if (!own) {
      for (std::uint32_t x : nbrs) {
        if (c.qs.rows[x] & ubit) res.push_back(x);
      }
      own = true;
    } else {
      tmp.clear();
      const bool res_small = res.size() <= nbrs.size();
      const auto& small = res_small ? res : nbrs;
      const auto& large = res_small ? nbrs : res;
      for (std::uint32_t x : small) {
        if (std::binary_search(large.begin(), large.end(), x)) tmp.push_back(x);
      }
      res.swap(tmp);
    }
    cur = res.size();
  }
  if (!own && cur != 0) {  // no backward neighbour (unreachable for a prefix-connected order)
    for (std::uint32_t v = 0; v < c.qs.rows.size(); ++v) {
      if (c.qs.rows[v] & ubit) res.push_back(v);
    }
  }
  erase_assigned(res, assign, level);
}

// gen_candidates (matcher.cpp:87-108) without edge labels.  The reference
// intersects column(u) with N_0, then the result with N_1, ... (ascending i);
// the candidate set is the same whatever the order, so it is computed from
// the shorter lists, while intersection_ops is charged on the reference's
// sequence of operand sizes: |column(u)|, then |column ∩ N_0| (memoised for
// long N_0), |column ∩ N_0 ∩ N_1|, ...
void gen_candidates(const Ctx& c, const std::vector<std::uint32_t>& order,
                    const std::uint32_t* assign, std::size_t level,
                    std::vector<std::uint32_t>& res, Stats& st) {
  ++st.calls;
  if (!c.fast) {
    gen_candidates_labelled(c, order, assign, level, res, st);
    return;
  }
  const std::uint32_t u = order[level];
  const std::uint32_t ubit = 1u << u;
  const auto& rows = c.qs.rows;
  BackLists bl;
  back_lists(c, order, assign, level, bl, st);
  static thread_local std::vector<std::uint32_t> tmp;
  res.clear();
  std::uint64_t cur = c.qs.colsize[u];
  if (bl.m == 0) {  // unreachable for a prefix-connected order
    for (std::uint32_t v = 0; cur != 0 && v < rows.size(); ++v) {
      if (rows[v] & ubit) res.push_back(v);
    }
    erase_assigned(res, assign, level);
    return;
  }
  if (cur == 0) return;
  const auto& n0 = *bl.l[0];
  st.iops += iops_of(cur, n0.size());
  std::size_t k = 1;
  if (n0.size() >= memo_min()) {
    // column ∩ N_0 from the memo
    const auto& f = col_list(c, bl.who[0], u);
    cur = f.size();
    if (cur == 0) return;
    if (bl.m >= 2) {  // ∩ N_1 from the shorter side
      const auto& n1 = *bl.l[1];
      st.iops += iops_of(cur, n1.size());
      const bool f_small = f.size() <= n1.size();
      const auto& small = f_small ? f : n1;
      const auto& large = f_small ? n1 : f;
      gallop_intersect(small, large, res, [&](std::uint32_t x) { return f_small || (rows[x] & ubit); });
      k = 2;
    } else {
      res.assign(f.begin(), f.end());
    }
    cur = res.size();
  } else {
    for (std::uint32_t x : n0) {
      if (rows[x] & ubit) res.push_back(x);
    }
    cur = res.size();
  }
  for (; k < bl.m && cur != 0; ++k) {
    const auto& nk = *bl.l[k];
    st.iops += iops_of(cur, nk.size());
    tmp.clear();
    const bool res_small = res.size() <= nk.size();
    gallop_intersect(res_small ? res : nk, res_small ? nk : res, tmp, [](std::uint32_t) { return true; });
    res.swap(tmp);
    cur = res.size();
  }
  erase_assigned(res, assign, level);
}

// dedupe_by_order (matcher.cpp:110-117) for one query edge's image: rejected
// iff the pair is a same-kind update of the batch with a lower order.  A pair
// with an endpoint outside the batch cannot be in the UpdateIndex.
inline bool edge_hidden(const Ctx& c, std::uint32_t x, std::uint32_t y, std::uint32_t anchor_order) {
  if (!c.endpoint[x] || !c.endpoint[y]) return false;
  auto it = c.order_by_pair.find(pair_key(x, y));
  return it != c.order_by_pair.end() && it->second < anchor_order;
}

struct TaskRun {
  const Ctx* c = nullptr;
  const std::vector<std::uint32_t>* order = nullptr;
  std::uint32_t anchor_order = 0;
  std::size_t n = 0;
  std::vector<std::uint32_t> pos_of;  // query vertex -> position in order
};

// Per-thread accumulators (padded against false sharing).
struct alignas(64) ThreadAcc {
  Stats st;
  std::uint64_t count = 0;
};

// The final level of run_match_task (matcher.cpp:258-309): every candidate is
// one dfs_visit and one emit_with_joins -> dedupe_by_order (matcher.cpp:169-217);
// the edges not incident to the last position are the same for every
// candidate, so they are checked once for the prefix.
void count_last(const TaskRun& tr, const std::uint32_t* assign, const std::vector<std::uint32_t>& last,
                Stats& st, std::uint64_t& count, bool pruned) {
  const Ctx& c = *tr.c;
  const Query& q = c.qs.q;
  st.visits += last.size();
  if (last.empty()) return;
  const std::uint32_t ul = (*tr.order)[tr.n - 1];
  for (const QEdge& e : q.edges) {
    if (e.a == ul || e.b == ul) continue;
    if (edge_hidden(c, assign[tr.pos_of[e.a]], assign[tr.pos_of[e.b]], tr.anchor_order)) return;
  }
  std::uint64_t ok = 0;
  for (std::uint32_t x : last) {
    bool pass = true;
    if (c.endpoint[x]) {
      for (const QEdge& e : q.edges) {
        if (e.a != ul && e.b != ul) continue;
        std::uint32_t other = assign[tr.pos_of[e.a == ul ? e.b : e.a]];
        if (edge_hidden(c, x, other, tr.anchor_order)) {
          pass = false;
          break;
        }
      }
    }
    ok += pass;
  }
  st.emitted += ok;
  count += ok;
  if (!pruned) st.vpruned += ok;
}

// The last position L of the order: gen_candidates for L, then count_last.
// With one backward neighbour x (every query edge of π[L] goes to it) and a
// long N(x), the candidate set is column(u) ∩ N(x) minus the assigned
// vertices, so its size is the memoised count minus the assigned vertices in
// it, and the matches dedupe_by_order rejects are the candidates c whose edge
// (x, c) is a same-kind update of lower order: they are enumerated from x's
// updates instead of from N(x).  Same counts and MatchStats as the list path.
void count_level_last(const TaskRun& tr, std::uint32_t* assign, std::size_t L, Stats& st,
                      std::uint64_t& count, bool pruned) {
  const Ctx& c = *tr.c;
  const auto& order = *tr.order;
  const std::uint32_t u = order[L];
  const Query& q = c.qs.q;
  if (c.fast && std::popcount(q.adjmask[u]) == 1) {
    std::size_t i0 = 0;
    while (!q.adjacent(order[i0], u)) ++i0;
    const std::uint32_t x = assign[i0];
    const auto& nx = c.g.adj[x];
    if (nx.size() >= memo_min()) {
      ++st.calls;
      st.balg += 4ull * nx.size();
      const std::uint64_t col = c.qs.colsize[u];
      if (col == 0) return;
      st.iops += iops_of(col, nx.size());
      const std::uint32_t ubit = 1u << u;
      std::uint64_t k = col_list(c, x, u).size();
      for (std::size_t i = 0; i < L; ++i) {
        std::uint32_t a = assign[i];
        if ((c.qs.rows[a] & ubit) && std::binary_search(nx.begin(), nx.end(), a)) --k;
      }
      st.visits += k;
      if (k == 0) return;
      for (const QEdge& e : q.edges) {
        if (e.a == u || e.b == u) continue;
        if (edge_hidden(c, assign[tr.pos_of[e.a]], assign[tr.pos_of[e.b]], tr.anchor_order)) return;
      }
      std::uint64_t hidden = 0;
      c.upd_adj.for_each(x, [&](std::uint32_t y, std::uint32_t ord) {
        if (ord >= tr.anchor_order || !(c.qs.rows[y] & ubit)) return;
        for (std::size_t i = 0; i < L; ++i) {
          if (assign[i] == y) return;
        }
        ++hidden;
      });
      st.emitted += k - hidden;
      count += k - hidden;
      if (!pruned) st.vpruned += k - hidden;
      return;
    }
  }
  static thread_local std::vector<std::uint32_t> last;
  gen_candidates(c, order, assign, L, last, st);
  count_last(tr, assign, last, st, count, pruned);
}

// Some query edge from an earlier position to position `level` maps onto a
// hidden pair (dedupe_by_order would reject every match below).
bool back_hidden(const TaskRun& tr, const std::uint32_t* assign, std::size_t level, std::uint32_t cand) {
  const Ctx& c = *tr.c;
  if (!c.endpoint[cand]) return false;
  const std::uint32_t u = (*tr.order)[level];
  for (std::size_t i = 0; i < level; ++i) {
    if (c.qs.q.adjacent((*tr.order)[i], u) && edge_hidden(c, assign[i], cand, tr.anchor_order)) return true;
  }
  return false;
}

// The DFS below `level` over that level's candidates.  The subtrees of the two
// shallowest levels run as separate OpenMP tasks, so a hub-anchored task
// spreads over the threads (the results are sums).
void dfs(const TaskRun& tr, std::uint32_t* assign, std::size_t level, const std::uint32_t* cands,
         std::size_t ncands, ThreadAcc* acc, bool pruned) {
  const std::size_t n = tr.n;
  const bool spawn = level + 2 < n && ncands > 1 && (level == 2 || (level == 3 && ncands > 64));
  if (spawn) {
    const std::size_t grain = level == 2 ? 1 : 16;
    for (std::size_t b = 0; b < ncands; b += grain) {
      std::size_t e = std::min(ncands, b + grain);
      std::array<std::uint32_t, 32> a{};
      std::copy(assign, assign + level, a.begin());
      std::vector<std::uint32_t> part(cands + b, cands + e);
#pragma omp task firstprivate(a, part, level, pruned) shared(tr) untied
      dfs(tr, a.data(), level, part.data(), part.size(), acc, pruned);
    }
    return;
  }
  std::vector<std::uint32_t> next;
  for (std::size_t k = 0; k < ncands; ++k) {
    ThreadAcc& me = acc[omp_get_thread_num()];
    assign[level] = cands[k];
    ++me.st.visits;
    const bool hid = pruned || back_hidden(tr, assign, level, cands[k]);
    if (!hid) ++me.st.vpruned;
    if (level + 2 == n) {
      count_level_last(tr, assign, level + 1, me.st, me.count, hid);
      continue;
    }
    gen_candidates(*tr.c, *tr.order, assign, level + 1, next, me.st);
    if (!next.empty()) {
      std::vector<std::uint32_t> mine;
      mine.swap(next);
      dfs(tr, assign, level + 1, mine.data(), mine.size(), acc, hid);
      next.swap(mine);
    }
  }
}

// Level-2 driver of a task: the smallest-degree backward neighbour of
// order[2] among the anchor positions (ties: position 0).  Shared with the
// CUDA engine's work-item split (paper_2401_17018_b200/csrc/match.cu).
std::uint32_t driver_vertex(const Graph& g, const QState& qs, const Task& t, const Update& up) {
  const auto& order = qs.orders[t.edge];
  std::uint32_t a0 = t.flipped ? up.v : up.u, a1 = t.flipped ? up.u : up.v;
  bool b0 = qs.q.adjacent(order[0], order[2]);
  bool b1 = qs.q.adjacent(order[1], order[2]);
  if (b0 && b1) return g.adj[a1].size() < g.adj[a0].size() ? a1 : a0;
  return b0 ? a0 : a1;
}

// run_match_task (matcher.cpp:219-310) for one anchor task, coalesce off:
// level-2 candidates (matcher.cpp:243-247), then the DFS.
void run_task(const Ctx& c, const Task& t, TaskRun& tr, ThreadAcc* acc) {
  const Update& up = c.ups[t.upd];
  const std::vector<std::uint32_t>& order = c.qs.orders[t.edge];
  const std::size_t n = order.size();
  tr.c = &c;
  tr.order = &order;
  tr.anchor_order = up.order;
  tr.n = n;
  tr.pos_of.assign(c.qs.q.n, 0);
  for (std::size_t i = 0; i < n; ++i) tr.pos_of[order[i]] = std::uint32_t(i);
  ThreadAcc& me = acc[omp_get_thread_num()];
  ++me.st.tasks;
  std::array<std::uint32_t, 32> assign{};
  assign[0] = t.flipped ? up.v : up.u;
  assign[1] = t.flipped ? up.u : up.v;
  if (n <= 2) {
    // a 2-vertex query's only match is the anchor itself (emit at matcher.cpp:237-241)
    bool hidden = false;
    for (const QEdge& e : c.qs.q.edges) {
      hidden = hidden || edge_hidden(c, assign[tr.pos_of[e.a]], assign[tr.pos_of[e.b]], tr.anchor_order);
    }
    if (!hidden) {
      ++me.count;
      ++me.st.emitted;
    }
    return;
  }
  std::vector<std::uint32_t> l2;
  gen_candidates(c, order, assign.data(), 2, l2, me.st);
  if (!t.whole) {  // shard restriction: level-2 values inside the owned driver range
    std::erase_if(l2, [&](std::uint32_t v) { return v < t.lo || v > t.hi; });
  }
  if (n == 3) {
    count_last(tr, assign.data(), l2, me.st, me.count, false);
    return;
  }
  dfs(tr, assign.data(), 2, l2.data(), l2.size(), acc, false);
}

std::uint64_t run_phase(orc_engine* h, QState& qs, const std::vector<Update>& ups, bool inserts,
                        std::uint32_t nthreads, std::uint32_t rank, std::uint32_t world,
                        Stats& total) {
  const Graph& g = h->g;
  const Query& q = qs.q;
  std::unordered_map<std::uint64_t, std::uint32_t> order_by_pair;  // UpdateIndex::build
  std::vector<std::uint8_t> endpoint(g.labels.size(), 0);
  for (const Update& up : ups) {
    if (up.insert != inserts) continue;
    order_by_pair.emplace(pair_key(up.u, up.v), up.order);
    endpoint[up.u] = endpoint[up.v] = 1;
  }
  // match_phase task construction (matcher.cpp:334-354).
  std::vector<Task> tasks;
  for (std::uint32_t i = 0; i < ups.size(); ++i) {
    const Update& up = ups[i];
    if (up.insert != inserts) continue;
    std::uint32_t el = up.insert ? up.label : g.edge_label(up.u, up.v);
    std::uint32_t lu = g.labels[up.u], lv = g.labels[up.v];
    for (std::uint32_t e = 0; e < q.edges.size(); ++e) {
      const QEdge& qe = q.edges[e];
      if (qe.label != el) continue;
      if (q.labels[qe.a] == lu && q.labels[qe.b] == lv) tasks.push_back({i, e, false, 0, kNone, true});
      if (q.labels[qe.a] == lv && q.labels[qe.b] == lu) tasks.push_back({i, e, true, 0, kNone, true});
    }
  }
  if (world > 1) {
    // Cost-balanced split over (task, level-2 driver chunk) items in canonical
    // order; item k goes to rank floor(world * prefix_k / total).
    constexpr std::uint64_t kChunk = 64;
    struct Item {
      std::uint32_t task;
      std::uint64_t begin, end;
    };
    std::vector<Item> items;
    std::vector<std::uint64_t> cost;
    for (std::uint32_t ti = 0; ti < tasks.size(); ++ti) {
      const Task& t = tasks[ti];
      if (q.n <= 2) {
        items.push_back({ti, 0, 1});
        cost.push_back(1);
        continue;
      }
      std::uint64_t d = g.adj[driver_vertex(g, qs, t, ups[t.upd])].size();
      for (std::uint64_t b = 0; b < d; b += kChunk) {
        items.push_back({ti, b, std::min(d, b + kChunk)});
        cost.push_back(std::min(d, b + kChunk) - b);
      }
    }
    std::uint64_t T = 0;
    for (auto c : cost) T += c;
    std::vector<Task> mine;
    std::uint64_t P = 0;
    for (std::size_t k = 0; k < items.size(); ++k) {
      std::uint64_t owner = T ? (P * world) / T : 0;
      P += cost[k];
      if (owner != rank) continue;
      Task t = tasks[items[k].task];
      if (q.n > 2) {
        const auto& dl = g.adj[driver_vertex(g, qs, t, ups[t.upd])];
        t.whole = false;
        t.lo = dl[items[k].begin];
        t.hi = dl[items[k].end - 1];
      }
      mine.push_back(t);
    }
    tasks.swap(mine);
  }
  UpdAdj upd_adj;
  for (const Update& up : ups) {
    if (up.insert != inserts) continue;
    upd_adj.e.push_back({(std::uint64_t(up.u) << 32) | up.v, up.order});
    upd_adj.e.push_back({(std::uint64_t(up.v) << 32) | up.u, up.order});
  }
  std::sort(upd_adj.e.begin(), upd_adj.e.end());
  bool fast = g.elab.empty();
  for (const QEdge& e : q.edges) fast = fast && e.label == kNone;
  qs.memo->reset(g.labels.size(), q.n);
  Ctx ctx{g, qs, ups, order_by_pair, endpoint, upd_adj, *qs.memo, fast};
  const std::uint32_t nt = std::max(1u, nthreads);
  std::vector<ThreadAcc> acc(nt);
  std::vector<TaskRun> runs(tasks.size());
#pragma omp parallel num_threads(nt)
#pragma omp single
  for (std::size_t i = 0; i < tasks.size(); ++i) {
#pragma omp task firstprivate(i) shared(ctx, tasks, runs, acc) untied
    run_task(ctx, tasks[i], runs[i], acc.data());
  }
  std::uint64_t count = 0;
  for (auto& a : acc) {
    total.add(a.st);
    count += a.count;
  }
  return count;
}

void insert_sorted(std::vector<std::uint32_t>& v, std::uint32_t x) {
  v.insert(std::lower_bound(v.begin(), v.end(), x), x);
}
void erase_sorted(std::vector<std::uint32_t>& v, std::uint32_t x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it != v.end() && *it == x) v.erase(it);
}

}  // namespace

extern "C" {

orc_engine* orc_create(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                       const std::uint32_t* eu, const std::uint32_t* ev,
                       const std::uint32_t* elab, std::uint32_t group_bits, char* err,
                       std::size_t errcap) {
  try {
    auto* h = new orc_engine();
    h->group_bits = group_bits;
    Graph& g = h->g;
    g.labels.assign(vlabels, vlabels + nv);
    g.adj.assign(nv, {});
    // graph.cpp:52-68 (self-loops, unknown vertices and duplicates rejected),
    // built in parallel: degree count, fill, per-list sort
    std::uint64_t first_bad = ne;
#pragma omp parallel for reduction(min : first_bad) schedule(static)
    for (std::uint64_t i = 0; i < ne; ++i) {
      if (eu[i] == ev[i] || eu[i] >= nv || ev[i] >= nv) first_bad = std::min(first_bad, i);
    }
    if (first_bad < ne) {
      std::uint32_t u = eu[first_bad], v = ev[first_bad];
      if (u == v) throw std::invalid_argument("self-loop edge (" + std::to_string(u) + "," + std::to_string(v) + ")");
      throw std::invalid_argument("edge references unknown vertex");
    }
    if (elab) {
      for (std::uint64_t i = 0; i < ne; ++i) {
        if (elab[i] != kNone) g.elab[pair_key(eu[i], ev[i])] = elab[i];
      }
    }
    std::vector<std::uint64_t> deg(nv, 0);
#pragma omp parallel for schedule(static)
    for (std::uint64_t i = 0; i < ne; ++i) {
      std::atomic_ref<std::uint64_t>(deg[eu[i]]).fetch_add(1, std::memory_order_relaxed);
      std::atomic_ref<std::uint64_t>(deg[ev[i]]).fetch_add(1, std::memory_order_relaxed);
    }
#pragma omp parallel for schedule(dynamic, 4096)
    for (std::uint64_t v = 0; v < nv; ++v) {
      g.adj[v].resize(deg[v]);
      deg[v] = 0;
    }
#pragma omp parallel for schedule(static)
    for (std::uint64_t i = 0; i < ne; ++i) {
      std::uint32_t u = eu[i], v = ev[i];
      g.adj[u][std::atomic_ref<std::uint64_t>(deg[u]).fetch_add(1, std::memory_order_relaxed)] = v;
      g.adj[v][std::atomic_ref<std::uint64_t>(deg[v]).fetch_add(1, std::memory_order_relaxed)] = u;
    }
    int dup = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : dup)
    for (std::uint64_t v = 0; v < nv; ++v) {
      auto& a = g.adj[v];
      std::sort(a.begin(), a.end());
      for (std::size_t i = 1; i < a.size(); ++i) dup |= a[i] == a[i - 1];
    }
    if (dup) throw std::invalid_argument("duplicate edge");
    return h;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return nullptr;
  }
}

int orc_add_query(orc_engine* h, std::uint32_t n, const std::uint32_t* qlabels, std::uint32_t m,
                  const std::uint32_t* qa, const std::uint32_t* qb, const std::uint32_t* qlab,
                  char* err, std::size_t errcap) {
  try {
    QState qs;
    Query& q = qs.q;
    if (n == 0) throw std::invalid_argument("empty query graph");
    if (n > 32) throw std::invalid_argument("query graph too large");
    q.n = n;
    q.labels.assign(qlabels, qlabels + n);
    q.adjmask.assign(n, 0);
    q.degree.assign(n, 0);
    for (std::uint32_t i = 0; i < m; ++i) {  // query_graph.cpp:10-27
      QEdge e{qa[i], qb[i], qlab ? qlab[i] : kNone};
      if (e.a >= n || e.b >= n) throw std::invalid_argument("query edge references unknown vertex");
      if (e.a == e.b) throw std::invalid_argument("query self-loop");
      if (q.adjacent(e.a, e.b)) throw std::invalid_argument("duplicate query edge");
      q.adjmask[e.a] |= 1u << e.b;
      q.adjmask[e.b] |= 1u << e.a;
      ++q.degree[e.a];
      ++q.degree[e.b];
      q.edges.push_back(e);
    }
    {  // connected() (query_graph.cpp:43-55)
      std::uint32_t seen = 1, frontier = 1;
      while (frontier) {
        std::uint32_t next = 0;
        for (std::uint32_t u = 0; u < n; ++u) {
          if ((frontier >> u) & 1u) next |= q.adjmask[u];
        }
        frontier = next & ~seen;
        seen |= next;
      }
      if (seen != (n == 32 ? ~0u : (1u << n) - 1)) throw std::invalid_argument("disconnected query graph");
    }
    // build_scheme / encode_query / encode_all / CandidateTable::build.
    qs.group_labels = q.labels;
    std::sort(qs.group_labels.begin(), qs.group_labels.end());
    qs.group_labels.erase(std::unique(qs.group_labels.begin(), qs.group_labels.end()), qs.group_labels.end());
    qs.cap = (1u << h->group_bits) - 1;
    std::size_t G = qs.G();
    qs.qcnt.assign(std::size_t(n) * G, 0);
    for (std::uint32_t u = 0; u < n; ++u) {
      std::vector<std::uint32_t> c(G, 0);
      for (std::uint32_t w = 0; w < n; ++w) {
        if (q.adjacent(u, w)) ++c[std::size_t(qs.group_index(q.labels[w]))];
      }
      for (std::size_t gi = 0; gi < G; ++gi) qs.qcnt[u * G + gi] = std::uint8_t(std::min(c[gi], qs.cap));
    }
    const Graph& g = h->g;
    std::size_t V = g.labels.size();
    qs.vcnt.assign(V * G, 0);
    qs.rows.assign(V, 0);
    qs.colsize.assign(n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
    for (std::size_t v = 0; v < V; ++v) {
      qs.encode_vertex(g, std::uint32_t(v), &qs.vcnt[v * G]);
      qs.rows[v] = qs.compute_row(g, std::uint32_t(v));
    }
    for (std::size_t v = 0; v < V; ++v) {
      for (std::uint32_t r = qs.rows[v]; r; r &= r - 1) ++qs.colsize[std::countr_zero(r)];
    }
    for (std::uint32_t e = 0; e < m; ++e) qs.orders.push_back(matching_order(qs, e));
    h->queries.push_back(std::move(qs));
    return int(h->queries.size() - 1);
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return -ORC_INVALID_ARGUMENT;
  }
}

int orc_apply_batch(orc_engine* h, std::uint64_t n, const std::uint32_t* uu,
                    const std::uint32_t* uv, const std::uint8_t* uop, const std::uint32_t* ulab,
                    std::uint32_t nthreads, std::uint32_t shard_rank, std::uint32_t shard_world,
                    std::uint64_t* pos, std::uint64_t* neg, std::uint64_t* stats, char* err,
                    std::size_t errcap) {
  try {
    Graph& g = h->g;
    h->errors.clear();
    std::vector<Update> ups(n);
    std::unordered_set<std::uint64_t> seen;  // UpdateBatch ctor (graph.cpp:8-23)
    for (std::uint64_t i = 0; i < n; ++i) {
      Update& up = ups[i];
      up = {uu[i], uv[i], ulab ? ulab[i] : kNone, std::uint32_t(i), uop[i] == 0};
      if (up.u == up.v) {
        set_err(err, errcap, "self-loop update (" + std::to_string(up.u) + "," + std::to_string(up.v) + ")");
        return ORC_INVALID_ARGUMENT;
      }
      if (!seen.insert(pair_key(up.u, up.v)).second) {
        set_err(err, errcap, "conflicting updates on edge (" + std::to_string(up.u) + "," +
                                 std::to_string(up.v) + ") within one batch");
        return ORC_INVALID_ARGUMENT;
      }
    }
    std::size_t V = g.labels.size();
    for (std::uint64_t i = 0; i < n; ++i) {  // validate_batch (graph.cpp:117-135)
      const Update& up = ups[i];
      if (up.u >= V || up.v >= V) {
        h->errors.push_back({i, 1});
        continue;
      }
      bool present = g.has_edge(up.u, up.v);
      if (up.insert && present) h->errors.push_back({i, 2});
      else if (!up.insert && !present) h->errors.push_back({i, 3});
    }
    if (!h->errors.empty()) {
      set_err(err, errcap, "batch rejected: " + std::to_string(h->errors.size()) +
                               " invalid update(s), none applied");
      return ORC_BATCH_ERROR;
    }
    Stats st;
    if (shard_world == 0) shard_world = 1;
    const bool match = pos != nullptr && neg != nullptr;  // null: apply + refresh only
    for (std::size_t qi = 0; match && qi < h->queries.size(); ++qi) {
      neg[qi] = run_phase(h, h->queries[qi], ups, false, nthreads, shard_rank, shard_world, st);
    }
    // apply_batch (graph.cpp:137-158) + B_upd bookkeeping.
    std::unordered_set<std::uint32_t> touched;
    for (const Update& up : ups) {
      touched.insert(up.u);
      touched.insert(up.v);
    }
    std::uint64_t bupd = 16ull * n;
    for (std::uint32_t v : touched) bupd += 4ull * g.adj[v].size();
    for (const Update& up : ups) {
      if (up.insert) {
        insert_sorted(g.adj[up.u], up.v);
        insert_sorted(g.adj[up.v], up.u);
        if (up.label != kNone) g.elab[pair_key(up.u, up.v)] = up.label;
      } else {
        erase_sorted(g.adj[up.u], up.v);
        erase_sorted(g.adj[up.v], up.u);
        g.elab.erase(pair_key(up.u, up.v));
      }
    }
    for (std::uint32_t v : touched) bupd += 4ull * g.adj[v].size();
    // incremental_reencode + CandidateTable::refresh.
    std::vector<std::uint32_t> tv(touched.begin(), touched.end());
    std::sort(tv.begin(), tv.end());
    for (QState& qs : h->queries) {
      std::size_t G = qs.G();
      std::vector<std::uint8_t> fresh(G);
      for (std::uint32_t v : tv) {
        qs.encode_vertex(g, v, fresh.data());
        std::uint8_t* cur = &qs.vcnt[std::size_t(v) * G];
        if (std::equal(fresh.begin(), fresh.end(), cur)) continue;
        std::copy(fresh.begin(), fresh.end(), cur);
        std::uint32_t before = qs.rows[v], after = qs.compute_row(g, v);
        if (before == after) continue;
        qs.rows[v] = after;
        for (std::uint32_t u = 0; u < qs.q.n; ++u) {
          if (((after & ~before) >> u) & 1u) ++qs.colsize[u];
          else if (((before & ~after) >> u) & 1u) --qs.colsize[u];
        }
      }
    }
    for (std::size_t qi = 0; match && qi < h->queries.size(); ++qi) {
      pos[qi] = run_phase(h, h->queries[qi], ups, true, nthreads, shard_rank, shard_world, st);
    }
    if (stats) {
      stats[0] = st.visits;
      stats[1] = st.iops;
      stats[2] = st.tasks;
      stats[3] = st.calls;
      stats[4] = st.balg;
      stats[5] = bupd;
      stats[6] = st.vpruned;
    }
    return ORC_OK;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return ORC_RUNTIME_ERROR;
  }
}

std::size_t orc_last_errors(orc_engine* h, std::uint64_t* idx, std::uint32_t* code,
                            std::size_t cap) {
  std::size_t n = std::min(cap, h->errors.size());
  for (std::size_t i = 0; i < n; ++i) {
    idx[i] = h->errors[i].first;
    code[i] = h->errors[i].second;
  }
  return h->errors.size();
}

int orc_order(orc_engine* h, int q, std::uint32_t e, std::uint32_t* out, std::size_t cap) {
  const auto& o = h->queries.at(std::size_t(q)).orders.at(e);
  for (std::size_t i = 0; i < o.size() && i < cap; ++i) out[i] = o[i];
  return int(o.size());
}

std::uint32_t orc_row(orc_engine* h, int q, std::uint32_t v) {
  return h->queries.at(std::size_t(q)).rows.at(v);
}

std::uint64_t orc_degree(orc_engine* h, std::uint32_t v) { return h->g.adj.at(v).size(); }

void orc_destroy(orc_engine* h) { delete h; }

}  // extern "C"
