// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
// See oracle.hpp for the contract and the reference lines each part follows.

#include "oracle.hpp"

#include <algorithm>
#include <atomic>
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

// Per-query filter state: encoding.cpp's scheme + per-vertex saturated
// neighbour-label counters + CandidateTable rows and sorted columns.
struct QState {
  Query q;
  std::vector<std::uint32_t> group_labels;  // sorted distinct query labels
  std::uint32_t cap = 3;
  std::vector<std::uint8_t> qcnt;           // [n][G]
  std::vector<std::uint8_t> vcnt;           // [V][G]
  std::vector<std::uint32_t> rows;          // [V]
  std::vector<std::vector<std::uint32_t>> columns;
  std::vector<std::vector<std::uint32_t>> orders;  // per query edge

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
  void add(const Stats& o) {
    visits += o.visits;
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
    return double(qs.columns[u].size()) / double(std::max<std::uint32_t>(q.degree[u], 1));
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

// Reference intersect_sorted (matcher.cpp:59-73): binary-search each element
// of the smaller list in the larger; counts the same intersection_ops.
void intersect(const std::vector<std::uint32_t>& a, const std::vector<std::uint32_t>& b,
               std::vector<std::uint32_t>& out, Stats& st) {
  const auto& small = a.size() <= b.size() ? a : b;
  const auto& large = a.size() <= b.size() ? b : a;
  out.clear();
  std::uint64_t probe = 1 + std::uint64_t(std::bit_width(large.size()));
  st.iops += probe * small.size();
  for (std::uint32_t x : small) {
    if (std::binary_search(large.begin(), large.end(), x)) out.push_back(x);
  }
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

struct Ctx {
  const Graph& g;
  const QState& qs;
  const std::vector<Update>& ups;
  const std::unordered_map<std::uint64_t, std::uint32_t>& order_by_pair;  // UpdateIndex
};

// gen_candidates (matcher.cpp:87-108).
void gen_candidates(const Ctx& c, const std::vector<std::uint32_t>& order,
                    const std::uint32_t* assign, std::size_t level,
                    std::vector<std::uint32_t>& res, Stats& st) {
  const Query& q = c.qs.q;
  std::uint32_t u = order[level];
  ++st.calls;
  for (std::size_t i = 0; i < level; ++i) {
    if (q.adjacent(order[i], u)) st.balg += 4ull * c.g.adj[assign[i]].size();
  }
  const std::vector<std::uint32_t>* cur = &c.qs.columns[u];
  bool own = false;
  std::vector<std::uint32_t> scratch, tmp;
  for (std::size_t i = 0; i < level && !cur->empty(); ++i) {
    std::uint32_t prev = order[i];
    if (!q.adjacent(prev, u)) continue;
    const auto& nbrs = labeled_neighbors(c.g, assign[i], q.edge_label(prev, u), scratch);
    intersect(*cur, nbrs, tmp, st);
    res.swap(tmp);
    cur = &res;
    own = true;
  }
  if (!own) res = *cur;
  if (!res.empty()) {
    std::erase_if(res, [&](std::uint32_t v) {
      for (std::size_t i = 0; i < level; ++i) {
        if (assign[i] == v) return true;
      }
      return false;
    });
  }
}

// dedupe_by_order (matcher.cpp:110-117) over the image by query vertex.
bool dedupe(const Ctx& c, const std::uint32_t* image, std::uint32_t anchor_order) {
  for (const QEdge& e : c.qs.q.edges) {
    auto it = c.order_by_pair.find(pair_key(image[e.a], image[e.b]));
    if (it != c.order_by_pair.end() && it->second < anchor_order) return false;
  }
  return true;
}

// run_match_task (matcher.cpp:219-310) with workers = 1, no coalescing.
std::uint64_t run_task(const Ctx& c, const Task& t, Stats& st) {
  const Query& q = c.qs.q;
  const Update& up = c.ups[t.upd];
  const std::vector<std::uint32_t>& order = c.qs.orders[t.edge];
  std::size_t n = order.size();
  std::uint32_t assign[32];
  std::uint32_t image[32];
  assign[0] = t.flipped ? up.v : up.u;
  assign[1] = t.flipped ? up.u : up.v;
  ++st.tasks;
  std::uint64_t count = 0;
  auto emit = [&]() {
    for (std::size_t i = 0; i < n; ++i) image[order[i]] = assign[i];
    if (dedupe(c, image, up.order)) {
      ++count;
      ++st.emitted;
    }
  };
  if (n <= 2) {
    emit();
    return count;
  }
  std::vector<std::vector<std::uint32_t>> levels(n);
  std::vector<std::size_t> cursor(n, 0);
  gen_candidates(c, order, assign, 2, levels[2], st);
  if (!t.whole) {  // shard restriction: level-2 values inside the owned driver range
    std::erase_if(levels[2], [&](std::uint32_t v) { return v < t.lo || v > t.hi; });
  }
  std::size_t l = 2;
  while (true) {
    while (cursor[l] >= levels[l].size()) {
      if (l == 2) return count;
      --l;
    }
    std::uint32_t cand = levels[l][cursor[l]++];
    ++st.visits;
    assign[l] = cand;
    if (l + 1 == n) {
      emit();
      continue;
    }
    gen_candidates(c, order, assign, l + 1, levels[l + 1], st);
    if (levels[l + 1].empty()) continue;
    cursor[l + 1] = 0;
    ++l;
  }
  (void)q;
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

std::uint64_t run_phase(orc_engine* h, QState& qs, const std::vector<Update>& ups, bool inserts,
                        std::uint32_t nthreads, std::uint32_t rank, std::uint32_t world,
                        Stats& total) {
  const Graph& g = h->g;
  const Query& q = qs.q;
  std::unordered_map<std::uint64_t, std::uint32_t> order_by_pair;  // UpdateIndex::build
  for (const Update& up : ups) {
    if (up.insert == inserts) order_by_pair.emplace(pair_key(up.u, up.v), up.order);
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
  Ctx ctx{g, qs, ups, order_by_pair};
  std::atomic<std::size_t> next{0};
  std::atomic<std::uint64_t> count{0};
  std::vector<Stats> per(std::max(1u, nthreads));
  auto worker = [&](std::size_t w) {
    std::uint64_t local = 0;
    for (std::size_t i; (i = next.fetch_add(1)) < tasks.size();) local += run_task(ctx, tasks[i], per[w]);
    count += local;
  };
  if (nthreads <= 1 || tasks.size() < 2) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (std::size_t w = 0; w < nthreads; ++w) th.emplace_back(worker, w);
    for (auto& t : th) t.join();
  }
  for (auto& s : per) total.add(s);
  return count.load();
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
    std::vector<std::uint64_t> keys;
    keys.reserve(2 * ne);
    for (std::uint64_t i = 0; i < ne; ++i) {  // graph.cpp:52-68
      std::uint32_t u = eu[i], v = ev[i];
      if (u == v) throw std::invalid_argument("self-loop edge (" + std::to_string(u) + "," + std::to_string(v) + ")");
      if (u >= nv || v >= nv) throw std::invalid_argument("edge references unknown vertex");
      keys.push_back((std::uint64_t(u) << 32) | v);
      keys.push_back((std::uint64_t(v) << 32) | u);
      if (elab && elab[i] != kNone) g.elab[pair_key(u, v)] = elab[i];
    }
    std::sort(keys.begin(), keys.end());
    for (std::size_t i = 1; i < keys.size(); ++i) {
      if (keys[i] == keys[i - 1]) throw std::invalid_argument("duplicate edge");
    }
    std::vector<std::uint64_t> deg(nv, 0);
    for (auto k : keys) ++deg[k >> 32];
    for (std::uint32_t v = 0; v < nv; ++v) g.adj[v].reserve(deg[v]);
    for (auto k : keys) g.adj[k >> 32].push_back(std::uint32_t(k));
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
    qs.columns.assign(n, {});
    for (std::uint32_t v = 0; v < V; ++v) {
      qs.encode_vertex(g, v, &qs.vcnt[std::size_t(v) * G]);
      qs.rows[v] = qs.compute_row(g, v);
      for (std::uint32_t u = 0; u < n; ++u) {
        if ((qs.rows[v] >> u) & 1u) qs.columns[u].push_back(v);
      }
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
          if (((after & ~before) >> u) & 1u) insert_sorted(qs.columns[u], v);
          else if (((before & ~after) >> u) & 1u) erase_sorted(qs.columns[u], v);
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
