// Text formats (src/io.cpp:16-148) and seeded generators (src/bench.cpp:67-289)
// of the `bdsm run` CLI.  See textio.hpp.
#include "textio.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>

namespace bdsm::text {

namespace {

std::uint64_t pair_key(std::uint32_t u, std::uint32_t v) {  // types.hpp edge_pair_key
  if (u > v) std::swap(u, v);
  return (std::uint64_t(u) << 32) | v;
}

std::ifstream open_or_throw(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  return in;
}

// `v id label` / `e u v [label]` records, `#` comments, blank lines ignored.
Graph parse_records(std::istream& in) {
  Graph out;
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      std::uint32_t id, label;
      if (!(ls >> id >> label)) throw std::runtime_error("bad vertex record at line " + std::to_string(lineno));
      out.vertices.push_back({id, label});
    } else if (tag == "e") {
      std::uint32_t u, v;
      if (!(ls >> u >> v)) throw std::runtime_error("bad edge record at line " + std::to_string(lineno));
      gpu::EdgeRecord rec{u, v, std::nullopt};
      std::uint32_t el;
      if (ls >> el) rec.label = el;
      out.edges.push_back(rec);
    } else {
      throw std::runtime_error("unknown record '" + tag + "' at line " + std::to_string(lineno));
    }
  }
  return out;
}

// Host adjacency of the loaded graph (sorted lists), for the generators.
struct HostGraph {
  std::vector<std::uint32_t> label;
  std::vector<std::vector<std::uint32_t>> nbr;
  std::unordered_map<std::uint64_t, std::uint32_t> elabel;
  explicit HostGraph(const Graph& g) {
    label.assign(g.vertices.size(), 0xffffffffu);
    for (const auto& r : g.vertices) {
      if (r.id >= label.size())
        throw std::invalid_argument("vertex ids must be dense 0-based and unique (got " + std::to_string(r.id) + ")");
      label[r.id] = r.label;
    }
    nbr.resize(label.size());
    for (const auto& e : g.edges) {
      if (e.u >= label.size() || e.v >= label.size() || e.u == e.v)
        throw std::invalid_argument("edge (" + std::to_string(e.u) + "," + std::to_string(e.v) + ") is invalid");
      nbr[e.u].push_back(e.v);
      nbr[e.v].push_back(e.u);
      if (e.label) elabel[pair_key(e.u, e.v)] = *e.label;
    }
    for (auto& l : nbr) std::sort(l.begin(), l.end());
  }
  std::optional<std::uint32_t> edge_label(std::uint32_t u, std::uint32_t v) const {
    auto it = elabel.find(pair_key(u, v));
    if (it == elabel.end()) return std::nullopt;
    return it->second;
  }
};

// Batagelj-Zaversnik peeling in the reference's bucket order (core_numbers,
// src/bench.cpp:142-177): the same stale-entry handling and neighbour order.
std::vector<std::uint32_t> core_numbers(const HostGraph& g) {
  const std::size_t n = g.label.size();
  std::vector<std::uint32_t> deg(n), core(n, 0);
  std::size_t max_deg = 0;
  for (std::size_t v = 0; v < n; ++v) {
    deg[v] = std::uint32_t(g.nbr[v].size());
    max_deg = std::max<std::size_t>(max_deg, deg[v]);
  }
  std::vector<std::vector<std::uint32_t>> buckets(max_deg + 1);
  for (std::uint32_t v = 0; v < n; ++v) buckets[deg[v]].push_back(v);
  std::vector<bool> done(n, false);
  std::size_t processed = 0, b = 0;
  std::uint32_t current = 0;
  while (processed < n) {
    while (b <= max_deg && buckets[b].empty()) ++b;
    if (b > max_deg) break;
    std::uint32_t v = buckets[b].back();
    buckets[b].pop_back();
    if (done[v] || deg[v] != b) continue;
    done[v] = true;
    ++processed;
    current = std::max(current, std::uint32_t(b));
    core[v] = current;
    for (std::uint32_t w : g.nbr[v]) {
      if (done[w] || deg[w] == 0) continue;
      if (deg[w] > deg[v]) {
        --deg[w];
        buckets[deg[w]].push_back(w);
        if (deg[w] < b) b = deg[w];
      }
    }
  }
  return core;
}

}  // namespace

Graph load_graph(std::istream& in) { return parse_records(in); }

Graph load_graph_file(const std::string& path) {
  auto in = open_or_throw(path);
  return load_graph(in);
}

Query load_query(std::istream& in) {
  Graph p = parse_records(in);
  Query q;
  q.labels.assign(p.vertices.size(), 0xffffffffu);
  for (const auto& r : p.vertices) {
    if (r.id >= q.labels.size()) throw std::runtime_error("query vertex ids must be dense");
    q.labels[r.id] = r.label;
  }
  for (const auto& e : p.edges) q.edges.push_back({e.u, e.v, e.label});
  return q;
}

Query load_query_file(const std::string& path) {
  auto in = open_or_throw(path);
  return load_query(in);
}

std::vector<Batch> load_stream(std::istream& in) {
  std::vector<Batch> batches;
  Batch cur;
  std::string line;
  std::size_t lineno = 0;
  auto flush = [&] {
    if (!cur.empty()) {
      batches.push_back(std::move(cur));
      cur.clear();
    }
  };
  while (std::getline(in, line)) {
    ++lineno;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag)) {
      flush();
      continue;
    }
    if (tag[0] == '#') continue;
    if (tag != "+" && tag != "-") throw std::runtime_error("bad update at line " + std::to_string(lineno));
    std::uint32_t u, v;
    if (!(ls >> u >> v)) throw std::runtime_error("bad update at line " + std::to_string(lineno));
    gpu::EdgeUpdate up{tag == "+" ? gpu::EdgeUpdate::Op::kInsert : gpu::EdgeUpdate::Op::kDelete, u, v,
                       std::nullopt};
    std::uint32_t el;
    if (tag == "+" && (ls >> el)) up.edge_label = el;
    cur.push_back(up);
  }
  flush();
  return batches;
}

std::vector<Batch> load_stream_file(const std::string& path) {
  auto in = open_or_throw(path);
  return load_stream(in);
}

void save_query(std::ostream& out, const Query& q) {
  for (std::size_t u = 0; u < q.labels.size(); ++u) out << "v " << u << ' ' << q.labels[u] << '\n';
  for (const auto& e : q.edges) {
    out << "e " << e.a << ' ' << e.b;
    if (e.label) out << ' ' << *e.label;
    out << '\n';
  }
}

void save_stream(std::ostream& out, const std::vector<Batch>& stream) {
  for (std::size_t i = 0; i < stream.size(); ++i) {
    if (i > 0) out << '\n';
    for (const auto& up : stream[i]) {
      out << (up.is_insert() ? '+' : '-') << ' ' << up.u << ' ' << up.v;
      if (up.is_insert() && up.edge_label) out << ' ' << *up.edge_label;
      out << '\n';
    }
  }
}

// Random-walk query extraction with per-category rejection
// (generate_queries, src/bench.cpp:67-140).
std::vector<Query> generate_queries(const Graph& graph, const std::string& category, std::size_t size,
                                    std::size_t count, std::uint64_t seed) {
  if (category != "dense" && category != "sparse" && category != "tree")
    throw std::invalid_argument("unknown query category: " + category);
  HostGraph g(graph);
  const std::size_t n = g.label.size();
  if (size < 2 || size > 32) throw std::invalid_argument("query size out of range");
  if (size > n) throw std::invalid_argument("query larger than graph");
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<std::uint32_t> pick(0, std::uint32_t(n - 1));
  std::vector<Query> out;
  for (std::size_t qi = 0; qi < count; ++qi) {
    bool made = false;
    for (std::size_t attempt = 0; attempt < 4000 && !made; ++attempt) {
      std::uint32_t start = pick(rng);
      if (g.nbr[start].empty()) continue;
      std::vector<std::uint32_t> members{start};
      std::unordered_set<std::uint32_t> in_set{start};
      std::vector<std::pair<std::uint32_t, std::uint32_t>> walk;
      std::size_t stuck = 0;
      while (members.size() < size && stuck < 64 * size) {
        std::uint32_t u = members[rng() % members.size()];
        const auto& nb = g.nbr[u];
        if (nb.empty()) {
          ++stuck;
          continue;
        }
        std::uint32_t w = nb[rng() % nb.size()];
        if (in_set.count(w)) {
          ++stuck;
          continue;
        }
        members.push_back(w);
        in_set.insert(w);
        walk.emplace_back(u, w);
        stuck = 0;
      }
      if (members.size() < size) continue;
      std::sort(members.begin(), members.end());
      std::unordered_map<std::uint32_t, std::uint32_t> local;
      Query q;
      q.labels.resize(members.size());
      for (std::size_t i = 0; i < members.size(); ++i) {
        local[members[i]] = std::uint32_t(i);
        q.labels[i] = g.label[members[i]];
      }
      if (category == "tree") {
        for (auto& [u, w] : walk) q.edges.push_back({local[u], local[w], g.edge_label(u, w)});
      } else {
        for (std::uint32_t u : members)
          for (std::uint32_t w : g.nbr[u])
            if (w > u && in_set.count(w)) q.edges.push_back({local[u], local[w], g.edge_label(u, w)});
        double d_avg = 2.0 * double(q.edges.size()) / double(size);
        if (category == "dense" && d_avg < 3.0) continue;
        if (category == "sparse" && (d_avg >= 3.0 || q.edges.size() < size)) continue;
      }
      out.push_back(std::move(q));
      made = true;
    }
    if (!made)
      throw std::runtime_error("could not extract a " + category + " query of size " + std::to_string(size));
  }
  return out;
}

// Update stream valid against the evolving graph (generate_stream,
// src/bench.cpp:179-289): inserts are uniform non-edge pairs whose label pair
// occurs in G, deletes uniform over the current edge list, mixed 2:1.  The
// edge list keeps the reference's swap-with-last removal (found through an
// index instead of a linear scan; the list contents are identical).
std::vector<Batch> generate_stream(const Graph& graph, const StreamSpec& spec) {
  if (spec.rate <= 0.0 || spec.rate > 1.0) throw std::invalid_argument("rate must be in (0,1]");
  if (spec.batches == 0) throw std::invalid_argument("batches must be >= 1");
  if (spec.mode != "insert" && spec.mode != "delete" && spec.mode != "mixed")
    throw std::invalid_argument("unknown stream mode: " + spec.mode);
  HostGraph g(graph);
  std::mt19937_64 rng(spec.seed);
  const std::size_t n = g.label.size();
  std::unordered_set<std::uint64_t> present;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> edge_list;
  std::unordered_map<std::uint64_t, std::size_t> where;
  std::unordered_map<std::uint64_t, std::vector<std::uint32_t>> labels_by_pair;
  std::set<std::uint64_t> label_pairs;
  for (std::uint32_t v = 0; v < n; ++v) {
    for (std::uint32_t w : g.nbr[v]) {
      if (v < w) {
        present.insert(pair_key(v, w));
        where[pair_key(v, w)] = edge_list.size();
        edge_list.emplace_back(v, w);
        std::uint64_t lp = pair_key(g.label[v], g.label[w]);
        label_pairs.insert(lp);
        if (auto el = g.edge_label(v, w)) labels_by_pair[lp].push_back(*el);
      }
    }
  }
  std::vector<bool> in_core(n, true);
  if (spec.kcore) {
    auto cores = core_numbers(g);
    std::size_t kept = 0;
    for (std::size_t v = 0; v < n; ++v) {
      in_core[v] = cores[v] >= *spec.kcore;
      kept += in_core[v];
    }
    if (kept < 2) throw std::runtime_error("k-core too small for density mode");
  }
  std::size_t total = std::size_t(std::llround(spec.rate * double(edge_list.size())));
  total = std::max<std::size_t>(total, 1);
  std::uniform_int_distribution<std::uint32_t> pick(0, std::uint32_t(n - 1));
  std::vector<Batch> stream;
  std::size_t emitted = 0;
  for (std::size_t bi = 0; bi < spec.batches; ++bi) {
    std::size_t want = total / spec.batches + (bi < total % spec.batches ? 1 : 0);
    if (want == 0) continue;
    Batch ups;
    std::unordered_set<std::uint64_t> in_batch;
    for (std::size_t s = 0; s < want; ++s, ++emitted) {
      bool insert = spec.mode == "insert" || (spec.mode == "mixed" && emitted % 3 != 2);
      bool found = false;
      if (insert) {
        for (std::size_t attempt = 0; attempt < 20000 && !found; ++attempt) {
          std::uint32_t u = pick(rng), v = pick(rng);
          if (u == v || !in_core[u] || !in_core[v]) continue;
          std::uint64_t pk = pair_key(u, v);
          if (present.count(pk) || in_batch.count(pk)) continue;
          std::uint64_t lp = pair_key(g.label[u], g.label[v]);
          if (!label_pairs.count(lp)) continue;
          std::optional<std::uint32_t> el;
          auto it = labels_by_pair.find(lp);
          if (it != labels_by_pair.end() && !it->second.empty()) el = it->second[rng() % it->second.size()];
          ups.push_back({gpu::EdgeUpdate::Op::kInsert, u, v, el});
          in_batch.insert(pk);
          found = true;
        }
        if (!found) throw std::runtime_error("insufficient label-compatible non-edges");
      } else {
        for (std::size_t attempt = 0; attempt < 20000 && !found; ++attempt) {
          if (edge_list.empty()) break;
          auto [u, v] = edge_list[rng() % edge_list.size()];
          if (!in_core[u] || !in_core[v]) continue;
          std::uint64_t pk = pair_key(u, v);
          if (in_batch.count(pk)) continue;
          ups.push_back({gpu::EdgeUpdate::Op::kDelete, u, v, std::nullopt});
          in_batch.insert(pk);
          found = true;
        }
        if (!found) throw std::runtime_error("no deletable edges left");
      }
    }
    for (const auto& up : ups) {  // advance the replica to the post-batch state
      std::uint64_t pk = pair_key(up.u, up.v);
      if (up.is_insert()) {
        present.insert(pk);
        where[pk] = edge_list.size();
        edge_list.emplace_back(std::min(up.u, up.v), std::max(up.u, up.v));
      } else {
        present.erase(pk);
        auto it = where.find(pk);
        if (it != where.end()) {
          std::size_t i = it->second;
          where.erase(it);
          if (i + 1 != edge_list.size()) {
            edge_list[i] = edge_list.back();
            where[pair_key(edge_list[i].first, edge_list[i].second)] = i;
          }
          edge_list.pop_back();
        }
      }
    }
    stream.push_back(std::move(ups));
  }
  return stream;
}

}  // namespace bdsm::text
