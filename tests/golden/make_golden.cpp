// Golden-vector generator (run here, where /root/reference exists; see
// make_golden.sh).  It rebuilds the reference's OWN test instances with the
// reference's own seeded generators — tests/support/random_instances.hpp,
// tests/support/fig1.hpp, bench.cpp generate_queries — and records what the
// UNMODIFIED reference computes on them:
//   * match_batch with MatchOptions{coalesce=false, workers=1} and a plan of
//     generate_matching_order per query edge: |positive|, |negative|,
//     dfs_visits, intersection_ops, tasks_run per batch;
//   * the brute-force oracle incremental_diff_oracle (<= 60 vertices).
// The fixtures are committed so the GPU box (which has no /root/reference)
// can check the CUDA engine and the CPU restatement against them.

#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "bdsm/bench.hpp"
#include "bdsm/matcher.hpp"
#include "bdsm/oracle.hpp"
#include "bdsm/query_analysis.hpp"
#include "support/fig1.hpp"
#include "support/random_instances.hpp"

using namespace bdsm;

namespace {

long long lab(const std::optional<LabelId>& l) { return l ? static_cast<long long>(*l) : -1; }

struct Out {
  std::FILE* f;
  bool first = true;
};

QueryPlan plain_plan(const QueryGraph& q, const CandidateTable& table) {
  QueryPlan plan;
  plan.coalescing = false;
  plan.edge_plans.resize(q.edge_count());
  for (std::size_t e = 0; e < q.edge_count(); ++e) {
    plan.edge_plans[e].order = generate_matching_order(q, e, table);
  }
  return plan;
}

// Writes one instance: graph, query, batches and the reference's results.
void emit(Out& out, const std::string& name, const LabeledGraph& g0, const QueryGraph& q,
          const std::vector<UpdateBatch>& stream, bool brute) {
  std::FILE* f = out.f;
  std::fprintf(f, "%s\n{\"name\": \"%s\", \"nv\": %zu, \"vlabels\": [", out.first ? "" : ",",
               name.c_str(), g0.vertex_count());
  out.first = false;
  for (VertexId v = 0; v < g0.vertex_count(); ++v) std::fprintf(f, "%s%u", v ? "," : "", g0.label(v));
  std::fprintf(f, "], \"edges\": [");
  bool fe = true;
  for (VertexId v = 0; v < g0.vertex_count(); ++v) {
    for (VertexId w : g0.neighbors(v)) {
      if (w < v) continue;
      std::fprintf(f, "%s[%u,%u,%lld]", fe ? "" : ",", v, w, lab(g0.edge_label(v, w)));
      fe = false;
    }
  }
  std::fprintf(f, "], \"qlabels\": [");
  for (QueryVertexId u = 0; u < q.vertex_count(); ++u) std::fprintf(f, "%s%u", u ? "," : "", q.label(u));
  std::fprintf(f, "], \"qedges\": [");
  for (std::size_t e = 0; e < q.edge_count(); ++e) {
    std::fprintf(f, "%s[%u,%u,%lld]", e ? "," : "", q.edge(e).a, q.edge(e).b, lab(q.edge(e).label));
  }
  std::fprintf(f, "], \"batches\": [");
  for (std::size_t b = 0; b < stream.size(); ++b) {
    std::fprintf(f, "%s[", b ? "," : "");
    const auto& ups = stream[b].updates();
    for (std::size_t i = 0; i < ups.size(); ++i) {
      std::fprintf(f, "%s[%d,%u,%u,%lld]", i ? "," : "", ups[i].is_insert() ? 0 : 1, ups[i].u, ups[i].v,
                   lab(ups[i].edge_label));
    }
    std::fprintf(f, "]");
  }
  std::fprintf(f, "], \"expect\": [");
  LabeledGraph g = g0;
  auto enc = QueryEncodingState::initialize(g, q);
  QueryPlan plan = plain_plan(q, enc.table);
  MatchOptions opts;
  opts.coalesce = false;
  opts.scheduler.workers = 1;
  for (std::size_t b = 0; b < stream.size(); ++b) {
    long long bpos = -1, bneg = -1;
    if (brute) {
      auto d = oracle::incremental_diff_oracle(g, stream[b], q);
      bpos = static_cast<long long>(d.positive.size());
      bneg = static_cast<long long>(d.negative.size());
    }
    MatchStats st;
    auto r = match_batch(g, q, plan, enc, stream[b], opts, &st);
    std::fprintf(f,
                 "%s{\"pos\": %zu, \"neg\": %zu, \"visits\": %llu, \"iops\": %llu, \"tasks\": %llu, "
                 "\"brute_pos\": %lld, \"brute_neg\": %lld}",
                 b ? "," : "", r.positive.size(), r.negative.size(),
                 (unsigned long long)st.dfs_visits, (unsigned long long)st.intersection_ops,
                 (unsigned long long)st.tasks_run, bpos, bneg);
  }
  std::fprintf(f, "]}");
}

void suite(const char* path, const std::function<void(Out&)>& body) {
  Out out{std::fopen(path, "w")};
  std::fprintf(out.f, "[");
  body(out);
  std::fprintf(out.f, "\n]\n");
  std::fclose(out.f);
}

}  // namespace

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";

  // Running example (tests/support/fig1.hpp; test_matcher.cpp:49-78).
  suite((dir + "/fig1.json").c_str(), [](Out& out) {
    emit(out, "fig1_batch", fig1::data_graph(), fig1::query(), {fig1::batch()}, true);
    emit(out, "fig1_singletons", fig1::data_graph(), fig1::query(),
         {fig1::insert_v0_v2(), fig1::insert_v1_v4(), fig1::delete_v4_v5()}, true);
    emit(out, "fig1_empty", fig1::data_graph(), fig1::query(), {UpdateBatch{std::vector<EdgeUpdate>{}}}, true);
    // Static KATs from test_oracle.cpp:24-42 restated incrementally: insert
    // every edge of the data graph into an edgeless graph.
    {
      std::vector<VertexRecord> vs = {{0, 1}, {1, 1}, {2, 1}, {3, 1}};
      std::vector<EdgeUpdate> ups;
      for (VertexId u = 0; u < 4; ++u)
        for (VertexId v = u + 1; v < 4; ++v) ups.push_back({EdgeUpdate::Op::kInsert, u, v, {}, 0});
      QueryGraph q({1, 1, 1}, {{0, 1, {}}, {1, 2, {}}, {0, 2, {}}});
      UpdateBatch ins(ups);
      emit(out, "k3_on_k4", LabeledGraph::build_from_edges(vs, {}), q, {ins, ins.inverse()}, true);
    }
    {
      std::vector<VertexRecord> vs = {{0, 0}, {1, 1}, {2, 0}, {3, 1}};
      QueryGraph q({0, 1, 0}, {{0, 1, {}}, {1, 2, {}}});
      UpdateBatch ins({{EdgeUpdate::Op::kInsert, 0, 1, {}, 0}, {EdgeUpdate::Op::kInsert, 1, 2, {}, 0},
                       {EdgeUpdate::Op::kInsert, 2, 3, {}, 0}, {EdgeUpdate::Op::kInsert, 3, 0, {}, 0}});
      emit(out, "path_on_square", LabeledGraph::build_from_edges(vs, {}), q, {ins, ins.inverse()}, true);
    }
    {  // single-edge query: every anchor is a complete match
      std::vector<VertexRecord> vs = {{0, 0}, {1, 0}, {2, 1}};
      QueryGraph q({0, 0}, {{0, 1, {}}});
      UpdateBatch ins({{EdgeUpdate::Op::kInsert, 0, 1, {}, 0}, {EdgeUpdate::Op::kInsert, 1, 2, {}, 0}});
      emit(out, "single_edge", LabeledGraph::build_from_edges(vs, {}), q, {ins, ins.inverse()}, true);
    }
  });

  // Skewed hub (test_scheduler.cpp:59-97, :174-188): 400*120+3 positives.
  suite((dir + "/skewed.json").c_str(), [](Out& out) {
    std::vector<VertexRecord> vs;
    std::vector<EdgeRecord> es;
    VertexId next = 0;
    VertexId a = next++;
    vs.push_back({a, 0});
    VertexId hub = next++;
    vs.push_back({hub, 1});
    for (std::size_t s = 0; s < 400; ++s) {
      VertexId sv = next++;
      vs.push_back({sv, 1});
      es.push_back({hub, sv, {}});
      for (std::size_t l = 0; l < 120; ++l) {
        VertexId lv = next++;
        vs.push_back({lv, 1});
        es.push_back({sv, lv, {}});
      }
    }
    std::vector<EdgeUpdate> ups{{EdgeUpdate::Op::kInsert, a, hub, {}, 0}};
    for (int i = 0; i < 3; ++i) {
      VertexId la = next++, lb = next++, lc = next++, ld = next++;
      vs.push_back({la, 0});
      vs.push_back({lb, 1});
      vs.push_back({lc, 1});
      vs.push_back({ld, 1});
      es.push_back({lb, lc, {}});
      es.push_back({lc, ld, {}});
      ups.push_back({EdgeUpdate::Op::kInsert, la, lb, {}, 0});
    }
    QueryGraph q({0, 1, 1, 1}, {{0, 1, {}}, {1, 2, {}}, {2, 3, {}}});
    UpdateBatch b(ups);
    emit(out, "skewed_400x120", LabeledGraph::build_from_edges(vs, es), q, {b, b.inverse()}, false);
  });

  // test_matcher.cpp:214-234 (seed 61 x 120).
  suite((dir + "/matcher_random.json").c_str(), [](Out& out) {
    std::mt19937_64 rng(61);
    for (int round = 0; round < 120; ++round) {
      testgen::GraphSpec spec;
      spec.vertices = 10 + rng() % 15;
      spec.edges = 20 + rng() % 40;
      spec.labels = 1 + rng() % 3;
      auto g = testgen::random_graph(spec, rng);
      auto q = testgen::random_query(3 + rng() % 3, spec.labels, rng, 0.35);
      auto batch = testgen::random_batch(g, 1 + rng() % 6, rng);
      if (batch.empty()) continue;
      emit(out, "matcher61_" + std::to_string(round), g, q, {batch}, true);
    }
  });

  // test_matcher.cpp:236-282 (seed 67 x 40, edge labels).
  suite((dir + "/edge_labeled.json").c_str(), [](Out& out) {
    std::mt19937_64 rng(67);
    for (int round = 0; round < 40; ++round) {
      testgen::GraphSpec spec;
      spec.vertices = 12;
      spec.edges = 28;
      spec.labels = 2;
      spec.edge_labels = true;
      auto g = testgen::random_graph(spec, rng);
      std::vector<VertexId> members;
      VertexId start = rng() % g.vertex_count();
      if (g.degree(start) == 0) continue;
      members.push_back(start);
      while (members.size() < 3) {
        VertexId u = members[rng() % members.size()];
        auto nbrs = g.neighbors(u);
        VertexId w = nbrs[rng() % nbrs.size()];
        if (std::find(members.begin(), members.end(), w) == members.end()) members.push_back(w);
      }
      std::sort(members.begin(), members.end());
      members.erase(std::unique(members.begin(), members.end()), members.end());
      if (members.size() < 3) continue;
      std::vector<LabelId> labels;
      std::vector<QueryEdge> qedges;
      for (std::size_t i = 0; i < members.size(); ++i) labels.push_back(g.label(members[i]));
      for (std::size_t i = 0; i < members.size(); ++i) {
        for (std::size_t j = i + 1; j < members.size(); ++j) {
          if (g.has_edge(members[i], members[j])) {
            qedges.push_back({static_cast<QueryVertexId>(i), static_cast<QueryVertexId>(j),
                              g.edge_label(members[i], members[j])});
          }
        }
      }
      QueryGraph q(std::move(labels), std::move(qedges));
      if (!q.connected()) continue;
      auto batch = testgen::random_batch(g, 1 + rng() % 5, rng, true);
      if (batch.empty()) continue;
      emit(out, "elab67_" + std::to_string(round), g, q, {batch}, true);
    }
  });

  // acceptance.cpp:55-85 random_suite(500, 1001) — criterion 2.
  suite((dir + "/acceptance_random.json").c_str(), [](Out& out) {
    std::mt19937_64 rng(1001);
    const QueryCategory cats[] = {QueryCategory::kTree, QueryCategory::kSparse, QueryCategory::kDense};
    std::size_t made = 0, attempts = 0;
    while (made < 500 && attempts < 500 * 30) {
      ++attempts;
      testgen::GraphSpec spec;
      spec.vertices = 12 + rng() % 19;
      spec.edges = 20 + rng() % 71;
      spec.labels = 1 + rng() % 3;
      auto g = testgen::random_graph(spec, rng);
      QueryCategory cat = cats[made % 3];
      std::size_t size = cat == QueryCategory::kDense ? 4 + rng() % 3 : 3 + rng() % 4;
      std::vector<QueryGraph> qs;
      try {
        qs = generate_queries(g, {cat, size, 1}, rng());
      } catch (const std::exception&) {
        continue;
      }
      auto batch = testgen::random_batch(g, 1 + rng() % 8, rng);
      if (batch.empty()) continue;
      emit(out, "acc1001_" + std::to_string(made), g, qs[0], {batch}, true);
      ++made;
    }
  });

  // Evolving-graph streams: several consecutive batches on one graph, with
  // medium graphs where only the reference engine (not brute force) runs.
  suite((dir + "/streams.json").c_str(), [](Out& out) {
    std::mt19937_64 rng(2024);
    for (int round = 0; round < 40; ++round) {
      testgen::GraphSpec spec;
      spec.vertices = 14 + rng() % 16;
      spec.edges = 30 + rng() % 50;
      spec.labels = 1 + rng() % 2;
      auto g = testgen::random_graph(spec, rng);
      auto q = testgen::random_query(3 + rng() % 4, spec.labels, rng, 0.4, 2);
      std::vector<UpdateBatch> stream;
      LabeledGraph cur = g;
      for (int b = 0; b < 4; ++b) {
        auto batch = testgen::random_batch(cur, 2 + rng() % 10, rng);
        cur.apply_batch(batch);
        stream.push_back(std::move(batch));
      }
      emit(out, "stream_small_" + std::to_string(round), g, q, stream, true);
    }
    for (int round = 0; round < 12; ++round) {
      testgen::GraphSpec spec;
      spec.vertices = 1500 + rng() % 1500;
      spec.edges = 6000 + rng() % 10000;
      spec.labels = 2 + rng() % 3;
      auto g = testgen::random_graph(spec, rng);
      auto q = testgen::random_query(4 + rng() % 3, spec.labels, rng, 0.35);
      std::vector<UpdateBatch> stream;
      LabeledGraph cur = g;
      for (int b = 0; b < 3; ++b) {
        auto batch = testgen::random_batch(cur, 50 + rng() % 200, rng);
        cur.apply_batch(batch);
        stream.push_back(std::move(batch));
      }
      emit(out, "stream_medium_" + std::to_string(round), g, q, stream, false);
    }
  });
  return 0;
}
