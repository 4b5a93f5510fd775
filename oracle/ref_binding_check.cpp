// TEST INFRASTRUCTURE ONLY — exercises include/bdsm_gpu_reference.hpp (the
// reference-side binding) the way the reference's own tests would: with the
// reference's fixtures (tests/support/fig1.hpp, random_instances.hpp), its
// types, and its own match_batch (coalesce off) as the expected result.
// Built by `make -C oracle ref` against /root/reference/proj/include and the
// unmodified reference library; linked with libbdsm_b200.so.
//
// Prints one JSON line.  Exit 0: every check equal.  Exit 3: no usable GPU —
// the binding raised std::runtime_error from the engine's BDSM_CUDA_ERROR
// (the CPU test checks exactly that).  Exit 1: a mismatch.

#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../include/bdsm_gpu_reference.hpp"
#include "bdsm/matcher.hpp"
#include "bdsm/query_analysis.hpp"
#include "tests/support/fig1.hpp"             // reference fixtures (-I$(REF))
#include "tests/support/random_instances.hpp"

using namespace bdsm;

namespace {

struct RefRun {
  LabeledGraph g;
  QueryGraph q;
  QueryEncodingState enc;
  QueryPlan plan;
  RefRun(LabeledGraph g0, QueryGraph q0)
      : g(std::move(g0)), q(std::move(q0)), enc(QueryEncodingState::initialize(g, q)),
        plan(build_query_plan(q, enc.table, PlanOptions{false, {}})) {}
  gpu_ref::DeltaCounts step(const UpdateBatch& b) {
    MatchOptions o;
    o.coalesce = false;  // the parity configuration
    IncrementalMatchSet r = match_batch(g, q, plan, enc, b, o);
    return {r.positive.size(), r.negative.size()};
  }
};

std::vector<VertexRecord> vertices_of(const LabeledGraph& g) {
  std::vector<VertexRecord> vs;
  for (VertexId v = 0; v < g.vertex_count(); ++v) vs.push_back({v, g.label(v)});
  return vs;
}

}  // namespace

int main() {
  int checks = 0, bad = 0;
  auto expect = [&](bool ok, const std::string& what) {
    ++checks;
    if (!ok) {
      ++bad;
      std::fprintf(stderr, "MISMATCH: %s\n", what.c_str());
    }
  };
  try {
    // Fig. 1: one batch -> +4/-0 (tests/test_matcher.cpp:49-78)
    {
      gpu_ref::DeviceMatcher dm(fig1::data_graph());
      dm.add_query(fig1::query());
      RefRun ref(fig1::data_graph(), fig1::query());
      auto got = dm.match_batch(fig1::batch());
      auto exp = ref.step(fig1::batch());
      expect(got.size() == 1 && got[0].positive == 4 && got[0].negative == 0, "fig1 batch +4/-0");
      expect(got[0].positive == exp.positive && got[0].negative == exp.negative, "fig1 batch vs reference");
    }
    // Fig. 1 singletons -> +4, +2, -2; BatchError contract (all-or-nothing)
    {
      std::vector<EdgeRecord> es;
      const LabeledGraph g0 = fig1::data_graph();
      for (VertexId v = 0; v < g0.vertex_count(); ++v)
        for (VertexId w : g0.neighbors(v))
          if (v < w) es.push_back({v, w, {}});
      gpu_ref::DeviceMatcher dm(vertices_of(g0), es);
      dm.add_query(fig1::query());
      RefRun ref(fig1::data_graph(), fig1::query());
      using Op = EdgeUpdate::Op;
      UpdateBatch bad_batch({{Op::kInsert, 0, 2, {}, 0}, {Op::kDelete, 0, 1, {}, 0}, {Op::kInsert, 0, 3, {}, 0}});
      std::vector<UpdateError> ref_fail = ref.g.validate_batch(bad_batch);
      bool threw = false;
      try {
        dm.match_batch(bad_batch);
      } catch (const BatchError& e) {
        threw = e.failures.size() == ref_fail.size();
        for (std::size_t i = 0; threw && i < ref_fail.size(); ++i)
          threw = e.failures[i].index == ref_fail[i].index && e.failures[i].reason == ref_fail[i].reason;
      }
      expect(threw, "BatchError failures equal validate_batch's");
      bool inval = false;
      try {
        dm.match_batch(UpdateBatch({{Op::kInsert, 7, 9, {}, 0}, {Op::kDelete, 4, 5, {}, 0},
                                    {Op::kInsert, 3, 3, {}, 0}}));
      } catch (const std::invalid_argument&) {
        inval = true;
      }
      expect(inval, "self-loop -> std::invalid_argument");
      const int want[3][2] = {{4, 0}, {2, 0}, {0, 2}};
      const UpdateBatch singles[3] = {fig1::insert_v0_v2(), fig1::insert_v1_v4(), fig1::delete_v4_v5()};
      for (int i = 0; i < 3; ++i) {
        auto got = dm.match_batch(singles[i]);
        auto exp = ref.step(singles[i]);
        expect(got[0].positive == std::uint64_t(want[i][0]) && got[0].negative == std::uint64_t(want[i][1]),
               "fig1 singleton " + std::to_string(i));
        expect(got[0].positive == exp.positive && got[0].negative == exp.negative,
               "fig1 singleton vs reference " + std::to_string(i));
      }
    }
    // randomized suite (seeded, reference generators): several queries per
    // engine, multi-batch streams, against the reference's match_batch
    std::mt19937_64 rng(4242);
    int streams = 0;
    for (int inst = 0; inst < 40; ++inst) {
      testgen::GraphSpec spec;
      spec.vertices = 30 + rng() % 50;
      spec.edges = spec.vertices * (2 + rng() % 3);
      spec.labels = 2 + rng() % 2;
      LabeledGraph g = testgen::random_graph(spec, rng);
      const std::size_t nq = 1 + rng() % 4;
      std::vector<QueryGraph> qs;
      for (std::size_t k = 0; k < nq; ++k) qs.push_back(testgen::random_query(3 + rng() % 3, spec.labels, rng));
      gpu_ref::DeviceMatcher dm(g);
      std::vector<RefRun> refs;
      for (const QueryGraph& q : qs) {
        dm.add_query(q);
        refs.emplace_back(g, q);
      }
      for (int b = 0; b < 3; ++b) {
        UpdateBatch batch = testgen::random_batch(refs[0].g, 4 + rng() % 12, rng);
        auto got = dm.match_batch(batch);
        for (std::size_t k = 0; k < nq; ++k) {
          auto exp = refs[k].step(batch);
          expect(got[k].positive == exp.positive && got[k].negative == exp.negative,
                 "random instance " + std::to_string(inst) + " batch " + std::to_string(b) + " query " +
                     std::to_string(k));
        }
      }
      ++streams;
    }
    std::printf("{\"checks\": %d, \"mismatches\": %d, \"random_streams\": %d}\n", checks, bad, streams);
    return bad ? 1 : 0;
  } catch (const BatchError& e) {
    std::printf("{\"error\": \"unexpected BatchError: %s\"}\n", e.what());
    return 1;
  } catch (const std::runtime_error& e) {
    // BDSM_CUDA_ERROR without a device maps to std::runtime_error
    const std::string w = e.what();
    std::printf("{\"no_gpu\": %s, \"error\": \"%s\"}\n",
                w.find("CUDA") != std::string::npos || w.find("device") != std::string::npos ? "true" : "false",
                w.c_str());
    return 3;
  }
}
