// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// The reference's own `bdsm run` path (tools/bdsm.cpp:66-150) driven without
// CLI11 (absent here): load_graph_file, load_query_file or
// generate_queries, load_stream_file or generate_stream, run_pipeline with
// MatchOptions{coalesce=false}, emit_report and the summary
// line.  Built by `make -C oracle ref` against the unmodified reference; used
// by tests/golden/make_cli_golden.sh to produce the CLI fixtures the B200
// CLI is checked against.
//
//   ref_cli GRAPH (q:FILE | g:cat,size,count) (s:FILE | s:rate,mode,batches[,k]) SEED OUTDIR [dump]
//   (dump: --dump-matches, matches_batch<i>.txt in OUTDIR)
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "bdsm/bench.hpp"
#include "bdsm/io.hpp"

namespace {
std::vector<std::string> csv(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, ',')) out.push_back(x);
  return out;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 6 && argc != 7) {
    std::cerr << "usage: ref_cli GRAPH q:FILE|g:cat,size,count s:FILE|s:rate,mode,batches[,k] SEED OUT\n";
    return 2;
  }
  const std::string qspec = argv[2], sspec = argv[3], out = argv[5];
  const std::uint64_t seed = std::stoull(argv[4]);
  try {
    bdsm::LabeledGraph g = bdsm::load_graph_file(argv[1]);
    std::filesystem::create_directories(out);
    std::vector<bdsm::QueryGraph> queries;
    std::vector<std::string> cats;
    if (qspec.rfind("q:", 0) == 0) {
      queries.push_back(bdsm::load_query_file(qspec.substr(2)));
      cats.push_back("file");
    } else {
      auto p = csv(qspec.substr(2));
      bdsm::QuerySpec spec;
      spec.category = bdsm::parse_query_category(p.at(0));
      spec.size = std::stoul(p.at(1));
      spec.count = std::stoul(p.at(2));
      queries = bdsm::generate_queries(g, spec, seed);
      cats.assign(queries.size(), p[0]);
      for (std::size_t i = 0; i < queries.size(); ++i) {
        std::ofstream f(std::filesystem::path(out) / ("query_" + std::to_string(i) + ".txt"));
        bdsm::save_query(f, queries[i]);
      }
    }
    std::vector<bdsm::UpdateBatch> stream;
    const std::string sv = sspec.substr(2);
    if (sv.find(',') == std::string::npos) {
      stream = bdsm::load_stream_file(sv);
    } else {
      auto p = csv(sv);
      bdsm::StreamSpec spec;
      spec.rate = std::stod(p.at(0));
      spec.mode = bdsm::parse_stream_mode(p.at(1));
      spec.batches = std::stoul(p.at(2));
      if (p.size() > 3) spec.kcore = std::uint32_t(std::stoul(p[3]));
      spec.seed = seed;
      stream = bdsm::generate_stream(g, spec);
      std::ofstream f(std::filesystem::path(out) / "stream.txt");
      bdsm::save_stream(f, stream);
    }
    bdsm::PipelineConfig config;
    config.match.coalesce = false;
    config.query_categories = cats;
    if (argc == 7) config.dump_matches_dir = out;
    bdsm::RunReport report = bdsm::run_pipeline(g, queries, stream, config);
    bdsm::emit_report(report, out);
    std::size_t pos = 0, neg = 0, unsolved = 0;
    for (const auto& d : report.deltas) {
      pos += d.positive;
      neg += d.negative;
    }
    for (const auto& q : report.queries) unsolved += q.solved ? 0 : 1;
    std::cout << "batches=" << report.deltas.size() << " positive=" << pos << " negative=" << neg
              << " unsolved_queries=" << unsolved << " reports=" << out << "/\n";
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return 0;
}
