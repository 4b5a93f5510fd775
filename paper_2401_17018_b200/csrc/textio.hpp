// Host text formats and workload generators of the `bdsm run` CLI.
//
// Formats restate src/io.cpp:16-148 (same records, comments, error messages);
// generators restate generate_queries / generate_stream (src/bench.cpp:67-140,
// :179-289) with the same RNG (std::mt19937_64) and the same draw order, so a
// seeded `--gen-queries` / `--gen-stream` run yields the reference's queries
// and stream (checked by tests/test_cli.py against the reference's own CLI).
#pragma once

#include <cstdint>
#include <istream>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "bdsm_gpu.hpp"

namespace bdsm::text {

struct Graph {
  std::vector<gpu::VertexRecord> vertices;
  std::vector<gpu::EdgeRecord> edges;
};

struct Query {
  std::vector<std::uint32_t> labels;
  std::vector<gpu::QueryEdge> edges;
};

using Batch = std::vector<gpu::EdgeUpdate>;

Graph load_graph(std::istream& in);
Graph load_graph_file(const std::string& path);
Query load_query(std::istream& in);
Query load_query_file(const std::string& path);
std::vector<Batch> load_stream(std::istream& in);
std::vector<Batch> load_stream_file(const std::string& path);
void save_query(std::ostream& out, const Query& q);
void save_stream(std::ostream& out, const std::vector<Batch>& stream);

struct StreamSpec {
  double rate = 0.10;
  std::string mode = "insert";  // insert | delete | mixed
  std::size_t batches = 1;
  std::optional<std::uint32_t> kcore;
  std::uint64_t seed = 1;
};

std::vector<Query> generate_queries(const Graph& g, const std::string& category, std::size_t size,
                                    std::size_t count, std::uint64_t seed);
std::vector<Batch> generate_stream(const Graph& g, const StreamSpec& spec);

}  // namespace bdsm::text
