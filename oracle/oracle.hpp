// TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the reference's
// per-batch hot path, used by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg as the CHECKER.  Nothing in paper_2401_17018_b200/ links or
// calls it.
//
// It restates bdsm::match_batch (reference src/matcher.cpp:370-389) with
// MatchOptions{coalesce=false} as a count-only engine:
//   validate (src/graph.cpp:8-23, :117-135) -> negative phase on G with the
//   pre-batch candidate table -> apply (src/graph.cpp:137-158) -> incremental
//   re-encode + table refresh (src/encoding.cpp:124-143, :171-191) -> positive
//   phase on G'.
// Each phase mirrors match_phase / run_match_task / gen_candidates /
// intersect_sorted / dedupe_by_order (src/matcher.cpp:27-117, :219-310,
// :328-368) and the plan is generate_matching_order per query edge
// (src/query_analysis.cpp:295-363).  Matches are counted, never materialised,
// which is exact because with coalescing off every match is emitted exactly
// once.  It reproduces the reference's MatchStats.dfs_visits,
// intersection_ops and tasks_run, which is how it is pinned to the reference
// (tests/test_oracle_vs_reference.py, tests/golden/).
//
// Semantics follow the reference's brute-force oracle where the engine
// diverges from it: an unlabelled query edge matches only
// an unlabelled data edge, and labels are compared exactly.
#pragma once

#include <cstddef>
#include <cstdint>

extern "C" {

typedef struct orc_engine orc_engine;

// Status codes shared with the CUDA engine's C ABI (include/bdsm_gpu.h).
enum {
  ORC_OK = 0,
  ORC_BATCH_ERROR = 1,      // all-or-nothing validation failure (BatchError)
  ORC_INVALID_ARGUMENT = 2, // self-loop / conflicting pair / bad query
  ORC_RUNTIME_ERROR = 3,
};

// Stats layout for orc_apply_batch (all summed over queries and both phases):
//   [0] dfs_visits  [1] intersection_ops  [2] tasks_run  [3] gen_candidates calls
//   [4] algorithmic adjacency bytes of the phases (SURVEY.md §8(d) B_phase)
//   [5] algorithmic bytes of the graph update (B_upd)
//   [6] dfs_visits outside the subtrees the visibility rule prunes (the tree
//       the CUDA engine walks: it applies dedupe_by_order at generation time)
enum { ORC_NSTATS = 7 };

orc_engine* orc_create(std::uint32_t nv, const std::uint32_t* vlabels, std::uint64_t ne,
                       const std::uint32_t* eu, const std::uint32_t* ev,
                       const std::uint32_t* elab /* nullable, 0xffffffff = none */,
                       std::uint32_t group_bits, char* err, std::size_t errcap);

// Returns the query index (>= 0) or -ORC_INVALID_ARGUMENT.
int orc_add_query(orc_engine* h, std::uint32_t n, const std::uint32_t* qlabels, std::uint32_t m,
                  const std::uint32_t* qa, const std::uint32_t* qb,
                  const std::uint32_t* qlab /* nullable */, char* err, std::size_t errcap);

// op: 0 insert, 1 delete.  pos/neg: one entry per query (both null: validate,
// apply and refresh without matching).  shard_rank/world:
// count only the anchor tasks this rank owns under the cost-balanced split
// (world 1 = everything).
int orc_apply_batch(orc_engine* h, std::uint64_t n, const std::uint32_t* uu,
                    const std::uint32_t* uv, const std::uint8_t* uop,
                    const std::uint32_t* ulab /* nullable */, std::uint32_t nthreads,
                    std::uint32_t shard_rank, std::uint32_t shard_world, std::uint64_t* pos,
                    std::uint64_t* neg, std::uint64_t* stats, char* err, std::size_t errcap);

// After ORC_BATCH_ERROR: failing update indices and reason codes
// (1 unknown vertex, 2 insert of existing edge, 3 delete of missing edge).
std::size_t orc_last_errors(orc_engine* h, std::uint64_t* idx, std::uint32_t* code,
                            std::size_t cap);

// Plan introspection: matching order of query q anchored at edge e.
int orc_order(orc_engine* h, int q, std::uint32_t e, std::uint32_t* out, std::size_t cap);
// Candidate row of data vertex v for query q.
std::uint32_t orc_row(orc_engine* h, int q, std::uint32_t v);
std::uint64_t orc_degree(orc_engine* h, std::uint32_t v);

void orc_destroy(orc_engine* h);
}
