/* bdsm_gpu.h — C ABI of the B200-native batch-dynamic subgraph matching engine
 * (libbdsm_b200.so).  Plain pointers and sizes only; no CUDA or torch types.
 *
 * The reference has no FFI: its boundary is the bdsm_core C++ API
 * (SURVEY.md §8(b)).  Each entry point below replaces the reference call
 * named beside it; INTEGRATION.md shows the bindings (C++ wrapper, ctypes).
 *
 * Semantics are the reference's with MatchOptions{coalesce=false} (SURVEY.md
 * F1), with its brute-force oracle's edge-label and vertex-label rules
 * (F4, F5): per batch the engine returns |positive| = |Matches(G') \ Matches(G)|
 * and |negative| = |Matches(G) \ Matches(G')| for every registered query.
 */
#ifndef BDSM_GPU_H_
#define BDSM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BDSM_API __attribute__((visibility("default")))
#else
#define BDSM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BDSM_NO_LABEL 0xffffffffu /* "no edge label" (reference: std::nullopt) */

/* Status codes map one-to-one onto the reference's exceptions. */
typedef enum bdsm_status {
  BDSM_OK = 0,
  BDSM_BATCH_ERROR = 1,      /* bdsm::BatchError (src/graph.cpp:117-143, src/matcher.cpp:373-378) */
  BDSM_INVALID_ARGUMENT = 2, /* std::invalid_argument: self-loop / conflicting pair in a batch
                                (src/graph.cpp:13-20), bad graph (src/graph.cpp:38-64) or query
                                (src/query_graph.cpp:14-22, src/query_analysis.cpp:361,367) */
  BDSM_RUNTIME_ERROR = 3,    /* std::runtime_error (src/scheduler.cpp:281-283) */
  BDSM_CUDA_ERROR = 4,       /* device failure (no reference counterpart) */
  BDSM_OUT_OF_MEMORY = 5     /* std::bad_alloc */
} bdsm_status;

typedef struct bdsm_engine bdsm_engine;

/* Data graph: replaces LabeledGraph::build_from_edges(vertices, edges)
 * (include/bdsm/graph.hpp:69-70, src/graph.cpp:35-72).  Vertex ids are dense
 * 0..num_vertices-1; edges are undirected, simple, without self-loops. */
typedef struct bdsm_graph_desc {
  uint32_t num_vertices;
  const uint32_t* vertex_labels; /* [num_vertices] */
  uint64_t num_edges;
  const uint32_t* src;           /* [num_edges] */
  const uint32_t* dst;           /* [num_edges] */
  const uint32_t* edge_labels;   /* [num_edges] or NULL; BDSM_NO_LABEL = none */
} bdsm_graph_desc;

/* Query: replaces QueryGraph(labels, edges) (include/bdsm/query_graph.hpp:24). */
typedef struct bdsm_query_desc {
  uint32_t num_vertices;         /* <= 16 on the GPU engine (the reference allows 32,
                                    src/query_graph.cpp:14); connected */
  const uint32_t* vertex_labels;
  uint32_t num_edges;
  const uint32_t* a;
  const uint32_t* b;
  const uint32_t* edge_labels;   /* [num_edges] or NULL */
} bdsm_query_desc;

typedef struct bdsm_options {
  uint32_t group_bits;   /* NLF counter width M (reference default 2; PipelineConfig::group_bits) */
  uint32_t coalesce;     /* 1: exact coalesced search (MatchOptions::coalesce, src/matcher.cpp:119-140, done
                            right): one anchored orientation per automorphism orbit of directed query
                            edges, counted with the orbit size — the counts equal coalesce 0 on every
                            batch (the reference's version misses matches).  dfs_visits
                            then describe the search done, not the reference tree. */
  int32_t device;        /* CUDA device ordinal */
  uint32_t shard_rank;   /* multi-GPU: this rank's share of the work units */
  uint32_t shard_world;  /* 0 or 1 = whole batch */
  float slack;           /* per-vertex adjacency slack fraction (default 0.25) */
  float pool_reserve;    /* extra adjacency pool for relocations, fraction of 2|E| (default 0.5) */
  uint32_t chunk;        /* level-2 work-unit size, multiple of 8 (default 32) */
  uint32_t zero_copy;    /* 1: adjacency pool in mapped pinned host memory (graphs beyond HBM) */
  uint32_t l2_hot_mb;    /* > 0: hot-list L2 persistence budget in MB (K8 estimator + access-policy window) */
} bdsm_options;

/* One update: replaces EdgeUpdate (include/bdsm/graph.hpp:14-22).  The batch
 * order is the array index, as in UpdateBatch (src/graph.cpp:21). */
typedef struct bdsm_update {
  uint32_t u;
  uint32_t v;
  uint32_t op;          /* 0 insert, 1 delete */
  uint32_t edge_label;  /* inserts only; BDSM_NO_LABEL = none */
} bdsm_update;

/* Replaces UpdateError{index, reason} (include/bdsm/graph.hpp:36-39). */
typedef struct bdsm_update_error {
  uint64_t index;
  uint32_t reason;      /* 1 unknown vertex, 2 insert of existing edge, 3 delete of missing edge */
} bdsm_update_error;

/* Per-batch counters (MatchStats, include/bdsm/search.hpp:18-36, plus
 * device timing and the SURVEY.md §8(d) algorithmic byte counts). */
typedef struct bdsm_batch_stats {
  double ms_total;        /* host wall time of the call */
  double ms_device;       /* CUDA-event time of the whole device sequence, every attempt and rerun */
  double ms_negative;     /* matching kernel, negative phase(s) */
  double ms_update;       /* sort + merge + refresh */
  double ms_positive;     /* matching kernel, positive phase(s) */
  uint64_t dfs_visits;    /* candidates accepted at levels >= 2 */
  uint64_t tasks;         /* (update, query edge, orientation) anchors */
  uint64_t work_items;    /* level-2 chunks scheduled */
  uint64_t gen_calls;     /* GenCandidates calls (levels whose candidates were generated) */
  uint64_t bytes_phase;   /* B_phase: 4 B x backward-neighbour degrees per GenCandidates call */
  uint64_t bytes_update;  /* B_upd: 16|dB| + 4 x (old + new degree) of touched vertices */
  uint64_t touched;       /* distinct batch endpoints */
  uint64_t relocations;   /* adjacency lists moved to the append pool */
  uint32_t compactions;   /* pool compactions triggered by this batch */
  uint32_t timed_out;     /* bitmask of queries 0..31 whose deadline passed in this batch (counts
                             dropped); any query: bdsm_engine_query_timed_out */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  double ms_match_kernel;  /* CUDA-event time of the K6 matching kernels (both phases) */
  double ms_merge_kernel;  /* CUDA-event time of K3 alloc + merge/refresh */
  uint32_t kernel_launches;/* launches of this library's own kernels (CUB sort/scan excluded) */
  uint32_t cub_launches;   /* CUB sort / select / scan calls */
  uint64_t bytes_kernel;   /* 4 B x backward degrees of the GenCandidates calls the kernel actually made
                              (bytes_phase counts them on the reference's DFS tree; the kernel counts
                              independent query tails once per prefix instead of enumerating them) */
  uint32_t attempts;       /* device launches of the whole batch sequence (> 1: pool compaction, work-item
                              regrowth, edge-label array or full-width sort rerun); ms_device spans all */
  uint32_t reruns;         /* positive-phase reruns after a work-item regrowth (inside ms_device) */
} bdsm_batch_stats;

/* Engine lifecycle.  Replaces LabeledGraph::build_from_edges plus the
 * device-resident copy of the graph (PackedMemoryArray, src/pma.cpp). */
BDSM_API bdsm_status bdsm_engine_create(const bdsm_graph_desc* graph, const bdsm_options* opts,
                               bdsm_engine** out);
BDSM_API void bdsm_engine_destroy(bdsm_engine* engine);

/* Registers a query: QueryEncodingState::initialize (src/matcher.cpp:10-18) +
 * build_query_plan with coalescing off (src/query_analysis.cpp:358-363,
 * :437-441).  Returns the query index (>= 0) or -status.  Up to 256 queries
 * per engine (run_pipeline's query set, src/bench.cpp:370-479); each batch
 * reports one count per query. */
BDSM_API int bdsm_engine_add_query(bdsm_engine* engine, const bdsm_query_desc* query);

/* match_batch (src/matcher.cpp:370-389) over every registered query: validate,
 * negative phase on G, apply, refresh, positive phase on G'.  `updates` is
 * HOST memory.  pos/neg receive one count per query.  All-or-nothing: on
 * BDSM_BATCH_ERROR / BDSM_INVALID_ARGUMENT the graph is unchanged. */
BDSM_API bdsm_status bdsm_engine_apply_batch(bdsm_engine* engine, const bdsm_update* updates, size_t n,
                                    uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats);

/* Same, with `updates` already resident in device memory (HBM). */
BDSM_API bdsm_status bdsm_engine_apply_batch_device(bdsm_engine* engine, const bdsm_update* d_updates,
                                           size_t n, uint64_t* pos, uint64_t* neg,
                                           bdsm_batch_stats* stats);

/* Pipelined form of bdsm_engine_apply_batch (run_pipeline's stage overlap,
 * src/bench.cpp:370-564): submit copies the host batch into the engine's
 * page-locked staging buffer, enqueues its H2D and every phase, and returns
 * without waiting — the caller may reuse `updates` at once and prepare the
 * next batch while this one matches.  wait blocks until the batch is done,
 * runs any rerun it needs and reports exactly as bdsm_engine_apply_batch
 * (same counts, errors and all-or-nothing contract).  One batch in flight per
 * engine: submit while one is in flight, or wait with none, is
 * BDSM_INVALID_ARGUMENT. */
BDSM_API bdsm_status bdsm_engine_submit_batch(bdsm_engine* engine, const bdsm_update* updates, size_t n);
BDSM_API bdsm_status bdsm_engine_wait(bdsm_engine* engine, uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats);

/* Pipelined stream: k batches in order, with the same counts, errors and
 * all-or-nothing contract as k bdsm_engine_apply_batch calls.  The positive
 * phase of batch i and the negative phase of batch i+1 read the same graph
 * (after batch i's merge), so they run as one launch of the matching kernel
 * (run_pipeline's stage overlap, src/bench.cpp:495-545, on the device); the
 * host synchronises once per stream.  batches[i] is host memory, or device
 * memory with device_input != 0.  pos/neg: [k * num_queries] (batch-major);
 * stats: [k] or NULL (ms_device per batch is the pipeline step: from the end
 * of batch i-1 to the end of batch i).  On an error *done = the number of
 * batches applied before the failing one (whose error is returned, nothing of
 * it applied).  Batches must be non-empty.  Queries with a deadline, match
 * collection and the K8 L2 window fall back to one batch at a time. */
BDSM_API bdsm_status bdsm_engine_apply_stream(bdsm_engine* engine, const bdsm_update* const* batches,
                                             const size_t* sizes, size_t k, int device_input, uint64_t* pos,
                                             uint64_t* neg, bdsm_batch_stats* stats, size_t* done);

/* Per-query time budget in seconds for subsequent batches (MatchOptions::
 * deadline, PipelineConfig::timeout_seconds); <= 0 disables. */
BDSM_API bdsm_status bdsm_engine_set_deadline(bdsm_engine* engine, int query, double seconds_from_now);

/* Whether `query` is matched by later batches (default 1).  run_pipeline
 * stops matching a query once it is unsolved (src/bench.cpp:420-432, :463-467);
 * an inactive query reports 0/0. */
BDSM_API bdsm_status bdsm_engine_set_query_active(bdsm_engine* engine, int query, int active);

/* 1 if the deadline of `query` fired during the last batch (its counts of
 * that batch were dropped, MatchStats::timed_out), 0 if not, -status on a bad
 * index.  A deadline applies per batch; the engine keeps matching the query
 * in later batches until the caller deactivates it. */
BDSM_API int bdsm_engine_query_timed_out(bdsm_engine* engine, int query);

/* After BDSM_BATCH_ERROR: the failures in batch order (BatchError::failures).
 * Returns the total number of failures. */
BDSM_API size_t bdsm_last_batch_errors(bdsm_engine* engine, bdsm_update_error* out, size_t cap);

/* Message of the last failing call on this thread (exception::what()). */
BDSM_API const char* bdsm_last_error(void);

/* Introspection (tests, CLI): sorted neighbours of v (returns the degree),
 * candidate rows of a query, matching order for (query, edge), counts. */
BDSM_API size_t bdsm_engine_neighbors(bdsm_engine* engine, uint32_t v, uint32_t* out, size_t cap);
BDSM_API bdsm_status bdsm_engine_rows(bdsm_engine* engine, int query, uint32_t* out /* [V] */);
BDSM_API int bdsm_engine_order(bdsm_engine* engine, int query, uint32_t edge, uint32_t* out /* [32] */);
/* Host-only planner (no device): the matching order of `query` anchored at
 * query edge `edge` for the given candidate column sizes — build_query_plan's
 * per-edge order with coalescing off (src/query_analysis.cpp:295-363,
 * :437-441) — into order[num_vertices], and optionally the counted-tail level.
 * Returns num_vertices or -status. */
BDSM_API int bdsm_plan_order(const bdsm_query_desc* query, const uint64_t* column_sizes, uint32_t edge,
                             uint32_t* order, uint32_t* tail);
/* First level T of the independent tail of that order: levels > T are counted
 * once per prefix and multiplied instead of enumerated (no reference counterpart). */
BDSM_API int bdsm_engine_tail(bdsm_engine* engine, int query, uint32_t edge);
BDSM_API bdsm_status bdsm_engine_column_sizes(bdsm_engine* engine, int query, uint64_t* out /* [n] */);
BDSM_API uint64_t bdsm_engine_num_edges(bdsm_engine* engine);
BDSM_API uint32_t bdsm_engine_num_vertices(bdsm_engine* engine);
/* Rebuild the plan of a query from the current candidate columns
 * (drift replanning, src/bench.cpp:451-453). */
BDSM_API bdsm_status bdsm_engine_replan(bdsm_engine* engine, int query);

/* Host-only planner: the automorphism orbits of the query's directed edges
 * (d = 2*edge + flip; flip 0 = (a, b), 1 = (b, a)) used by exact coalescing.
 * mult[d] = orbit size when d is its orbit's representative (its lowest
 * index), 0 otherwise; all 1 when the query has more than 20,000
 * automorphisms (the reference's KDegenOptions limit).  mult has 2*num_edges
 * entries.  Returns the number of automorphisms (or 0 when truncated), -status. */
BDSM_API int64_t bdsm_plan_edge_orbits(const bdsm_query_desc* query, uint32_t* mult);

/* Multi-GPU work split: owner rank of each work unit given
 * its cost, in canonical order.  owner = floor(world * prefix / total).
 * Pure host function, used by the engine and by the CPU tests. */
BDSM_API void bdsm_shard_owners(const uint64_t* costs, size_t n, uint32_t world, uint32_t* owners);

/* Bounded match materialisation (the reference's match vectors, for
 * --dump-matches, src/bench.cpp:484-491): with cap > 0 every later batch also
 * records up to `cap` matches per (query, phase); 0 returns to counts only. */
BDSM_API bdsm_status bdsm_engine_collect_matches(bdsm_engine* engine, uint64_t cap);
/* Matches of the last batch for (query, phase: 0 negative, 1 positive), in
 * external ids, query vertex order, sorted ascending (src/matcher.cpp:365-366);
 * copies up to `cap` matches (num_vertices words each) and returns the total
 * number of matches (> collected when the engine's cap was exceeded), or -status. */
BDSM_API int64_t bdsm_engine_matches(bdsm_engine* engine, int query, int phase, uint32_t* out, size_t cap);

/* Diagnostics of -DBDSM_TRACE builds: per-phase matching-kernel trace words
 * of the last batch (zeros otherwise).  Returns the number of words. */
BDSM_API size_t bdsm_engine_debug_trace(bdsm_engine* engine, uint64_t* out, size_t cap);

/* Multi-device engine group (SURVEY.md §8(e) in one process; the devices[]
 * option of §8(b)).  One engine per listed device (a device may repeat), each
 * holding a replica of the graph and applying every batch to it, and counting
 * only its share (shard r of n) of the canonical cost-balanced work-unit order;
 * a batch's counts are the sums over the engines.  The reference has no
 * multi-device mode; every call keeps the semantics of the engine call it is
 * named after (same counts, errors, all-or-nothing contract).  bdsm_options'
 * device / shard fields are set per engine.  Stats: times of the slowest engine,
 * work counters summed.  A query whose deadline fires on any device reports 0/0
 * for that batch.  apply_stream takes host batches only.  After a device failure
 * (BDSM_CUDA_ERROR / BDSM_OUT_OF_MEMORY) on any engine the replicas may differ:
 * destroy the group. */
typedef struct bdsm_group bdsm_group;
BDSM_API bdsm_status bdsm_group_create(const bdsm_graph_desc* graph, const bdsm_options* opts,
                                       const int32_t* devices, uint32_t num_devices, bdsm_group** out);
BDSM_API void bdsm_group_destroy(bdsm_group* group);
BDSM_API uint32_t bdsm_group_size(bdsm_group* group);
/* Engine r of the group (introspection: neighbours, rows, column sizes). */
BDSM_API bdsm_engine* bdsm_group_engine(bdsm_group* group, uint32_t r);
BDSM_API int bdsm_group_add_query(bdsm_group* group, const bdsm_query_desc* query);
BDSM_API bdsm_status bdsm_group_apply_batch(bdsm_group* group, const bdsm_update* updates, size_t n,
                                            uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats);
BDSM_API bdsm_status bdsm_group_submit_batch(bdsm_group* group, const bdsm_update* updates, size_t n);
BDSM_API bdsm_status bdsm_group_wait(bdsm_group* group, uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats);
BDSM_API bdsm_status bdsm_group_apply_stream(bdsm_group* group, const bdsm_update* const* batches,
                                             const size_t* sizes, size_t k, uint64_t* pos, uint64_t* neg,
                                             bdsm_batch_stats* stats, size_t* done);
BDSM_API size_t bdsm_group_last_batch_errors(bdsm_group* group, bdsm_update_error* out, size_t cap);
BDSM_API bdsm_status bdsm_group_set_deadline(bdsm_group* group, int query, double seconds_from_now);
BDSM_API bdsm_status bdsm_group_set_query_active(bdsm_group* group, int query, int active);
BDSM_API int bdsm_group_query_timed_out(bdsm_group* group, int query);
BDSM_API bdsm_status bdsm_group_replan(bdsm_group* group, int query);
/* Matches of the last batch over all engines, merged into one sorted list. */
BDSM_API bdsm_status bdsm_group_collect_matches(bdsm_group* group, uint64_t cap);
BDSM_API int64_t bdsm_group_matches(bdsm_group* group, int query, int phase, uint32_t* out, size_t cap);

BDSM_API const char* bdsm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BDSM_GPU_H_ */
