// Kernel entry points of libbdsm_b200.so (definitions in store.cu, match.cu).
#pragma once

#include "common.cuh"

namespace bdsm_b200 {

struct bdsm_update_dev {  // mirrors bdsm_update (include/bdsm_gpu.h)
  uint32_t u, v, op, elab;
};

// Per-query filter tables on the device (candidate rows, encodings).
struct DevQueryEnc {
  uint32_t n;                    // query vertices
  uint32_t G;                    // counter groups
  uint32_t cap;                  // saturation cap
  uint32_t qlabel[kMaxQ];
  uint32_t glabel[kMaxQ];
  uint32_t glo[kMaxQ], ghi[kMaxQ];  // internal-id range of each group's label (ids are label-ordered)
  uint32_t gcls[kMaxQ];          // label class index of each group's label (kNone: absent from the graph)
  uint32_t nsig;                 // memo signatures of this query's weighted levels (invalidation)
  uint32_t sig[kMaxQ * 2];
  uint8_t qcnt[kMaxQ][kMaxQ];    // [u][g]
};

// Mutable device graph (owner's view).
struct DevGraphMut {
  uint32_t V;
  uint64_t* off;
  uint32_t* deg;
  uint32_t* cap;
  uint32_t* adj;
  uint32_t* elab;
  uint32_t* vlabel;
  uint64_t pool_size;
  uint32_t* loff;                // label index (see DevGraph), or nullptr
  uint32_t nlab;
  const uint32_t* class_lo;      // first internal id of each label class [nlab]
  const uint32_t* hub_slot;      // membership bitmaps (see DevGraph), or nullptr
  uint32_t* bitmaps;
  uint64_t bm_words;
  uint32_t* memo_bits;           // see DevGraph
};

// ---- store.cu: build ------------------------------------------------------
void launch_build_keys(const uint32_t* src, const uint32_t* dst, uint64_t E, uint32_t V,
                       uint64_t* keys, uint64_t* vals, uint32_t* bad, cudaStream_t s);
void launch_check_sorted_dups(const uint64_t* keys, uint64_t n, uint32_t* bad, cudaStream_t s);
void launch_degrees(const uint64_t* keys, uint64_t n, uint32_t* deg, cudaStream_t s);
void launch_caps(const uint32_t* deg, uint32_t V, float slack, uint32_t* cap, uint64_t* cap64,
                 cudaStream_t s);
void launch_scatter(const uint64_t* keys, const uint64_t* vals, uint64_t n, const uint64_t* dense_off,
                    const uint64_t* off, uint32_t* adj, const uint32_t* edge_labels, uint32_t* elab,
                    cudaStream_t s);
void launch_compact(DevGraphMut g_old, const uint64_t* new_off, const uint32_t* new_cap,
                    uint32_t* new_adj, uint32_t* new_elab, cudaStream_t s);

// ---- store.cu: per batch ---------------------------------------------------
void launch_prepare(const bdsm_update_dev* ups, uint32_t n, DevGraph g, const uint32_t* new_of,
                    bdsm_update_dev* iups, BatchState* st, uint64_t* keys, uint32_t* vals, uint32_t* dlab,
                    uint8_t* ecode, uint32_t id_limit, uint32_t key_bits, cudaStream_t s);
// pipelined stream: K1 split around the previous batch's merge (store.cu)
void launch_translate(const bdsm_update_dev* ups, uint32_t n, uint32_t V, bool has_elab, const uint32_t* new_of,
                      bdsm_update_dev* iups, BatchState* st, uint64_t* keys, uint32_t* vals, uint8_t* ecode,
                      uint32_t id_limit, uint32_t key_bits, cudaStream_t s);
void launch_validate(const bdsm_update_dev* iups, uint32_t n, DevGraph g, BatchState* st, uint32_t* dlab,
                     uint8_t* ecode, uint32_t* const* rows, uint32_t nq, uint32_t slot, cudaStream_t s);
void launch_post_sort(const uint64_t* in_keys, const uint32_t* in_vals, uint32_t key_bits, uint64_t* out_keys,
                      uint32_t* out_vals, uint32_t m, BatchState* st, uint8_t* head, uint32_t* insflag,
                      uint32_t* const* rows, uint32_t nq, uint32_t V, unsigned long long* hkeys, uint32_t* hvals,
                      uint32_t hmask, uint32_t slot, cudaStream_t s);
void launch_clear_flags(const uint64_t* skeys, uint32_t m, uint32_t* const* rows, uint32_t nq, uint32_t V,
                        uint32_t slot, cudaStream_t s, BatchState* next = nullptr);
void launch_alloc(const uint32_t* heads, const uint64_t* skeys, const uint32_t* ins_prefix,
                  uint32_t m, DevGraph g, float slack, BatchState* st, uint64_t* new_off,
                  uint32_t* new_cap, uint32_t* big_list, uint32_t* small_list, uint32_t* mid_list,
                  uint32_t small_max, uint32_t big_min, cudaStream_t s);
void launch_merge_refresh(const uint32_t* heads, const uint64_t* skeys, const uint32_t* svals,
                          const uint32_t* ins_prefix, uint32_t m, const bdsm_update_dev* ups,
                          DevGraphMut g, const uint64_t* new_off, const uint32_t* new_cap,
                          uint32_t* ipos, const DevQueryEnc* qenc, uint32_t nq, uint32_t* const* rows,
                          uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
                          uint32_t memo_mask, const uint32_t* big_list, const uint32_t* small_list,
                          const uint32_t* mid_list, uint32_t small_mode, int num_sms, cudaStream_t s,
                          cudaStream_t s_big);
void launch_encode_all(DevGraph g, const DevQueryEnc* qenc, uint32_t* rows, int num_sms, cudaStream_t s);
void launch_column_sizes(const uint32_t* rows, uint32_t V, uint32_t n, uint64_t* out, cudaStream_t s);
void launch_label_index(DevGraphMut g, int num_sms, cudaStream_t s);
void launch_build_bitmaps(DevGraphMut g, const uint32_t* hubs, uint32_t nhubs, cudaStream_t s);
void launch_hot_walks(const uint32_t* heads, const uint64_t* skeys, const BatchState* st, DevGraph g,
                      uint32_t* heat, uint32_t walks, uint32_t depth, uint32_t seed, int num_sms, cudaStream_t s);
void launch_hot_pack(DevGraphMut g, uint32_t* heat, unsigned long long* hist, unsigned long long budget,
                     BatchState* st, int num_sms, cudaStream_t s);

// ---- match.cu ---------------------------------------------------------------
// Per-update anchor counts (K5 pass 1) and their exclusive scan (one CUB scan).
struct AnchorCount {
  uint32_t tasks, items;
  uint64_t cost;
};
struct AnchorCountSum {
  __host__ __device__ AnchorCount operator()(const AnchorCount& x, const AnchorCount& y) const {
    return AnchorCount{x.tasks + y.tasks, x.items + y.items, x.cost + y.cost};
  }
};

struct PhaseArgs {
  DevGraph g;
  const bdsm_update_dev* ups;
  uint32_t n_ups;
  const uint32_t* dlab;          // pre-batch edge labels of deletes
  const AnchorEdge* anchors;     // anchor table of this query
  uint32_t n_anchor;
  const EdgeProg* progs;
  const uint32_t* rows;          // candidate rows of this query
  const uint64_t* skeys;         // sorted directed batch keys
  const uint32_t* svals;
  uint32_t m_keys;
  const unsigned long long* hkeys;  // visibility table (pair_hash, linear probing)
  const uint32_t* hvals;
  uint32_t hmask;
  uint32_t phase;                // 0 negative (deletes), 1 positive (inserts)
  uint32_t flag;                 // candidate-row flag of this phase's batch endpoints (row_del/ins_flag(slot))
  uint32_t query;
  uint32_t qn;                   // query vertex count
  uint32_t chunk;
  uint32_t shard_rank, shard_world;
  AnchorCount* upd_cnt;          // [n_ups + 1] per-update anchors / items / driver mass (scan input)
  AnchorCount* upd_off;          // its exclusive scan
  uint32_t self_scan;            // small batch: k_anchor_emit scans upd_cnt itself (upd_off unused)
  Task* tasks;
  Item* items;
  uint32_t max_items;
  BatchState* st;
  unsigned long long* count_out; // this (query, phase)'s match count (after the BatchState)
  uint32_t* timed_out;           // this query's deadline flag
  uint64_t deadline_ns;          // 0: none
  QueueState* q;                 // work-queue counters (reset before each launch)
  DynItem* dyn;                  // donated-subtree queue
  uint32_t* dyn_ready;           // per-slot epoch: slot is readable when == epoch
  uint32_t dyn_cap;
  uint32_t epoch;
  uint32_t merge_ratio;          // merge-window intersection when |other| <= ratio x |driver|
  uint32_t backoff_max;          // idle warps' longest sleep between donation polls (ns)
  unsigned long long* memo;      // weight memo (persistent; common.cuh)
  uint32_t memo_mask;
  unsigned long long* memo_fill; // slots taken (the engine resets the memo when it fills up)
  const uint32_t* heads;         // segment heads of the sorted batch keys (touched vertices)
  unsigned long long* task_tail; // per-task counts of anchor-only tail levels ([task][natail_stride], ~0 = unset)
  uint32_t natail_stride;
  uint32_t* match_out;           // non-null: materialise matches ([match_cap][n], query vertex order)
  unsigned long long* match_count;
  unsigned long long match_cap;
};

void launch_anchor_count(const PhaseArgs& a, cudaStream_t s);
void launch_anchor_emit(const PhaseArgs& a, cudaStream_t s);
// Two phases of one launch (k_wbm): the pipelined stream's positive phase of
// batch i and negative phase of batch i+1, on the same graph.
struct PhasePair {
  PhaseArgs p[2];
  uint32_t n;  // phases in use (1 or 2)
};
// ctas_per_sm: 2 (104 registers, launches bound by their longest subtree), 3 (80), 4 (64, many work items).
// second: a phase of the next batch on the same graph, run in the same launch (nullptr: one phase).
void launch_wbm(const PhaseArgs& a, const PhaseArgs* second, int num_sms, int ctas_per_sm, cudaStream_t s);
void launch_leaf_prefill(const PhaseArgs& a, const LeafSig* sigs, uint32_t nsig, const uint32_t* hubs,
                         const uint32_t* n_hubs, int num_sms, cudaStream_t s);
void launch_select_hubs(const uint32_t* deg, uint32_t V, uint32_t min_deg, uint32_t* hubs, uint32_t* n_hubs,
                        void* tmp, size_t tmp_bytes, cudaStream_t s);
size_t select_hubs_tmp_bytes(uint32_t V);

}  // namespace bdsm_b200
