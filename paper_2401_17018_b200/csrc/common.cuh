// Shared host/device definitions of the B200 engine (libbdsm_b200.so).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bdsm_b200 {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kMaxQ = 16;          // query vertices handled by the matching kernel
constexpr int kMaxQEdges = kMaxQ * (kMaxQ - 1) / 2;
constexpr int kWarpsPerBlock = 8;  // matching kernel: 256 threads
constexpr uint32_t kMaxQueries = 256;  // queries per engine (the memo tag's query field is 8 bits)
constexpr uint32_t kFull = 0xffffffffu;

// Device view of the slack-padded dynamic CSR:
// adj[off[v] .. off[v] + deg[v]) is v's sorted neighbour list, with room up to
// cap[v] for in-place merges; offsets are 64-bit (F9) and 16-byte aligned.
struct DevGraph {
  uint32_t V;
  const uint64_t* off;
  const uint32_t* deg;
  const uint32_t* cap;
  const uint32_t* adj;
  const uint32_t* elab;    // parallel to adj, or nullptr when no edge labels exist
  const uint32_t* vlabel;
  // Label index: loff[v * (nlab + 1) + k] = position in v's list of the first
  // neighbour of label class >= k (ids are label-ordered), so a label
  // sub-range is two loads instead of two binary searches; nullptr when the
  // graph has more than kMaxLabelIndex label classes.
  const uint32_t* loff;
  uint32_t nlab;
  // Hub membership bitmaps: hub_slot[v] = bitmap index of a high-degree vertex
  // (kNone otherwise); bitmap h holds bit y set iff y is a neighbour, so a
  // membership test in a hub's list is one load instead of a binary search.
  const uint32_t* hub_slot;
  const uint32_t* bitmaps;
  uint64_t bm_words;       // words per bitmap ((V + 31) / 32)
  // bit v set: the weight memo may hold entries of vertex v (set by memo_put,
  // cleared with the memo); the merge's invalidations skip the others
  uint32_t* memo_bits;
};

constexpr uint32_t kMaxLabelIndex = 64;
constexpr uint32_t kBitmapMinDeg = 1024;  // lists this long get a membership bitmap (within the budget)

#ifdef __CUDACC__
// Label sub-range [lo, hi) of label class `cls` (id range [vlo, vhi)) in x's
// sorted list lst[0, d): from the label index when present, else by binary
// search.  `which` 0 -> lo, 1 -> hi.
__device__ __forceinline__ uint32_t label_bound(const DevGraph& g, uint32_t x, const uint32_t* lst, uint32_t d,
                                                uint32_t cls, uint32_t vlo, uint32_t vhi, uint32_t which) {
  if (cls == kNone) return 0;
  if (g.loff) return __ldg(g.loff + uint64_t(x) * (g.nlab + 1) + cls + which);
  const uint32_t key = which ? vhi : vlo;
  uint32_t lo = 0, hi = d;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(lst + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
#endif

// Matching program of one (query, anchor edge): the matching order and, per
// level l >= 2, the backward neighbours (positions j < l adjacent to order[l]),
// the positions holding the same query label (injectivity candidates) and
// the query-edge label of each backward edge.  Built by the host planner.
struct LevelProg {
  uint32_t qbit;                 // 1 << order[l] (candidate-row bit)
  uint32_t vlo, vhi;             // internal-id range of label(order[l]) (ids are label-ordered)
  uint32_t lcls;                 // label class index of label(order[l]) (kNone: absent from the graph)
  uint32_t backmask;             // positions j < l adjacent to order[l]
  uint32_t eqmask;               // positions j < l with label(order[j]) == label(order[l])
  uint32_t nback;
  uint8_t back[kMaxQ];           // ascending positions
  uint32_t elab[kMaxQ];          // query edge label of (order[back[b]], order[l])
};

struct EdgeProg {
  uint32_t n;                    // query vertex count
  uint32_t query;                // query index
  uint32_t tail;                 // first level T of the independent tail (levels > T are counted, not enumerated)
  uint32_t order[kMaxQ];
  uint32_t inval[kMaxQ];         // position j -> independent tail levels whose cached count depends on M[j]
  uint32_t leafmask;             // tail levels that are leaves of level `tail` (weight f(M[tail]))
  uint32_t singlemask;           // independent tail levels with one backward neighbour j (weight f(M[j]))
  uint32_t sig[kMaxQ];           // weighted level t: (order[parent] << 4) | order[t], the weight's memo tag
  uint32_t natail;               // independent tail levels that depend on the anchor pair only
  uint8_t atail_slot[kMaxQ];     // level t -> its slot in the per-task count cache (0xff: none)
  LevelProg lv[kMaxQ];
};

// A distinct leaf signature of a query's programs (EdgeProg::sig): the
// parent query vertex p = order[T] (candidate bit, label id range) and the
// leaf's level program (candidate bit, label range, edge label in elab[0]).
struct LeafSig {
  uint32_t sig;
  uint32_t pbit;
  uint32_t plo, phi;
  LevelProg leaf;
};

// Anchor-mapping table entry (map_update_to_query_edges, src/matcher.cpp:42-55).
struct AnchorEdge {
  uint32_t la, lb;               // labels of query endpoints a, b
  uint32_t elab;                 // query edge label (kNone: unlabelled)
  uint32_t prog;                 // EdgeProg index
  uint32_t mult[2];              // per orientation (0: a->u, 1: a->v): matches each found one stands for
                                 // (1 without coalescing; the orbit size / 0 with exact coalescing, planner.hpp)
};

// One anchor: (update, query edge, orientation) with its level-2 driver length.
struct Task {
  uint32_t upd;
  uint32_t prog;
  uint32_t flip;
  uint32_t d;                    // level-2 driver range length (0 for 2-vertex queries)
  uint32_t base;                 // start of that range in the driver list (label sub-range)
  uint32_t mult;                 // AnchorEdge::mult of this orientation
};

// One work unit: a chunk [begin, begin + chunk) of a task's level-2 driver.
struct Item {
  uint32_t task;
  uint32_t begin;
};

// A donated DFS subtree (work sharing): the prefix
// assignment M[0..level), and the driver-index range [begin, end) of `level`.
// Either a driver range (ncand == 0) or an explicit list of already-filtered
// candidates of `level` taken from the donor's current chunk.
struct DynItem {
  uint32_t task;
  uint32_t level;
  uint32_t begin;
  uint32_t end;
  uint32_t ncand;
  uint32_t pad[3];
  uint32_t M[kMaxQ];
  uint32_t cand[32];
};

// Work-queue counters of one matching launch, each on its own 128-byte line
// so idle warps polling the queue do not contend with the busy warps' atomics.
struct alignas(128) PaddedU32 {
  uint32_t v;
  uint32_t pad[31];
};
// Ticket queue: an idle warp takes ticket t once and waits on slot t's own
// ready flag; donors reserve slots from `tail` when tickets > tail (a warp is
// waiting).  `holders` counts warps working plus donated items not yet
// finished, so holders == 0 means no work exists or can appear.
struct alignas(128) TicketTail {
  uint32_t tickets;     // tickets handed to idle warps
  uint32_t tail;        // donated slots reserved
  uint32_t pad[30];
};
struct QueueState {
  PaddedU32 next_item;  // static work-item head
  TicketTail tt;        // one 64-bit poll reads both (donors' demand check)
  PaddedU32 holders;
};

// Candidate rows carry the query-vertex bits in the low 16 bits (kMaxQ) and
// per-batch flags in the top bits: the vertex is an endpoint of an insert
// (positive phase) / delete (negative phase) of a batch in flight.  Two
// batches can be in flight (the pipelined stream: batch i's positive phase
// and batch i+1's negative phase share one launch), so each batch buffer slot
// has its own pair of bits.  The matching kernel gets the visibility-rule
// prefilter from the same load.
__host__ __device__ constexpr uint32_t row_ins_flag(uint32_t slot) { return 1u << (31 - 2 * slot); }
__host__ __device__ constexpr uint32_t row_del_flag(uint32_t slot) { return 1u << (30 - 2 * slot); }
constexpr uint32_t kRowFlags = 0xf0000000u;  // every slot's flags (kept by the merge's row refresh)

// Per-batch open-addressing table of the directed update keys (x << 32 | y)
// -> (batch index | op << 31), for O(1) visibility-rule lookups.
constexpr unsigned long long kEmptyKey = ~0ull;
__host__ __device__ __forceinline__ uint32_t pair_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return uint32_t(k);
}

// Persistent weight memo (matching kernel, invalidated by the merge): one
// 64-bit word per (vertex x, query q, signature sig) = x << 32 | q << 24 |
// sig << 16 | weight (a weight counts neighbours of x, so it is < 2^16 below
// degree 65535; larger ones are recomputed, never stored).  Weights >= kMemoInvalid are never stored; an entry
// whose weight field is kMemoInvalid was invalidated (its list or a
// neighbour's candidate row changed) and reads as a miss.  Linear probing,
// at most kMemoProbes slots.
constexpr int kMemoProbes = 8;
constexpr unsigned long long kMemoEmpty = ~0ull;
constexpr uint32_t kMemoWeightBits = 16;
constexpr unsigned long long kMemoWeightMask = (1ull << kMemoWeightBits) - 1;
constexpr unsigned long long kMemoInvalid = kMemoWeightMask;

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long memo_tag(uint32_t x, uint32_t q, uint32_t sig) {
  return (uint64_t(x) << 32) | (uint64_t(q & 0xff) << 24) | (uint64_t(sig & 0xff) << kMemoWeightBits);
}

__device__ __forceinline__ bool memo_get(const unsigned long long* memo, uint32_t mask, uint32_t x, uint32_t q,
                                         uint32_t sig, unsigned long long* w) {
  const unsigned long long tag = memo_tag(x, q, sig);
  uint32_t pos = pair_hash(tag) & mask;
  for (int i = 0; i < kMemoProbes; ++i) {
    const unsigned long long e = __ldcg(memo + pos);
    if (e == kMemoEmpty) return false;
    if ((e & ~kMemoWeightMask) == tag) {
      if ((e & kMemoWeightMask) == kMemoInvalid) return false;
      *w = e & kMemoWeightMask;
      return true;
    }
    pos = (pos + 1) & mask;
  }
  return false;
}

// Returns true when a fresh slot was taken (fill accounting).
__device__ __forceinline__ bool memo_put(unsigned long long* memo, uint32_t mask, uint32_t x, uint32_t q,
                                         uint32_t sig, unsigned long long w) {
  if (w >= kMemoInvalid) return false;
  const unsigned long long tag = memo_tag(x, q, sig);
  uint32_t pos = pair_hash(tag) & mask;
  for (int i = 0; i < kMemoProbes; ++i) {
    const unsigned long long prev = atomicCAS(memo + pos, kMemoEmpty, tag | w);
    if (prev == kMemoEmpty) return true;
    if ((prev & ~kMemoWeightMask) == tag) {
      if ((prev & kMemoWeightMask) == kMemoInvalid) atomicCAS(memo + pos, prev, tag | w);
      return false;
    }
    pos = (pos + 1) & mask;
  }
  return false;
}

__device__ __forceinline__ void memo_invalidate(unsigned long long* memo, uint32_t mask, uint32_t x, uint32_t q,
                                                uint32_t sig);
// The merge's invalidation of x's entries: a probe only when x ever had one
// (most touched vertices of a large batch never did: one bit load instead of a
// random probe of the memo per signature).
__device__ __forceinline__ void memo_invalidate_v(const uint32_t* memo_bits, unsigned long long* memo,
                                                  uint32_t mask, uint32_t x, uint32_t q, uint32_t sig) {
  if (memo_bits && !((__ldcg(memo_bits + (x >> 5)) >> (x & 31)) & 1u)) return;
  memo_invalidate(memo, mask, x, q, sig);
}
__device__ __forceinline__ void memo_invalidate(unsigned long long* memo, uint32_t mask, uint32_t x, uint32_t q,
                                                uint32_t sig) {
  const unsigned long long tag = memo_tag(x, q, sig);
  uint32_t pos = pair_hash(tag) & mask;
  for (int i = 0; i < kMemoProbes; ++i) {
    const unsigned long long e = __ldcg(memo + pos);
    if (e == kMemoEmpty) return;
    if ((e & ~kMemoWeightMask) == tag) {
      atomicExch(memo + pos, tag | kMemoInvalid);
      return;
    }
    pos = (pos + 1) & mask;
  }
}
#endif

// Device-side batch bookkeeping, copied back once per batch.  The per-query
// results follow it in the same allocation (one D2H): u64 counts[2][nq]
// ([phase][query] matches) and u32 timed_out[nq] (deadline fired).
struct BatchState {
  BatchState* prev;              // the preceding batch of a pipelined stream (nullptr: none); a batch
                                 // whose predecessor aborted aborts too (overflow 6).  When the
                                 // predecessor completes (its k_clear_flags, after the launch that ran
                                 // its positive phase) its abort is folded into this batch's flags and
                                 // the pointer cleared, before the predecessor's slot is reused
  uint32_t err_count;            // validate_batch failures
  uint32_t selfloop_min;         // first self-loop update index (kNone: none)
  uint32_t conflict_min;         // first conflicting update index (kNone: none)
  uint32_t n_touched;            // distinct endpoints
  uint32_t overflow;             // 1 pool exhausted (merge skipped), 2/3 work items of the negative /
                                 // positive phase, 4 labelled insert into an unlabelled graph, 5 id beyond
                                 // the sorted bits, 6 a preceding batch of the stream aborted
  uint32_t n_tasks[2];           // per phase (0 negative, 1 positive), last query
  uint32_t n_items[2];
  uint32_t item_lo[2], item_hi[2];  // multi-GPU: this rank's work items per phase, a contiguous index range
                                    // (owners are monotone in the canonical order), so k_wbm never walks
                                    // the other ranks' items
  uint32_t donations;            // statistics: donated subtrees
  uint32_t n_big;                // long lists this batch (k_alloc -> k_merge_big)
  uint32_t n_small;              // short lists this batch (k_alloc -> k_merge_small)
  uint32_t n_mid;                // the other lists (k_alloc -> k_merge_refresh)
  uint64_t pool_top;             // adjacency pool bump pointer (elements)
  uint64_t relocations;
  uint64_t bytes_update;
  uint64_t visits;
  uint64_t tasks_total;
  uint64_t items_total;
  uint64_t gen_calls;
  uint64_t bytes_phase;
  uint64_t bytes_kernel;         // 4 B x backward degrees of the GenCandidates calls the kernel made
  // -DBDSM_TRACE builds only, per phase: busy ns summed over items, longest
  // item ns, its (kind << 8 | start level), static items, donated items,
  // first item start / last item end (%globaltimer), and for the longest
  // item: main-loop chunks, tail chunks, warp-counted leaf misses, donations,
  // anchor endpoint degrees (deg0 << 32 | deg1), SM cycles spent donating,
  // filtering chunks, weighting leaves, in setups (incl. tail factors)
  uint64_t trace[2][16];
  uint64_t trace_chunks[2][kMaxQ];  // -DBDSM_TRACE: 32-candidate chunks filtered per level
  uint64_t trace_setups[2][kMaxQ];  // -DBDSM_TRACE: GenCandidates setups per level
};

#ifdef __CUDACC__
__device__ __forceinline__ bool batch_aborted_own(const BatchState* st) {
  return st->err_count || st->selfloop_min != kNone || st->conflict_min != kNone || st->overflow;
}
// Every kernel of a batch returns at once when the batch was rejected or must
// be rerun, or when the batch before it in a pipelined stream was (then this
// batch is marked as well, so the chain propagates).
__device__ __forceinline__ bool batch_aborted(BatchState* st) {
  if (batch_aborted_own(st)) return true;
  if (st->prev && batch_aborted_own(st->prev)) {
    st->overflow = 6;
    return true;
  }
  return false;
}
#endif

}  // namespace bdsm_b200
