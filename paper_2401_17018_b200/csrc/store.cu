// Graph store kernels: initial CSR build, batch validation and canonicalisation
// (K1), per-vertex merge into slack-padded adjacency (K3) fused with the
// incremental NLF re-encode and candidate-row refresh (K4).
//
// Replaces LabeledGraph::build_from_edges / validate_batch / apply_batch
// (reference src/graph.cpp:35-72, :117-158) over the PMA (src/pma.cpp), and
// incremental_reencode + CandidateTable::refresh (src/encoding.cpp:124-143,
// :171-191).  The invariant kept is "sorted, duplicate-free, symmetric
// adjacency"; the PMA density rules are not carried over.
#include "kernels.cuh"

#include <cub/cub.cuh>

#include <mutex>
#include <unordered_map>

namespace bdsm_b200 {

namespace {

constexpr int kThreads = 256;

// CTAs of `kernel` resident on the whole GPU at `threads` per CTA (one wave).
// The merge kernels stride over their lists statically, so a grid of 1.33
// waves (1184 CTAs where 888 fit) takes two waves' time.
template <typename K>
uint64_t resident_ctas(K kernel, int threads, int num_sms) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;  // (kernel) -> CTAs per SM at `threads`
  const void* key = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_sm.find(key);
  if (it == per_sm.end()) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, 0) != cudaSuccess || n < 1) n = 1;
    it = per_sm.emplace(key, n).first;
  }
  return uint64_t(num_sms) * uint64_t(it->second);
}

inline unsigned blocks_for(uint64_t n, int threads = kThreads) {
  uint64_t b = (n + threads - 1) / threads;
  if (b == 0) b = 1;
  if (b > (1u << 30)) b = 1u << 30;
  return unsigned(b);
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ a, uint32_t n,
                                                    uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// lower_bound by a whole warp: 32 probes per round narrow the range 32-fold,
// so a list of up to 1024 entries takes two dependent loads instead of ten.
// Every lane returns the same position.
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t x,
                                                     uint32_t lane) {
  uint32_t lo = 0, len = n;
  while (len > 32) {
    const uint32_t b = (len + 31) >> 5;  // bucket size; lane i probes bucket i's last entry
    const uint32_t idx = lo + (lane + 1) * b - 1;
    const bool less = idx < lo + len && __ldg(a + idx) < x;
    const uint32_t c = __popc(__ballot_sync(kFull, less));  // buckets entirely below x
    const uint32_t end = lo + len;
    lo += c * b;
    len = lo >= end ? 0u : (end - lo < b ? end - lo : b);
  }
  const bool less = lane < len && __ldg(a + lo + lane) < x;
  return lo + __popc(__ballot_sync(kFull, less));
}

__device__ __forceinline__ uint32_t slack_cap(uint32_t d, float slack) {
  uint64_t extra = uint64_t(float(d) * slack);
  if (extra < 4) extra = 4;
  uint64_t c = uint64_t(d) + extra;
  c = (c + 3) & ~uint64_t(3);  // 16-byte aligned lists (128-bit loads)
  if (c > 0x3ffffff0ull) c = 0x3ffffff0ull;  // new_cap[] keeps two flag bits above the capacity
  return uint32_t(c);
}

// ---------------------------------------------------------------- build ----

__global__ void k_build_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                             uint64_t E, uint32_t V, uint64_t* keys, uint64_t* vals, uint32_t* bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t u = src[i], v = dst[i];
    if (u == v) atomicOr(bad, 1u);                 // self-loop
    if (u >= V || v >= V) atomicOr(bad, 2u);       // unknown vertex
    keys[2 * i] = (uint64_t(u) << 32) | v;
    keys[2 * i + 1] = (uint64_t(v) << 32) | u;
    if (vals) {
      vals[2 * i] = i;
      vals[2 * i + 1] = i;
    }
  }
}

__global__ void k_check_dups(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x + 1; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (keys[i] == keys[i - 1]) atomicOr(bad, 4u);  // duplicate edge
  }
}

__global__ void k_degrees(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* deg) {
  // keys are sorted: count run lengths at run ends.
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t s = uint32_t(keys[i] >> 32);
    bool last = (i + 1 == n) || uint32_t(keys[i + 1] >> 32) != s;
    if (last) {
      // binary search the run start
      uint64_t lo = 0, hi = i;
      while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (uint32_t(keys[mid] >> 32) < s) lo = mid + 1;
        else hi = mid;
      }
      deg[s] = uint32_t(i + 1 - lo);
    }
  }
}

__global__ void k_caps(const uint32_t* __restrict__ deg, uint32_t V, float slack, uint32_t* cap,
                       uint64_t* cap64) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    uint32_t c = slack_cap(deg[v], slack);
    cap[v] = c;
    cap64[v] = c;
  }
}

__global__ void k_scatter(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                          uint64_t n, const uint64_t* __restrict__ dense_off,
                          const uint64_t* __restrict__ off, uint32_t* adj,
                          const uint32_t* __restrict__ edge_labels, uint32_t* elab) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t k = keys[i];
    uint32_t s = uint32_t(k >> 32);
    uint64_t p = off[s] + (i - dense_off[s]);
    adj[p] = uint32_t(k);
    if (elab) elab[p] = edge_labels ? edge_labels[vals[i]] : kNone;
  }
}

// Warp per vertex: copy every list into a fresh pool with fresh slack.
__global__ void k_compact(DevGraphMut g, const uint64_t* __restrict__ new_off,
                          const uint32_t* __restrict__ new_cap, uint32_t* new_adj, uint32_t* new_elab) {
  uint32_t lane = threadIdx.x & 31;
  uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t v = warp; v < g.V; v += nwarps) {
    uint32_t d = g.deg[v];
    const uint32_t* src = g.adj + g.off[v];
    uint32_t* dst = new_adj + new_off[v];
    for (uint32_t i = lane; i < d; i += 32) dst[i] = src[i];
    if (new_elab) {
      const uint32_t* es = g.elab + g.off[v];
      uint32_t* ed = new_elab + new_off[v];
      for (uint32_t i = lane; i < d; i += 32) ed[i] = es[i];
    }
  }
}

// ------------------------------------------------------------- per batch ---

// K1: canonicalise and validate each update (UpdateBatch ctor,
// src/graph.cpp:8-23; validate_batch, src/graph.cpp:117-135).  Presence is a
// binary search in the lower-degree endpoint's sorted list.
// External vertex ids are translated to the internal label-ordered ids here;
// every later kernel reads the translated copy `iups`.
// id_limit: the radix sort only orders the low bits of the source id; an
// (invalid) id at or above it sets overflow 5 and the host reruns the batch
// with the full 64-bit sort, so its error is reported exactly.
__global__ void k_prepare(const bdsm_update_dev* __restrict__ ups, uint32_t n, DevGraph g,
                          const uint32_t* __restrict__ new_of, bdsm_update_dev* iups, BatchState* st,
                          uint64_t* keys, uint32_t* vals, uint32_t* dlab, uint8_t* ecode, uint32_t id_limit,
                          uint32_t key_bits) {
  // pipelined stream: this batch allocates from where its predecessor's merge
  // left the pool's bump pointer (k_prepare runs after that merge)
  if (blockIdx.x == 0 && threadIdx.x == 0 && st->prev) st->pool_top = st->prev->pool_top;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    bdsm_update_dev up = ups[i];
    if (up.u < g.V) up.u = new_of[up.u];
    if (up.v < g.V) up.v = new_of[up.v];
    iups[i] = up;
    if (up.u >= id_limit || up.v >= id_limit) st->overflow = 5;
    uint32_t del = up.op != 0 ? 1u : 0u;
    // sort keys (source << key_bits | destination); key_bits < 32 packs both
    // ids into the bits the radix sort orders (k_post_sort widens them back)
    keys[2 * i] = (uint64_t(up.u) << key_bits) | up.v;
    keys[2 * i + 1] = (uint64_t(up.v) << key_bits) | up.u;
    vals[2 * i] = i | (del << 31);
    vals[2 * i + 1] = i | (del << 31);
    uint32_t lab = kNone;
    uint8_t code = 0;
    if (up.u == up.v) {
      atomicMin(&st->selfloop_min, i);
    } else if (up.u >= g.V || up.v >= g.V) {
      code = 1;  // unknown vertex
    } else {
      uint32_t du = g.deg[up.u], dv = g.deg[up.v];
      uint32_t x = du <= dv ? up.u : up.v, y = du <= dv ? up.v : up.u;
      uint32_t dx = du <= dv ? du : dv;
      const uint32_t* lst = g.adj + g.off[x];
      uint32_t p = lower_bound_u32(lst, dx, y);
      bool present = p < dx && lst[p] == y;
      if (present && !del) code = 2;  // insert of existing edge
      if (!present && del) code = 3;  // delete of missing edge
      if (present && g.elab) lab = g.elab[g.off[x] + p];
    }
    if (code) atomicAdd(&st->err_count, 1u);
    // labelled insert while the graph keeps no label array: abort, the host
    // materialises the labels and reruns the batch (nothing applied yet)
    if (!del && up.elab != kNone && !g.elab) st->overflow = 4;
    ecode[i] = code;
    dlab[i] = lab;
  }
}

// Pipelined stream, K1 in two parts.  k_translate is the graph-independent
// part of k_prepare (ids, sort keys, self-loops, unknown vertices, labelled
// inserts into an unlabelled graph), so the next batch's key sort can run on a
// side stream while the current batch merges; k_validate is the rest, after
// that merge: presence of every update in G (insert of an existing / delete of
// a missing edge, src/graph.cpp:117-135), the pre-batch labels of deleted
// edges, the batch-endpoint flags in the candidate rows, and the pool's bump
// pointer taken over from the predecessor's merge.
__global__ void k_translate(const bdsm_update_dev* __restrict__ ups, uint32_t n, uint32_t V, bool has_elab,
                            const uint32_t* __restrict__ new_of, bdsm_update_dev* iups, BatchState* st,
                            uint64_t* keys, uint32_t* vals, uint8_t* ecode, uint32_t id_limit, uint32_t key_bits) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    bdsm_update_dev up = ups[i];
    if (up.u < V) up.u = new_of[up.u];
    if (up.v < V) up.v = new_of[up.v];
    iups[i] = up;
    if (up.u >= id_limit || up.v >= id_limit) st->overflow = 5;
    const uint32_t del = up.op != 0 ? 1u : 0u;
    keys[2 * i] = (uint64_t(up.u) << key_bits) | up.v;
    keys[2 * i + 1] = (uint64_t(up.v) << key_bits) | up.u;
    vals[2 * i] = i | (del << 31);
    vals[2 * i + 1] = i | (del << 31);
    uint8_t code = 0;
    if (up.u == up.v) atomicMin(&st->selfloop_min, i);
    else if (up.u >= V || up.v >= V) code = 1;  // unknown vertex
    if (code) atomicAdd(&st->err_count, 1u);
    if (!del && up.elab != kNone && !has_elab) st->overflow = 4;
    ecode[i] = code;
  }
}

__global__ void k_validate(const bdsm_update_dev* __restrict__ iups, uint32_t n, DevGraph g, BatchState* st,
                           uint32_t* dlab, uint8_t* ecode, uint32_t* const* rows, uint32_t nq, uint32_t flag_ins,
                           uint32_t flag_del) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && st->prev) st->pool_top = st->prev->pool_top;  // see k_prepare
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bdsm_update_dev up = iups[i];
    const bool del = up.op != 0;
    uint32_t lab = kNone;
    if (up.u != up.v && up.u < g.V && up.v < g.V) {
      const uint32_t du = g.deg[up.u], dv = g.deg[up.v];
      const uint32_t x = du <= dv ? up.u : up.v, y = du <= dv ? up.v : up.u;
      const uint32_t dx = du <= dv ? du : dv;
      const uint32_t* lst = g.adj + g.off[x];
      const uint32_t p = lower_bound_u32(lst, dx, y);
      const bool present = p < dx && lst[p] == y;
      uint8_t code = 0;
      if (present && !del) code = 2;  // insert of existing edge
      if (!present && del) code = 3;  // delete of missing edge
      if (present && g.elab) lab = g.elab[g.off[x] + p];
      if (code) {
        ecode[i] = code;
        atomicAdd(&st->err_count, 1u);
      }
      for (uint32_t q = 0; q < nq; ++q) {
        atomicOr(rows[q] + up.u, del ? flag_del : flag_ins);
        atomicOr(rows[q] + up.v, del ? flag_del : flag_ins);
      }
    }
    dlab[i] = lab;
  }
}

// After the radix sort of the 2n directed keys: conflicting pairs, segment
// heads (distinct sources = touched vertices), insert flags for the merge
// prefix, and the per-phase same-kind endpoint flags in the candidate rows
// used to prefilter the visibility rule (UpdateIndex, src/matcher.cpp:27-40).
// in_keys/in_vals: the sort's output, keys packed as (source << key_bits |
// destination); out_keys/out_vals (non-null): where the widened
// (source << 32 | destination) keys and the values are written for every
// later kernel.  (rerun_positive passes the widened keys, key_bits 32, no out.)
__global__ void k_post_sort(const uint64_t* __restrict__ in_keys, const uint32_t* __restrict__ in_vals,
                            uint32_t key_bits, uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_vals,
                            uint32_t m, BatchState* st, uint8_t* head, uint32_t* insflag,
                            uint32_t* const* rows, uint32_t nq, uint32_t V, unsigned long long* hkeys,
                            uint32_t* hvals, uint32_t hmask, uint32_t flag_ins, uint32_t flag_del) {
  const uint64_t dmask = key_bits >= 32 ? 0xffffffffull : (1ull << key_bits) - 1;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= m; j += gridDim.x * blockDim.x) {
    if (j == m) {
      insflag[j] = 0;
      continue;
    }
    const uint64_t ck = in_keys[j];
    uint32_t val = in_vals[j];
    uint32_t src = uint32_t(ck >> key_bits);
    const uint64_t k = (uint64_t(src) << 32) | (ck & dmask);
    if (out_keys) {
      out_keys[j] = k;
      out_vals[j] = val;
    }
    bool is_del = val >> 31;
    if (j > 0 && in_keys[j - 1] == ck) {
      uint32_t a = in_vals[j - 1] & 0x7fffffffu, b = val & 0x7fffffffu;
      atomicMin(&st->conflict_min, a > b ? a : b);
    }
    bool h = j == 0 || uint32_t(in_keys[j - 1] >> key_bits) != src;
    head[j] = h ? 1 : 0;
    insflag[j] = is_del ? 0u : 1u;
    if (src < V)
      for (uint32_t q = 0; rows && q < nq; ++q) atomicOr(rows[q] + src, is_del ? flag_del : flag_ins);
    // visibility table: linear probing (duplicates only in rejected batches);
    // segment heads also map (src, kNone) -> the segment's first index
    for (int pass = 0; pass < (h ? 2 : 1); ++pass) {
      const unsigned long long key = pass ? ((uint64_t(src) << 32) | kNone) : (unsigned long long)k;
      uint32_t pos = pair_hash(key) & hmask;
      for (uint32_t probe = 0; probe <= hmask; ++probe) {
        unsigned long long prev = atomicCAS(hkeys + pos, kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) {
          hvals[pos] = pass ? j : val;
          break;
        }
        pos = (pos + 1) & hmask;
      }
    }
  }
}

// End of batch (also after a rejected one): clear the per-batch row flags of
// every touched vertex.
// Pipelined stream: `next` is the following batch's state.  This batch is
// complete now, so `next` folds this batch's abort into its own flags and
// stops looking back — before this batch's slot is handed to the batch after
// `next` (whose state overwrites it).
__global__ void k_clear_flags(const uint64_t* __restrict__ skeys, uint32_t m, uint32_t* const* rows,
                              uint32_t nq, uint32_t V, uint32_t flags, BatchState* next) {
  if (next && blockIdx.x == 0 && threadIdx.x == 0 && next->prev) {
    if (batch_aborted_own(next->prev)) next->overflow = 6;
    next->prev = nullptr;
  }
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    uint32_t src = uint32_t(skeys[j] >> 32);
    if (src < V && (j == 0 || uint32_t(skeys[j - 1] >> 32) != src))
      for (uint32_t q = 0; q < nq; ++q) rows[q][src] &= ~flags;
  }
}

#ifndef BDSM_BIG_LIST
#define BDSM_BIG_LIST 1024
#endif
#ifndef BDSM_SMALL_LIST
#define BDSM_SMALL_LIST 256
#endif
#ifndef BDSM_BIG_THREADS
#define BDSM_BIG_THREADS 256
#endif
constexpr uint32_t kBigList = BDSM_BIG_LIST;  // lists this long are merged by a whole CTA (k_merge_big)
constexpr uint32_t kBigFlag = 0x80000000u;  // new_cap[t]: the list is merged by k_merge_big
constexpr uint32_t kSmallList = BDSM_SMALL_LIST;  // lists up to this long (before and after): one thread each
constexpr uint32_t kSmallFlag = 0x40000000u;  // new_cap[t]: the list is merged by k_merge_small
// batch keys of a short list at most (k_merge_small keeps their positions in a
// per-thread array; a list with more keys goes to k_merge_refresh)
constexpr uint32_t kSmallKeys = 32;
constexpr uint32_t kCapMask = 0x3fffffffu;

__device__ __forceinline__ uint32_t seg_end(const uint32_t* heads, uint32_t t, uint32_t nt, uint32_t m) {
  return t + 1 < nt ? heads[t + 1] : m;
}

// K3 (part 1): per touched vertex, new degree and relocation when the merged
// list no longer fits its slack; the list goes to the kernel for its length.
// List appends and pool allocations are aggregated per CTA (warp ballots and
// scans into shared counters, then one global atomic per counter per CTA): a
// 1M-update batch touches 2M lists, and per-warp atomics on the same five
// counters serialise in L2.  In-place lists keep their offset, which the merge
// kernels read themselves (new_off is only written for relocations).
__global__ void __launch_bounds__(kThreads) k_alloc(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ ins_prefix,
    uint32_t m, DevGraph g, float slack, BatchState* st, uint64_t* new_off, uint32_t* new_cap, uint32_t* big_list,
    uint32_t* small_list, uint32_t* mid_list, uint32_t small_max, uint32_t big_min) {
  if (batch_aborted(st)) return;
  __shared__ uint32_t s_cnt[3];  // mid, big, small lists of this CTA round
  __shared__ unsigned long long s_pool, s_reloc;
  __shared__ uint32_t s_base[3];
  __shared__ unsigned long long s_pbase;
  const uint32_t nt = st->n_touched;
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  for (uint32_t c0 = blockIdx.x * blockDim.x; c0 < nt; c0 += gridDim.x * blockDim.x) {  // CTA-uniform
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_pool = s_reloc = 0;
    __syncthreads();
    const uint32_t t = c0 + threadIdx.x;
    uint32_t big = 0, small = 0, c = 0;
    if (t < nt) {
      const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
      const uint32_t x = uint32_t(skeys[s] >> 32);
      const uint32_t nins = ins_prefix[e] - ins_prefix[s];
      const uint32_t ndel = (e - s) - nins;
      const uint32_t dold = g.deg[x];
      const uint32_t dnew = dold + nins - ndel;
      // the pre-batch list is long (k_merge_big) / both lists are short (k_merge_small)
      big = dold >= big_min ? kBigFlag : 0u;
      small = !big && dold <= small_max && dnew <= small_max && e - s <= kSmallKeys ? kSmallFlag : 0u;
      if (dnew > g.cap[x] || (nins && ndel)) c = slack_cap(dnew, slack);  // overflow, or a mixed segment
    }
    const uint32_t bm = __ballot_sync(kFull, t < nt && !big && !small);
    const uint32_t bb = __ballot_sync(kFull, big != 0), bs = __ballot_sync(kFull, small != 0);
    const uint32_t br = __ballot_sync(kFull, c != 0);
    // warp offsets within the CTA
    uint32_t wo = 0;
    if (lane < 3) {
      const uint32_t b = lane == 0 ? bm : lane == 1 ? bb : bs;
      if (b) wo = atomicAdd(&s_cnt[lane], __popc(b));
    }
    const uint32_t wo_mid = __shfl_sync(kFull, wo, 0), wo_big = __shfl_sync(kFull, wo, 1);
    const uint32_t wo_small = __shfl_sync(kFull, wo, 2);
    uint64_t inc = c, wpool = 0;
    if (br) {  // relocations: the warp's slots carved by an inclusive scan
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) {
        wpool = atomicAdd(&s_pool, (unsigned long long)inc);
        atomicAdd(&s_reloc, (unsigned long long)__popc(br));
      }
      wpool = __shfl_sync(kFull, wpool, 31);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_base[0] = s_cnt[0] ? atomicAdd(&st->n_mid, s_cnt[0]) : 0u;
      s_base[1] = s_cnt[1] ? atomicAdd(&st->n_big, s_cnt[1]) : 0u;
      s_base[2] = s_cnt[2] ? atomicAdd(&st->n_small, s_cnt[2]) : 0u;
      s_pbase = s_pool ? atomicAdd((unsigned long long*)&st->pool_top, s_pool) : 0ull;
      if (s_reloc) atomicAdd((unsigned long long*)&st->relocations, s_reloc);
    }
    __syncthreads();
    if ((bm >> lane) & 1u) mid_list[s_base[0] + wo_mid + __popc(bm & lt)] = t;
    if (big) big_list[s_base[1] + wo_big + __popc(bb & lt)] = t;
    if (small) small_list[s_base[2] + wo_small + __popc(bs & lt)] = t;
    if (t < nt) {
      if (c) new_off[t] = s_pbase + wpool + inc - c;
      new_cap[t] = c | big | small;  // capacity 0: in place
    }
    __syncthreads();  // the shared counters are reset for the next round
  }
}

// Position of old element `a` (index i) in the merged list, and whether the
// batch deletes it.  seg/segn: the vertex's sorted batch keys (destination
// ids); ipre: insert prefix at the segment start.
__device__ __forceinline__ void merged_pos(const uint64_t* seg, uint32_t segn,
                                           const uint32_t* ins_prefix, uint32_t s, uint32_t a,
                                           uint32_t i, uint32_t& p, bool& deleted) {
  // lower_bound on the low 32 bits (same source throughout the segment)
  uint32_t lo = 0, hi = segn;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (uint32_t(seg[mid]) < a) lo = mid + 1;
    else hi = mid;
  }
  uint32_t I = ins_prefix[s + lo] - ins_prefix[s];
  uint32_t D = lo - I;
  deleted = lo < segn && uint32_t(seg[lo]) == a;
  p = i - D + I;
}

// Saturated neighbour counts of one query's label groups for a sorted list
// (encode_vertex, src/encoding.cpp:70-87): internal ids are label-ordered, so
// group g's count is the size of the id range [glo[g], ghi[g]) inside the
// list — two binary searches (lanes 2g / 2g+1) instead of a label gather per
// neighbour.  Returns lane g's count of group g.
__device__ __forceinline__ uint32_t group_counts(const uint32_t* lst, uint32_t d, const DevQueryEnc& qe,
                                                 uint32_t lane) {
  const uint32_t gi = lane >> 1;
  uint32_t bnd = 0;
  if (gi < qe.G) bnd = lower_bound_u32(lst, d, (lane & 1) ? qe.ghi[gi] : qe.glo[gi]);
  const uint32_t lo = __shfl_sync(kFull, bnd, (2 * lane) & 31);
  const uint32_t hi = __shfl_sync(kFull, bnd, (2 * lane + 1) & 31);
  uint32_t cnt = lane < qe.G ? hi - lo : 0;
  return cnt > qe.cap ? qe.cap : cnt;
}

// Candidate row of a vertex with label vl from lane g's saturated counts
// (encoding_contains, src/encoding.cpp:115-122).
__device__ __forceinline__ uint32_t row_of(const DevQueryEnc& qe, uint32_t vl, uint32_t cnt, uint32_t lane) {
  uint32_t row = 0;
  for (uint32_t u = 0; u < qe.n; ++u) {
    bool ok = lane >= qe.G || cnt >= qe.qcnt[u][lane];
    if (__all_sync(kFull, ok) && vl == qe.qlabel[u]) row |= 1u << u;
  }
  return row;
}

// Column-size deltas (CandidateTable column |C(u)|, read by the planner) of
// the first kColAggQ queries are summed per block in shared memory and added
// to the global counters once per block: a large batch flips thousands of
// rows, and per-list atomics on the same few counters serialise in L2.
constexpr uint32_t kColAggQ = 2;
struct ColAgg {
  int (*s)[kMaxQ];  // [kColAggQ][kMaxQ] shared accumulators
  uint32_t* done;   // shared: warps of the CTA that have finished
  __device__ __forceinline__ void init() {
    for (uint32_t i = threadIdx.x; i < kColAggQ * kMaxQ; i += blockDim.x) s[i / kMaxQ][i % kMaxQ] = 0;
    if (threadIdx.x == 0) *done = 0;
    __syncthreads();
  }
  __device__ __forceinline__ void add(uint64_t* const* colsize, uint32_t q, uint32_t u, bool up) {
    if (q < kColAggQ) atomicAdd(&s[q][u], up ? 1 : -1);
    else atomicAdd((unsigned long long*)(colsize[q] + u), up ? 1ull : (unsigned long long)(-1ll));
  }
  // Warp-collective, once per warp at its end: the CTA's last warp to finish
  // adds the sums, so finished warps exit instead of waiting at a barrier for
  // the CTA's slowest list.
  __device__ __forceinline__ void flush(uint64_t* const* colsize, uint32_t nq) {
    __threadfence_block();
    __syncwarp();
    uint32_t last = 0;
    if ((threadIdx.x & 31) == 0) last = atomicAdd(done, 1u) == (blockDim.x >> 5) - 1u;
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence_block();
    for (uint32_t i = threadIdx.x & 31; i < kColAggQ * kMaxQ; i += 32) {
      const uint32_t q = i / kMaxQ, u = i % kMaxQ;
      const int v = atomicAdd(&s[q][u], 0);
      if (q < nq && v) atomicAdd((unsigned long long*)(colsize[q] + u), (unsigned long long)(long long)v);
    }
  }
};

// After a list's merge (warp-collective): keep its membership bitmap in step,
// rewrite its label index, and recompute every query's candidate row from the
// label-range counts of the new list (K4).
__device__ __forceinline__ void finish_vertex(DevGraphMut& g, uint32_t x, const uint32_t* dst, uint32_t dnew,
                                              const uint64_t* seg, uint32_t segn, const uint32_t* segvals,
                                              const DevQueryEnc* __restrict__ qenc, uint32_t nq,
                                              uint32_t* const* rows, uint64_t* const* colsize,
                                              unsigned long long* memo, uint32_t memo_mask, uint32_t lane,
                                              ColAgg agg) {
  // the memoised weights of x (its list changed) are stale in every query
  for (uint32_t q = 0; q < nq; ++q)
    for (uint32_t k = lane; k < qenc[q].nsig; k += 32) memo_invalidate_v(g.memo_bits, memo, memo_mask, x, q, qenc[q].sig[k]);
    // membership bitmap of a hub: set inserted, clear deleted neighbours
    if (g.hub_slot) {
      const uint32_t hs = g.hub_slot[x];
      if (hs != kNone) {
        uint32_t* bm = g.bitmaps + uint64_t(hs) * g.bm_words;
        for (uint32_t k = lane; k < segn; k += 32) {
          const uint32_t y = uint32_t(seg[k]);
          if (segvals[k] >> 31) atomicAnd(bm + (y >> 5), ~(1u << (y & 31)));
          else atomicOr(bm + (y >> 5), 1u << (y & 31));
        }
      }
    }
    // label index of the new list (lane k: class k's first position): the
    // old position moved by the batch's inserts minus deletes below
    // class_lo[k] (the segment is sorted), no search of the new list
    uint32_t lpos = 0;
    if (g.loff)
      for (uint32_t k = lane; k <= g.nlab; k += 32) {
        uint32_t* cell = g.loff + uint64_t(x) * (g.nlab + 1) + k;
        if (k < g.nlab) {
          const uint32_t lo = g.class_lo[k];
          int acc = 0;
          for (uint32_t j = 0; j < segn && uint32_t(seg[j]) < lo; ++j) acc += (segvals[j] >> 31) ? -1 : 1;
          lpos = uint32_t(int(*cell) + acc);
        } else {
          lpos = dnew;
        }
        *cell = lpos;
      }
    const bool from_index = g.loff && g.nlab < 32;  // the whole index sits in lanes 0..nlab
    // 4. refresh: saturated per-group neighbour counts -> candidate rows (K4)
    const uint32_t vl = g.vlabel[x];
    for (uint32_t q = 0; q < nq; ++q) {
      const DevQueryEnc& qe = qenc[q];
      uint32_t cnt;
      if (from_index) {  // group g's count = the size of its label class's range
        const uint32_t cls = lane < qe.G ? qe.gcls[lane] : kNone;
        const uint32_t lo = __shfl_sync(kFull, lpos, cls == kNone ? 0 : cls);
        const uint32_t hi = __shfl_sync(kFull, lpos, cls == kNone ? 0 : cls + 1);
        cnt = cls == kNone ? 0 : hi - lo;
        if (cnt > qe.cap) cnt = qe.cap;
      } else {
        cnt = group_counts(dst, dnew, qe, lane);
      }
      const uint32_t row = row_of(qe, vl, cnt, lane);
      uint32_t word = 0;
      if (lane == 0) word = rows[q][x];
      word = __shfl_sync(kFull, word, 0);
      const uint32_t before = word & ~kRowFlags;  // keep the batch flags
      if (before != row) {
        const uint32_t diff = before ^ row;
        if (lane == 0) {
          rows[q][x] = row | (word & kRowFlags);
          uint32_t d = diff;
          while (d) {
            uint32_t u = __ffs(d) - 1;
            d &= d - 1;
            agg.add(colsize, q, u, (row >> u) & 1u);
          }
        }
        // x's candidate bits changed: the memoised weights of its neighbours
        // that count a query vertex among those bits are stale (a signature's
        // low nibble is the counted child vertex)
        for (uint32_t k = 0; k < qe.nsig; ++k) {
          const uint32_t sg = qe.sig[k];
          if (!((diff >> (sg & 15)) & 1u)) continue;
          for (uint32_t i = lane; i < dnew; i += 32) memo_invalidate_v(g.memo_bits, memo, memo_mask, dst[i], q, sg);
        }
      }
    }
}

constexpr uint32_t kMoveUnroll = 8;      // old elements per thread in flight per sweep step (k_merge_big)
constexpr uint32_t kWarpMoveUnroll = 4;  // the same for k_merge_refresh (lists < kBigList)
constexpr uint32_t kWarpSearchKeys = 4;  // k_merge_refresh: segments up to this many keys use warp searches
// k_merge_refresh is latency-bound over many lists: its register budget sets
// how many are in flight per SM.  5 CTAs: 48 registers (C4 279.2M updates/s,
// C2 12.38M); 6: 40 with 116 B of spills (280.8M, 12.17M); 4: 61 (277.8M)
#ifndef BDSM_MERGE_WARP_BLOCKS
#define BDSM_MERGE_WARP_BLOCKS 5
#endif
constexpr int kMergeWarpBlocks = BDSM_MERGE_WARP_BLOCKS;

// K3 (part 2) + K4: one warp per touched vertex.  Insert slots are computed
// first against the intact old list.  In place (merged list fits the slack)
// the old elements move in two sweeps — ascending for left-movers, descending
// for right-movers — in steps of 32 x kMoveUnroll elements: a step is read
// completely before it is written, and it only writes slots of its own step
// or of steps already read (the merged order is a monotone map of the old
// order and single-kind segments shift in one direction), so hub lists move
// with kMoveUnroll loads in flight per lane.  Relocated lists are merged out
// of place.  The same warp then recomputes the candidate row of every query
// from label-range counts of the new list (K4).
__global__ void __launch_bounds__(256, kMergeWarpBlocks) k_merge_refresh(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
    const uint32_t* __restrict__ svals, const uint32_t* __restrict__ ins_prefix, uint32_t m,
    const bdsm_update_dev* __restrict__ ups, DevGraphMut g, const uint64_t* __restrict__ new_off,
    const uint32_t* __restrict__ new_cap, uint32_t* ipos, const DevQueryEnc* __restrict__ qenc,
    uint32_t nq, uint32_t* const* rows, uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
    uint32_t memo_mask, const uint32_t* __restrict__ mid_list) {
  if (batch_aborted(st)) return;
  if (st->pool_top > g.pool_size) {
    if (threadIdx.x == 0 && blockIdx.x == 0) st->overflow = 1;
    return;
  }
  __shared__ int s_colagg[kColAggQ][kMaxQ];
  __shared__ uint32_t s_agg_done;
  ColAgg agg{s_colagg, &s_agg_done};
  agg.init();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nt = st->n_touched, nmid = st->n_mid;
  uint64_t bytes = 0;
  for (uint32_t mi = warp; mi < nmid; mi += nwarps) {
    const uint32_t t = mid_list[mi];  // neither long nor short (k_alloc's list)
    const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
    const uint64_t* seg = skeys + s;
    const uint32_t segn = e - s;
    const uint32_t x = uint32_t(seg[0] >> 32);
    const uint32_t dold = g.deg[x];
    const uint64_t ooff = g.off[x];
    const uint32_t nins = ins_prefix[e] - ins_prefix[s];
    const uint32_t dnew = dold + nins - (segn - nins);
    const uint32_t ncap = new_cap[t] & kCapMask;
    const bool reloc = ncap != 0;
    const uint64_t noff = reloc ? new_off[t] : ooff;
    uint32_t* src = g.adj + ooff;
    uint32_t* dst = g.adj + noff;
    uint32_t* esrc = g.elab ? g.elab + ooff : nullptr;
    uint32_t* edst = g.elab ? g.elab + noff : nullptr;

    // 1. insert slots against the intact old list, and the first position
    // that can move (entries below the first batch key never move).  A few
    // keys are searched one after another by the whole warp (two dependent
    // loads each below 1024 entries); many keys by one lane each.
    // With <= 32 keys, lane k also keeps key k's position in the old list
    // (k_lb) and kind (k_del): a moved element's merged position then comes
    // from ballots over the keys instead of a search per element.
    uint32_t start = 0, k_lb = 0;
    bool k_del = false;
#ifdef BDSM_NO_KEY_LANES
    const bool keys_in_lanes = false;
#else
    const bool keys_in_lanes = segn <= 32;
#endif
    if (segn <= kWarpSearchKeys) {
      for (uint32_t k = 0; k < segn; ++k) {
        const bool del = svals[s + k] >> 31;
        const uint32_t lb = warp_lower_bound(src, dold, uint32_t(seg[k]), lane);
        if (lane == k) {
          k_lb = lb;
          k_del = del;
        }
        if (k == 0 && !reloc) start = lb;
        if (!del && lane == 0) {
          const uint32_t ib = ins_prefix[s + k] - ins_prefix[s];
          ipos[s + k] = ib + (lb - (k - ib));
        }
      }
    } else {
      for (uint32_t k = lane; k < segn; k += 32) {
        const bool del = svals[s + k] >> 31;
        const uint32_t lb = lower_bound_u32(src, dold, uint32_t(seg[k]));
        if (k < 32) {
          k_lb = lb;
          k_del = del;
        }
        if (del) continue;
        const uint32_t ib = ins_prefix[s + k] - ins_prefix[s];
        ipos[s + k] = ib + (lb - (k - ib));
      }
      if (!reloc && dold) start = __shfl_sync(kFull, k_lb, 0);
    }
    __syncwarp();
    // 2. move old elements
    const bool ascending = reloc || nins == 0;  // left-movers ascend, right-movers descend
    const uint32_t step = 32 * kWarpMoveUnroll;
    const uint32_t nsteps = dold > start ? (dold - start + step - 1) / step : 0;
    for (uint32_t si = 0; si < nsteps; ++si) {
      const uint32_t base = start + (ascending ? si : nsteps - 1 - si) * step;
      uint32_t a[kWarpMoveUnroll], p[kWarpMoveUnroll], el[kWarpMoveUnroll];
      bool mv[kWarpMoveUnroll];
#pragma unroll
      for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
        const uint32_t i = base + k * 32 + lane;
        mv[k] = false;
        el[k] = kNone;
        if (i < dold) {
          a[k] = src[i];
          if (esrc) el[k] = esrc[i];
        }
      }
      if (keys_in_lanes) {
        // old element i: inserts before it = insert keys with position <= i,
        // deletes before it = delete keys with position < i, deleted if a
        // delete key sits at i.  Keys before the window by ballot, the few
        // inside it one by one.
        const bool live = lane < segn;
        const uint32_t ins_before = __popc(__ballot_sync(kFull, live && !k_del && k_lb < base));
        const uint32_t del_before = __popc(__ballot_sync(kFull, live && k_del && k_lb < base));
        uint32_t win = __ballot_sync(kFull, live && k_lb >= base && k_lb < base + step);
        uint32_t I[kWarpMoveUnroll], D[kWarpMoveUnroll];
        bool dl[kWarpMoveUnroll];
#pragma unroll
        for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
          I[k] = ins_before;
          D[k] = del_before;
          dl[k] = false;
        }
        while (win) {
          const uint32_t kk = __ffs(win) - 1;
          win &= win - 1;
          const uint32_t lb = __shfl_sync(kFull, k_lb, kk);
          const bool del = __shfl_sync(kFull, k_del ? 1u : 0u, kk);
#pragma unroll
          for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
            const uint32_t i = base + k * 32 + lane;
            if (del) {
              D[k] += lb < i;
              dl[k] |= lb == i;
            } else {
              I[k] += lb <= i;
            }
          }
        }
#pragma unroll
        for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
          const uint32_t i = base + k * 32 + lane;
          if (i < dold) {
            p[k] = i - D[k] + I[k];
            mv[k] = !dl[k] && (reloc || p[k] != i);
          }
        }
      } else {
#pragma unroll
        for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
          const uint32_t i = base + k * 32 + lane;
          if (i < dold) {
            bool dl;
            merged_pos(seg, segn, ins_prefix, s, a[k], i, p[k], dl);
            mv[k] = !dl && (reloc || p[k] != i);
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (uint32_t k = 0; k < kWarpMoveUnroll; ++k) {
        if (mv[k]) {
          dst[p[k]] = a[k];
          if (edst) edst[p[k]] = el[k];
        }
      }
      __syncwarp();
    }
    // 3. inserts
    for (uint32_t k = lane; k < segn; k += 32) {
      uint32_t val = svals[s + k];
      if (val >> 31) continue;
      uint32_t p = ipos[s + k];
      dst[p] = uint32_t(seg[k]);
      if (edst) edst[p] = ups[val & 0x7fffffffu].elab;
    }
    __syncwarp();
    if (lane == 0) {
      g.deg[x] = dnew;
      if (reloc) {
        g.off[x] = noff;
        g.cap[x] = ncap;
      }
    }
    bytes += 4ull * (uint64_t(dold) + dnew);
    finish_vertex(g, x, dst, dnew, seg, segn, svals + s, qenc, nq, rows, colsize, memo, memo_mask, lane, agg);
  }
  if (lane == 0 && bytes) atomicAdd((unsigned long long*)&st->bytes_update, (unsigned long long)bytes);
  agg.flush(colsize, nq);
}

// k_merge_small's run copies: full blocks of kRunUnroll entries without
// predicates (kRunUnroll loads in flight, then the stores), the remainder in
// predicated blocks of 8; kLab: the graph has edge labels, moved alongside.
#ifndef BDSM_RUN_UNROLL
#define BDSM_RUN_UNROLL 16
#endif
constexpr uint32_t kRunUnroll = BDSM_RUN_UNROLL;
template <bool kLab>
__device__ __forceinline__ void run_up(const uint32_t* src, uint32_t* dst, const uint32_t* esrc, uint32_t* edst,
                                       uint32_t from, uint32_t to, uint32_t len) {
  constexpr uint32_t U = kLab ? 8 : kRunUnroll;
  uint32_t b = 0;
  for (; b + U <= len; b += U) {
    uint32_t v[U], l[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      v[k] = src[from + b + k];
      if (kLab) l[k] = esrc[from + b + k];
    }
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      dst[to + b + k] = v[k];
      if (kLab) edst[to + b + k] = l[k];
    }
  }
  for (; b < len; b += 8) {
    uint32_t v[8], l[8];
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
      v[k] = b + k < len ? src[from + b + k] : 0u;
      if (kLab) l[k] = b + k < len ? esrc[from + b + k] : 0u;
    }
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k)
      if (b + k < len) {
        dst[to + b + k] = v[k];
        if (kLab) edst[to + b + k] = l[k];
      }
  }
}
template <bool kLab>
__device__ __forceinline__ void run_down(const uint32_t* src, uint32_t* dst, const uint32_t* esrc, uint32_t* edst,
                                         uint32_t from, uint32_t to, uint32_t len) {
  constexpr uint32_t U = kLab ? 8 : kRunUnroll;
  uint32_t b = len;
  for (; b >= U; b -= U) {
    uint32_t v[U], l[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      v[k] = src[from + b - U + k];
      if (kLab) l[k] = esrc[from + b - U + k];
    }
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      dst[to + b - U + k] = v[k];
      if (kLab) edst[to + b - U + k] = l[k];
    }
  }
  while (b) {  // the remainder, highest block first (in place the entries move right)
    const uint32_t nb = b < 8 ? b : 8;
    b -= nb;
    uint32_t v[8], l[8];
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
      v[k] = k < nb ? src[from + b + k] : 0u;
      if (kLab) l[k] = k < nb ? esrc[from + b + k] : 0u;
    }
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k)
      if (k < nb) {
        dst[to + b + k] = v[k];
        if (kLab) edst[to + b + k] = l[k];
      }
  }
}

// Short lists (<= kSmallList entries before and after the batch; most touched
// lists at the C2-C4 shapes) are merged by ONE thread each, so a warp merges
// 32 of them at once instead of one.  The batch keys' positions in the old
// list are found first (independent searches); the old entries then move as
// runs between them, 8 loads in flight (ascending in place for delete-only
// lists, descending in place for insert-only ones, out of place for relocated
// ones), so no load waits on the previous comparison.  The finish is
// finish_vertex's done serially: the label index comes from the old one
// shifted by the batch keys below each class (no pass over the new list),
// then candidate rows, memo invalidations and hub bitmap bits.
__global__ void __launch_bounds__(256) k_merge_small(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
    const uint32_t* __restrict__ svals, const uint32_t* __restrict__ ins_prefix, uint32_t m,
    const bdsm_update_dev* __restrict__ ups, DevGraphMut g, const uint64_t* __restrict__ new_off,
    const uint32_t* __restrict__ new_cap, const DevQueryEnc* __restrict__ qenc, uint32_t nq,
    uint32_t* const* rows, uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
    uint32_t memo_mask, const uint32_t* __restrict__ small_list) {
  if (batch_aborted(st)) return;
  if (st->pool_top > g.pool_size) return;  // k_merge_refresh flags the overflow
  __shared__ int s_colagg[kColAggQ][kMaxQ];
  __shared__ uint32_t s_agg_done;
  ColAgg agg{s_colagg, &s_agg_done};
  agg.init();
  const uint32_t nt = st->n_touched, nsmall = st->n_small;
  uint64_t bytes = 0;
  for (uint32_t si = blockIdx.x * blockDim.x + threadIdx.x; si < nsmall; si += gridDim.x * blockDim.x) {
    const uint32_t t = small_list[si];
    const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
    const uint64_t* seg = skeys + s;
    const uint32_t segn = e - s;
    const uint32_t x = uint32_t(seg[0] >> 32);
    const uint32_t dold = g.deg[x];
    const uint64_t ooff = g.off[x];
    const uint32_t nins = ins_prefix[e] - ins_prefix[s];
    const uint32_t dnew = dold + nins - (segn - nins);
    const uint32_t ncap = new_cap[t] & kCapMask;
    const bool reloc = ncap != 0;
    const uint64_t noff = reloc ? new_off[t] : ooff;
    const uint32_t* src = g.adj + ooff;
    uint32_t* dst = g.adj + noff;
    const uint32_t* esrc = g.elab ? g.elab + ooff : nullptr;
    uint32_t* edst = g.elab ? g.elab + noff : nullptr;
    auto ins_label = [&](uint32_t k) { return ups[svals[s + k] & 0x7fffffffu].elab; };
    // where each batch key falls in the old list (independent searches)
    uint32_t ypos[kSmallKeys];
    for (uint32_t k = 0; k < segn; ++k) ypos[k] = lower_bound_u32(src, dold, uint32_t(seg[k]));
    // copy a run of old entries, 8 loads in flight; in place the runs move
    // left in ascending order or right in descending order, and a block is
    // read completely before it is written, so overlapping runs are safe
    auto copy_up = [&](uint32_t from, uint32_t to, uint32_t len) {
      if (esrc) run_up<true>(src, dst, esrc, edst, from, to, len);
      else run_up<false>(src, dst, nullptr, nullptr, from, to, len);
    };
    auto copy_down = [&](uint32_t from, uint32_t to, uint32_t len) {
      if (esrc) run_down<true>(src, dst, esrc, edst, from, to, len);
      else run_down<false>(src, dst, nullptr, nullptr, from, to, len);
    };
    if (reloc || nins == 0) {  // ascending: out of place, or delete-only in place (moves left)
      // in place the entries below the first batch key do not move
      uint32_t r = reloc || segn == 0 ? 0 : ypos[0], w = r;
      for (uint32_t k = 0; k < segn; ++k) {
        const uint32_t pk = ypos[k];
        copy_up(r, w, pk - r);
        w += pk - r;
        r = pk;
        if (svals[s + k] >> 31) {
          ++r;  // the deleted entry
        } else {
          dst[w] = uint32_t(seg[k]);
          if (edst) edst[w] = ins_label(k);
          ++w;
        }
      }
      if (r < dold) copy_up(r, w, dold - r);
    } else {  // insert-only in place: descending (moves right)
      uint32_t r = dold, w = dnew;
      for (int k = int(segn) - 1; k >= 0; --k) {
        const uint32_t pk = ypos[k];
        copy_down(pk, w - (r - pk), r - pk);
        w -= r - pk;
        r = pk;
        --w;
        dst[w] = uint32_t(seg[k]);
        if (edst) edst[w] = ins_label(uint32_t(k));
      }
    }
    g.deg[x] = dnew;
    if (reloc) {
      g.off[x] = noff;
      g.cap[x] = ncap;
    }
    bytes += 4ull * (uint64_t(dold) + dnew);
    // --- finish (finish_vertex, serially) ---
    if (g.hub_slot) {
      const uint32_t hs = g.hub_slot[x];
      if (hs != kNone) {
        uint32_t* bm = g.bitmaps + uint64_t(hs) * g.bm_words;
        for (uint32_t k = 0; k < segn; ++k) {
          const uint32_t y = uint32_t(seg[k]);
          if (svals[s + k] >> 31) atomicAnd(bm + (y >> 5), ~(1u << (y & 31)));
          else atomicOr(bm + (y >> 5), 1u << (y & 31));
        }
      }
    }
    for (uint32_t q = 0; q < nq; ++q)
      for (uint32_t k = 0; k < qenc[q].nsig; ++k) memo_invalidate_v(g.memo_bits, memo, memo_mask, x, q, qenc[q].sig[k]);
    // label index of the new list from the old one: class k's first
    // position moves by the inserts minus the deletes below class_lo[k]
    // (a two-pointer walk over the sorted keys, the row rewritten in place;
    // no per-thread array, which lived in local memory)
    const bool indexed = g.loff != nullptr;
    uint32_t* lrow = indexed ? g.loff + uint64_t(x) * (g.nlab + 1) : nullptr;
    if (indexed) {
      int acc = 0;
      uint32_t j = 0;
      for (uint32_t k = 0; k < g.nlab; ++k) {
        const uint32_t lo = g.class_lo[k];
        for (; j < segn && uint32_t(seg[j]) < lo; ++j) acc += (svals[s + j] >> 31) ? -1 : 1;
        lrow[k] = uint32_t(int(lrow[k]) + acc);
      }
      lrow[g.nlab] = dnew;
    }
    const uint32_t vl = g.vlabel[x];
    for (uint32_t q = 0; q < nq; ++q) {
      const DevQueryEnc& qe = qenc[q];
      uint32_t cnt[kMaxQ];
      for (uint32_t gi = 0; gi < qe.G; ++gi) {
        uint32_t c = 0;
        if (indexed) {
          const uint32_t cls = qe.gcls[gi];
          c = cls == kNone ? 0u : lrow[cls + 1] - lrow[cls];
        } else {
          for (uint32_t i = 0; i < dnew; ++i) c += dst[i] >= qe.glo[gi] && dst[i] < qe.ghi[gi];
        }
        cnt[gi] = c > qe.cap ? qe.cap : c;
      }
      uint32_t row = 0;
      for (uint32_t u = 0; u < qe.n; ++u) {
        if (vl != qe.qlabel[u]) continue;
        bool ok = true;
        for (uint32_t gi = 0; gi < qe.G && ok; ++gi) ok = cnt[gi] >= qe.qcnt[u][gi];
        if (ok) row |= 1u << u;
      }
      const uint32_t word = rows[q][x];
      const uint32_t before = word & ~kRowFlags;
      if (before != row) {
        rows[q][x] = row | (word & kRowFlags);
        const uint32_t diff = before ^ row;
        uint32_t d = diff;
        while (d) {
          const uint32_t u = __ffs(d) - 1;
          d &= d - 1;
          agg.add(colsize, q, u, (row >> u) & 1u);
        }
        for (uint32_t k = 0; k < qe.nsig; ++k) {  // neighbours' weights that count a flipped bit
          const uint32_t sg = qe.sig[k];
          if ((diff >> (sg & 15)) & 1u)
            for (uint32_t i = 0; i < dnew; ++i) memo_invalidate_v(g.memo_bits, memo, memo_mask, dst[i], q, sg);
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(kFull, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd((unsigned long long*)&st->bytes_update, (unsigned long long)bytes);
  agg.flush(colsize, nq);
}

// Lower bound of x in the sorted a[0, n) by a group of GS lanes (sub = lane
// index within the group): each round the GS lanes test the last element of
// GS equal blocks, so a list of <= GS^3 entries takes three dependent loads.
template <uint32_t GS>
__device__ __forceinline__ uint32_t group_lower_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t x,
                                                      uint32_t sub, uint32_t gbase, uint32_t gmask) {
  uint32_t lo = 0, len = n;
  while (len > GS) {
    const uint32_t stride = (len + GS - 1) / GS;
    const uint32_t last = lo + (sub + 1) * stride - 1;
    const bool lt = last < lo + len && a[last] < x;
    const uint32_t c = __popc((__ballot_sync(gmask, lt) >> gbase) & ((GS == 32 ? 0u : 1u << GS) - 1u));
    const uint32_t nlo = lo + c * stride;
    len = min(stride, lo + len - nlo);
    lo = nlo;
  }
  const bool lt = sub < len && a[lo + sub] < x;
  return lo + __popc((__ballot_sync(gmask, lt) >> gbase) & ((GS == 32 ? 0u : 1u << GS) - 1u));
}

constexpr uint32_t kGroupMoveUnroll = 4;  // k_merge_group: old elements per lane in flight per step

// Short lists (<= kSmallList entries before and after the batch; most touched
// lists of the 1M-update batches) merged by a group of GS lanes each, so a warp
// merges 32 / GS lists at once and every load and store of the moves is a
// GS x 4-byte run (one 32-byte sector at GS = 8) instead of a 4-byte access per
// lane to 32 different lists (k_merge_small: eight L2 sectors written per
// sector of list data).  The steps are k_merge_refresh's (insert slots against
// the intact old list, by GS-ary group searches; in place, left-movers ascend
// and right-movers descend in steps that are read completely before they are
// written), and the finish is finish_vertex's spread over the group: memo
// invalidations and hub bits by key, the label index by class (staged in shared
// memory), candidate rows by query.
template <uint32_t GS>
__global__ void __launch_bounds__(256) k_merge_group(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
    const uint32_t* __restrict__ svals, const uint32_t* __restrict__ ins_prefix, uint32_t m,
    const bdsm_update_dev* __restrict__ ups, DevGraphMut g, const uint64_t* __restrict__ new_off,
    const uint32_t* __restrict__ new_cap, uint32_t* ipos, const DevQueryEnc* __restrict__ qenc, uint32_t nq,
    uint32_t* const* rows, uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
    uint32_t memo_mask, const uint32_t* __restrict__ small_list) {
  if (batch_aborted(st)) return;
  if (st->pool_top > g.pool_size) return;  // k_merge_refresh flags the overflow
  __shared__ int s_colagg[kColAggQ][kMaxQ];
  __shared__ uint32_t s_agg_done;
  __shared__ uint32_t s_lpos[256 / GS][kMaxLabelIndex + 1];
  ColAgg agg{s_colagg, &s_agg_done};
  agg.init();
  const uint32_t lane = threadIdx.x & 31, sub = lane % GS, gbase = lane - sub;
  const uint32_t gmask = GS == 32 ? kFull : ((1u << GS) - 1u) << gbase;
  uint32_t* lpos = s_lpos[threadIdx.x / GS];
  const uint32_t ngroups = gridDim.x * (blockDim.x / GS);
  const uint32_t nt = st->n_touched, nsmall = st->n_small;
  uint64_t bytes = 0;
  for (uint32_t si = (blockIdx.x * blockDim.x + threadIdx.x) / GS; si < nsmall; si += ngroups) {
    const uint32_t t = small_list[si];
    const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
    const uint64_t* seg = skeys + s;
    const uint32_t segn = e - s;
    const uint32_t x = uint32_t(seg[0] >> 32);
    const uint32_t dold = g.deg[x];
    const uint64_t ooff = g.off[x];
    const uint32_t nins = ins_prefix[e] - ins_prefix[s];
    const uint32_t dnew = dold + nins - (segn - nins);
    const uint32_t ncap = new_cap[t] & kCapMask;
    const bool reloc = ncap != 0;
    const uint64_t noff = reloc ? new_off[t] : ooff;
    const uint32_t* src = g.adj + ooff;
    uint32_t* dst = g.adj + noff;
    const uint32_t* esrc = g.elab ? g.elab + ooff : nullptr;
    uint32_t* edst = g.elab ? g.elab + noff : nullptr;

    // 1. insert slots against the intact old list, and the first position that
    // can move in place (entries below the first batch key never move)
    uint32_t start = 0;
    if (segn <= GS) {
      for (uint32_t k = 0; k < segn; ++k) {
        const bool del = svals[s + k] >> 31;
        if (del && (k || reloc)) continue;
        const uint32_t lb = group_lower_bound<GS>(src, dold, uint32_t(seg[k]), sub, gbase, gmask);
        if (k == 0 && !reloc) start = lb;
        if (!del && sub == 0) {
          const uint32_t ib = ins_prefix[s + k] - ins_prefix[s];
          ipos[s + k] = ib + (lb - (k - ib));
        }
      }
    } else {
      if (sub == GS - 1 && !reloc && dold) start = lower_bound_u32(src, dold, uint32_t(seg[0]));
      for (uint32_t k = sub; k < segn; k += GS) {
        if (svals[s + k] >> 31) continue;
        const uint32_t ib = ins_prefix[s + k] - ins_prefix[s];
        ipos[s + k] = ib + (lower_bound_u32(src, dold, uint32_t(seg[k])) - (k - ib));
      }
      start = __shfl_sync(gmask, start, gbase + GS - 1);
    }
    __syncwarp(gmask);
    // 2. move the old elements
    const bool ascending = reloc || nins == 0;
    const uint32_t step = GS * kGroupMoveUnroll;
    const uint32_t nsteps = dold > start ? (dold - start + step - 1) / step : 0;
    for (uint32_t sj = 0; sj < nsteps; ++sj) {
      const uint32_t base = start + (ascending ? sj : nsteps - 1 - sj) * step;
      uint32_t a[kGroupMoveUnroll], p[kGroupMoveUnroll], el[kGroupMoveUnroll];
      bool mv[kGroupMoveUnroll];
#pragma unroll
      for (uint32_t k = 0; k < kGroupMoveUnroll; ++k) {
        const uint32_t i = base + k * GS + sub;
        mv[k] = false;
        el[k] = kNone;
        a[k] = 0;
        if (i < dold) {
          a[k] = src[i];
          if (esrc) el[k] = esrc[i];
        }
      }
#pragma unroll
      for (uint32_t k = 0; k < kGroupMoveUnroll; ++k) {
        const uint32_t i = base + k * GS + sub;
        p[k] = 0;
        if (i < dold) {
          bool dl;
          merged_pos(seg, segn, ins_prefix, s, a[k], i, p[k], dl);
          mv[k] = !dl && (reloc || p[k] != i);
        }
      }
      __syncwarp(gmask);
#pragma unroll
      for (uint32_t k = 0; k < kGroupMoveUnroll; ++k)
        if (mv[k]) {
          dst[p[k]] = a[k];
          if (edst) edst[p[k]] = el[k];
        }
      __syncwarp(gmask);
    }
    // 3. inserts
    for (uint32_t k = sub; k < segn; k += GS) {
      const uint32_t val = svals[s + k];
      if (val >> 31) continue;
      const uint32_t pp = ipos[s + k];
      dst[pp] = uint32_t(seg[k]);
      if (edst) edst[pp] = ups[val & 0x7fffffffu].elab;
    }
    __syncwarp(gmask);
    if (sub == 0) {
      g.deg[x] = dnew;
      if (reloc) {
        g.off[x] = noff;
        g.cap[x] = ncap;
      }
      bytes += 4ull * (uint64_t(dold) + dnew);
    }
    // 4. finish (finish_vertex over the group)
    for (uint32_t q = 0; q < nq; ++q)
      for (uint32_t k = sub; k < qenc[q].nsig; k += GS)
        memo_invalidate_v(g.memo_bits, memo, memo_mask, x, q, qenc[q].sig[k]);
    if (g.hub_slot) {
      const uint32_t hs = g.hub_slot[x];
      if (hs != kNone) {
        uint32_t* bm = g.bitmaps + uint64_t(hs) * g.bm_words;
        for (uint32_t k = sub; k < segn; k += GS) {
          const uint32_t y = uint32_t(seg[k]);
          if (svals[s + k] >> 31) atomicAnd(bm + (y >> 5), ~(1u << (y & 31)));
          else atomicOr(bm + (y >> 5), 1u << (y & 31));
        }
      }
    }
    // label index: class k's first position moves by the inserts minus the
    // deletes below class_lo[k] (the segment is sorted)
    const bool indexed = g.loff != nullptr;
    if (indexed) {
      uint32_t* lrow = g.loff + uint64_t(x) * (g.nlab + 1);
      for (uint32_t k = sub; k <= g.nlab; k += GS) {
        uint32_t v = dnew;
        if (k < g.nlab) {
          const uint32_t lo = g.class_lo[k];
          int acc = 0;
          for (uint32_t j = 0; j < segn && uint32_t(seg[j]) < lo; ++j) acc += (svals[s + j] >> 31) ? -1 : 1;
          v = uint32_t(int(lrow[k]) + acc);
        }
        lrow[k] = v;
        lpos[k] = v;
      }
      __syncwarp(gmask);
    }
    // candidate rows, one query per lane
    const uint32_t vl = g.vlabel[x];
    for (uint32_t q = sub; q < nq; q += GS) {
      const DevQueryEnc& qe = qenc[q];
      uint32_t row = 0;
      bool any = false;
      for (uint32_t u = 0; u < qe.n; ++u) any |= vl == qe.qlabel[u];
      if (any) {
        uint32_t cnt[kMaxQ];
        for (uint32_t gi = 0; gi < qe.G; ++gi) {
          uint32_t c = 0;
          if (indexed) {
            const uint32_t cls = qe.gcls[gi];
            c = cls == kNone ? 0u : lpos[cls + 1] - lpos[cls];
          } else {
            for (uint32_t i = 0; i < dnew; ++i) c += dst[i] >= qe.glo[gi] && dst[i] < qe.ghi[gi];
          }
          cnt[gi] = c > qe.cap ? qe.cap : c;
        }
        for (uint32_t u = 0; u < qe.n; ++u) {
          if (vl != qe.qlabel[u]) continue;
          bool ok = true;
          for (uint32_t gi = 0; gi < qe.G && ok; ++gi) ok = cnt[gi] >= qe.qcnt[u][gi];
          if (ok) row |= 1u << u;
        }
      }
      const uint32_t word = rows[q][x];
      const uint32_t before = word & ~kRowFlags;
      if (before != row) {
        rows[q][x] = row | (word & kRowFlags);
        const uint32_t diff = before ^ row;
        uint32_t d = diff;
        while (d) {
          const uint32_t u = __ffs(d) - 1;
          d &= d - 1;
          agg.add(colsize, q, u, (row >> u) & 1u);
        }
        for (uint32_t k = 0; k < qe.nsig; ++k) {  // neighbours' weights that count a flipped bit
          const uint32_t sg = qe.sig[k];
          if ((diff >> (sg & 15)) & 1u)
            for (uint32_t i = 0; i < dnew; ++i) memo_invalidate_v(g.memo_bits, memo, memo_mask, dst[i], q, sg);
        }
      }
    }
    __syncwarp(gmask);  // lpos is reused by the group's next list
  }
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(kFull, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd((unsigned long long*)&st->bytes_update, (unsigned long long)bytes);
  agg.flush(colsize, nq);
}

// The same merge for lists of >= kBigList entries, one CTA per list: each
// sweep step moves 256 threads x kMoveUnroll elements (read completely, then
// written, with a CTA barrier between), so an 18K-neighbour hub moves in a
// handful of steps instead of ~75 warp steps; warp 0 then finishes the vertex.
__global__ void __launch_bounds__(256) k_merge_big(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
    const uint32_t* __restrict__ svals, const uint32_t* __restrict__ ins_prefix, uint32_t m,
    const bdsm_update_dev* __restrict__ ups, DevGraphMut g, const uint64_t* __restrict__ new_off,
    const uint32_t* __restrict__ new_cap, uint32_t* ipos, const DevQueryEnc* __restrict__ qenc,
    uint32_t nq, uint32_t* const* rows, uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
    uint32_t memo_mask, const uint32_t* __restrict__ big_list) {
  if (batch_aborted(st)) return;
  if (st->pool_top > g.pool_size) return;  // k_merge_refresh flags the overflow
  __shared__ uint32_t s_start;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t nt = st->n_touched;
  uint64_t bytes = 0;
  const uint32_t nbig = st->n_big;
  for (uint32_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
    const uint32_t t = big_list[bi];  // long lists, listed by k_alloc
    const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
    const uint64_t* seg = skeys + s;
    const uint32_t segn = e - s;
    const uint32_t x = uint32_t(seg[0] >> 32);
    const uint32_t ncap = new_cap[t] & kCapMask;
    const uint32_t dold = g.deg[x];
    const uint64_t ooff = g.off[x];
    const uint32_t nins = ins_prefix[e] - ins_prefix[s];
    const uint32_t dnew = dold + nins - (segn - nins);
    const bool reloc = ncap != 0;
    const uint64_t noff = reloc ? new_off[t] : ooff;
    uint32_t* src = g.adj + ooff;
    uint32_t* dst = g.adj + noff;
    uint32_t* esrc = g.elab ? g.elab + ooff : nullptr;
    uint32_t* edst = g.elab ? g.elab + noff : nullptr;
    // insert slots against the intact old list; key 0's search also gives
    // the first position that can move (entries below it never move)
    // (a few keys: one warp-cooperative search per key, spread over the
    // warps, three dependent loads each below 32K entries instead of 15)
    if (tid == 0 && reloc) s_start = 0u;
    const uint32_t nw = blockDim.x >> 5;
    const bool warp_search = segn <= 2 * nw;
    for (uint32_t k = warp_search ? tid >> 5 : tid; k < segn; k += warp_search ? nw : blockDim.x) {
      const bool del = svals[s + k] >> 31;
      if (del && (k || reloc)) continue;
      const uint32_t lb = warp_search ? warp_lower_bound(src, dold, uint32_t(seg[k]), lane)
                                      : lower_bound_u32(src, dold, uint32_t(seg[k]));
      if (warp_search && lane) continue;
      if (k == 0 && !reloc) s_start = lb;
      if (!del) {
        const uint32_t ib = ins_prefix[s + k] - ins_prefix[s];
        ipos[s + k] = ib + (lb - (k - ib));
      }
    }
    __syncthreads();
    const uint32_t start = s_start;
    const bool ascending = reloc || nins == 0;
    const uint32_t step = blockDim.x * kMoveUnroll;
    const uint32_t nsteps = dold > start ? (dold - start + step - 1) / step : 0;
    for (uint32_t si = 0; si < nsteps; ++si) {
      const uint32_t base = start + (ascending ? si : nsteps - 1 - si) * step;
      uint32_t a[kMoveUnroll], p[kMoveUnroll], el[kMoveUnroll];
      bool mv[kMoveUnroll];
#pragma unroll
      for (uint32_t k = 0; k < kMoveUnroll; ++k) {
        const uint32_t i = base + k * blockDim.x + tid;
        mv[k] = false;
        el[k] = kNone;
        if (i < dold) {
          a[k] = src[i];
          if (esrc) el[k] = esrc[i];
        }
      }
#pragma unroll
      for (uint32_t k = 0; k < kMoveUnroll; ++k) {
        const uint32_t i = base + k * blockDim.x + tid;
        if (i < dold) {
          bool dl;
          merged_pos(seg, segn, ins_prefix, s, a[k], i, p[k], dl);
          mv[k] = !dl && (reloc || p[k] != i);
        }
      }
      // in place, a step's writes may land on entries the step read; they
      // never reach the next step's reads (left moves ascend, right moves
      // descend), so one barrier per step suffices, none when relocating
      if (!reloc) __syncthreads();
#pragma unroll
      for (uint32_t k = 0; k < kMoveUnroll; ++k) {
        if (mv[k]) {
          dst[p[k]] = a[k];
          if (edst) edst[p[k]] = el[k];
        }
      }
    }
    for (uint32_t k = tid; k < segn; k += blockDim.x) {
      const uint32_t val = svals[s + k];
      if (val >> 31) continue;
      const uint32_t pp = ipos[s + k];
      dst[pp] = uint32_t(seg[k]);
      if (edst) edst[pp] = ups[val & 0x7fffffffu].elab;
    }
    if (tid == 0) {
      g.deg[x] = dnew;
      if (reloc) {
        g.off[x] = noff;
        g.cap[x] = ncap;
      }
      bytes += 4ull * (uint64_t(dold) + dnew);
    }
    __syncthreads();  // s_start and this list's reads are done before the next list
  }
  if (tid == 0 && bytes) atomicAdd((unsigned long long*)&st->bytes_update, (unsigned long long)bytes);
}

// finish_vertex of the long lists k_merge_big moved, a warp per list, so a
// CTA's other warps do not wait on one warp's serial finish between lists.
__global__ void __launch_bounds__(256) k_finish_big(
    const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
    const uint32_t* __restrict__ svals, uint32_t m, DevGraphMut g, const DevQueryEnc* __restrict__ qenc,
    uint32_t nq, uint32_t* const* rows, uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
    uint32_t memo_mask, const uint32_t* __restrict__ big_list) {
  if (batch_aborted(st)) return;
  if (st->pool_top > g.pool_size) return;
  __shared__ int s_colagg[kColAggQ][kMaxQ];
  __shared__ uint32_t s_agg_done;
  ColAgg agg{s_colagg, &s_agg_done};
  agg.init();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nt = st->n_touched, nbig = st->n_big;
  for (uint32_t bi = warp; bi < nbig; bi += nwarps) {
    const uint32_t t = big_list[bi];
    const uint32_t s = heads[t], e = seg_end(heads, t, nt, m);
    const uint64_t* seg = skeys + s;
    const uint32_t x = uint32_t(seg[0] >> 32);
    finish_vertex(g, x, g.adj + g.off[x], g.deg[x], seg, e - s, svals + s, qenc, nq, rows, colsize, memo,
                  memo_mask, lane, agg);
  }
  agg.flush(colsize, nq);
}

// Full encode (QueryEncodingState::initialize, src/matcher.cpp:10-18):
// warp per vertex computes the candidate row of one query.
__global__ void __launch_bounds__(256) k_encode_all(DevGraph g, const DevQueryEnc* __restrict__ qenc,
                                                    uint32_t* rows) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const DevQueryEnc& qe = *qenc;
  for (uint64_t v = warp; v < g.V; v += nwarps) {
    uint32_t vl = g.vlabel[v];
    bool any = false;
    for (uint32_t u = 0; u < qe.n; ++u) any |= vl == qe.qlabel[u];
    if (!any) {  // label absent from the query: empty row without a scan
      if (lane == 0) rows[v] = 0;
      continue;
    }
    const uint32_t cnt = group_counts(g.adj + g.off[v], g.deg[v], qe, lane);
    const uint32_t row = row_of(qe, vl, cnt, lane);
    if (lane == 0) rows[v] = row;
  }
}

// ---- K8: hot-list estimator, packing into an L2-persisting arena ----------
// (north_star item 4; no reference counterpart).  Random walks
// from the batch's touched vertices estimate which adjacency lists the next
// batches' DFS will read; the hottest lists (by visits, within a byte budget)
// are copied contiguously into an arena of the pool that an access-policy
// window marks persisting in L2.  Performance only: list contents never change.

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_hot_walks(const uint32_t* __restrict__ heads, const uint64_t* __restrict__ skeys,
                            const BatchState* st, DevGraph g, uint32_t* heat, uint32_t walks, uint32_t depth,
                            uint32_t seed) {
  if (batch_aborted_own(st)) return;
  const uint64_t total = uint64_t(st->n_touched) * walks;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t v = uint32_t(skeys[heads[i / walks]] >> 32);
    uint32_t h = mix32(seed ^ uint32_t(i * 0x9e3779b9u));
    atomicAdd(heat + v, 1u);
    for (uint32_t s = 0; s < depth; ++s) {
      const uint32_t d = g.deg[v];
      if (!d) break;
      h = mix32(h + s);
      v = g.adj[g.off[v] + h % d];
      atomicAdd(heat + v, 1u);
    }
  }
}

// Bytes of lists per heat bucket (bucket = bit length of the heat).
__global__ void k_hot_hist(DevGraph g, const uint32_t* __restrict__ heat, unsigned long long* hist) {
  __shared__ unsigned long long sh[33];
  if (threadIdx.x < 33) sh[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.V; v += gridDim.x * blockDim.x) {
    const uint32_t h = heat[v];
    if (h) atomicAdd(&sh[32 - __clz(h)], 4ull * g.deg[v]);
  }
  __syncthreads();
  if (threadIdx.x < 33 && sh[threadIdx.x]) atomicAdd(hist + threadIdx.x, sh[threadIdx.x]);
}

// Threshold bucket: the hottest buckets whose lists fit the budget.
__global__ void k_hot_select(unsigned long long* hist, unsigned long long budget) {
  if (threadIdx.x != 0) return;
  unsigned long long acc = 0;
  uint32_t tb = 33;
  for (int b = 32; b >= 1; --b) {
    if (acc + hist[b] > budget) break;
    acc += hist[b];
    tb = uint32_t(b);
  }
  hist[33] = tb;  // read by k_hot_pack
}

// Warp per hot vertex: copy the list (and labels) to the arena slot reserved
// from the pool bump pointer, repoint off/cap; decay every vertex's heat.
__global__ void k_hot_pack(DevGraphMut g, uint32_t* heat, const unsigned long long* hist, BatchState* st) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t tb = uint32_t(hist[33]);
  for (uint64_t v = warp; v < g.V; v += nwarps) {
    const uint32_t h = heat[v];
    const uint32_t d = g.deg[v];
    const bool hot = h && (32 - __clz(h)) >= tb && d >= 32;
    __syncwarp();
    if (lane == 0) heat[v] = h >> 1;
    if (!hot) continue;
    const uint32_t c = (d + 3) & ~3u;  // no slack: the next insert relocates it out of the arena
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd((unsigned long long*)&st->pool_top, (unsigned long long)c);
    slot = __shfl_sync(kFull, slot, 0);
    if (slot + c > g.pool_size) continue;  // pool exhausted: leave it in place
    const uint64_t o = g.off[v];
    for (uint32_t i = lane; i < d; i += 32) g.adj[slot + i] = g.adj[o + i];
    if (g.elab)
      for (uint32_t i = lane; i < d; i += 32) g.elab[slot + i] = g.elab[o + i];
    __syncwarp();
    if (lane == 0) {
      g.off[v] = slot;
      g.cap[v] = c;
    }
  }
}

// Label index of every vertex (DevGraph::loff): warp per vertex, lane k
// finds label class k's first position by binary search.
__global__ void __launch_bounds__(256) k_label_index(DevGraphMut g) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t v = warp; v < g.V; v += nwarps) {
    const uint32_t d = g.deg[v];
    const uint32_t* lst = g.adj + g.off[v];
    for (uint32_t k = lane; k <= g.nlab; k += 32)
      g.loff[v * (g.nlab + 1) + k] = k < g.nlab ? lower_bound_u32(lst, d, g.class_lo[k]) : d;
  }
}

__global__ void k_column_sizes(const uint32_t* __restrict__ rows, uint32_t V, uint32_t n, uint64_t* out) {
  __shared__ unsigned long long acc[32];
  if (threadIdx.x < 32) acc[threadIdx.x] = 0;
  __syncthreads();
  uint32_t local[kMaxQ] = {0};
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    uint32_t r = rows[v];
    for (uint32_t u = 0; u < n && u < kMaxQ; ++u) local[u] += (r >> u) & 1u;
  }
  for (uint32_t u = 0; u < n && u < kMaxQ; ++u) {
    uint32_t c = local[u];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&acc[u], (unsigned long long)c);
  }
  __syncthreads();
  if (threadIdx.x < n && threadIdx.x < kMaxQ && acc[threadIdx.x])
    atomicAdd((unsigned long long*)out + threadIdx.x, acc[threadIdx.x]);
}

}  // namespace

// ------------------------------------------------------------ launchers ----

void launch_build_keys(const uint32_t* src, const uint32_t* dst, uint64_t E, uint32_t V,
                       uint64_t* keys, uint64_t* vals, uint32_t* bad, cudaStream_t s) {
  k_build_keys<<<blocks_for(E), kThreads, 0, s>>>(src, dst, E, V, keys, vals, bad);
}
void launch_check_sorted_dups(const uint64_t* keys, uint64_t n, uint32_t* bad, cudaStream_t s) {
  k_check_dups<<<blocks_for(n), kThreads, 0, s>>>(keys, n, bad);
}
void launch_degrees(const uint64_t* keys, uint64_t n, uint32_t* deg, cudaStream_t s) {
  k_degrees<<<blocks_for(n), kThreads, 0, s>>>(keys, n, deg);
}
void launch_caps(const uint32_t* deg, uint32_t V, float slack, uint32_t* cap, uint64_t* cap64,
                 cudaStream_t s) {
  k_caps<<<blocks_for(V), kThreads, 0, s>>>(deg, V, slack, cap, cap64);
}
void launch_scatter(const uint64_t* keys, const uint64_t* vals, uint64_t n, const uint64_t* dense_off,
                    const uint64_t* off, uint32_t* adj, const uint32_t* edge_labels, uint32_t* elab,
                    cudaStream_t s) {
  k_scatter<<<blocks_for(n), kThreads, 0, s>>>(keys, vals, n, dense_off, off, adj, edge_labels, elab);
}
void launch_compact(DevGraphMut g_old, const uint64_t* new_off, const uint32_t* new_cap,
                    uint32_t* new_adj, uint32_t* new_elab, cudaStream_t s) {
  (void)new_cap;
  k_compact<<<blocks_for(uint64_t(g_old.V) * 32), kThreads, 0, s>>>(g_old, new_off, new_cap, new_adj,
                                                                    new_elab);
}
void launch_prepare(const bdsm_update_dev* ups, uint32_t n, DevGraph g, const uint32_t* new_of,
                    bdsm_update_dev* iups, BatchState* st, uint64_t* keys, uint32_t* vals, uint32_t* dlab,
                    uint8_t* ecode, uint32_t id_limit, uint32_t key_bits, cudaStream_t s) {
  k_prepare<<<blocks_for(n), kThreads, 0, s>>>(ups, n, g, new_of, iups, st, keys, vals, dlab, ecode, id_limit,
                                               key_bits);
}
void launch_translate(const bdsm_update_dev* ups, uint32_t n, uint32_t V, bool has_elab, const uint32_t* new_of,
                      bdsm_update_dev* iups, BatchState* st, uint64_t* keys, uint32_t* vals, uint8_t* ecode,
                      uint32_t id_limit, uint32_t key_bits, cudaStream_t s) {
  k_translate<<<blocks_for(n), kThreads, 0, s>>>(ups, n, V, has_elab, new_of, iups, st, keys, vals, ecode, id_limit,
                                                 key_bits);
}
void launch_validate(const bdsm_update_dev* iups, uint32_t n, DevGraph g, BatchState* st, uint32_t* dlab,
                     uint8_t* ecode, uint32_t* const* rows, uint32_t nq, uint32_t slot, cudaStream_t s) {
  k_validate<<<blocks_for(n), kThreads, 0, s>>>(iups, n, g, st, dlab, ecode, rows, nq, row_ins_flag(slot),
                                                row_del_flag(slot));
}
void launch_post_sort(const uint64_t* in_keys, const uint32_t* in_vals, uint32_t key_bits, uint64_t* out_keys,
                      uint32_t* out_vals, uint32_t m, BatchState* st, uint8_t* head, uint32_t* insflag,
                      uint32_t* const* rows, uint32_t nq, uint32_t V, unsigned long long* hkeys, uint32_t* hvals,
                      uint32_t hmask, uint32_t slot, cudaStream_t s) {
  k_post_sort<<<blocks_for(uint64_t(m) + 1), kThreads, 0, s>>>(in_keys, in_vals, key_bits, out_keys, out_vals, m,
                                                              st, head, insflag, rows, nq, V, hkeys, hvals, hmask,
                                                              row_ins_flag(slot), row_del_flag(slot));
}
void launch_clear_flags(const uint64_t* skeys, uint32_t m, uint32_t* const* rows, uint32_t nq, uint32_t V,
                        uint32_t slot, cudaStream_t s, BatchState* next) {
  k_clear_flags<<<blocks_for(m), kThreads, 0, s>>>(skeys, m, rows, nq, V, row_ins_flag(slot) | row_del_flag(slot),
                                                   next);
}
void launch_alloc(const uint32_t* heads, const uint64_t* skeys, const uint32_t* ins_prefix,
                  uint32_t m, DevGraph g, float slack, BatchState* st, uint64_t* new_off,
                  uint32_t* new_cap, uint32_t* big_list, uint32_t* small_list, uint32_t* mid_list,
                  uint32_t small_max, uint32_t big_min, cudaStream_t s) {
  // small_max: longest list (before and after) of the short-list kernel, 0 =
  // none; k_merge_small's position array bounds it at kSmallList
  k_alloc<<<blocks_for(m), kThreads, 0, s>>>(heads, skeys, ins_prefix, m, g, slack, st, new_off, new_cap,
                                             big_list, small_list, mid_list, small_max, big_min ? big_min : kBigList);
}
void launch_merge_refresh(const uint32_t* heads, const uint64_t* skeys, const uint32_t* svals,
                          const uint32_t* ins_prefix, uint32_t m, const bdsm_update_dev* ups,
                          DevGraphMut g, const uint64_t* new_off, const uint32_t* new_cap,
                          uint32_t* ipos, const DevQueryEnc* qenc, uint32_t nq, uint32_t* const* rows,
                          uint64_t* const* colsize, BatchState* st, unsigned long long* memo,
                          uint32_t memo_mask, const uint32_t* big_list, const uint32_t* small_list,
                          const uint32_t* mid_list, uint32_t small_mode, int num_sms, cudaStream_t s,
                          cudaStream_t s_big) {
  // one warp per touched vertex (<= m), persistent over a bounded grid
  uint64_t warps = m ? m : 1;
  uint64_t blocks = (warps * 32 + 255) / 256;
  const uint64_t cap = resident_ctas(k_merge_refresh, 256, num_sms);
  if (blocks > cap) blocks = cap;
  k_merge_refresh<<<unsigned(blocks), 256, 0, s>>>(heads, skeys, svals, ins_prefix, m, ups, g, new_off,
                                                  new_cap, ipos, qenc, nq, rows, colsize, st, memo, memo_mask,
                                                  mid_list);
  // short lists: small_mode 1 = a thread per list (k_merge_small), 8 / 16 = a
  // group of that many lanes per list (k_merge_group), 0 = none (k_alloc did
  // not split them off)
  if (small_mode == 1)
    k_merge_small<<<unsigned(std::min<uint64_t>((uint64_t(m ? m : 1) + 255) / 256,
                                                resident_ctas(k_merge_small, 256, num_sms))), 256,
                    0, s>>>(heads, skeys, svals, ins_prefix, m, ups, g, new_off, new_cap, qenc, nq, rows, colsize,
                            st, memo, memo_mask, small_list);
  else if (small_mode == 8 || small_mode == 16) {
    const unsigned gb = unsigned(std::min<uint64_t>(
        (uint64_t(m ? m : 1) * small_mode + 255) / 256,
        small_mode == 8 ? resident_ctas(k_merge_group<8>, 256, num_sms) : resident_ctas(k_merge_group<16>, 256, num_sms)));
    if (small_mode == 8)
      k_merge_group<8><<<gb, 256, 0, s>>>(heads, skeys, svals, ins_prefix, m, ups, g, new_off, new_cap, ipos, qenc,
                                          nq, rows, colsize, st, memo, memo_mask, small_list);
    else
      k_merge_group<16><<<gb, 256, 0, s>>>(heads, skeys, svals, ins_prefix, m, ups, g, new_off, new_cap, ipos, qenc,
                                           nq, rows, colsize, st, memo, memo_mask, small_list);
  }
  // a CTA per long list (k_alloc's list), so long lists merge concurrently
  // long lists (disjoint from the others; shared structures are updated with
  // atomics) on s_big, which the caller may run beside s
  k_merge_big<<<unsigned(std::min<uint64_t>(m ? m : 1, resident_ctas(k_merge_big, BDSM_BIG_THREADS, num_sms))),
                BDSM_BIG_THREADS, 0, s_big>>>(heads, skeys, svals, ins_prefix, m, ups, g, new_off, new_cap, ipos, qenc,
                                          nq, rows, colsize, st, memo, memo_mask, big_list);
  k_finish_big<<<unsigned(std::min<uint64_t>((uint64_t(m ? m : 1) * 32 + 255) / 256,
                                             resident_ctas(k_finish_big, 256, num_sms))), 256, 0,
                 s_big>>>(heads, skeys, svals, m, g, qenc, nq, rows, colsize, st, memo, memo_mask, big_list);
}
void launch_encode_all(DevGraph g, const DevQueryEnc* qenc, uint32_t* rows, int num_sms, cudaStream_t s) {
  k_encode_all<<<unsigned(num_sms * 16), 256, 0, s>>>(g, qenc, rows);
}
void launch_hot_walks(const uint32_t* heads, const uint64_t* skeys, const BatchState* st, DevGraph g,
                      uint32_t* heat, uint32_t walks, uint32_t depth, uint32_t seed, int num_sms, cudaStream_t s) {
  k_hot_walks<<<unsigned(num_sms * 4), kThreads, 0, s>>>(heads, skeys, st, g, heat, walks, depth, seed);
}
void launch_hot_pack(DevGraphMut g, uint32_t* heat, unsigned long long* hist, unsigned long long budget,
                     BatchState* st, int num_sms, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, 34 * sizeof(unsigned long long), s);
  DevGraph v{g.V, g.off, g.deg, g.cap, g.adj, g.elab, g.vlabel, g.loff, g.nlab, g.hub_slot, g.bitmaps, g.bm_words};
  k_hot_hist<<<unsigned(num_sms * 8), kThreads, 0, s>>>(v, heat, hist);
  k_hot_select<<<1, 32, 0, s>>>(hist, budget);
  k_hot_pack<<<unsigned(num_sms * 16), kThreads, 0, s>>>(g, heat, hist, st);
}
struct DegAbove {
  const uint32_t* deg;
  uint32_t min_deg;
  __host__ __device__ bool operator()(uint32_t v) const { return deg[v] > min_deg; }
};
// Hub list (ascending ids with more than min_deg neighbours) for the leaf prefill.
size_t select_hubs_tmp_bytes(uint32_t V) {
  size_t tmp = 0;
  cub::DeviceSelect::If(nullptr, tmp, cub::CountingInputIterator<uint32_t>(0), (uint32_t*)nullptr,
                        (uint32_t*)nullptr, int(V), DegAbove{nullptr, 0});
  return tmp;
}
void launch_select_hubs(const uint32_t* deg, uint32_t V, uint32_t min_deg, uint32_t* hubs, uint32_t* n_hubs,
                        void* tmp, size_t tmp_bytes, cudaStream_t s) {
  cub::DeviceSelect::If(tmp, tmp_bytes, cub::CountingInputIterator<uint32_t>(0), hubs, n_hubs, int(V),
                        DegAbove{deg, min_deg}, s);
}
// Warp per hub: set the bit of every neighbour.
__global__ void k_build_bitmaps(DevGraphMut g, const uint32_t* __restrict__ hubs, uint32_t nhubs) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t h = warp; h < nhubs; h += nwarps) {
    const uint32_t v = hubs[h];
    uint32_t* bm = g.bitmaps + uint64_t(g.hub_slot[v]) * g.bm_words;
    const uint32_t* lst = g.adj + g.off[v];
    for (uint32_t i = lane; i < g.deg[v]; i += 32) {
      const uint32_t y = lst[i];
      atomicOr(bm + (y >> 5), 1u << (y & 31));
    }
  }
}
void launch_build_bitmaps(DevGraphMut g, const uint32_t* hubs, uint32_t nhubs, cudaStream_t s) {
  if (nhubs) k_build_bitmaps<<<blocks_for(uint64_t(nhubs) * 32), kThreads, 0, s>>>(g, hubs, nhubs);
}
void launch_label_index(DevGraphMut g, int num_sms, cudaStream_t s) {
  if (g.loff && g.V) k_label_index<<<unsigned(num_sms * 16), 256, 0, s>>>(g);
}
void launch_column_sizes(const uint32_t* rows, uint32_t V, uint32_t n, uint64_t* out, cudaStream_t s) {
  k_column_sizes<<<blocks_for(V), kThreads, 0, s>>>(rows, V, n, out);
}

}  // namespace bdsm_b200
