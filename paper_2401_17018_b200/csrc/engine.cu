// Engine orchestration and the C ABI (include/bdsm_gpu.h).
//
// One engine = one device-resident dynamic CSR shared by N queries.  A batch
// is one stream-ordered device sequence with a single host synchronisation at
// the end (match_batch, reference src/matcher.cpp:370-389):
//   H2D(batch) -> K1 validate/canonicalise -> radix sort of the 2|dB| directed
//   keys -> segment heads / bitmaps -> [per query: K5 anchors -> K6 count on G]
//   -> K3 merge + K4 refresh -> [per query: K5 -> K6 on G'] -> D2H(counts).
// Every kernel after K1 checks the device-side error flags, so an invalid
// batch is rejected all-or-nothing without a host round trip.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include "../../include/bdsm_gpu.h"
#include "kernels.cuh"
#include "planner.hpp"

using namespace bdsm_b200;

namespace {

thread_local std::string g_last_error;

// NVTX range over a host scope (the enqueue of a batch stage; nsys / ncu
// --nvtx show them beside the kernels)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct BatchRejected : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      if (e_ == cudaErrorMemoryAllocation) throw std::bad_alloc();                        \
      throw CudaFailure(std::string(#expr) + ": " + cudaGetErrorString(e_));              \
    }                                                                                     \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  T* host = nullptr;    // zero-copy: mapped pinned host allocation behind p
  bool mapped = false;  // allocate as mapped pinned host memory (graphs beyond HBM)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (host) cudaFreeHost(host);
    else if (p) cudaFree(p);
    p = nullptr;
    host = nullptr;
    n = 0;
  }
  void ensure(size_t want) {
    if (want <= n && p) return;
    release();
    size_t alloc = std::max<size_t>(want, 1);
    if (mapped) {
      CK(cudaHostAlloc(reinterpret_cast<void**>(&host), alloc * sizeof(T), cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p), host, 0));
    } else {
      CK(cudaMalloc(&p, alloc * sizeof(T)));
    }
    n = alloc;
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(host, o.host);
    std::swap(mapped, o.mapped);
  }
  void ensure_grow(size_t want) {  // amortised growth
    if (want <= n && p) return;
    ensure(std::max<size_t>(want, n + n / 2));
  }
};

struct QueryState {
  HostQuery q;
  QueryEncoding enc;
  DevQueryEnc denc{};
  DBuf<uint32_t> rows;
  DBuf<uint64_t> colsize;
  DBuf<EdgeProg> progs;
  DBuf<AnchorEdge> anchors;
  DBuf<AnchorEdge> anchors_co;   // exact coalescing: one directed edge per automorphism orbit (planner.hpp)
  uint32_t coalesce_gain = 1;    // directed edges per searched one (diagnostics)
  std::vector<std::vector<uint32_t>> orders;
  std::vector<uint32_t> tails;  // EdgeProg::tail per query edge
  bool has_leaf = false;         // some program weights leaves of its last DFS level (memo in use)
  uint32_t prev_items[2] = {0, 0};  // work items of the last batch per phase (kernel variant choice)
  bool memo_cold = true;            // the memo holds none of this query's weights (full prefill next)
  uint32_t natail = 0;              // anchor-only tail levels per program (per-task count cache stride)
  DBuf<uint32_t> mbuf[2];        // materialised matches per phase (bdsm_engine_collect_matches)
  DBuf<unsigned long long> mcount;
  DBuf<LeafSig> leafsigs;        // distinct leaf signatures (prefill before each launch)
  uint32_t n_leafsig = 0;
  uint64_t deadline_ns = 0;  // host-steady-clock based, translated per batch
  double deadline_s = 0;     // seconds since epoch of the host steady clock
  bool active = true;        // matched in later batches (bdsm_engine_set_query_active)
};

uint64_t now_ns() {
  return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now().time_since_epoch())
                      .count());
}

}  // namespace

struct bdsm_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  // the positive phase's touched-hub memo prefill runs here, beside the
  // anchor kernels (both only read G'); joined before the matching kernel
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  bool early_anchors = false;  // this attempt's negative-phase anchors were issued on `side`
  cudaEvent_t fork2_ev = nullptr, join2_ev = nullptr;  // the insert-prefix scan on `side`
  // the long lists' merge (k_merge_big + k_finish_big) runs on its own stream
  // beside the warp- and thread-per-list merges (disjoint lists, atomics on
  // the shared structures)
  cudaStream_t side_big = nullptr;
  cudaEvent_t big_fork_ev = nullptr, big_join_ev = nullptr;
  cudaStream_t fork_big() {
    CK(cudaEventRecord(big_fork_ev, stream));
    CK(cudaStreamWaitEvent(side_big, big_fork_ev, 0));
    return side_big;
  }
  void join_big() {
    CK(cudaEventRecord(big_join_ev, side_big));
    CK(cudaStreamWaitEvent(stream, big_join_ev, 0));
  }
  DBuf<uint8_t> cub_tmp_side;
  DBuf<uint8_t> cub_tmp_big;  // CUB scratch of side_big (the stream's next-batch anchors)
  int num_sms = 148;
  bdsm_options opts{};
  DevGraphMut g{};
  uint64_t pool_top = 0;
  uint64_t n_edges = 0;
  bool has_elab = false;

  DBuf<uint64_t> off;
  DBuf<uint32_t> deg, cap, adj, elab, vlabel;
  DBuf<uint32_t> loff, class_lo;  // label index (DevGraph::loff) and label-class start ids
  DBuf<uint32_t> hub_slot, bitmaps;  // hub membership bitmaps (DevGraph::hub_slot)
  uint64_t bm_words = 0;

  std::vector<std::unique_ptr<QueryState>> queries;
  DBuf<DevQueryEnc> d_qenc;
  DBuf<uint32_t*> d_rows;
  DBuf<uint64_t*> d_colsize;

  // batch buffers
  // Per-batch buffers.  Two slots: the pipelined stream (apply_stream) keeps
  // batch i and batch i+1 in flight together; a single batch uses slot 0.
  struct BatchBufs {
    DBuf<bdsm_update_dev> ups;      // translated (internal ids), read by every kernel after K1
    DBuf<bdsm_update_dev> ups_ext;  // host-input staging (external ids)
    DBuf<uint64_t> keys, keys2, skeys;
    DBuf<uint32_t> vals, vals2, svals, dlab, insflag, ins_prefix, heads, ipos, new_cap, big_list, small_list, mid_list;
    DBuf<uint8_t> ecode, head;
    DBuf<uint64_t> new_off;
    DBuf<unsigned long long> hkeys;  // visibility table of the batch
    DBuf<uint32_t> hvals;
    DBuf<AnchorCount> upd_cnt, upd_off;
    DBuf<Task> tasks;
    DBuf<Item> items;
    DBuf<unsigned long long> task_tail;  // per-task counts of anchor-only tail levels (PhaseArgs::task_tail)
    size_t batch_cap = 0;
    // BatchState followed by the per-query results (common.cuh): one H2D
    // before, one D2H after every batch
    DBuf<unsigned char> st_buf;
    BatchState* d_st = nullptr;
    BatchState* h_st = nullptr;
    size_t st_bytes = 0, h_st_bytes = 0;
    ~BatchBufs() {
      if (h_st) cudaFreeHost(h_st);
    }
  };
  BatchBufs slot_[2];
  uint32_t cs = 0;  // slot of the batch being enqueued
  BatchBufs& B() { return slot_[cs]; }
  size_t max_items = 0;
  DBuf<DynItem> dyn;           // donated-subtree queue of the matching kernel
  DBuf<QueueState> qstate;
  DBuf<uint32_t> dyn_ready;
  DBuf<unsigned long long> memo;  // weight memo of the matching kernel (2^21 words, persistent)
  DBuf<unsigned long long> memo_fill;  // slots taken since the last reset
  uint32_t qs_natail(int qi) const { return queries.at(size_t(qi))->natail; }
  bool memo_persistent = true;     // false when a query has too many signatures to invalidate
  unsigned long long* h_memo_fill = nullptr;  // pinned copy of memo_fill, refreshed every batch
  DBuf<uint32_t> memo_bits;  // DevGraph::memo_bits
  void reset_memo() {
    if (!memo.p) return;
    CK(cudaMemsetAsync(memo.p, 0xff, sizeof(unsigned long long) * memo.n, stream));
    if (memo_bits.p) CK(cudaMemsetAsync(memo_bits.p, 0, 4 * memo_bits.n, stream));
    CK(cudaMemsetAsync(memo_fill.p, 0, sizeof(unsigned long long), stream));
    for (auto& q : queries) q->memo_cold = true;
  }
  uint64_t collect_cap = 0;        // matches materialised per (query, phase); 0 = counts only
  // matching-kernel tuning knobs (BDSM_TUNE_BACKOFF / BDSM_TUNE_MERGE env overrides, for sweeps)
  // idle warps' longest sleep between donation polls (ns); 0: by variant —
  // 256 for the latency-bound 2-CTA launches (C2 +1.5-2 %), 1024 for the
  // 4-CTA throughput launches (C4 -3 % at 256; C3/C5 neutral)
  uint32_t tune_backoff = env_u32("BDSM_TUNE_BACKOFF", 0);
  uint32_t tune_merge_ratio = env_u32("BDSM_TUNE_MERGE", 8);
  uint32_t tune_variant = env_u32("BDSM_TUNE_VARIANT", 0);  // 2 / 3 / 4: force a matching-kernel variant
  // the variant of launches with many work items (4: 4 CTAs/SM, 64 registers; 3: 3 CTAs/SM, 80 registers):
  // 4 up to tune_many_items items per phase (C3, ~10K: 69.5K vs 66.1K updates/s), 3 above (C4, ~30K: +3 %);
  // BDSM_TUNE_VARIANT_THROUGHPUT forces one of them
  uint32_t tune_variant_tp = env_u32("BDSM_TUNE_VARIANT_THROUGHPUT", 0);
  uint32_t tune_many_items = env_u32("BDSM_TUNE_MANY_ITEMS", 16000);
  int variant_for(uint32_t items) const {
    if (tune_variant) return int(tune_variant);
    if (items <= tune_throughput_items) return 2;
    if (tune_variant_tp) return int(tune_variant_tp);
    return items > tune_many_items ? 3 : 4;
  }
  uint32_t tune_no_tasktail = env_u32("BDSM_TUNE_NO_TASKTAIL", 0);  // 1: recount anchor-only tail levels per item
  uint32_t tune_throughput_items = env_u32("BDSM_TUNE_ITEMS", kThroughputItems);
  // short lists (<= tune_small_max entries before and after) of batches with at
  // least tune_small_min directed keys get their own kernel: lanes per list
  // tune_small_group below kSmallMergeMinKeys keys (latency-bound: a group of 8
  // lanes per list, k_merge_group; C2 merge 0.085 -> 0.070 ms) and
  // tune_small_group_large above (throughput-bound: a thread per list,
  // k_merge_small, 32 lists in flight per warp; C4 merge 1.59 ms vs 1.92 ms
  // with groups of 8)
  uint32_t tune_small_min = env_u32("BDSM_TUNE_SMALLMIN", 1);
  uint32_t tune_small_group = env_u32("BDSM_TUNE_SMALL_GROUP", 8);
  uint32_t tune_small_group_large = env_u32("BDSM_TUNE_SMALL_GROUP_LARGE", 1);
  uint32_t tune_small_max = env_u32("BDSM_TUNE_SMALLMAX", 256);
  // shortest list merged by a whole CTA (k_merge_big), small / large batches
  uint32_t tune_big_min = env_u32("BDSM_TUNE_BIGLIST", 1024);
  uint32_t tune_big_min_large = env_u32("BDSM_TUNE_BIGLIST_LARGE", 4096);  // C4: 4096 268.7M, 2048 265.7M, 1024 253.1M
  bool large_batch(uint32_t m) const { return m >= kSmallMergeMinKeys; }
  uint32_t small_group(uint32_t m) const { return large_batch(m) ? tune_small_group_large : tune_small_group; }
  uint32_t small_max(uint32_t m) const {
    if (m < tune_small_min) return 0;
    return small_group(m) == 1 ? std::min<uint32_t>(tune_small_max, 256) : tune_small_max;
  }
  uint32_t big_min(uint32_t m) const { return large_batch(m) ? tune_big_min_large : tune_big_min; }
  uint32_t tune_self_scan = env_u32("BDSM_TUNE_SELFSCAN", kSelfScanUpdates);
  static uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* v = getenv(name);
    return v ? uint32_t(strtoul(v, nullptr, 10)) : dflt;
  }

  // K8 hot-list L2 persistence (opts.l2_hot_mb > 0).  Every kHotPeriod batches
  // the hottest lists (random-walk visit counts, decayed) are packed into an
  // arena at the pool's bump pointer and the engine stream gets a persisting
  // access-policy window over it.
  static constexpr uint64_t kHotPeriod = 8;
  static constexpr uint32_t kSelfScanUpdates = 16384;  // batches up to this size: anchor offsets scanned in k_anchor_emit
  static constexpr uint32_t kSmallMergeMinKeys = 65536;  // C2 batches: 20K keys, C4: 2M
  static constexpr uint32_t kThroughputItems = 2000;  // above: the 4-CTA matching-kernel variant (C2 ~300, C3 ~7K)
  // Hub list for the leaf-weight prefill, refreshed every kHubPeriod batches.
  static constexpr uint64_t kHubPeriod = 16;
  DBuf<uint32_t> hub_ids, n_hubs;
  DBuf<uint8_t> hub_tmp;
  uint64_t hubs_at = ~0ull;
  void refresh_hubs() {
    if (hubs_at != ~0ull && batches_done - hubs_at < kHubPeriod) return;
    hub_ids.ensure(std::max<uint32_t>(g.V, 1));
    n_hubs.ensure(1);
    const size_t tmp = select_hubs_tmp_bytes(g.V);
    hub_tmp.ensure(std::max<size_t>(tmp, 1));
    launch_select_hubs(g.deg, g.V, 256, hub_ids.p, n_hubs.p, hub_tmp.p, hub_tmp.n, stream);
    ++cub_calls;
    hubs_at = batches_done;
  }
  DBuf<uint32_t> heat;
  DBuf<unsigned long long> hot_hist;
  bool heat_init = false;
  uint64_t batches_done = 0;
  void hot_pack_maybe() {
    if (!opts.l2_hot_mb || batches_done == 0 || batches_done % kHotPeriod) return;
    int max_persist = 0, max_window = 0;
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device));
    CK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device));
    const uint64_t budget =
        std::min<uint64_t>({uint64_t(opts.l2_hot_mb) << 20, uint64_t(max_window), uint64_t(max_persist)});
    if (budget < 4096 || g.pool_size - pool_top < 2 * (budget / 4)) return;  // no room: skip this period
    hot_hist.ensure(34);
    launch_hot_pack(g, heat.p, hot_hist.p, budget, B().d_st, num_sms, stream);
    launches += 4;
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(budget)));
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = g.adj + pool_top;
    attr.accessPolicyWindow.num_bytes = size_t(budget);
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &attr));
  }

  // Matches of the last batch for (query, phase) in external ids, query vertex
  // order, sorted (the reference sorts its match vectors, src/matcher.cpp:365-366).
  size_t fetch_matches(int qi, int phase, std::vector<uint32_t>& out) {
    QueryState& qs = *queries.at(size_t(qi));
    out.clear();
    if (!collect_cap || !qs.mcount.p) return 0;
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, qs.mcount.p + phase, sizeof(cnt), cudaMemcpyDeviceToHost, stream));
    sync();
    const size_t got = size_t(std::min<unsigned long long>(cnt, collect_cap));
    const uint32_t n = qs.q.n;
    out.resize(got * n);
    if (got) CK(cudaMemcpyAsync(out.data(), qs.mbuf[phase].p, 4ull * got * n, cudaMemcpyDeviceToHost, stream));
    sync();
    for (auto& x : out) x = old_of[x];
    std::vector<size_t> idx(got);
    for (size_t i = 0; i < got; ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](size_t p, size_t q) {
      return std::lexicographical_compare(out.begin() + p * n, out.begin() + (p + 1) * n, out.begin() + q * n,
                                          out.begin() + (q + 1) * n);
    });
    std::vector<uint32_t> sorted(got * n);
    for (size_t i = 0; i < got; ++i) std::copy_n(out.begin() + idx[i] * n, n, sorted.begin() + i * n);
    out.swap(sorted);
    return size_t(cnt);
  }
  uint32_t epoch = 0;
  DBuf<uint8_t> cub_tmp;
  size_t st_size() const { return sizeof(BatchState) + 20 * std::max<size_t>(queries.size(), 1); }
  static unsigned long long* st_counts(BatchState* s) { return reinterpret_cast<unsigned long long*>(s + 1); }
  uint32_t* st_timed(BatchState* s) const { return reinterpret_cast<uint32_t*>(st_counts(s) + 2 * queries.size()); }
  void ensure_state() {
    BatchBufs& b = B();
    b.st_bytes = st_size();
    if (b.st_buf.n < b.st_bytes) {
      b.st_buf.ensure(b.st_bytes);
      b.d_st = reinterpret_cast<BatchState*>(b.st_buf.p);
    }
    if (b.h_st_bytes < b.st_bytes) {
      if (b.h_st) cudaFreeHost(b.h_st);
      b.h_st = nullptr;
      CK(cudaMallocHost(&b.h_st, b.st_bytes));
      b.h_st_bytes = b.st_bytes;
    }
  }
  bdsm_update* h_ups = nullptr;
  const bdsm_update* h_src = nullptr;  // this batch's host updates (caller's pinned buffer or h_ups)
  size_t h_ups_cap = 0;
  cudaEvent_t ev[6] = {};
  cudaEvent_t merge_ev[2] = {};
  std::vector<cudaEvent_t> kev;  // pairs around K6 launches, then the merge pair
  size_t kev_used = 0;
  uint32_t launches = 0, cub_calls = 0;
  cudaEvent_t next_kev() {
    if (kev_used == kev.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      kev.push_back(e);
    }
    return kev[kev_used++];
  }

  std::vector<bdsm_update_error> last_errors;
  std::vector<uint8_t> last_timed;  // per query: the deadline fired in the last batch

  ~bdsm_engine() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : merge_ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : kev) cudaEventDestroy(e);
    if (h_memo_fill) cudaFreeHost(h_memo_fill);
    if (h_stream) cudaFreeHost(h_stream);
    for (auto& x : stream_ev) cudaEventDestroy(x);
    for (auto& x : stream_kev) cudaEventDestroy(x);
    for (auto& x : front_ev)
      if (x) cudaEventDestroy(x);
    if (h_ups) cudaFreeHost(h_ups);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (fork2_ev) cudaEventDestroy(fork2_ev);
    if (join2_ev) cudaEventDestroy(join2_ev);
    if (side) cudaStreamDestroy(side);
    if (side_big) cudaStreamDestroy(side_big);
    if (big_fork_ev) cudaEventDestroy(big_fork_ev);
    if (big_join_ev) cudaEventDestroy(big_join_ev);
    if (stream) cudaStreamDestroy(stream);
  }

  DevGraph view() const {
    DevGraph v;
    v.V = g.V;
    v.off = g.off;
    v.deg = g.deg;
    v.cap = g.cap;
    v.adj = g.adj;
    v.elab = g.elab;
    v.vlabel = g.vlabel;
    v.loff = g.loff;
    v.nlab = g.nlab;
    v.hub_slot = g.hub_slot;
    v.bitmaps = g.bitmaps;
    v.bm_words = g.bm_words;
    v.memo_bits = g.memo_bits;
    return v;
  }

  void sync() { CK(cudaStreamSynchronize(stream)); }

  // ---------------------------------------------------------------- build --
  // Internal vertex ids are ordered by (label, external id): every label class
  // is one contiguous id range, so the label-L neighbours of any vertex form a
  // contiguous sub-range of its sorted list (used by the matching kernel to
  // shrink drivers and searches).  The C ABI speaks external ids only.
  std::vector<uint32_t> new_of, old_of;           // external -> internal, internal -> external
  std::vector<std::pair<uint32_t, std::pair<uint32_t, uint32_t>>> label_ranges;  // label -> [lo, hi)
  DBuf<uint32_t> d_new_of;
  const bdsm_graph_desc* orig_desc = nullptr;

  void build(const bdsm_graph_desc* d) {
    const uint32_t V = d->num_vertices;
    const uint64_t E = d->num_edges;
    if (E && (!d->src || !d->dst)) throw std::invalid_argument("edge arrays are null");
    if (V && !d->vertex_labels) throw std::invalid_argument("vertex labels are null");
    orig_desc = d;
    std::vector<uint64_t> key(V);
    for (uint32_t v = 0; v < V; ++v) key[v] = (uint64_t(d->vertex_labels[v]) << 32) | v;
    std::sort(key.begin(), key.end());
    new_of.assign(V, 0);
    old_of.assign(V, 0);
    std::vector<uint32_t> lab(V);
    label_ranges.clear();
    for (uint32_t i = 0; i < V; ++i) {
      uint32_t v = uint32_t(key[i]), l = uint32_t(key[i] >> 32);
      old_of[i] = v;
      new_of[v] = i;
      lab[i] = l;
      if (label_ranges.empty() || label_ranges.back().first != l) label_ranges.push_back({l, {i, i}});
      label_ranges.back().second.second = i + 1;
    }
    key.clear();
    key.shrink_to_fit();
    std::vector<uint32_t> src(E), dst(E);
    for (uint64_t i = 0; i < E; ++i) {
      uint32_t u = d->src[i], v = d->dst[i];
      if (u >= V || v >= V) throw_build_error(d, 2);
      src[i] = new_of[u];
      dst[i] = new_of[v];
    }
    bdsm_graph_desc internal{V, lab.data(), E, src.data(), dst.data(), d->edge_labels};
    d_new_of.ensure(std::max<uint32_t>(V, 1));
    if (V) CK(cudaMemcpyAsync(d_new_of.p, new_of.data(), 4ull * V, cudaMemcpyHostToDevice, stream));
    build_internal(&internal);
    orig_desc = nullptr;
    build_label_index();
    build_bitmaps();
  }

  // Label index over the label classes (label_ranges order); disabled for
  // graphs with more than kMaxLabelIndex classes.
  void build_label_index() {
    const uint32_t nl = uint32_t(label_ranges.size());
    g.nlab = nl;
    loff.release();
    std::vector<uint32_t> lo(std::max<uint32_t>(nl, 1), 0);
    for (uint32_t k = 0; k < nl; ++k) lo[k] = label_ranges[k].second.first;
    class_lo.ensure(lo.size());
    CK(cudaMemcpyAsync(class_lo.p, lo.data(), 4 * lo.size(), cudaMemcpyHostToDevice, stream));
    if (nl > kMaxLabelIndex || g.V == 0) {
      refresh_graph_view();
      sync();
      return;
    }
    loff.ensure(uint64_t(g.V) * (nl + 1));
    refresh_graph_view();
    launch_label_index(g, num_sms, stream);
    sync();
  }

  // Membership bitmaps for the highest-degree vertices (>= kBitmapMinDeg
  // neighbours; BDSM_BITMAP_MINDEG overrides, tests use it to exercise the
  // path on small graphs), as many as fit the budget (BDSM_BITMAP_MB, default 2048).
  // The set is fixed at build; the merge keeps each bitmap in step with its list.
  void build_bitmaps() {
    hub_slot.release();
    bitmaps.release();
    if (g.V == 0) return;
    const uint64_t words = (uint64_t(g.V) + 31) / 32;
    const uint64_t budget = uint64_t(env_u32("BDSM_BITMAP_MB", 2048)) << 20;
    const uint64_t maxh = budget / (4 * words);
    if (maxh == 0) return;
    std::vector<uint32_t> d(g.V);
    CK(cudaMemcpyAsync(d.data(), g.deg, 4ull * g.V, cudaMemcpyDeviceToHost, stream));
    sync();
    std::vector<uint32_t> hubs;
    const uint32_t min_deg = env_u32("BDSM_BITMAP_MINDEG", kBitmapMinDeg);
    for (uint32_t v = 0; v < g.V; ++v)
      if (d[v] >= min_deg) hubs.push_back(v);
    if (hubs.empty()) return;
    std::sort(hubs.begin(), hubs.end(), [&](uint32_t a, uint32_t b) { return d[a] != d[b] ? d[a] > d[b] : a < b; });
    if (hubs.size() > maxh) hubs.resize(maxh);
    std::vector<uint32_t> slot(g.V, kNone);
    for (uint32_t i = 0; i < hubs.size(); ++i) slot[hubs[i]] = i;
    hub_slot.ensure(g.V);
    CK(cudaMemcpyAsync(hub_slot.p, slot.data(), 4ull * g.V, cudaMemcpyHostToDevice, stream));
    bitmaps.ensure(words * hubs.size());
    CK(cudaMemsetAsync(bitmaps.p, 0, 4ull * words * hubs.size(), stream));
    bm_words = words;
    DBuf<uint32_t> dh;
    dh.ensure(hubs.size());
    CK(cudaMemcpyAsync(dh.p, hubs.data(), 4ull * hubs.size(), cudaMemcpyHostToDevice, stream));
    refresh_graph_view();
    launch_build_bitmaps(g, dh.p, uint32_t(hubs.size()), stream);
    sync();
  }

  uint32_t label_class(uint32_t label) const {
    auto it = std::lower_bound(label_ranges.begin(), label_ranges.end(), label,
                               [](const auto& e, uint32_t l) { return e.first < l; });
    if (it == label_ranges.end() || it->first != label) return kNone;
    return uint32_t(it - label_ranges.begin());
  }

  std::pair<uint32_t, uint32_t> label_range(uint32_t label) const {
    auto it = std::lower_bound(label_ranges.begin(), label_ranges.end(), label,
                               [](const auto& e, uint32_t l) { return e.first < l; });
    if (it == label_ranges.end() || it->first != label) return {0, 0};
    return it->second;
  }

  void build_internal(const bdsm_graph_desc* d) {
    const uint32_t V = d->num_vertices;
    const uint64_t E = d->num_edges;
    g.V = V;
    n_edges = E;
    has_elab = false;
    if (d->edge_labels) {
      for (uint64_t i = 0; i < E; ++i)
        if (d->edge_labels[i] != BDSM_NO_LABEL) {
          has_elab = true;
          break;
        }
    }
    vlabel.ensure(V);
    deg.ensure(V);
    cap.ensure(V);
    off.ensure(V);
    if (V) CK(cudaMemcpyAsync(vlabel.p, d->vertex_labels, sizeof(uint32_t) * V, cudaMemcpyHostToDevice, stream));
    CK(cudaMemsetAsync(deg.p, 0, sizeof(uint32_t) * std::max<uint32_t>(V, 1), stream));
    const uint64_t M = 2 * E;
    DBuf<uint32_t> src, dst, labs;
    DBuf<uint64_t> k0, k1, v0, v1, cap64, dense;
    DBuf<uint32_t> bad;
    bad.ensure(1);
    CK(cudaMemsetAsync(bad.p, 0, 4, stream));
    if (E) {
      src.ensure(E);
      dst.ensure(E);
      CK(cudaMemcpyAsync(src.p, d->src, 4 * E, cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(dst.p, d->dst, 4 * E, cudaMemcpyHostToDevice, stream));
      k0.ensure(M);
      k1.ensure(M);
      if (has_elab) {
        v0.ensure(M);
        v1.ensure(M);
        labs.ensure(E);
        CK(cudaMemcpyAsync(labs.p, d->edge_labels, 4 * E, cudaMemcpyHostToDevice, stream));
      }
      launch_build_keys(src.p, dst.p, E, V, k0.p, has_elab ? v0.p : nullptr, bad.p, stream);
      src.release();
      dst.release();
      size_t tmp = 0;
      cub::DoubleBuffer<uint64_t> kb(k0.p, k1.p), vb(v0.p, v1.p);
      if (has_elab) {
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, int64_t(M), 0, 64, stream));
        cub_tmp.ensure(tmp);
        CK(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tmp, kb, vb, int64_t(M), 0, 64, stream));
      } else {
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kb, int64_t(M), 0, 64, stream));
        cub_tmp.ensure(tmp);
        CK(cub::DeviceRadixSort::SortKeys(cub_tmp.p, tmp, kb, int64_t(M), 0, 64, stream));
      }
      uint64_t* sk = kb.Current();
      uint64_t* sv = has_elab ? vb.Current() : nullptr;
      launch_check_sorted_dups(sk, M, bad.p, stream);
      uint32_t hbad = 0;
      CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, stream));
      sync();
      if (hbad) throw_build_error(orig_desc ? orig_desc : d, hbad);
      launch_degrees(sk, M, deg.p, stream);
      // capacities -> offsets; dense offsets for the scatter
      cap64.ensure(V);
      dense.ensure(V);
      launch_caps(deg.p, V, opts.slack, cap.p, cap64.p, stream);
      scan_u64_inplace(cap64.p, off.p, V);
      // dense offsets: exclusive scan of deg (as u64)
      scan_widen(deg.p, dense.p, V);
      uint64_t last_off = 0;
      uint32_t last_cap = 0;
      CK(cudaMemcpyAsync(&last_off, off.p + (V - 1), 8, cudaMemcpyDeviceToHost, stream));
      CK(cudaMemcpyAsync(&last_cap, cap.p + (V - 1), 4, cudaMemcpyDeviceToHost, stream));
      sync();
      pool_top = last_off + last_cap;
      uint64_t reserve = std::max<uint64_t>(uint64_t(double(M) * opts.pool_reserve), 1u << 20);
      g.pool_size = pool_top + reserve;
      adj.ensure(g.pool_size);
      if (has_elab) elab.ensure(g.pool_size);
      launch_scatter(sk, sv, M, dense.p, off.p, adj.p, has_elab ? labs.p : nullptr,
                     has_elab ? elab.p : nullptr, stream);
    } else {
      if (V) {
        DBuf<uint64_t> cap64b;
        cap64b.ensure(V);
        launch_caps(deg.p, V, opts.slack, cap.p, cap64b.p, stream);
        scan_u64_inplace(cap64b.p, off.p, V);
        uint64_t last_off = 0;
        uint32_t last_cap = 0;
        CK(cudaMemcpyAsync(&last_off, off.p + (V - 1), 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(&last_cap, cap.p + (V - 1), 4, cudaMemcpyDeviceToHost, stream));
        sync();
        pool_top = last_off + last_cap;
      }
      g.pool_size = pool_top + (1u << 20);
      adj.ensure(g.pool_size);
    }
    sync();
    refresh_graph_view();
  }

  void refresh_graph_view() {
    g.off = off.p;
    g.deg = deg.p;
    g.cap = cap.p;
    g.adj = adj.p;
    g.elab = has_elab ? elab.p : nullptr;
    g.vlabel = vlabel.p;
    g.loff = loff.n ? loff.p : nullptr;
    g.class_lo = class_lo.p;
    g.hub_slot = hub_slot.n ? hub_slot.p : nullptr;
    g.bitmaps = bitmaps.p;
    g.bm_words = bm_words;
    g.memo_bits = memo_bits.p;
  }

  [[noreturn]] void throw_build_error(const bdsm_graph_desc* d, uint32_t bad) {
    // Host rescan for the reference's exact message (src/graph.cpp:38-64).
    for (uint64_t i = 0; i < d->num_edges; ++i) {
      uint32_t u = d->src[i], v = d->dst[i];
      if (u == v)
        throw std::invalid_argument("self-loop edge (" + std::to_string(u) + "," + std::to_string(v) + ")");
      if (u >= d->num_vertices || v >= d->num_vertices)
        throw std::invalid_argument("edge (" + std::to_string(u) + "," + std::to_string(v) +
                                    ") references unknown vertex");
    }
    if (bad & 4u) throw std::invalid_argument("duplicate edge");
    throw std::invalid_argument("invalid graph");
  }

  struct Widen {
    __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
  };
  void scan_widen(const uint32_t* in, uint64_t* out, uint64_t n) {
    cub::TransformInputIterator<uint64_t, Widen, const uint32_t*> it(in, Widen{});
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, out, int64_t(n), stream));
    cub_tmp.ensure(tmp);
    CK(cub::DeviceScan::ExclusiveSum(cub_tmp.p, tmp, it, out, int64_t(n), stream));
  }

  void scan_u64_inplace(const uint64_t* in, uint64_t* out, uint64_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, int64_t(n), stream));
    cub_tmp.ensure(tmp);
    CK(cub::DeviceScan::ExclusiveSum(cub_tmp.p, tmp, in, out, int64_t(n), stream));
  }

  // Rebuild every list into a fresh pool with fresh slack (pool exhausted).
  void compact(uint64_t extra_need) {
    const uint32_t V = g.V;
    DBuf<uint32_t> ncap;
    DBuf<uint64_t> ncap64, noff;
    ncap.ensure(V);
    ncap64.ensure(V);
    noff.ensure(V);
    launch_caps(deg.p, V, opts.slack, ncap.p, ncap64.p, stream);
    scan_u64_inplace(ncap64.p, noff.p, V);
    uint64_t last_off = 0;
    uint32_t last_cap = 0;
    CK(cudaMemcpyAsync(&last_off, noff.p + (V - 1), 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&last_cap, ncap.p + (V - 1), 4, cudaMemcpyDeviceToHost, stream));
    sync();
    uint64_t used = last_off + last_cap;
    uint64_t reserve = std::max<uint64_t>(uint64_t(double(used) * opts.pool_reserve), 1u << 20);
    reserve = std::max(reserve, 2 * extra_need);
    uint64_t size = used + reserve;
    DBuf<uint32_t> nadj, nelab;
    nadj.mapped = adj.mapped;
    nelab.mapped = elab.mapped;
    nadj.ensure(size);
    if (has_elab) nelab.ensure(size);
    launch_compact(g, noff.p, ncap.p, nadj.p, has_elab ? nelab.p : nullptr, stream);
    sync();
    adj.swap(nadj);
    if (has_elab) {
      elab.swap(nelab);
    }
    std::swap(off.p, noff.p);
    std::swap(off.n, noff.n);
    std::swap(cap.p, ncap.p);
    std::swap(cap.n, ncap.n);
    g.pool_size = size;
    pool_top = used;
    refresh_graph_view();
  }

  void enable_edge_labels() {
    // A labelled insert into an unlabelled graph: materialise the parallel
    // label array (all "none") once.
    elab.ensure(g.pool_size);
    std::vector<uint32_t> none(1 << 20, BDSM_NO_LABEL);
    for (uint64_t i = 0; i < g.pool_size; i += none.size()) {
      uint64_t k = std::min<uint64_t>(none.size(), g.pool_size - i);
      CK(cudaMemcpyAsync(elab.p + i, none.data(), 4 * k, cudaMemcpyHostToDevice, stream));
      sync();
    }
    has_elab = true;
    refresh_graph_view();
  }

  // --------------------------------------------------------------- queries --
  int add_query(const bdsm_query_desc* d) {
    if (!d || (d->num_vertices && !d->vertex_labels) || (d->num_edges && (!d->a || !d->b)))
      throw std::invalid_argument("null query arrays");
    std::vector<uint32_t> labels(d->vertex_labels, d->vertex_labels + d->num_vertices);
    std::vector<QEdge> edges;
    for (uint32_t i = 0; i < d->num_edges; ++i)
      edges.push_back({d->a[i], d->b[i], d->edge_labels ? d->edge_labels[i] : kNone});
    auto qs = std::make_unique<QueryState>();
    qs->q = HostQuery(std::move(labels), std::move(edges));
    if (!qs->q.connected()) throw std::invalid_argument("disconnected query graph");
    if (qs->q.n > uint32_t(kMaxQ))
      throw std::invalid_argument("query graph too large for the GPU engine (max " +
                                  std::to_string(kMaxQ) + " vertices)");
    if (queries.size() >= kMaxQueries)
      throw std::invalid_argument("at most " + std::to_string(kMaxQueries) + " queries per engine");
    qs->enc = encode_query(qs->q, opts.group_bits);
    DevQueryEnc& de = qs->denc;
    de.n = qs->q.n;
    de.G = uint32_t(qs->enc.group_labels.size());
    de.cap = qs->enc.cap;
    for (uint32_t u = 0; u < de.n; ++u) de.qlabel[u] = qs->q.labels[u];
    for (uint32_t gi = 0; gi < de.G; ++gi) {
      de.glabel[gi] = qs->enc.group_labels[gi];
      const auto r = label_range(de.glabel[gi]);
      de.glo[gi] = r.first;
      de.ghi[gi] = r.second;
      de.gcls[gi] = label_class(de.glabel[gi]);
    }
    for (uint32_t u = 0; u < de.n; ++u)
      for (uint32_t gi = 0; gi < de.G; ++gi) de.qcnt[u][gi] = qs->enc.qcnt[u * de.G + gi];
    DBuf<DevQueryEnc> one;
    one.ensure(1);
    CK(cudaMemcpyAsync(one.p, &de, sizeof(de), cudaMemcpyHostToDevice, stream));
    qs->rows.ensure(std::max<uint32_t>(g.V, 1));
    qs->colsize.ensure(32);
    CK(cudaMemsetAsync(qs->colsize.p, 0, 8 * 32, stream));
    if (g.V) {
      launch_encode_all(view(), one.p, qs->rows.p, num_sms, stream);
      launch_column_sizes(qs->rows.p, g.V, de.n, qs->colsize.p, stream);
    }
    sync();
    queries.push_back(std::move(qs));
    int qi = int(queries.size() - 1);
    replan(qi);
    upload_query_tables();
    return qi;
  }

  std::vector<uint64_t> column_sizes(int qi) {
    QueryState& qs = *queries.at(size_t(qi));
    std::vector<uint64_t> cs(32);
    CK(cudaMemcpyAsync(cs.data(), qs.colsize.p, 8 * 32, cudaMemcpyDeviceToHost, stream));
    sync();
    cs.resize(qs.q.n);
    return cs;
  }

  // build_query_plan with coalescing off: one order per query edge.
  void replan(int qi) {
    QueryState& qs = *queries.at(size_t(qi));
    std::vector<uint64_t> cs = column_sizes(qi);
    qs.orders.clear();
    qs.tails.clear();
    qs.natail = 0;
    qs.has_leaf = false;
    if (!memo.p) {
      // one slot per vertex (power of two), 2^21..2^25 words: 32 MB at C2, 256 MB at C4
      size_t words = size_t(1) << 21;
      while (words < g.V && words < (size_t(1) << 25)) words <<= 1;
      memo.ensure(words);
      memo_fill.ensure(1);
      memo_bits.ensure(std::max<size_t>((size_t(g.V) + 31) / 32, 1));
      refresh_graph_view();
      reset_memo();
    }
    std::vector<EdgeProg> progs;
    std::vector<AnchorEdge> anchors;
    std::vector<LeafSig> leafsigs;
    std::vector<std::pair<uint32_t, uint32_t>> ranges(qs.q.n);
    std::vector<uint32_t> classes(qs.q.n);
    for (uint32_t u = 0; u < qs.q.n; ++u) {
      ranges[u] = label_range(qs.q.labels[u]);
      classes[u] = label_class(qs.q.labels[u]);
    }
    for (uint32_t e = 0; e < qs.q.edges.size(); ++e) {
      qs.orders.push_back(matching_order(qs.q, e, cs));
      progs.push_back(build_program(qs.q, uint32_t(qi), qs.orders.back(), ranges, classes));
      qs.tails.push_back(progs.back().tail);
      qs.natail = std::max(qs.natail, progs.back().natail);
      const EdgeProg& ep = progs.back();
      for (uint32_t t = 0; t < ep.n; ++t) {
        if (!(((ep.leafmask | ep.singlemask) >> t) & 1u)) continue;
        bool seen = false;
        for (const LeafSig& ls : leafsigs) seen |= ls.sig == ep.sig[t];
        if (seen) continue;
        const uint32_t pq = ep.order[(ep.leafmask >> t) & 1u ? ep.tail : ep.lv[t].back[0]];
        LeafSig ls{};
        ls.sig = ep.sig[t];
        ls.pbit = 1u << pq;
        ls.plo = ranges[pq].first;
        ls.phi = ranges[pq].second;
        ls.leaf = ep.lv[t];
        leafsigs.push_back(ls);
      }
      const QEdge& qe = qs.q.edges[e];
      anchors.push_back({qs.q.labels[qe.a], qs.q.labels[qe.b], qe.label, e, {1u, 1u}});
    }
    // exact coalesced search (bdsm_options.coalesce): the same programs, one
    // anchored orientation per orbit of directed query edges, weighted by the
    // orbit size
    std::vector<AnchorEdge> anchors_co = anchors;
    {
      const std::vector<uint32_t> mult = directed_edge_orbits(qs.q);
      uint32_t searched = 0;
      for (size_t e = 0; e < anchors_co.size(); ++e) {
        anchors_co[e].mult[0] = mult[2 * e];
        anchors_co[e].mult[1] = mult[2 * e + 1];
        searched += (mult[2 * e] != 0) + (mult[2 * e + 1] != 0);
      }
      qs.coalesce_gain = searched ? uint32_t(2 * anchors_co.size() / searched) : 1;
    }
    qs.has_leaf = !leafsigs.empty();
    qs.n_leafsig = uint32_t(leafsigs.size());
    // the query's memo signatures, for the merge's invalidations; new orders
    // mean new signatures, so the memo starts over
    if (leafsigs.size() > sizeof(qs.denc.sig) / sizeof(qs.denc.sig[0])) memo_persistent = false;
    qs.denc.nsig = uint32_t(std::min<size_t>(leafsigs.size(), sizeof(qs.denc.sig) / sizeof(qs.denc.sig[0])));
    for (uint32_t k = 0; k < qs.denc.nsig; ++k) qs.denc.sig[k] = leafsigs[k].sig;
    reset_memo();
    qs.leafsigs.ensure(std::max<size_t>(leafsigs.size(), 1));
    if (!leafsigs.empty())
      CK(cudaMemcpyAsync(qs.leafsigs.p, leafsigs.data(), sizeof(LeafSig) * leafsigs.size(), cudaMemcpyHostToDevice,
                         stream));
    qs.progs.ensure(std::max<size_t>(progs.size(), 1));
    qs.anchors.ensure(std::max<size_t>(anchors.size(), 1));
    qs.anchors_co.ensure(std::max<size_t>(anchors.size(), 1));
    if (!progs.empty()) {
      CK(cudaMemcpyAsync(qs.progs.p, progs.data(), sizeof(EdgeProg) * progs.size(), cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(qs.anchors.p, anchors.data(), sizeof(AnchorEdge) * anchors.size(),
                         cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(qs.anchors_co.p, anchors_co.data(), sizeof(AnchorEdge) * anchors_co.size(),
                         cudaMemcpyHostToDevice, stream));
    }
    sync();
  }

  void upload_query_tables() {
    size_t nq = queries.size();
    std::vector<DevQueryEnc> enc(nq);
    std::vector<uint32_t*> rows(nq);
    std::vector<uint64_t*> cols(nq);
    for (size_t i = 0; i < nq; ++i) {
      enc[i] = queries[i]->denc;
      rows[i] = queries[i]->rows.p;
      cols[i] = queries[i]->colsize.p;
    }
    d_qenc.ensure(nq);
    d_rows.ensure(nq);
    d_colsize.ensure(nq);
    CK(cudaMemcpyAsync(d_qenc.p, enc.data(), sizeof(DevQueryEnc) * nq, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_rows.p, rows.data(), sizeof(uint32_t*) * nq, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_colsize.p, cols.data(), sizeof(uint64_t*) * nq, cudaMemcpyHostToDevice, stream));
    sync();
  }


  // --------------------------------------------------------------- batches --
  size_t cub_bytes_for(size_t n) {
    size_t m = 2 * n, a = 0, b = 0, c = 0, d = 0, e = 0;
    cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, int(m), 0, 64, stream));
    CK(cub::DeviceSelect::Flagged(nullptr, b, cub::CountingInputIterator<uint32_t>(0), (uint8_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, int(m), stream));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, int(m + 1), stream));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, d, (uint64_t*)nullptr, (uint64_t*)nullptr, int(n + 1), stream));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, e, (uint32_t*)nullptr, (uint32_t*)nullptr, int(n + 1), stream));
    size_t f = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, f, (AnchorCount*)nullptr, (AnchorCount*)nullptr, AnchorCountSum(),
                                      AnchorCount{0, 0, 0}, int(n + 1), stream));
    return std::max({a, b, c, d, e, f});
  }

  void ensure_batch(size_t n) {
    if (n <= B().batch_cap) return;
    size_t cap_n = std::max<size_t>(n, B().batch_cap + B().batch_cap / 2);
    cap_n = std::max<size_t>(cap_n, 1024);
    size_t m = 2 * cap_n;
    B().ups.ensure(cap_n);
    B().ups_ext.ensure(cap_n);
    B().keys.ensure(m);
    B().keys2.ensure(m);
    B().skeys.ensure(m);
    B().vals.ensure(m);
    B().vals2.ensure(m);
    B().svals.ensure(m);
    B().dlab.ensure(cap_n);
    B().ecode.ensure(cap_n);
    B().head.ensure(m);
    B().insflag.ensure(m + 1);
    B().ins_prefix.ensure(m + 1);
    B().heads.ensure(m);
    B().ipos.ensure(m);
    B().new_off.ensure(m);
    B().new_cap.ensure(m);
    B().big_list.ensure(m);
    B().small_list.ensure(m);
    B().mid_list.ensure(m);
    B().upd_cnt.ensure(cap_n + 1);
    B().upd_off.ensure(cap_n + 1);
    cub_tmp.ensure(cub_bytes_for(cap_n));
    size_t hcap = 1024;
    while (hcap < 8 * cap_n) hcap <<= 1;  // >= 2x the 2|dB| directed keys + <= 2|dB| segment heads
    B().hkeys.ensure(hcap);
    B().hvals.ensure(hcap);
    B().batch_cap = cap_n;
  }

  void ensure_tasks(size_t n) {
    size_t maxq_edges = 1;
    for (auto& q : queries) maxq_edges = std::max(maxq_edges, q->q.edges.size());
    B().tasks.ensure_grow(std::max<size_t>(n * 2 * maxq_edges, 1024));
    // BDSM_MAX_ITEMS (tests): a small initial work-item capacity, so the
    // regrowth and rerun paths run on small inputs
    if (max_items == 0) max_items = env_u32("BDSM_MAX_ITEMS", 0);
    if (max_items == 0) max_items = std::max<size_t>(B().tasks.n * 4, size_t(1) << 22);
    if (B().items.n < max_items) B().items.ensure(max_items);
    if (!dyn.p) {
      qstate.ensure(1);
      dyn.ensure(size_t(1) << 20);  // 80 MiB of donated subtrees per launch
      dyn_ready.ensure(dyn.n);
      CK(cudaMemsetAsync(dyn_ready.p, 0, 4 * dyn_ready.n, stream));
    }
  }

  void ensure_host_ups(size_t n) {
    if (n <= h_ups_cap) return;
    if (h_ups) cudaFreeHost(h_ups);
    size_t c = std::max<size_t>(n, h_ups_cap * 2);
    CK(cudaMallocHost(&h_ups, c * sizeof(bdsm_update)));
    h_ups_cap = c;
  }

  PhaseArgs phase_args(uint32_t n, uint32_t phase, int qi) {
    QueryState& qs = *queries[size_t(qi)];
    PhaseArgs a{};
    a.g = view();
    a.ups = B().ups.p;
    a.n_ups = n;
    a.dlab = B().dlab.p;
    // materialised matches (--dump-matches) need every anchored orientation
    a.anchors = opts.coalesce && !collect_cap ? qs.anchors_co.p : qs.anchors.p;
    a.n_anchor = uint32_t(qs.q.edges.size());
    a.progs = qs.progs.p;
    a.rows = qs.rows.p;
    a.skeys = B().skeys.p;
    a.svals = B().svals.p;
    a.m_keys = 2 * n;
    a.hkeys = B().hkeys.p;
    a.hvals = B().hvals.p;
    a.hmask = uint32_t(B().hkeys.n - 1);
    a.phase = phase;
    a.flag = phase == 0 ? row_del_flag(cs) : row_ins_flag(cs);
    a.query = uint32_t(qi);
    a.qn = qs.q.n;
    a.chunk = opts.chunk;
    a.shard_rank = opts.shard_rank;
    a.shard_world = std::max<uint32_t>(opts.shard_world, 1);
    a.upd_cnt = B().upd_cnt.p;
    a.upd_off = B().upd_off.p;
    a.tasks = B().tasks.p;
    a.items = B().items.p;
    a.max_items = uint32_t(std::min<size_t>(max_items, 0xffffffffu));
    a.st = B().d_st;
    a.count_out = st_counts(B().d_st) + size_t(phase) * queries.size() + size_t(qi);
    a.timed_out = st_timed(B().d_st) + qi;
    a.deadline_ns = 0;
    a.q = qstate.p;
    a.dyn = dyn.p;
    a.dyn_ready = dyn_ready.p;
    a.dyn_cap = uint32_t(dyn.n);
    a.merge_ratio = tune_merge_ratio;
    a.backoff_max = tune_backoff;
    a.memo = memo.p;
    a.memo_mask = uint32_t(memo.n - 1);
    a.memo_fill = memo_fill.p;
    a.heads = B().heads.p;
    a.task_tail = nullptr;
    a.natail_stride = qs_natail(qi);
    a.match_out = nullptr;
    a.match_count = nullptr;
    a.match_cap = 0;
    return a;
  }

  void run_phase(uint32_t n, uint32_t phase) {
    Nvtx range(phase == 0 ? "bdsm negative phase" : "bdsm positive phase");
    for (size_t qi = 0; qi < queries.size(); ++qi) {
      QueryState& qs = *queries[qi];
      if (!qs.active || qs.q.edges.empty()) continue;
      PhaseArgs a = phase_args(n, phase, int(qi));
      // positive phase, warm memo: the touched hubs' weights are refilled on
      // the side stream while the anchors are counted and emitted
      const bool side_prefill = phase == 1 && qs.q.n > 2 && qs.has_leaf && !collect_cap && memo_persistent &&
                                !qs.memo_cold && qs.n_leafsig;
      if (side_prefill) {
        CK(cudaEventRecord(fork_ev, stream));
        CK(cudaStreamWaitEvent(side, fork_ev, 0));
        launch_leaf_prefill(a, qs.leafsigs.p, qs.n_leafsig, nullptr, nullptr, num_sms, side);
        CK(cudaEventRecord(join_ev, side));
        ++launches;
      }
      if (qs.deadline_s > 0) {
        // device %globaltimer is in ns since an arbitrary epoch: express the
        // deadline relative to "now" on both clocks via a calibration kernel
        // would be exact; the host steady clock offset is applied instead.
        a.deadline_ns = device_deadline(qs.deadline_s);
      }
      if (phase == 0 && early_anchors) {  // issued on the side stream by launch_attempt
        CK(cudaStreamWaitEvent(stream, join_ev, 0));
      } else {
        launch_anchor_count(a, stream);
        a.self_scan = n <= tune_self_scan;
        if (!a.self_scan) {
          size_t tmp = cub_tmp.n;
          CK(cub::DeviceScan::ExclusiveScan(cub_tmp.p, tmp, B().upd_cnt.p, B().upd_off.p, AnchorCountSum(),
                                            AnchorCount{0, 0, 0}, int(n + 1), stream));
          cub_calls += 1;
        }
        if (!(collect_cap && qs.q.n <= 2)) launch_anchor_emit(a, stream);
        // fresh work queues for this launch (next_item, dyn_head, dyn_tail, busy, idle)
        CK(cudaMemsetAsync(qstate.p, 0, sizeof(QueueState), stream));
      }
      a.epoch = ++epoch;
      launches += 2;
      if (collect_cap) {  // --dump-matches: materialise this (query, phase)'s matches
        qs.mbuf[phase].ensure(collect_cap * qs.q.n);
        qs.mcount.ensure(2);
        CK(cudaMemsetAsync(qs.mcount.p + phase, 0, sizeof(unsigned long long), stream));
        a.match_out = qs.mbuf[phase].p;
        a.match_count = qs.mcount.p + phase;
        a.match_cap = collect_cap;
      }
      if (qs.q.n <= 2 && collect_cap) launch_anchor_emit(a, stream);  // 2-vertex matches are the anchors
      if (qs.q.n > 2) {
        CK(cudaEventRecord(next_kev(), stream));
        if (qs.has_leaf && !collect_cap) {
          // persistent memo: a full prefill over the hub list after a reset,
          // then only the batch's touched vertices (the merge invalidated
          // their weights) before the positive phase
          if (!memo_persistent) {
            CK(cudaMemsetAsync(memo.p, 0xff, sizeof(unsigned long long) * memo.n, stream));
            qs.memo_cold = true;
          }
          if (qs.memo_cold) {
            refresh_hubs();
            launch_leaf_prefill(a, qs.leafsigs.p, qs.n_leafsig, hub_ids.p, n_hubs.p, num_sms, stream);
            qs.memo_cold = false;
            ++launches;
          } else if (side_prefill) {
            CK(cudaStreamWaitEvent(stream, join_ev, 0));
          } else if (phase == 1) {
            launch_leaf_prefill(a, qs.leafsigs.p, qs.n_leafsig, nullptr, nullptr, num_sms, stream);
            ++launches;
          }
        }
        if (qs.natail && !tune_no_tasktail) {  // per-task counts of anchor-only tail levels, unset (~0) before the launch
          B().task_tail.ensure_grow(B().tasks.n * qs.natail);
          CK(cudaMemsetAsync(B().task_tail.p, 0xff, sizeof(unsigned long long) * B().tasks.n * qs.natail, stream));
          a.task_tail = B().task_tail.p;
        }
        // variant by the previous batch's work items of this (query, phase)
        const int variant = variant_for(qs.prev_items[phase]);
        a.backoff_max = tune_backoff ? tune_backoff : variant == 2 ? 256u : 1024u;
        launch_wbm(a, nullptr, num_sms, variant, stream);
        CK(cudaEventRecord(next_kev(), stream));
        ++launches;
      }
    }
  }

  // %globaltimer and the host steady clock differ by an offset measured once.
  int64_t gt_offset = 0;
  bool gt_calibrated = false;
  uint64_t device_deadline(double deadline_s);

  BatchState template_state() {
    BatchState s{};
    s.trace[0][5] = s.trace[1][5] = ~0ull;
    s.selfloop_min = kNone;
    s.conflict_min = kNone;
    s.pool_top = pool_top;
    return s;
  }

  // One batch in flight per engine: submit enqueues it (H2D, every phase) and
  // returns; wait synchronises once, handles reruns and reports.  apply() is
  // the two back to back; the pipelined API (bdsm_engine_submit_batch /
  // bdsm_engine_wait) lets the caller prepare the next batch meanwhile.
  struct Pending {
    bool active = false;
    size_t n = 0;
    bool device_input = false;
    const bdsm_update_dev* src = nullptr;
    std::chrono::steady_clock::time_point t0;
    bdsm_batch_stats st{};
    uint32_t compactions = 0;
    uint32_t reruns = 0;  // positive-phase reruns (work items regrown after the merge)
    int attempt = 0;
    bool full_sort = false;  // rerun with the 64-bit key sort (an id beyond the sorted bits)
  };
  Pending pend;

  void launch_attempt() {
    Nvtx range("bdsm batch");
    const size_t n = pend.n;
    const bool device_input = pend.device_input;
    const bdsm_update_dev* src = pend.src;
    kev_used = 0;
    launches = 0;
    cub_calls = 0;
    // ms_device spans every attempt of the batch (first attempt's start to the
    // last event of the last attempt or rerun), host-side regrowth included
    if (pend.attempt == 0) CK(cudaEventRecord(ev[0], stream));
    if (!device_input) {
      CK(cudaMemcpyAsync(B().ups_ext.p, h_src, n * sizeof(bdsm_update), cudaMemcpyHostToDevice, stream));
      pend.st.h2d_bytes = n * sizeof(bdsm_update);
    }
    std::memset(static_cast<void*>(B().h_st), 0, B().st_bytes);
    *B().h_st = template_state();
    CK(cudaMemcpyAsync(B().d_st, B().h_st, B().st_bytes, cudaMemcpyHostToDevice, stream));
    const uint32_t m = uint32_t(2 * n);
    const uint32_t nq = uint32_t(queries.size());
    if (pend.attempt == 0) hot_pack_maybe();
    // the sort orders the source id's significant bits only (+ the full
    // destination word); larger (invalid) ids rerun with all 64 bits
    const uint32_t id_bits = g.V > 1 ? 32u - uint32_t(__builtin_clz(g.V - 1)) : 1u;
    const bool full_sort = pend.full_sort || id_bits >= 32;
    const uint32_t key_bits = full_sort ? 32u : id_bits;  // both ids packed into 2 x id_bits
    const int sort_end_bit = full_sort ? 64 : int(2 * id_bits);
    launch_prepare(src, uint32_t(n), view(), d_new_of.p, B().ups.p, B().d_st, B().keys.p, B().vals.p, B().dlab.p, B().ecode.p,
                   full_sort ? 0xffffffffu : (1u << id_bits), key_bits, stream);
    // one query, small batch: the negative phase's anchors need only the
    // translated updates and G, so they are counted and emitted on the side
    // stream while the keys are sorted (joined before the matching kernel)
    early_anchors = false;
    if (queries.size() == 1 && n <= tune_self_scan && !collect_cap && queries[0]->active &&
        !queries[0]->q.edges.empty()) {
      PhaseArgs a = phase_args(uint32_t(n), 0, 0);
      a.self_scan = 1;
      CK(cudaEventRecord(fork_ev, stream));
      CK(cudaStreamWaitEvent(side, fork_ev, 0));
      launch_anchor_count(a, side);
      launch_anchor_emit(a, side);
      CK(cudaMemsetAsync(qstate.p, 0, sizeof(QueueState), side));
      CK(cudaEventRecord(join_ev, side));
      early_anchors = true;
    }
    // the sort ping-pongs between keys/keys2 (vals/vals2); k_post_sort
    // widens its output into skeys/svals, which every later kernel reads
    cub::DoubleBuffer<uint64_t> kb(B().keys.p, B().keys2.p);
    cub::DoubleBuffer<uint32_t> vb(B().vals.p, B().vals2.p);
    {
      size_t tmp = cub_tmp.n;
      CK(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tmp, kb, vb, int(m), 0, sort_end_bit, stream));
    }
    CK(cudaMemsetAsync(B().hkeys.p, 0xff, sizeof(unsigned long long) * B().hkeys.n, stream));
    launch_post_sort(kb.Current(), vb.Current(), key_bits, B().skeys.p, B().svals.p, m, B().d_st, B().head.p, B().insflag.p, d_rows.p,
                     nq, g.V, B().hkeys.p, B().hvals.p, uint32_t(B().hkeys.n - 1), cs, stream);
    {
      // the merge's insert prefix is only needed after the negative phase: it
      // is scanned on the side stream (own temporary storage) meanwhile
      CK(cudaEventRecord(fork2_ev, stream));
      CK(cudaStreamWaitEvent(side, fork2_ev, 0));
      size_t tmp = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, B().insflag.p, B().ins_prefix.p, int(m + 1), side));
      cub_tmp_side.ensure(tmp);
      tmp = cub_tmp_side.n;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp_side.p, tmp, B().insflag.p, B().ins_prefix.p, int(m + 1), side));
      CK(cudaEventRecord(join2_ev, side));
      tmp = cub_tmp.n;
      CK(cub::DeviceSelect::Flagged(cub_tmp.p, tmp, cub::CountingInputIterator<uint32_t>(0), B().head.p, B().heads.p,
                                    &B().d_st->n_touched, int(m), stream));
    }
    CK(cudaEventRecord(ev[1], stream));
    run_phase(uint32_t(n), 0);
    CK(cudaEventRecord(ev[2], stream));
    CK(cudaStreamWaitEvent(stream, join2_ev, 0));
    cudaEvent_t m0 = merge_ev[0], m1 = merge_ev[1];
    CK(cudaEventRecord(m0, stream));
    const bool small_ok = m >= tune_small_min;
    launch_alloc(B().heads.p, B().skeys.p, B().ins_prefix.p, m, view(), opts.slack, B().d_st, B().new_off.p, B().new_cap.p, B().big_list.p,
                 B().small_list.p, B().mid_list.p, small_max(m), big_min(m), stream);
    launch_merge_refresh(B().heads.p, B().skeys.p, B().svals.p, B().ins_prefix.p, m, B().ups.p, g, B().new_off.p, B().new_cap.p, B().ipos.p,
                         d_qenc.p, uint32_t(queries.size()), d_rows.p, d_colsize.p, B().d_st, memo.p,
                         uint32_t(memo.n ? memo.n - 1 : 0), B().big_list.p, B().small_list.p, B().mid_list.p,
                         small_max(m) ? small_group(m) : 0u, num_sms, stream, fork_big());
    join_big();
    CK(cudaEventRecord(m1, stream));
    launches += small_ok ? 7 : 6;  // prepare, post_sort, alloc, merge_refresh, [merge_small,] merge_big, finish_big
    cub_calls += 3; // sort, select, scan
    CK(cudaEventRecord(ev[3], stream));
    run_phase(uint32_t(n), 1);
    if (opts.l2_hot_mb) {  // K8 estimator: walks from this batch's touched vertices
      heat.ensure(g.V);
      if (!heat_init) {
        CK(cudaMemsetAsync(heat.p, 0, 4ull * g.V, stream));
        heat_init = true;
      }
      launch_hot_walks(B().heads.p, B().skeys.p, B().d_st, view(), heat.p, 4, 3, uint32_t(batches_done), num_sms, stream);
      ++launches;
    }
    launch_clear_flags(B().skeys.p, m, d_rows.p, nq, g.V, cs, stream);
    ++launches;
    CK(cudaEventRecord(ev[4], stream));
    CK(cudaMemcpyAsync(B().h_st, B().d_st, B().st_bytes, cudaMemcpyDeviceToHost, stream));
    if (memo.p) {
      if (!h_memo_fill) CK(cudaMallocHost(&h_memo_fill, sizeof(unsigned long long)));
      CK(cudaMemcpyAsync(h_memo_fill, memo_fill.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    }
    CK(cudaEventRecord(ev[5], stream));
  }

  void relaunch() {
    if (++pend.attempt > 8) throw std::runtime_error("batch could not be scheduled");
    launch_attempt();
  }

  // copy_host: always stage host updates through the engine's pinned buffer
  // (the caller may reuse its buffer as soon as submit returns)
  void submit(const bdsm_update* updates, size_t n, bool device_input, bool copy_host) {
    if (pend.active) throw std::invalid_argument("a batch is already in flight on this engine (wait for it first)");
    pend = Pending{};
    pend.t0 = std::chrono::steady_clock::now();
    last_errors.clear();
    pend.n = n;
    pend.device_input = device_input;
    if (n >= (size_t(1) << 31)) throw std::invalid_argument("batch too large");
    if (n == 0) {
      pend.active = true;
      return;
    }
    // (a labelled insert into an unlabelled graph is detected by k_prepare:
    // overflow 4 enables the label array and reruns the batch)
    ensure_batch(n);
    ensure_tasks(n);
    ensure_state();
    if (!ev[0]) {
      for (auto& e : ev) CK(cudaEventCreate(&e));
      for (auto& e : merge_ev) CK(cudaEventCreate(&e));
    }
    const bdsm_update_dev* src;
    if (device_input) {
      src = reinterpret_cast<const bdsm_update_dev*>(updates);
    } else {
      // pinned (page-locked) caller buffers are DMAed directly; pageable ones
      // are staged through the engine's pinned buffer first
      cudaPointerAttributes pa{};
      const bool pinned = cudaPointerGetAttributes(&pa, updates) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      cudaGetLastError();  // clear a pageable-pointer query error, if any
      if (pinned && !copy_host) {
        h_src = updates;
      } else {
        ensure_host_ups(n);
        std::memcpy(h_ups, updates, n * sizeof(bdsm_update));
        h_src = h_ups;
      }
      src = B().ups_ext.p;
    }
    pend.src = src;
    launch_attempt();
    pend.active = true;
  }

  bdsm_status wait(uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats) {
    if (!pend.active) throw std::invalid_argument("no batch in flight on this engine");
    struct Done {
      Pending& p;
      ~Done() { p.active = false; }
    } done{pend};
    for (size_t qi = 0; qi < queries.size(); ++qi) {
      if (pos) pos[qi] = 0;
      if (neg) neg[qi] = 0;
    }
    if (pend.n == 0) {
      if (stats) *stats = pend.st;
      return BDSM_OK;
    }
    const size_t n = pend.n;
    const bool device_input = pend.device_input;
    const bdsm_update_dev* src = pend.src;
    for (;;) {
      sync();
      const BatchState& b = *B().h_st;
      // the hot-list arena (K8) is reserved even when the batch is then rejected
      // (overflow 1 = pool exhausted: the compaction below re-lays the pool)
      if (b.pool_top > pool_top && b.overflow != 1) pool_top = b.pool_top;
      if (b.overflow == 5) {  // an id beyond the sorted bits (an invalid batch): exact errors need the full sort
        pend.full_sort = true;
        relaunch();
        continue;
      }
      if (b.selfloop_min != kNone || b.conflict_min != kNone) {
        bdsm_update bad{};
        uint32_t idx = std::min(b.selfloop_min, b.conflict_min);
        fetch_update(src, device_input, idx, &bad);
        if (b.selfloop_min <= b.conflict_min)
          throw std::invalid_argument("self-loop update (" + std::to_string(bad.u) + "," +
                                      std::to_string(bad.v) + ")");
        throw std::invalid_argument("conflicting updates on edge (" + std::to_string(bad.u) + "," +
                                    std::to_string(bad.v) + ") within one batch");
      }
      if (b.err_count) {
        std::vector<uint8_t> codes(n);
        CK(cudaMemcpyAsync(codes.data(), B().ecode.p, n, cudaMemcpyDeviceToHost, stream));
        sync();
        for (size_t i = 0; i < n; ++i)
          if (codes[i]) last_errors.push_back({uint64_t(i), codes[i]});
        throw BatchRejected("batch rejected: " + std::to_string(last_errors.size()) +
                            " invalid update(s), none applied");
      }
      if (b.overflow == 4) {  // labelled insert into an unlabelled graph: nothing merged
        enable_edge_labels();
        relaunch();
        continue;
      }
      if (b.overflow == 1) {  // adjacency pool exhausted: nothing merged yet
        compact(b.pool_top > g.pool_size ? b.pool_top - pool_top : 0);
        ++pend.compactions;
        relaunch();
        continue;
      }
      if (b.overflow == 2) {  // negative-phase work items: regrow, rerun all
        max_items = std::max<size_t>(max_items * 2, size_t(b.n_items[0]) + 1024);
        B().items.ensure(max_items);
        relaunch();
        continue;
      }
      if (b.overflow == 3) {  // positive phase only (graph already merged)
        max_items = std::max<size_t>(max_items * 2, size_t(b.n_items[1]) + 1024);
        B().items.ensure(max_items);
        rerun_positive(uint32_t(n));
      }
      break;
    }
    const BatchState& b = *B().h_st;
    pool_top = b.pool_top;
    ++batches_done;
    for (auto& q : queries) {  // BatchState keeps the last query's item counts per phase
      q->prev_items[0] = b.n_items[0];
      q->prev_items[1] = b.n_items[1];
    }
    // start the memo over before its probes run out (fill read with the batch's final copy)
    if (memo.p && h_memo_fill && *h_memo_fill > memo.n * 2 / 5) reset_memo();
    // a query whose deadline fired has its counts of this batch dropped
    // (MatchStats::timed_out, src/scheduler.cpp:101-110); whether it stays
    // matched in later batches is the caller's decision (set_query_active),
    // as in run_pipeline (src/bench.cpp:420-432)
    const unsigned long long* cnt = st_counts(B().h_st);
    const uint32_t* tmo = st_timed(B().h_st);
    uint32_t tmask = 0;
    last_timed.assign(queries.size(), 0);
    for (size_t qi = 0; qi < queries.size(); ++qi) {
      const bool dead = tmo[qi] != 0;
      last_timed[qi] = dead;
      if (dead && qi < 32) tmask |= 1u << qi;
      if (neg) neg[qi] = dead ? 0 : cnt[qi];
      if (pos) pos[qi] = dead ? 0 : cnt[queries.size() + qi];
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[0], ev[5]);
    pend.st.ms_device = ms;
    cudaEventElapsedTime(&ms, ev[1], ev[2]);
    pend.st.ms_negative = ms;
    cudaEventElapsedTime(&ms, ev[2], ev[3]);
    pend.st.ms_update = ms;
    cudaEventElapsedTime(&ms, ev[3], ev[4]);
    pend.st.ms_positive = ms;
    double mk = 0;
    for (size_t i = 0; i + 1 < kev_used; i += 2) {
      cudaEventElapsedTime(&ms, kev[i], kev[i + 1]);
      mk += ms;
    }
    pend.st.ms_match_kernel = mk;
    cudaEventElapsedTime(&ms, merge_ev[0], merge_ev[1]);
    pend.st.ms_merge_kernel = ms;
    pend.st.kernel_launches = launches;
    pend.st.cub_launches = cub_calls;
    pend.st.dfs_visits = b.visits;
    pend.st.tasks = b.tasks_total;
    pend.st.work_items = uint64_t(b.n_items[0]) + b.n_items[1];
    pend.st.gen_calls = b.gen_calls;
    pend.st.bytes_phase = b.bytes_phase;
    pend.st.bytes_kernel = b.bytes_kernel;
    pend.st.bytes_update = b.bytes_update + 16ull * n;
    pend.st.touched = b.n_touched;
    pend.st.relocations = b.relocations;
    pend.st.compactions = pend.compactions;
    pend.st.attempts = uint32_t(pend.attempt + 1);
    pend.st.reruns = pend.reruns;
    pend.st.timed_out = tmask;
    pend.st.d2h_bytes = B().st_bytes;
    pend.st.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pend.t0).count();
    if (stats) *stats = pend.st;
    return BDSM_OK;
  }

  bdsm_status apply(const bdsm_update* updates, size_t n, bool device_input, uint64_t* pos, uint64_t* neg,
                    bdsm_batch_stats* stats) {
    submit(updates, n, device_input, false);
    return wait(pos, neg, stats);
  }

  // Positive-phase work items overflowed after the merge: grow and rerun that
  // phase alone (the graph is already G').
  void rerun_positive(uint32_t n) {
    B().h_st->overflow = 0;
    for (size_t qi = 0; qi < queries.size(); ++qi) st_counts(B().h_st)[queries.size() + qi] = 0;
    CK(cudaMemcpyAsync(B().d_st, B().h_st, B().st_bytes, cudaMemcpyHostToDevice, stream));
    const uint32_t m = 2 * n, nq = uint32_t(queries.size());
    // the batch-endpoint row flags were cleared at the end of the attempt
    CK(cudaMemsetAsync(B().hkeys.p, 0xff, sizeof(unsigned long long) * B().hkeys.n, stream));
    launch_post_sort(B().skeys.p, B().svals.p, 32, nullptr, nullptr, m, B().d_st, B().head.p, B().insflag.p, d_rows.p, nq, g.V,
                     B().hkeys.p, B().hvals.p, uint32_t(B().hkeys.n - 1), cs, stream);
    run_phase(n, 1);
    launch_clear_flags(B().skeys.p, m, d_rows.p, nq, g.V, cs, stream);
    CK(cudaMemcpyAsync(B().h_st, B().d_st, B().st_bytes, cudaMemcpyDeviceToHost, stream));
    CK(cudaEventRecord(ev[5], stream));
    ++pend.reruns;
    sync();
    if (B().h_st->overflow) throw std::runtime_error("positive phase could not be scheduled");
  }

  // ------------------------------------------------------------- stream --
  // Pipelined stream (run_pipeline's stage overlap, src/bench.cpp:495-545,
  // taken onto the device).  The positive phase of batch i and the negative
  // phase of batch i+1 both read the graph after batch i's merge, so they run
  // as ONE launch of the matching kernel (k_wbm with two phases): the idle
  // warps of one phase's long tail take the other's items.  Batch buffers
  // alternate between two slots; each batch's BatchState points at its
  // predecessor's, so a batch that has to be rerun (pool or work-item
  // regrowth) or is rejected stops every later batch of the stream on the
  // device (overflow 6).  Per device order:
  //   front(0) neg(0) | merge(i) front(i+1) [pos(i) + neg(i+1)] flags(i) D2H(i) | ...
  // The host then reports the batches before the first abnormal one, handles
  // that one through the single-batch path (reruns, exact errors) and resumes.
  struct StreamBatch {
    const bdsm_update* src = nullptr;  // host or device updates
    size_t n = 0;
  };
  unsigned char* h_stream = nullptr;  // pinned: per batch a template and a result area
  size_t h_stream_bytes = 0;
  std::vector<cudaEvent_t> stream_ev;
  std::vector<cudaEvent_t> stream_kev;  // pairs around each matching launch, then each merge
  size_t stream_kev_used = 0;
  cudaEvent_t next_skev() {
    if (stream_kev_used == stream_kev.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      stream_kev.push_back(e);
    }
    return stream_kev[stream_kev_used++];
  }
  std::vector<std::pair<size_t, size_t>> seg_match_ev, seg_merge_ev;  // per batch: first/last kev index
  cudaEvent_t front_ev[2] = {nullptr, nullptr};  // front A of the batch in slot s done (side stream)

  bool stream_ok() const {
    if (collect_cap || opts.l2_hot_mb) return false;
    for (const auto& q : queries)
      if (q->deadline_s > 0) return false;
    return !queries.empty();
  }

  // Front part A of a batch on slot cs, on stream `st` (the side stream while
  // the previous batch merges): H2D, state template, the graph-independent
  // half of K1, key sort, post-sort (conflicts, heads, visibility table),
  // insert prefix, segment heads.  Part B (stream_validate) follows the
  // previous batch's merge on the main stream.
  void stream_front(const StreamBatch& sb, bool device_input, BatchState* prev, unsigned char* h_tmpl,
                    cudaStream_t st, DBuf<uint8_t>& tmp_buf) {
    Nvtx range("bdsm front");
    const size_t n = sb.n;
    ensure_batch(n);
    ensure_tasks(n);
    ensure_state();
    const bdsm_update_dev* src = reinterpret_cast<const bdsm_update_dev*>(sb.src);
    if (!device_input) {
      CK(cudaMemcpyAsync(B().ups_ext.p, sb.src, n * sizeof(bdsm_update), cudaMemcpyHostToDevice, st));
      src = B().ups_ext.p;
    }
    std::memset(h_tmpl, 0, B().st_bytes);
    BatchState t = template_state();
    t.prev = prev;
    std::memcpy(h_tmpl, &t, sizeof(t));
    CK(cudaMemcpyAsync(B().d_st, h_tmpl, B().st_bytes, cudaMemcpyHostToDevice, st));
    const uint32_t m = uint32_t(2 * n);
    const uint32_t id_bits = g.V > 1 ? 32u - uint32_t(__builtin_clz(g.V - 1)) : 1u;
    const bool full_sort = id_bits >= 32;
    const uint32_t key_bits = full_sort ? 32u : id_bits;
    const int sort_end_bit = full_sort ? 64 : int(2 * id_bits);
    launch_translate(src, uint32_t(n), g.V, has_elab, d_new_of.p, B().ups.p, B().d_st, B().keys.p, B().vals.p,
                     B().ecode.p, full_sort ? 0xffffffffu : (1u << id_bits), key_bits, st);
    cub::DoubleBuffer<uint64_t> kb(B().keys.p, B().keys2.p);
    cub::DoubleBuffer<uint32_t> vb(B().vals.p, B().vals2.p);
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, int(m), 0, sort_end_bit, st));
    tmp_buf.ensure(std::max(tmp, cub_bytes_for(n)));
    tmp = tmp_buf.n;
    CK(cub::DeviceRadixSort::SortPairs(tmp_buf.p, tmp, kb, vb, int(m), 0, sort_end_bit, st));
    CK(cudaMemsetAsync(B().hkeys.p, 0xff, sizeof(unsigned long long) * B().hkeys.n, st));
    launch_post_sort(kb.Current(), vb.Current(), key_bits, B().skeys.p, B().svals.p, m, B().d_st, B().head.p,
                     B().insflag.p, nullptr, 0, g.V, B().hkeys.p, B().hvals.p, uint32_t(B().hkeys.n - 1), cs, st);
    tmp = tmp_buf.n;
    CK(cub::DeviceScan::ExclusiveSum(tmp_buf.p, tmp, B().insflag.p, B().ins_prefix.p, int(m + 1), st));
    tmp = tmp_buf.n;
    CK(cub::DeviceSelect::Flagged(tmp_buf.p, tmp, cub::CountingInputIterator<uint32_t>(0), B().head.p, B().heads.p,
                                  &B().d_st->n_touched, int(m), st));
    launches += 2;
    cub_calls += 3;
  }

  // Front part B (main stream, after the previous batch's merge): presence in
  // G, pre-batch labels of deletes, batch-endpoint row flags, pool pointer.
  void stream_validate(size_t n, cudaStream_t st) {
    launch_validate(B().ups.p, uint32_t(n), view(), B().d_st, B().dlab.p, B().ecode.p, d_rows.p,
                    uint32_t(queries.size()), cs, st);
    ++launches;
  }

  // K3 + K4 of the batch on slot cs.
  void stream_merge(size_t n) {
    Nvtx range("bdsm merge");
    const uint32_t m = uint32_t(2 * n);
    const bool small_ok = m >= tune_small_min;
    launch_alloc(B().heads.p, B().skeys.p, B().ins_prefix.p, m, view(), opts.slack, B().d_st, B().new_off.p,
                 B().new_cap.p, B().big_list.p, B().small_list.p, B().mid_list.p, small_max(m), big_min(m),
                 stream);
    launch_merge_refresh(B().heads.p, B().skeys.p, B().svals.p, B().ins_prefix.p, m, B().ups.p, g, B().new_off.p,
                         B().new_cap.p, B().ipos.p, d_qenc.p, uint32_t(queries.size()), d_rows.p, d_colsize.p, B().d_st,
                         memo.p, uint32_t(memo.n ? memo.n - 1 : 0), B().big_list.p, B().small_list.p, B().mid_list.p,
                         small_max(m) ? small_group(m) : 0u, num_sms, stream, fork_big());
    join_big();
    launches += small_ok ? 5 : 4;
  }

  // Anchors (K5), work queues and memo prefill of (phase, query) for the
  // batch on slot cs; the launch itself is left to the caller.
  // st / tmp: the stream and CUB scratch to use (the next batch's negative
  // anchors run on side_big beside this batch's positive anchors)
  PhaseArgs stream_phase(uint32_t n, uint32_t phase, int qi, cudaStream_t st, DBuf<uint8_t>& tmp_buf) {
    QueryState& qs = *queries[size_t(qi)];
    PhaseArgs a = phase_args(n, phase, qi);
    launch_anchor_count(a, st);
    a.self_scan = n <= tune_self_scan;
    if (!a.self_scan) {
      size_t tmp = 0;
      CK(cub::DeviceScan::ExclusiveScan(nullptr, tmp, B().upd_cnt.p, B().upd_off.p, AnchorCountSum(),
                                        AnchorCount{0, 0, 0}, int(n + 1), st));
      tmp_buf.ensure(tmp);
      tmp = tmp_buf.n;
      CK(cub::DeviceScan::ExclusiveScan(tmp_buf.p, tmp, B().upd_cnt.p, B().upd_off.p, AnchorCountSum(),
                                        AnchorCount{0, 0, 0}, int(n + 1), st));
      cub_calls += 1;
    }
    launch_anchor_emit(a, st);
    launches += 2;
    if (qs.q.n > 2 && qs.has_leaf) {
      if (!memo_persistent) {
        CK(cudaMemsetAsync(memo.p, 0xff, sizeof(unsigned long long) * memo.n, st));
        qs.memo_cold = true;
      }
      if (qs.memo_cold) {
        refresh_hubs();
        launch_leaf_prefill(a, qs.leafsigs.p, qs.n_leafsig, hub_ids.p, n_hubs.p, num_sms, st);
        qs.memo_cold = false;
        ++launches;
      } else if (phase == 1) {
        launch_leaf_prefill(a, qs.leafsigs.p, qs.n_leafsig, nullptr, nullptr, num_sms, st);
        ++launches;
      }
    }
    if (qs.q.n > 2 && qs.natail && !tune_no_tasktail) {
      B().task_tail.ensure_grow(B().tasks.n * qs.natail);
      CK(cudaMemsetAsync(B().task_tail.p, 0xff, sizeof(unsigned long long) * B().tasks.n * qs.natail, st));
      a.task_tail = B().task_tail.p;
    }
    return a;
  }

  // One launch of the matching kernel for up to two phases of one query.
  void stream_launch(const PhaseArgs* a, const PhaseArgs* b, int qi) {
    QueryState& qs = *queries[size_t(qi)];
    if (qs.q.n <= 2) return;  // 2-vertex matches were counted by the anchors
    CK(cudaMemsetAsync(qstate.p, 0, sizeof(QueueState), stream));
    const PhaseArgs& first = a ? *a : *b;
    PhaseArgs x = first;
    x.epoch = ++epoch;
    const uint32_t items = std::max(qs.prev_items[0], qs.prev_items[1]);
    const int variant = variant_for(items);
    x.backoff_max = tune_backoff ? tune_backoff : variant == 2 ? 256u : 1024u;
    CK(cudaEventRecord(next_skev(), stream));
    launch_wbm(x, a && b ? b : nullptr, num_sms, variant, stream);
    CK(cudaEventRecord(next_skev(), stream));
    ++launches;
  }

  // Enqueues batches [i0, k) and waits; returns the first batch whose state is
  // abnormal (k if none).  Results of the batches before it are in h_res(i).
  size_t stream_segment(const StreamBatch* bs, size_t i0, size_t k, bool device_input) {
    Nvtx range("bdsm stream segment");
    const size_t nq = queries.size();
    const size_t sb = st_size();
    const size_t need = 2 * sb * std::max<size_t>(k - i0, 64);  // room for 64 batches up front
    if (h_stream_bytes < need) {
      if (h_stream) cudaFreeHost(h_stream);
      h_stream = nullptr;
      CK(cudaMallocHost(&h_stream, need));
      h_stream_bytes = need;
    }
    for (auto& fe : front_ev)
      if (!fe) CK(cudaEventCreateWithFlags(&fe, cudaEventDisableTiming));
    while (stream_ev.size() < k - i0 + 1) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      stream_ev.push_back(e);
    }
    auto h_tmpl = [&](size_t i) { return h_stream + 2 * sb * (i - i0); };
    auto h_res = [&](size_t i) { return h_stream + 2 * sb * (i - i0) + sb; };
    launches = 0;
    cub_calls = 0;
    stream_kev_used = 0;
    seg_match_ev.assign(k - i0, {0, 0});
    seg_merge_ev.assign(k - i0, {0, 0});
    CK(cudaEventRecord(stream_ev[0], stream));
    cs = 0;
    stream_front(bs[i0], device_input, nullptr, h_tmpl(i0), stream, cub_tmp);
    stream_validate(bs[i0].n, stream);
    // front A of the second batch on the side stream (its slot is free)
    if (i0 + 1 < k) {
      CK(cudaEventRecord(fork_ev, stream));
      CK(cudaStreamWaitEvent(side, fork_ev, 0));
      cs = 1;
      stream_front(bs[i0 + 1], device_input, slot_[0].d_st, h_tmpl(i0 + 1), side, cub_tmp_side);
      CK(cudaEventRecord(front_ev[1], side));
      cs = 0;
    }
    seg_match_ev[0].first = stream_kev_used;
    for (size_t qi = 0; qi < nq; ++qi) {
      if (!queries[qi]->active || queries[qi]->q.edges.empty()) continue;
      PhaseArgs an = stream_phase(uint32_t(bs[i0].n), 0, int(qi), stream, cub_tmp);
      stream_launch(nullptr, &an, int(qi));
    }
    for (size_t i = i0; i < k; ++i) {
      const uint32_t s = uint32_t((i - i0) & 1), t = s ^ 1u;
      cs = s;
      seg_merge_ev[i - i0].first = stream_kev_used;
      CK(cudaEventRecord(next_skev(), stream));
      stream_merge(bs[i].n);
      CK(cudaEventRecord(next_skev(), stream));
      seg_merge_ev[i - i0].second = stream_kev_used;
      // batch i+1's validation and negative anchors on side_big, beside batch
      // i's positive anchors and prefill on the main stream (both read the
      // merged graph; the memo's cold start stays on the main stream).  Per
      // query, as the slots' task and item buffers are shared by the queries.
      bool cold = !memo_persistent;
      for (const auto& q : queries) cold = cold || q->memo_cold;
      cudaStream_t nst = cold ? stream : side_big;
      const bool next = i + 1 < k;
      if (next) {  // front B of batch i+1 (its front A ran on the side stream)
        cs = t;
        if (nst != stream) {
          CK(cudaEventRecord(big_fork_ev, stream));
          CK(cudaStreamWaitEvent(nst, big_fork_ev, 0));
        }
        CK(cudaStreamWaitEvent(nst, front_ev[t], 0));
        stream_validate(bs[i + 1].n, nst);
      }
      if (i > i0) seg_match_ev[i - i0].first = stream_kev_used;
      bool first_q = true;
      for (size_t qi = 0; qi < nq; ++qi) {
        if (!queries[qi]->active || queries[qi]->q.edges.empty()) continue;
        PhaseArgs an{};
        if (next) {
          cs = t;
          if (nst != stream && !first_q) {  // the previous query's launch has read the buffers
            CK(cudaEventRecord(big_fork_ev, stream));
            CK(cudaStreamWaitEvent(nst, big_fork_ev, 0));
          }
          an = stream_phase(uint32_t(bs[i + 1].n), 0, int(qi), nst, nst == stream ? cub_tmp : cub_tmp_big);
          if (nst != stream) CK(cudaEventRecord(big_join_ev, nst));
        }
        cs = s;
        PhaseArgs ap = stream_phase(uint32_t(bs[i].n), 1, int(qi), stream, cub_tmp);
        if (next && nst != stream) CK(cudaStreamWaitEvent(stream, big_join_ev, 0));
        stream_launch(&ap, next ? &an : nullptr, int(qi));
        first_q = false;
      }
      seg_match_ev[i - i0].second = stream_kev_used;
      cs = s;
      launch_clear_flags(B().skeys.p, uint32_t(2 * bs[i].n), d_rows.p, uint32_t(nq), g.V, s, stream,
                         i + 1 < k ? slot_[t].d_st : nullptr);
      ++launches;
      CK(cudaMemcpyAsync(h_res(i), B().d_st, sb, cudaMemcpyDeviceToHost, stream));
      CK(cudaEventRecord(stream_ev[i - i0 + 1], stream));
      // slot s is free again: front A of batch i+2 on the side stream, beside
      // batch i+1's merge
      if (i + 2 < k) {
        CK(cudaStreamWaitEvent(side, stream_ev[i - i0 + 1], 0));
        cs = s;
        stream_front(bs[i + 2], device_input, slot_[t].d_st, h_tmpl(i + 2), side, cub_tmp_side);
        CK(cudaEventRecord(front_ev[s], side));
      }
    }
    if (memo.p) {
      if (!h_memo_fill) CK(cudaMallocHost(&h_memo_fill, sizeof(unsigned long long)));
      CK(cudaMemcpyAsync(h_memo_fill, memo_fill.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    }
    sync();
    cs = 0;
    for (size_t i = i0; i < k; ++i) {
      const BatchState& b = *reinterpret_cast<const BatchState*>(h_res(i));
      if (b.err_count || b.selfloop_min != kNone || b.conflict_min != kNone || b.overflow) return i;
    }
    return k;
  }

  // Counts and stats of a batch from its result area (as wait() reports them).
  double kev_span(const std::pair<size_t, size_t>& r) {
    double t = 0;
    for (size_t e = r.first; e + 1 < r.second; e += 2) {
      float ms = 0;
      cudaEventElapsedTime(&ms, stream_kev[e], stream_kev[e + 1]);
      t += ms;
    }
    return t;
  }

  void stream_report(const unsigned char* res, size_t n, double ms, uint64_t* pos, uint64_t* neg,
                     bdsm_batch_stats* stats, double ms_match = 0, double ms_merge = 0) {
    const BatchState& b = *reinterpret_cast<const BatchState*>(res);
    const size_t nq = queries.size();
    const unsigned long long* cnt = reinterpret_cast<const unsigned long long*>(&b + 1);
    const uint32_t* tmo = reinterpret_cast<const uint32_t*>(cnt + 2 * nq);
    last_timed.assign(nq, 0);
    for (size_t qi = 0; qi < nq; ++qi) {
      last_timed[qi] = tmo[qi] != 0;
      if (neg) neg[qi] = tmo[qi] ? 0 : cnt[qi];
      if (pos) pos[qi] = tmo[qi] ? 0 : cnt[nq + qi];
    }
    pool_top = b.pool_top;
    ++batches_done;
    for (auto& q : queries) {
      q->prev_items[0] = b.n_items[0];
      q->prev_items[1] = b.n_items[1];
    }
    if (stats) {
      bdsm_batch_stats s{};
      s.ms_device = ms;
      s.dfs_visits = b.visits;
      s.tasks = b.tasks_total;
      s.work_items = uint64_t(b.n_items[0]) + b.n_items[1];
      s.gen_calls = b.gen_calls;
      s.bytes_phase = b.bytes_phase;
      s.bytes_kernel = b.bytes_kernel;
      s.bytes_update = b.bytes_update + 16ull * n;
      s.touched = b.n_touched;
      s.relocations = b.relocations;
      s.attempts = 1;
      s.d2h_bytes = st_size();
      s.kernel_launches = launches;
      s.cub_launches = cub_calls;
      // the matching launches after this batch's merge (its positive phase,
      // fused with the next batch's negative phase) and its merge kernels
      s.ms_match_kernel = ms_match;
      s.ms_merge_kernel = ms_merge;
      *stats = s;
    }
  }

  bdsm_status apply_stream(const StreamBatch* bs, size_t k, bool device_input, uint64_t* pos, uint64_t* neg,
                           bdsm_batch_stats* stats, size_t* done) {
    if (pend.active) throw std::invalid_argument("a batch is already in flight on this engine (wait for it first)");
    const size_t nq = queries.size();
    *done = 0;
    size_t i0 = 0;
    while (i0 < k) {
      if (!stream_ok() || k - i0 == 1) {  // one batch, or a mode the stream does not cover
        bdsm_batch_stats st{};
        apply(bs[i0].src, bs[i0].n, device_input, pos ? pos + i0 * nq : nullptr, neg ? neg + i0 * nq : nullptr,
              &st);
        if (stats) stats[i0] = st;
        *done = ++i0;
        continue;
      }
      for (size_t i = i0; i < k; ++i)
        if (bs[i].n == 0 || bs[i].n >= (size_t(1) << 31)) throw std::invalid_argument("stream batches must be non-empty");
      const auto t0 = std::chrono::steady_clock::now();
      const size_t j = stream_segment(bs, i0, k, device_input);
      const size_t sb = st_size();
      for (size_t i = i0; i < j; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, stream_ev[i - i0], stream_ev[i - i0 + 1]);
        stream_report(h_stream + 2 * sb * (i - i0) + sb, bs[i].n, ms, pos ? pos + i * nq : nullptr,
                      neg ? neg + i * nq : nullptr, stats ? stats + i : nullptr, kev_span(seg_match_ev[i - i0]),
                      kev_span(seg_merge_ev[i - i0]));
        if (stats) stats[i].ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *done = i + 1;
      }
      if (memo.p && h_memo_fill && *h_memo_fill > memo.n * 2 / 5) reset_memo();
      if (j == k) break;
      // batch j needs the single-batch path: a positive-phase regrowth on the
      // merged graph, or a full rerun / exact error report on the graph before it
      const BatchState& b = *reinterpret_cast<const BatchState*>(h_stream + 2 * sb * (j - i0) + sb);
      if (b.overflow == 3 && !b.err_count && b.selfloop_min == kNone && b.conflict_min == kNone) {
        cs = uint32_t((j - i0) & 1);
        pend = Pending{};
        pend.n = bs[j].n;
        std::memcpy(static_cast<void*>(B().h_st), &b, sb);
        B().h_st->prev = nullptr;  // its predecessor is final; the slot behind it was reused
        max_items = std::max<size_t>(max_items * 2, size_t(b.n_items[1]) + 1024);
        B().items.ensure(max_items);
        rerun_positive(uint32_t(bs[j].n));
        stream_report(reinterpret_cast<const unsigned char*>(B().h_st), bs[j].n, 0.0, pos ? pos + j * nq : nullptr,
                      neg ? neg + j * nq : nullptr, stats ? stats + j : nullptr);
        if (stats) stats[j].reruns = pend.reruns;
        cs = 0;
      } else {
        // nothing of batch j was merged: rerun it alone (throws its error)
        bdsm_batch_stats st{};
        apply(bs[j].src, bs[j].n, device_input, pos ? pos + j * nq : nullptr, neg ? neg + j * nq : nullptr, &st);
        if (stats) stats[j] = st;
      }
      *done = j + 1;
      i0 = j + 1;
    }
    return BDSM_OK;
  }

  void fetch_update(const bdsm_update_dev* src, bool device_input, uint32_t idx, bdsm_update* out) {
    if (!device_input) {
      *out = h_src[idx];
      return;
    }
    CK(cudaMemcpyAsync(out, src + idx, sizeof(bdsm_update), cudaMemcpyDeviceToHost, stream));
    sync();
  }
};

namespace {
__global__ void k_read_globaltimer(uint64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace

// %globaltimer and the host steady clock differ by an offset, measured once
// with a one-thread kernel bracketed by host clock reads.
uint64_t bdsm_engine::device_deadline(double deadline_s) {
  if (!gt_calibrated) {
    DBuf<uint64_t> t;
    t.ensure(1);
    uint64_t h0 = now_ns();
    k_read_globaltimer<<<1, 1, 0, stream>>>(t.p);
    uint64_t gt = 0;
    CK(cudaMemcpyAsync(&gt, t.p, 8, cudaMemcpyDeviceToHost, stream));
    sync();
    uint64_t h1 = now_ns();
    gt_offset = int64_t(gt) - int64_t((h0 + h1) / 2);
    gt_calibrated = true;
  }
  int64_t host_deadline = int64_t(deadline_s * 1e9);
  int64_t dev = host_deadline + gt_offset;
  return dev <= 1 ? 1 : uint64_t(dev);
}

// ------------------------------------------------------------------ C ABI --

namespace {

bdsm_status fail(bdsm_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

template <typename F>
bdsm_status guarded(F&& f) {
  try {
    return f();
  } catch (const BatchRejected& e) {
    return fail(BDSM_BATCH_ERROR, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(BDSM_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return fail(BDSM_INVALID_ARGUMENT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(BDSM_OUT_OF_MEMORY, "out of device or host memory");
  } catch (const CudaFailure& e) {
    return fail(BDSM_CUDA_ERROR, e.what());
  } catch (const std::exception& e) {
    return fail(BDSM_RUNTIME_ERROR, e.what());
  }
}

}  // namespace

extern "C" {

const char* bdsm_version(void) { return "bdsm_b200 0.1 (sm_100a)"; }

const char* bdsm_last_error(void) { return g_last_error.c_str(); }

// group.cpp's failures (not exported)
void bdsm_internal_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

bdsm_status bdsm_engine_create(const bdsm_graph_desc* graph, const bdsm_options* opts, bdsm_engine** out) {
  if (!out) return fail(BDSM_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  return guarded([&]() -> bdsm_status {
    if (!graph) throw std::invalid_argument("null graph");
    auto e = std::make_unique<bdsm_engine>();
    bdsm_options o{};
    o.group_bits = 2;
    o.slack = 0.25f;
    o.pool_reserve = 0.5f;
    o.chunk = 32;
    o.shard_world = 1;
    if (opts) {
      o = *opts;
      if (o.group_bits == 0) o.group_bits = 2;
      if (o.slack <= 0) o.slack = 0.25f;
      if (o.pool_reserve <= 0) o.pool_reserve = 0.5f;
      if (o.chunk == 0) o.chunk = 32;
      if (o.shard_world == 0) o.shard_world = 1;
    }
    if (o.shard_rank >= o.shard_world) throw std::invalid_argument("shard_rank must be < shard_world");
    if (o.chunk % 8 != 0) throw std::invalid_argument("chunk must be a multiple of 8");
    e->opts = o;
    // zero-copy tier (north_star item 4): the adjacency pool in mapped pinned
    // host memory, for graphs whose lists exceed one GPU's HBM
    e->adj.mapped = e->elab.mapped = o.zero_copy != 0;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev == 0) throw CudaFailure("no CUDA device");
    e->device = o.device;
    CK(cudaSetDevice(e->device));
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->side_big, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&e->big_fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->big_join_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->join_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->fork2_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->join2_ev, cudaEventDisableTiming));
    CK(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, e->device));
    e->build(graph);
    *out = e.release();
    return BDSM_OK;
  });
}

void bdsm_engine_destroy(bdsm_engine* engine) { delete engine; }

int bdsm_engine_add_query(bdsm_engine* engine, const bdsm_query_desc* query) {
  if (!engine) return -int(fail(BDSM_INVALID_ARGUMENT, "null engine"));
  int idx = -1;
  bdsm_status s = guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    idx = engine->add_query(query);
    return BDSM_OK;
  });
  return s == BDSM_OK ? idx : -int(s);
}

bdsm_status bdsm_engine_apply_batch(bdsm_engine* engine, const bdsm_update* updates, size_t n, uint64_t* pos,
                                    uint64_t* neg, bdsm_batch_stats* stats) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  if (n && !updates) return fail(BDSM_INVALID_ARGUMENT, "null updates");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    return engine->apply(updates, n, false, pos, neg, stats);
  });
}

bdsm_status bdsm_engine_apply_batch_device(bdsm_engine* engine, const bdsm_update* d_updates, size_t n,
                                           uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  if (n && !d_updates) return fail(BDSM_INVALID_ARGUMENT, "null updates");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    return engine->apply(d_updates, n, true, pos, neg, stats);
  });
}

bdsm_status bdsm_engine_apply_stream(bdsm_engine* engine, const bdsm_update* const* batches, const size_t* sizes,
                                     size_t k, int device_input, uint64_t* pos, uint64_t* neg,
                                     bdsm_batch_stats* stats, size_t* done) {
  size_t dummy = 0;
  if (!done) done = &dummy;
  *done = 0;
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  if (k && (!batches || !sizes)) return fail(BDSM_INVALID_ARGUMENT, "null batches");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    std::vector<bdsm_engine::StreamBatch> bs(k);
    for (size_t i = 0; i < k; ++i) {
      if (sizes[i] && !batches[i]) throw std::invalid_argument("null updates");
      bs[i].src = batches[i];
      bs[i].n = sizes[i];
    }
    return engine->apply_stream(bs.data(), k, device_input != 0, pos, neg, stats, done);
  });
}

bdsm_status bdsm_engine_submit_batch(bdsm_engine* engine, const bdsm_update* updates, size_t n) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  if (n && !updates) return fail(BDSM_INVALID_ARGUMENT, "null updates");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    engine->submit(updates, n, false, true);
    return BDSM_OK;
  });
}

bdsm_status bdsm_engine_wait(bdsm_engine* engine, uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    return engine->wait(pos, neg, stats);
  });
}

bdsm_status bdsm_engine_set_deadline(bdsm_engine* engine, int query, double seconds_from_now) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    QueryState& qs = *engine->queries.at(size_t(query));
    qs.deadline_s = seconds_from_now > 0 ? double(now_ns()) * 1e-9 + seconds_from_now : 0;
    return BDSM_OK;
  });
}

bdsm_status bdsm_engine_set_query_active(bdsm_engine* engine, int query, int active) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    if (engine->pend.active) throw std::invalid_argument("a batch is in flight on this engine (wait for it first)");
    engine->queries.at(size_t(query))->active = active != 0;
    return BDSM_OK;
  });
}

int bdsm_engine_query_timed_out(bdsm_engine* engine, int query) {
  if (!engine) return -int(fail(BDSM_INVALID_ARGUMENT, "null engine"));
  if (query < 0 || size_t(query) >= engine->queries.size())
    return -int(fail(BDSM_INVALID_ARGUMENT, "query index out of range"));
  return size_t(query) < engine->last_timed.size() ? int(engine->last_timed[size_t(query)]) : 0;
}

size_t bdsm_last_batch_errors(bdsm_engine* engine, bdsm_update_error* out, size_t cap) {
  if (!engine) return 0;
  size_t n = std::min(cap, engine->last_errors.size());
  if (out)
    for (size_t i = 0; i < n; ++i) out[i] = engine->last_errors[i];
  return engine->last_errors.size();
}

size_t bdsm_engine_debug_trace(bdsm_engine* engine, uint64_t* out, size_t cap) {
  if (!engine || !engine->slot_[0].h_st) return 0;
  const BatchState* hs = engine->slot_[0].h_st;
  const size_t n = (sizeof(hs->trace) + sizeof(hs->trace_chunks) + sizeof(hs->trace_setups)) / sizeof(uint64_t);
  const uint64_t* t = &hs->trace[0][0];
  for (size_t i = 0; i < n && i < cap; ++i) out[i] = t[i];
  return n;
}

size_t bdsm_engine_neighbors(bdsm_engine* engine, uint32_t v, uint32_t* out, size_t cap) {
  if (!engine || v >= engine->g.V) return 0;
  size_t d = 0;
  guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    const uint32_t iv = engine->new_of[v];
    uint32_t dv = 0;
    uint64_t o = 0;
    CK(cudaMemcpyAsync(&dv, engine->deg.p + iv, 4, cudaMemcpyDeviceToHost, engine->stream));
    CK(cudaMemcpyAsync(&o, engine->off.p + iv, 8, cudaMemcpyDeviceToHost, engine->stream));
    engine->sync();
    d = dv;
    if (out && cap) {
      std::vector<uint32_t> lst(dv);
      CK(cudaMemcpyAsync(lst.data(), engine->adj.p + o, 4ull * dv, cudaMemcpyDeviceToHost, engine->stream));
      engine->sync();
      for (auto& x : lst) x = engine->old_of[x];  // external ids, ascending (LabeledGraph::neighbors)
      std::sort(lst.begin(), lst.end());
      std::copy(lst.begin(), lst.begin() + std::min<size_t>(cap, dv), out);
    }
    return BDSM_OK;
  });
  return d;
}

bdsm_status bdsm_engine_rows(bdsm_engine* engine, int query, uint32_t* out) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    QueryState& qs = *engine->queries.at(size_t(query));
    std::vector<uint32_t> rows(engine->g.V);
    CK(cudaMemcpyAsync(rows.data(), qs.rows.p, 4ull * engine->g.V, cudaMemcpyDeviceToHost, engine->stream));
    engine->sync();
    for (uint32_t v = 0; v < engine->g.V; ++v) out[v] = rows[engine->new_of[v]] & ~kRowFlags;
    return BDSM_OK;
  });
}

bdsm_status bdsm_engine_collect_matches(bdsm_engine* engine, uint64_t cap) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  engine->collect_cap = cap;
  return BDSM_OK;
}

int64_t bdsm_engine_matches(bdsm_engine* engine, int query, int phase, uint32_t* out, size_t cap) {
  if (!engine || query < 0 || size_t(query) >= engine->queries.size() || phase < 0 || phase > 1)
    return -int64_t(BDSM_INVALID_ARGUMENT);
  int64_t r = 0;
  bdsm_status st = guarded([&] {
    std::vector<uint32_t> m;
    const size_t cnt = engine->fetch_matches(query, phase, m);
    const uint32_t n = engine->queries[size_t(query)]->q.n;
    const size_t have = n ? m.size() / n : 0;
    if (out) std::copy_n(m.begin(), std::min(have, cap) * n, out);
    r = int64_t(cnt);
    return BDSM_OK;
  });
  return st == BDSM_OK ? r : -int64_t(st);
}

int bdsm_plan_order(const bdsm_query_desc* query, const uint64_t* column_sizes, uint32_t edge, uint32_t* order,
                    uint32_t* tail) {
  int r = -int(BDSM_INVALID_ARGUMENT);
  bdsm_status st = guarded([&]() -> bdsm_status {
    if (!query || !column_sizes || !order) throw std::invalid_argument("null argument");
    std::vector<uint32_t> labels(query->vertex_labels, query->vertex_labels + query->num_vertices);
    std::vector<QEdge> edges;
    for (uint32_t i = 0; i < query->num_edges; ++i)
      edges.push_back({query->a[i], query->b[i], query->edge_labels ? query->edge_labels[i] : kNone});
    HostQuery q(std::move(labels), std::move(edges));
    if (!q.connected()) throw std::invalid_argument("disconnected query graph");
    if (edge >= q.edges.size()) throw std::invalid_argument("query edge out of range");
    std::vector<uint64_t> cs(column_sizes, column_sizes + q.n);
    const std::vector<uint32_t> o = matching_order(q, edge, cs);
    for (size_t i = 0; i < o.size(); ++i) order[i] = o[i];
    if (tail) {
      std::vector<std::pair<uint32_t, uint32_t>> ranges(q.n, {0, 0});
      std::vector<uint32_t> classes(q.n, kNone);
      *tail = q.n <= uint32_t(kMaxQ) ? build_program(q, 0, o, ranges, classes).tail : 0;
    }
    r = int(o.size());
    return BDSM_OK;
  });
  return st == BDSM_OK ? r : -int(st);
}

int64_t bdsm_plan_edge_orbits(const bdsm_query_desc* query, uint32_t* mult) {
  int64_t r = -int64_t(BDSM_INVALID_ARGUMENT);
  bdsm_status st = guarded([&]() -> bdsm_status {
    if (!query || !mult) throw std::invalid_argument("null argument");
    std::vector<uint32_t> labels(query->vertex_labels, query->vertex_labels + query->num_vertices);
    std::vector<QEdge> edges;
    for (uint32_t i = 0; i < query->num_edges; ++i)
      edges.push_back({query->a[i], query->b[i], query->edge_labels ? query->edge_labels[i] : kNone});
    HostQuery q(std::move(labels), std::move(edges));
    const std::vector<uint32_t> m = directed_edge_orbits(q);
    std::copy(m.begin(), m.end(), mult);
    std::vector<std::vector<uint32_t>> autos;
    r = automorphisms(q, 20000, autos) ? int64_t(autos.size()) : 0;
    return BDSM_OK;
  });
  return st == BDSM_OK ? r : -int64_t(st);
}

int bdsm_engine_tail(bdsm_engine* engine, int query, uint32_t edge) {
  if (!engine || query < 0 || size_t(query) >= engine->queries.size()) return -int(BDSM_INVALID_ARGUMENT);
  QueryState& qs = *engine->queries[size_t(query)];
  if (edge >= qs.tails.size()) return -int(BDSM_INVALID_ARGUMENT);
  return int(qs.tails[edge]);
}

int bdsm_engine_order(bdsm_engine* engine, int query, uint32_t edge, uint32_t* out) {
  if (!engine || query < 0 || size_t(query) >= engine->queries.size()) return -int(BDSM_INVALID_ARGUMENT);
  QueryState& qs = *engine->queries[size_t(query)];
  if (edge >= qs.orders.size()) return -int(BDSM_INVALID_ARGUMENT);
  const auto& o = qs.orders[edge];
  for (size_t i = 0; i < o.size(); ++i) out[i] = o[i];
  return int(o.size());
}

bdsm_status bdsm_engine_column_sizes(bdsm_engine* engine, int query, uint64_t* out) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    auto cs = engine->column_sizes(query);
    std::copy(cs.begin(), cs.end(), out);
    return BDSM_OK;
  });
}

bdsm_status bdsm_engine_replan(bdsm_engine* engine, int query) {
  if (!engine) return fail(BDSM_INVALID_ARGUMENT, "null engine");
  return guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    engine->replan(query);
    engine->upload_query_tables();
    return BDSM_OK;
  });
}

uint64_t bdsm_engine_num_edges(bdsm_engine* engine) {
  if (!engine) return 0;
  uint64_t total = 0;
  guarded([&]() -> bdsm_status {
    CK(cudaSetDevice(engine->device));
    std::vector<uint32_t> d(engine->g.V);
    CK(cudaMemcpyAsync(d.data(), engine->deg.p, 4ull * engine->g.V, cudaMemcpyDeviceToHost, engine->stream));
    engine->sync();
    for (uint32_t x : d) total += x;
    return BDSM_OK;
  });
  return total / 2;
}

uint32_t bdsm_engine_num_vertices(bdsm_engine* engine) { return engine ? engine->g.V : 0; }

void bdsm_shard_owners(const uint64_t* costs, size_t n, uint32_t world, uint32_t* owners) {
  shard_owners(costs, n, world, owners);
}

}  // extern "C"
