// Incremental matching kernels (north_star item 3).
//
// K5 anchors (map_update_to_query_edges + task construction, reference
// src/matcher.cpp:42-55, :334-354): every update of the phase's kind is mapped
// to each (query edge, orientation) whose labels fit; each anchor's level-2
// driver list is cut into fixed-size work items.  Two passes with an
// exclusive scan in between give a deterministic canonical order
// (update, edge, orientation, chunk), which is what the multi-GPU split
// needs.
//
// K6 wbm_count (run_match_task / gen_candidates / intersect_sorted /
// dedupe_by_order, src/matcher.cpp:59-117, :219-310; WorkerPool,
// src/scheduler.cpp): a persistent grid whose warps pop work items from a
// global queue.  One warp owns one partial match at a time and walks the DFS
// with its stack staged in shared memory: per level the warp streams the
// smallest backward neighbour's sorted list in 32-wide chunks (coalesced
// 128-byte loads), each lane filters its candidate — candidate-row bit,
// injectivity against same-label assigned vertices, membership in every other
// backward list by binary search, edge labels, and the lowest-order
// visibility rule — and the survivors form a ballot mask.  The last level is
// counted with popc and never materialised.  Candidates are never copied from
// the candidate column (the reference copies it per call, matcher.cpp:92).
#include "kernels.cuh"

#include <cub/cub.cuh>

namespace bdsm_b200 {

namespace {

__device__ __forceinline__ uint32_t lb_u32(const uint32_t* __restrict__ a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t lb_u64(const uint64_t* __restrict__ a, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool batch_aborted(const BatchState* st) {
  return st->err_count || st->selfloop_min != kNone || st->conflict_min != kNone || st->overflow;
}

// Level-2 driver of an anchor: the lower-degree backward neighbour of
// order[2] among the two anchor positions (ties: position 0).  Shared with
// the CPU restatement's shard rule (oracle/oracle.cpp driver_vertex).
__device__ __forceinline__ uint32_t level2_driver(const EdgeProg& p, uint32_t m0, uint32_t m1,
                                                  const DevGraph& g, uint32_t* pos) {
  uint32_t bm = p.lv[2].backmask;
  bool b0 = bm & 1u, b1 = (bm >> 1) & 1u;
  if (b0 && b1) {
    bool pick1 = g.deg[m1] < g.deg[m0];
    *pos = pick1 ? 1 : 0;
    return pick1 ? m1 : m0;
  }
  *pos = b0 ? 0 : 1;
  return b0 ? m0 : m1;
}

// Level-2 driver range of an anchor: the sub-range of the driver list holding
// order[2]'s label (ids are label-ordered, so it is contiguous).
__device__ __forceinline__ void level2_range(const EdgeProg& p, uint32_t m0, uint32_t m1, const DevGraph& g,
                                             uint32_t* base, uint32_t* len) {
  uint32_t pos;
  const uint32_t drv = level2_driver(p, m0, m1, g, &pos);
  const uint32_t* lst = g.adj + g.off[drv];
  const uint32_t d = g.deg[drv];
  const uint32_t lo = lb_u32(lst, d, p.lv[2].vlo);
  const uint32_t hi = p.lv[2].vhi > p.lv[2].vlo ? lb_u32(lst, d, p.lv[2].vhi) : lo;
  *base = lo;
  *len = hi - lo;
}

// Visits every anchor of update i in canonical order.
template <typename F>
__device__ __forceinline__ void for_each_anchor(const PhaseArgs& a, uint32_t i, F&& f) {
  bdsm_update_dev up = a.ups[i];
  if ((up.op != 0) != (a.phase == 0)) return;  // negative phase: deletes; positive: inserts
  uint32_t el = a.phase == 0 ? a.dlab[i] : up.elab;
  uint32_t lu = a.g.vlabel[up.u], lv = a.g.vlabel[up.v];
  for (uint32_t e = 0; e < a.n_anchor; ++e) {
    AnchorEdge ae = a.anchors[e];
    if (ae.elab != el) continue;
    if (ae.la == lu && ae.lb == lv) f(ae.prog, 0u, up);
    if (ae.la == lv && ae.lb == lu) f(ae.prog, 1u, up);
  }
}

__global__ void k_anchor_count(PhaseArgs a) {
  if (batch_aborted(a.st)) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= a.n_ups; i += gridDim.x * blockDim.x) {
    uint32_t nt = 0, ni = 0;
    uint64_t cost = 0;
    if (i < a.n_ups) {
      for_each_anchor(a, i, [&](uint32_t prog, uint32_t flip, const bdsm_update_dev& up) {
        ++nt;
        if (a.qn <= 2) {
          cost += 1;
          return;
        }
        const EdgeProg& p = a.progs[prog];
        uint32_t m0 = flip ? up.v : up.u, m1 = flip ? up.u : up.v, base, d;
        level2_range(p, m0, m1, a.g, &base, &d);
        ni += (d + a.chunk - 1) / a.chunk;
        cost += d;
      });
    }
    a.upd_task_counts[i] = nt;
    a.upd_counts[i] = ni;
    a.upd_cost[i] = cost;
  }
}

__global__ void k_anchor_emit(PhaseArgs a) {
  if (batch_aborted(a.st)) return;
  const uint64_t total_cost = a.cost_off[a.n_ups];
  const uint32_t total_items = a.item_off[a.n_ups];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.st->n_tasks[a.phase] = a.task_off[a.n_ups];
    a.st->n_items[a.phase] = total_items;
    atomicAdd((unsigned long long*)&a.st->tasks_total, (unsigned long long)a.task_off[a.n_ups]);
    if (total_items > a.max_items) a.st->overflow = a.phase == 0 ? 2 : 3;  // host regrows, reruns
  }
  if (total_items > a.max_items) return;
  uint64_t direct = 0;    // 2-vertex queries: every anchor is a match
  uint64_t bytes = 0, calls = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ups; i += gridDim.x * blockDim.x) {
    uint32_t t = a.task_off[i], it = a.item_off[i];
    uint64_t c = a.cost_off[i];
    for_each_anchor(a, i, [&](uint32_t prog, uint32_t flip, const bdsm_update_dev& up) {
      if (a.qn <= 2) {
        uint32_t owner = a.shard_world > 1 ? uint32_t((unsigned __int128)c * a.shard_world / total_cost) : 0;
        if (owner == a.shard_rank) ++direct;
        a.tasks[t++] = Task{i, prog, flip, 0, 0};
        c += 1;
        return;
      }
      const EdgeProg& p = a.progs[prog];
      uint32_t m0 = flip ? up.v : up.u, m1 = flip ? up.u : up.v, base, d;
      level2_range(p, m0, m1, a.g, &base, &d);
      a.tasks[t] = Task{i, prog, flip, d, base};
      // level-2 GenCandidates call of this anchor (SURVEY.md §8(d) B_phase)
      uint32_t bm = p.lv[2].backmask;
      if (bm & 1u) bytes += 4ull * a.g.deg[m0];
      if (bm & 2u) bytes += 4ull * a.g.deg[m1];
      ++calls;
      for (uint32_t b = 0; b < d; b += a.chunk) {
        uint32_t owner = a.shard_world > 1
                             ? uint32_t((unsigned __int128)(c + b) * a.shard_world / total_cost)
                             : 0;
        a.items[it++] = Item{owner == a.shard_rank ? t : kNone, b};
      }
      ++t;
      c += d;
    });
  }
  if (direct) atomicAdd((unsigned long long*)&a.st->counts[a.phase][a.query], (unsigned long long)direct);
  if (a.shard_rank == 0 && bytes) {
    atomicAdd((unsigned long long*)&a.st->bytes_phase, (unsigned long long)bytes);
    atomicAdd((unsigned long long*)&a.st->gen_calls, (unsigned long long)calls);
  }
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Is the data edge (x, c) a same-kind batch update with order < anchor?
// (dedupe_by_order, src/matcher.cpp:110-117, applied at generation time.)
__device__ __forceinline__ bool hidden_edge(const PhaseArgs& a, uint32_t x, uint32_t c, uint32_t anchor) {
  const unsigned long long key = (uint64_t(x) << 32) | c;
  uint32_t pos = pair_hash(key) & a.hmask;
  while (true) {  // linear probing; the table is at most half full
    const unsigned long long k = __ldg(a.hkeys + pos);
    if (k == key) {
      const uint32_t val = __ldg(a.hvals + pos);
      const bool is_del = val >> 31;
      return is_del == (a.phase == 0) && (val & 0x7fffffffu) < anchor;
    }
    if (k == kEmptyKey) return false;
    pos = (pos + 1) & a.hmask;
  }
}

__device__ __forceinline__ bool bit_set(const uint32_t* bits, uint32_t v) {
  return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Donated-subtree ticket queue (slots are used once per launch).  A reserved
// slot counts as a holder until the warp that takes it finishes.
__device__ __forceinline__ uint32_t dyn_reserve(QueueState* q, uint32_t cap) {
  uint32_t t = atomicAdd(&q->tt.tail, 1u);
  if (t >= cap) return kNone;  // full: keep the work (tail overshoot is harmless)
  atomicAdd(&q->holders.v, 1u);
  return t;
}

constexpr int kFloorB = 8;  // backward lists per level with a tracked search floor

// Membership of each lane's candidate c in the sorted list L[0, n), for
// lanes with `want` (their candidates ascend with the lane id, and exceed
// every candidate of earlier chunks).  Merge-path style: the warp walks
// 32-element windows of L from the floor `fl` with one coalesced load per
// window and resolves candidates by a 5-step shuffle search; `fl` ends at the
// last window, a valid floor for the next chunk.
__device__ __forceinline__ bool member_merge(const uint32_t* __restrict__ L, uint32_t n, uint32_t& fl,
                                             uint32_t c, bool want, uint32_t lane, uint32_t* pos) {
  bool found = false;
  bool pending = want;
  uint32_t f = fl;
  while (__any_sync(kFull, pending)) {
    if (f >= n) break;
    uint32_t i = f + lane;
    uint32_t w = i < n ? __ldg(L + i) : 0xffffffffu;
    uint32_t wmax = __shfl_sync(kFull, w, 31);
    uint32_t lo = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      uint32_t v = __shfl_sync(kFull, w, lo + step - 1);
      if (v < c) lo += step;
    }
    uint32_t wl = __shfl_sync(kFull, w, lo);
    if (pending && c <= wmax) {
      found = wl == c;
      *pos = f + lo;
      pending = false;
    }
    if (__any_sync(kFull, pending)) f += 32;
  }
  fl = f;
  return found;
}

// K6: persistent warp-per-partial-match DFS counter with work donation.
//
// Work sources, in order: static items (level-2 chunks of every anchor),
// then subtrees donated by busy warps.  A busy warp checks every few chunk
// fetches whether warps are idle and the donation queue is short; if so it
// gives away the upper half of the remaining driver range at its shallowest
// splittable level (the reference's active stealing takes the same share,
// src/scheduler.cpp:49-64, claim_upper_half), pushing its prefix assignment.
// Ranges are disjoint, so counts are exact regardless of scheduling.
// GenCandidates setup for a level (warp-collective): the driver is the
// smallest backward list (ties: lower position, as the reference's order of
// intersection does not matter for the result); every backward list's label
// sub-range [lo, hi) of label(order[l]) is found by one parallel round of
// binary searches (lanes 2b / 2b+1), lists of <= 32 entries keep their whole
// extent (the candidate-row label test filters them).  The sub-ranges seed the
// membership-search floors / ceilings.
struct LevelSetup {
  uint64_t drv_off;
  uint32_t drv_b, lo, hi, deg_sum;
};

__device__ __forceinline__ LevelSetup setup_level(const LevelProg& lp, const DevGraph& g, const uint32_t* M,
                                                  uint32_t lane, uint32_t* floor_l, uint32_t* ceil_l) {
  const uint32_t nb = lp.nback;
  uint32_t myd = 0xffffffffu;
  uint64_t myo = 0;
  if (lane < nb) {
    const uint32_t x = M[lp.back[lane]];
    myd = __ldg(g.deg + x);
    myo = __ldg(g.off + x);
  }
  const uint32_t mn = __reduce_min_sync(kFull, myd);
  LevelSetup s;
  s.drv_b = __ffs(__ballot_sync(kFull, myd == mn)) - 1;
  s.deg_sum = __reduce_add_sync(kFull, lane < nb ? myd : 0u);
  const uint32_t lb_list = (lane >> 1) & 31;
  const uint32_t bd = __shfl_sync(kFull, myd, lb_list);
  const uint64_t bo = __shfl_sync(kFull, myo, lb_list);
  uint32_t bnd = 0;
  if (lane < 2 * nb) {
    if (bd <= 32) bnd = (lane & 1) ? bd : 0u;
    else bnd = lb_u32(g.adj + bo, bd, (lane & 1) ? lp.vhi : lp.vlo);
  }
  const uint32_t f = __shfl_sync(kFull, bnd, (2 * lane) & 31);
  const uint32_t c = __shfl_sync(kFull, bnd, (2 * lane + 1) & 31);
  if (lane < nb && lane < kFloorB) {
    floor_l[lane] = f;
    ceil_l[lane] = c;
  }
  s.lo = __shfl_sync(kFull, bnd, 2 * s.drv_b);
  s.hi = __shfl_sync(kFull, bnd, 2 * s.drv_b + 1);
  s.drv_off = __shfl_sync(kFull, myo, s.drv_b);
  return s;
}

// One 32-candidate chunk [cur, end2) of level l's driver list: each lane
// filters its candidate c — candidate-row bit (CandidateTable::is_candidate),
// edge label, injectivity against same-label assigned positions, membership
// in every other backward list (intersect_sorted, src/matcher.cpp:59-73) and
// the lowest-order visibility rule (dedupe_by_order, :110-117) — and the
// survivors are returned as a ballot.  `tc`: c is a same-kind batch endpoint.
__device__ __forceinline__ uint32_t filter_chunk(const PhaseArgs& a, const LevelProg& lp, const uint32_t* M,
                                                 uint32_t* floor_l, const uint32_t* ceil_l, uint64_t c_off,
                                                 uint32_t cur, uint32_t end2, uint32_t dpos, uint32_t touched,
                                                 uint32_t anchor, uint32_t flag, uint32_t lane, uint32_t& c_out,
                                                 bool& tc_out) {
  const DevGraph& g = a.g;
  const uint32_t idx = cur + lane;
  bool ok = idx < end2;
  uint32_t c = 0xffffffffu;
  if (ok) c = __ldg(g.adj + c_off + idx);
  uint32_t rw = 0;
  if (ok) rw = __ldg(a.rows + c);  // candidate bits + batch-endpoint flags
  ok = ok && (rw & lp.qbit) != 0;
  if (ok && g.elab) ok = __ldg(g.elab + c_off + idx) == lp.elab[dpos];
  if (ok) {  // injectivity: only same-label positions can collide
    uint32_t eq = lp.eqmask;
    while (eq) {
      uint32_t j = __ffs(eq) - 1;
      eq &= eq - 1;
      if (M[j] == c) {
        ok = false;
        break;
      }
    }
  }
  const uint32_t remain = end2 - cur;  // driver entries left in this range
  for (uint32_t b = 0; b < lp.nback; ++b) {  // other backward lists
    if (b == dpos) continue;
    if (!__any_sync(kFull, ok)) break;
    const uint32_t x = M[lp.back[b]];
    const uint64_t xo = __ldg(g.off + x);
    const uint32_t xd = __ldg(g.deg + x);
    // search window: label sub-range [floor, ceil), the floor advancing
    // with the (ascending) driver chunks
    uint32_t fl = b < kFloorB ? floor_l[b] : 0;
    const uint32_t ce = b < kFloorB ? ceil_l[b] : xd;
    uint32_t p = 0;
    bool hit;
    // comparable lengths: merge windows; skewed: floor-bounded binary search
    if (uint64_t(ce - min(fl, ce)) <= uint64_t(a.merge_ratio) * remain) {
      hit = member_merge(g.adj + xo, ce, fl, c, ok, lane, &p);
    } else {
      hit = false;
      if (ok) {
        p = fl + lb_u32(g.adj + xo + fl, ce - fl, c);
        hit = p < ce && __ldg(g.adj + xo + p) == c;
      }
      uint32_t mp = __reduce_max_sync(kFull, ok ? p : 0u);
      if (mp > fl) fl = mp;
    }
    if (b < kFloorB && lane == 0) floor_l[b] = min(fl, ce);
    if (ok && g.elab && hit) hit = __ldg(g.elab + xo + p) == lp.elab[b];
    ok = ok && hit;
  }
  const bool tc = (rw & flag) != 0;
  if (ok && (touched & lp.backmask) && tc) {
    uint32_t tb = touched & lp.backmask;
    while (tb && ok) {
      uint32_t j = __ffs(tb) - 1;
      tb &= tb - 1;
      if (hidden_edge(a, M[j], c, anchor)) ok = false;
    }
  }
  c_out = c;
  tc_out = tc;
  return __ballot_sync(kFull, ok);
}

// Independent tail (EdgeProg::tail): levels T+1..n-1 have all their backward
// neighbours in the prefix M[0..T) and pairwise distinct labels, so given the
// prefix their candidate sets are independent and every level-T candidate
// roots the same subtree: Π_{t>T} |C_t| matches.  The reference enumerates
// that subtree per level-T candidate; here it is counted once per prefix and
// multiplied.  Also returns, per level-T candidate, the DFS visits
// (1 + Σ_k Π_{T<s<=k} |C_s|), GenCandidates calls and B_phase bytes the
// reference tree spends below it, so MatchStats-style
// counters stay those of the reference tree.
struct TailFactor {
  unsigned long long f, v, b, c;
};

__device__ __forceinline__ void tail_factor(const PhaseArgs& a, const EdgeProg& P, uint32_t T, uint32_t w,
                                            const uint32_t* M, uint32_t (*s_floor)[kMaxQ][kFloorB],
                                            uint32_t (*s_ceil)[kMaxQ][kFloorB], uint32_t touched, uint32_t anchor,
                                            uint32_t flag, uint32_t lane, TailFactor* out,
                                            unsigned long long* stat) {
  unsigned long long prod = 1, v = 1, b = 0, c = 0;
  for (uint32_t t = T + 1; t < P.n; ++t) {
    const LevelProg& lp = P.lv[t];
    const LevelSetup su = setup_level(lp, a.g, M, lane, s_floor[w][t], s_ceil[w][t]);
    __syncwarp();
    b += prod * 4ull * su.deg_sum;  // one call per visit at level t-1
    c += prod;
    if (lane == 0) stat[4] += 4ull * su.deg_sum;
    unsigned long long cnt = 0;
    for (uint32_t cur = su.lo; cur < su.hi; cur += 32) {
      uint32_t cc;
      bool tc;
      cnt += __popc(filter_chunk(a, lp, M, s_floor[w][t], s_ceil[w][t], su.drv_off, cur, su.hi, su.drv_b, touched,
                                 anchor, flag, lane, cc, tc));
      __syncwarp();
    }
    prod *= cnt;
    v += prod;
    if (prod == 0) break;  // the reference tree has no deeper nodes either
  }
  if (lane == 0) *out = TailFactor{prod, v, b, c};
  __syncwarp();
}

#ifndef BDSM_WBM_MIN_BLOCKS
#define BDSM_WBM_MIN_BLOCKS 4  // resident 256-thread CTAs per SM the register budget must allow
#endif
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BDSM_WBM_MIN_BLOCKS) k_wbm(PhaseArgs a) {
  __shared__ uint32_t s_cand[kWarpsPerBlock][kMaxQ][32];
  __shared__ uint32_t s_M[kWarpsPerBlock][kMaxQ];
  __shared__ uint32_t s_floor[kWarpsPerBlock][kMaxQ][kFloorB];
  __shared__ uint32_t s_ceil[kWarpsPerBlock][kMaxQ][kFloorB];
  __shared__ TailFactor s_tail[kWarpsPerBlock];
  // per-warp counters (lane 0 updates them; kept out of the register budget)
  __shared__ unsigned long long s_stat[kWarpsPerBlock][5];  // count, visits, bytes, calls, kernel bytes
  if (batch_aborted(a.st)) return;
  BatchState* st = a.st;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t n_items = st->n_items[a.phase];
  const DevGraph& g = a.g;
  unsigned long long* stat = s_stat[threadIdx.x >> 5];
  if ((threadIdx.x & 31) < 5) stat[threadIdx.x & 31] = 0;
  __syncwarp();
  uint32_t dtick = 0;
  bool timed_out = false;
  bool static_done = false;
  uint32_t ticket = kNone;  // lane 0: outstanding ticket of this warp

  // Lane-distributed per-level DFS state: lane l holds level l's.
  uint64_t r_off = 0;   // driver list offset
  uint32_t r_cur = 0;   // next driver index to fetch
  uint32_t r_end = 0;   // end of driver range
  uint32_t r_mask = 0;  // unexplored candidates of the current chunk
  uint32_t r_drv = 0;   // index of the driver in the level's backward list
  uint32_t r_tmask = 0; // current chunk: which candidates are same-kind batch endpoints
  const uint32_t flag = a.phase == 0 ? kRowDelFlag : kRowInsFlag;

  while (true) {
    // ---- acquire work ----------------------------------------------------
    uint32_t kind = 0, ref = 0;  // 1 static item, 2 donated item, 3 exit
    QueueState* Q = a.q;
    if (lane == 0) {
      // Static items first (counted as held before the index is taken, so a
      // waiter never sees holders == 0 while a static item is in flight).
      if (!static_done) {
        atomicAdd(&Q->holders.v, 1u);
        uint32_t idx = atomicAdd(&Q->next_item.v, 1u);
        if (idx < n_items) {
          kind = 1;
          ref = idx;
        } else {
          static_done = true;
          atomicSub(&Q->holders.v, 1u);
        }
      }
      if (!kind) {
        // Donated work: one ticket per idle period, then wait on that slot.
        if (ticket == kNone) ticket = atomicAdd(&Q->tt.tickets, 1u);
        uint32_t backoff = 128, spins = 0;
        while (true) {
          if (ticket < a.dyn_cap && ld_volatile(a.dyn_ready + ticket) == a.epoch) {
            kind = 2;
            ref = ticket;
            ticket = kNone;
            break;
          }
          if ((++spins & 3u) == 0) {
            if (ld_volatile(&Q->holders.v) == 0) {
              kind = 3;
              break;
            }
            if (a.deadline_ns && globaltimer() > a.deadline_ns) {
              kind = 3;
              break;
            }
          }
          __nanosleep(backoff);
          if (backoff < 4096) backoff *= 2;
        }
      }
    }
    kind = __shfl_sync(kFull, kind, 0);
    ref = __shfl_sync(kFull, ref, 0);
    if (kind == 3) break;
    uint32_t task_id, lstart, rbegin, rend, ncand = 0;
    if (kind == 1) {
      const Item item = a.items[ref];
      task_id = item.task;
      lstart = 2;
      rbegin = item.begin;
      rend = 0;  // set below from the task
    } else {
      __syncwarp();
      __threadfence();
      // L2-coherent loads (.cg): the slot was written by another SM in this launch
      const DynItem* it = a.dyn + ref;
      task_id = __ldcg(&it->task);
      lstart = __ldcg(&it->level);
      rbegin = __ldcg(&it->begin);
      rend = __ldcg(&it->end);
      ncand = __ldcg(&it->ncand);
      if (lane < lstart) s_M[w][lane] = __ldcg(&it->M[lane]);
      if (lane < ncand) s_cand[w][lstart][lane] = __ldcg(&it->cand[lane]);
    }
    if (task_id == kNone) {  // another rank's share
      if (lane == 0) atomicSub(&Q->holders.v, 1u);
      continue;
    }
    const Task task = a.tasks[task_id];
    const EdgeProg& P = a.progs[task.prog];
    const uint32_t anchor = task.upd;
    const uint32_t T = P.tail;  // deepest DFS level; deeper levels are counted by tail_factor
    if (kind == 1) {
      const bdsm_update_dev up = a.ups[task.upd];
      const uint32_t m0 = task.flip ? up.v : up.u, m1 = task.flip ? up.u : up.v;
      if (lane == 0) {
        s_M[w][0] = m0;
        s_M[w][1] = m1;
      }
      rend = task.base + min(rbegin + a.chunk, task.d);
      rbegin = task.base + rbegin;
    }
    __syncwarp();
    // Positions whose assigned vertex is a same-kind batch endpoint (bit j <->
    // M[j]; the anchor endpoints always are), uniform across the warp.
    uint32_t touched = 3u | __ballot_sync(kFull, lane >= 2 && lane < lstart &&
                                                     (__ldg(a.rows + s_M[w][lane]) & flag));
    // The current level's state lives in uniform registers; shallower levels
    // are parked in the lane-distributed stack (lane j holds level j), so the
    // hot chunk loop needs no shuffles.
    uint64_t c_off;
    uint32_t c_cur, c_end, c_mask, c_drv, c_tmask;
    {
      c_tmask = __ballot_sync(kFull, lane < ncand && (__ldg(a.rows + s_cand[w][lstart][lane]) & flag));
      const LevelSetup su = setup_level(P.lv[lstart], g, s_M[w], lane, s_floor[w][lstart], s_ceil[w][lstart]);
      if (lane == 0) stat[4] += 4ull * su.deg_sum;
      c_off = su.drv_off;
      c_drv = su.drv_b;
      c_cur = rbegin;
      c_end = rend;
      c_mask = 0;
      if (ncand) {  // donated candidate list: no driver fetching at this level
        c_cur = c_end = 0;
        c_mask = ncand == 32 ? kFull : ((1u << ncand) - 1);
      }
      if (lstart == T) tail_factor(a, P, T, w, s_M[w], s_floor, s_ceil, touched, anchor, flag, lane, &s_tail[w], stat);
    }
    uint32_t l = lstart;
    while (true) {
      if (c_mask == 0) {
        if (c_cur >= c_end) {
          if (l == lstart) break;
          --l;  // backtrack: restore the parked state of level l
          c_off = __shfl_sync(kFull, r_off, l);
          c_cur = __shfl_sync(kFull, r_cur, l);
          c_end = __shfl_sync(kFull, r_end, l);
          c_mask = __shfl_sync(kFull, r_mask, l);
          c_drv = __shfl_sync(kFull, r_drv, l);
          c_tmask = __shfl_sync(kFull, r_tmask, l);
          touched &= (1u << l) - 1u;
          continue;
        }
        // ---- donate work at the shallowest splittable level ---------------
        // (upper half of the remaining driver range, or of the remaining
        // candidates of an already-fetched chunk); the deadline is polled on
        // the same cadence.
        if (((++dtick) & 7u) == 0) {
          if (a.deadline_ns && (dtick & 255u) == 0 &&
              __shfl_sync(kFull, uint32_t(globaltimer() > a.deadline_ns), 0)) {
            timed_out = true;
            break;
          }
          // demand: tickets handed out beyond the slots reserved so far
          const unsigned long long tt =
              *reinterpret_cast<const volatile unsigned long long*>(&a.q->tt.tickets);
          if (int32_t(uint32_t(tt) - uint32_t(tt >> 32)) > 0) {
            if (lane == l) {  // park the current level: the stack now covers [lstart, l]
              r_cur = c_cur;
              r_end = c_end;
              r_mask = 0;
            }
            bool can_r = lane >= lstart && lane <= l && r_end > r_cur && (r_end - r_cur) >= 64;
            bool can_m = lane >= lstart && lane < l && __popc(r_mask) >= 2;
            uint32_t cb = __ballot_sync(kFull, can_r || can_m);
            if (cb) {
              uint32_t j = __ffs(cb) - 1;
              bool by_range = (__ballot_sync(kFull, can_r) >> j) & 1u;
              uint32_t slot = 0;
              if (lane == 0) slot = dyn_reserve(a.q, a.dyn_cap);
              slot = __shfl_sync(kFull, slot, 0);
              if (slot != kNone) {
                DynItem* it = a.dyn + slot;
                if (lane < j) it->M[lane] = s_M[w][lane];
                if (by_range) {
                  uint32_t cj = __shfl_sync(kFull, r_cur, j), ej = __shfl_sync(kFull, r_end, j);
                  uint32_t mid = cj + (ej - cj) / 2;
                  if (lane == j) r_end = mid;
                  if (lane == 0) {
                    it->begin = mid;
                    it->end = ej;
                    it->ncand = 0;
                  }
                } else {
                  uint32_t mj = __shfl_sync(kFull, r_mask, j);
                  uint32_t keep_n = (__popc(mj) + 1) / 2, kept = 0, rest = mj;
                  for (uint32_t k = 0; k < keep_n; ++k) {
                    uint32_t bit = rest & (~rest + 1u);
                    kept |= bit;
                    rest &= ~bit;
                  }
                  if (lane == j) r_mask = kept;
                  // lane k < popc(rest) writes the k-th donated candidate
                  bool mine = (rest >> lane) & 1u;
                  uint32_t rank = __popc(rest & ((1u << lane) - 1u));
                  if (mine) it->cand[rank] = s_cand[w][j][lane];
                  if (lane == 0) {
                    it->begin = 0;
                    it->end = 0;
                    it->ncand = __popc(rest);
                  }
                }
                if (lane == 0) {
                  it->task = task_id;
                  it->level = j;
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                  atomicExch(a.dyn_ready + slot, a.epoch);
                  atomicAdd(&st->donations, 1u);
                }
                c_end = __shfl_sync(kFull, r_end, l);  // shrinks when j == l
              }
            }
          }
        }
        const uint32_t cur = c_cur;
        c_cur += 32;
        uint32_t c;
        bool tc;
        const uint32_t m = filter_chunk(a, P.lv[l], s_M[w], s_floor[w][l], s_ceil[w][l], c_off, cur, c_end, c_drv,
                                        touched, anchor, flag, lane, c, tc);
        if (l == T) {  // last DFS level: every survivor roots the counted tail
          const unsigned long long pm = __popc(m);
          if (pm && lane == 0) {
            const TailFactor tf = s_tail[w];
            stat[0] += pm * tf.f;
            stat[1] += pm * tf.v;
            stat[2] += pm * tf.b;
            stat[3] += pm * tf.c;
          }
          continue;
        }
        if (lane == 0) stat[1] += __popc(m);
        s_cand[w][l][lane] = c;
        c_mask = m;
        c_tmask = __ballot_sync(kFull, tc);
        __syncwarp();
      } else {
        const uint32_t k = __ffs(c_mask) - 1;
        c_mask &= c_mask - 1;
        const uint32_t c = s_cand[w][l][k];
        if (lane == 0) s_M[w][l] = c;
        touched |= ((c_tmask >> k) & 1u) << l;
        if (lane == l) {  // park level l
          r_off = c_off;
          r_cur = c_cur;
          r_end = c_end;
          r_mask = c_mask;
          r_drv = c_drv;
          r_tmask = c_tmask;
        }
        __syncwarp();
        ++l;
        // GenCandidates for level l: driver = smallest backward list, range =
        // its label sub-range
        const LevelSetup su = setup_level(P.lv[l], g, s_M[w], lane, s_floor[w][l], s_ceil[w][l]);
        if (lane == 0) {
          stat[2] += 4ull * su.deg_sum;
          stat[3] += 1;
          stat[4] += 4ull * su.deg_sum;
        }
        c_off = su.drv_off;
        c_cur = su.lo;
        c_end = su.hi;
        c_mask = 0;
        c_drv = su.drv_b;
        c_tmask = 0;
        if (l == T) tail_factor(a, P, T, w, s_M[w], s_floor, s_ceil, touched, anchor, flag, lane, &s_tail[w], stat);
      }
    }
    if (lane == 0) atomicSub(&a.q->holders.v, 1u);
    if (timed_out) break;
  }
  __syncwarp();
  if (lane == 0) {
    if (stat[0]) atomicAdd((unsigned long long*)&st->counts[a.phase][a.query], stat[0]);
    if (stat[1]) atomicAdd((unsigned long long*)&st->visits, stat[1]);
    if (stat[2]) atomicAdd((unsigned long long*)&st->bytes_phase, stat[2]);
    if (stat[3]) atomicAdd((unsigned long long*)&st->gen_calls, stat[3]);
    if (stat[4]) atomicAdd((unsigned long long*)&st->bytes_kernel, stat[4]);
    if (timed_out) atomicOr(&st->timed_out, 1u << a.query);
  }
}

}  // namespace

void launch_anchor_count(const PhaseArgs& a, cudaStream_t s) {
  unsigned blocks = unsigned((uint64_t(a.n_ups) + 1 + 255) / 256);
  k_anchor_count<<<blocks, 256, 0, s>>>(a);
}

void launch_anchor_emit(const PhaseArgs& a, cudaStream_t s) {
  unsigned blocks = unsigned((uint64_t(a.n_ups) + 255) / 256);
  if (blocks == 0) blocks = 1;
  k_anchor_emit<<<blocks, 256, 0, s>>>(a);
}

void launch_wbm(const PhaseArgs& a, int num_sms, cudaStream_t s) {
  // persistent: as many resident CTAs as the SMs hold
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wbm, kWarpsPerBlock * 32, 0);
    if (per_sm <= 0) per_sm = 1;
  }
  k_wbm<<<unsigned(num_sms * per_sm), kWarpsPerBlock * 32, 0, s>>>(a);
}

}  // namespace bdsm_b200
