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
  const LevelProg& lp = p.lv[2];
  const uint32_t lo = label_bound(g, drv, lst, d, lp.lcls, lp.vlo, lp.vhi, 0);
  const uint32_t hi = label_bound(g, drv, lst, d, lp.lcls, lp.vlo, lp.vhi, 1);
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
    if (ae.mult[0] && ae.la == lu && ae.lb == lv) f(ae.prog, 0u, up, ae.mult[0]);
    if (ae.mult[1] && ae.la == lv && ae.lb == lu) f(ae.prog, 1u, up, ae.mult[1]);
  }
}

__global__ void k_anchor_count(PhaseArgs a) {
  if (batch_aborted(a.st)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // k_anchor_emit narrows this rank's item range
    a.st->item_lo[a.phase] = kNone;
    a.st->item_hi[a.phase] = 0;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= a.n_ups; i += gridDim.x * blockDim.x) {
    uint32_t nt = 0, ni = 0;
    uint64_t cost = 0;
    if (i < a.n_ups) {
      for_each_anchor(a, i, [&](uint32_t prog, uint32_t flip, const bdsm_update_dev& up, uint32_t) {
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
    a.upd_cnt[i] = AnchorCount{nt, ni, cost};
  }
}

__device__ __forceinline__ AnchorCount ac_add(const AnchorCount& x, const AnchorCount& y) {
  return AnchorCount{x.tasks + y.tasks, x.items + y.items, x.cost + y.cost};
}
__device__ __forceinline__ AnchorCount ac_shfl_up(const AnchorCount& v, uint32_t o) {
  return AnchorCount{__shfl_up_sync(kFull, v.tasks, o), __shfl_up_sync(kFull, v.items, o),
                     __shfl_up_sync(kFull, v.cost, o)};
}
__device__ __forceinline__ AnchorCount ac_shfl_xor(const AnchorCount& v, uint32_t o) {
  return AnchorCount{__shfl_xor_sync(kFull, v.tasks, o), __shfl_xor_sync(kFull, v.items, o),
                     __shfl_xor_sync(kFull, v.cost, o)};
}

// Small batches (a.self_scan): the exclusive scan of the per-update counts is
// done here instead of by a separate device scan — every block sums the counts
// before its first update and the grand total (a few thousand 16-byte loads
// per block), then scans its own 256 updates.  Launched with one thread per
// update.
__device__ void anchor_self_scan(const PhaseArgs& a, AnchorCount& off, AnchorCount& tot) {
  __shared__ AnchorCount s_pre[8], s_tot[8], s_w[8];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t first = blockIdx.x * blockDim.x;
  AnchorCount pre{0, 0, 0}, all{0, 0, 0};
  // 8 independent loads in flight per thread (the sums do not wait on each other)
  constexpr uint32_t U = 8;
  for (uint32_t j0 = threadIdx.x; j0 < a.n_ups; j0 += blockDim.x * U) {
    AnchorCount v[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      const uint32_t j = j0 + k * blockDim.x;
      v[k] = j < a.n_ups ? a.upd_cnt[j] : AnchorCount{0, 0, 0};
    }
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      all = ac_add(all, v[k]);
      if (j0 + k * blockDim.x < first) pre = ac_add(pre, v[k]);
    }
  }
#pragma unroll
  for (uint32_t o = 16; o; o >>= 1) {
    pre = ac_add(pre, ac_shfl_xor(pre, o));
    all = ac_add(all, ac_shfl_xor(all, o));
  }
  const uint32_t i = first + threadIdx.x;
  const AnchorCount mine = i < a.n_ups ? a.upd_cnt[i] : AnchorCount{0, 0, 0};
  AnchorCount inc = mine;
#pragma unroll
  for (uint32_t o = 1; o < 32; o <<= 1) {
    const AnchorCount t = ac_shfl_up(inc, o);
    if (lane >= o) inc = ac_add(inc, t);
  }
  if (lane == 0) {
    s_pre[w] = pre;
    s_tot[w] = all;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  AnchorCount base{0, 0, 0};
  tot = AnchorCount{0, 0, 0};
  for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
    base = ac_add(base, s_pre[k]);
    tot = ac_add(tot, s_tot[k]);
    if (k < w) base = ac_add(base, s_w[k]);
  }
  off = AnchorCount{base.tasks + inc.tasks - mine.tasks, base.items + inc.items - mine.items,
                    base.cost + inc.cost - mine.cost};
}

__global__ void k_anchor_emit(PhaseArgs a) {
  if (batch_aborted(a.st)) return;
  AnchorCount tot, self_off{0, 0, 0};
  if (a.self_scan) anchor_self_scan(a, self_off, tot);
  else tot = a.upd_off[a.n_ups];
  const uint64_t total_cost = tot.cost;
  const uint32_t total_items = tot.items;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.st->n_tasks[a.phase] = tot.tasks;
    a.st->n_items[a.phase] = total_items;
    atomicAdd((unsigned long long*)&a.st->tasks_total, (unsigned long long)tot.tasks);
    if (total_items > a.max_items) a.st->overflow = a.phase == 0 ? 2 : 3;  // host regrows, reruns
  }
  if (total_items > a.max_items) return;
  uint64_t direct = 0;    // 2-vertex queries: every anchor is a match
  uint64_t bytes = 0, calls = 0;
  uint32_t my_lo = kNone, my_hi = 0;  // this thread's items owned by this rank
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_ups; i += gridDim.x * blockDim.x) {
    const AnchorCount off = a.self_scan ? self_off : a.upd_off[i];
    uint32_t t = off.tasks, it = off.items;
    uint64_t c = off.cost;
    for_each_anchor(a, i, [&](uint32_t prog, uint32_t flip, const bdsm_update_dev& up, uint32_t mult) {
      if (a.qn <= 2) {
        uint32_t owner = a.shard_world > 1 ? uint32_t((unsigned __int128)c * a.shard_world / total_cost) : 0;
        if (owner == a.shard_rank) direct += mult;
        if (owner == a.shard_rank && a.match_out) {  // materialise the 2-vertex match
          const EdgeProg& p = a.progs[prog];
          const unsigned long long k = atomicAdd(a.match_count, 1ull);
          if (k < a.match_cap) {
            a.match_out[k * 2 + p.order[0]] = flip ? up.v : up.u;
            a.match_out[k * 2 + p.order[1]] = flip ? up.u : up.v;
          }
        }
        a.tasks[t++] = Task{i, prog, flip, 0, 0, mult};
        c += 1;
        return;
      }
      const EdgeProg& p = a.progs[prog];
      uint32_t m0 = flip ? up.v : up.u, m1 = flip ? up.u : up.v, base, d;
      level2_range(p, m0, m1, a.g, &base, &d);
      a.tasks[t] = Task{i, prog, flip, d, base, mult};
      // level-2 GenCandidates call of this anchor (SURVEY.md §8(d) B_phase)
      uint32_t bm = p.lv[2].backmask;
      if (bm & 1u) bytes += 4ull * a.g.deg[m0];
      if (bm & 2u) bytes += 4ull * a.g.deg[m1];
      ++calls;
      for (uint32_t b = 0; b < d; b += a.chunk) {
        uint32_t owner = a.shard_world > 1
                             ? uint32_t((unsigned __int128)(c + b) * a.shard_world / total_cost)
                             : 0;
        if (owner == a.shard_rank) {
          my_lo = min(my_lo, it);
          my_hi = it + 1;
        }
        a.items[it++] = Item{owner == a.shard_rank ? t : kNone, b};
      }
      ++t;
      c += d;
    });
  }
  if (direct) atomicAdd(a.count_out, (unsigned long long)direct);
  if (a.shard_world > 1) {
    const uint32_t wlo = __reduce_min_sync(kFull, my_lo), whi = __reduce_max_sync(kFull, my_hi);
    if ((threadIdx.x & 31) == 0 && wlo != kNone) {
      atomicMin(&a.st->item_lo[a.phase], wlo);
      atomicMax(&a.st->item_hi[a.phase], whi);
    }
  }
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

constexpr uint32_t kSplitMin = 2;  // driver entries a parked range needs to be split for donation
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
  const uint32_t lb_list = (lane >> 1) & 31;
  // with a label index the sub-range bounds depend only on the list's vertex:
  // lanes 2b / 2b+1 load them in the same round trip as the degrees
  uint32_t ibnd = 0;
  if (g.loff && lp.lcls != kNone && lane < 2 * nb)
    ibnd = __ldg(g.loff + uint64_t(M[lp.back[lb_list]]) * (g.nlab + 1) + lp.lcls + (lane & 1));
  if (lane < nb) {
    const uint32_t x = M[lp.back[lane]];
    myd = __ldg(g.deg + x);
    myo = __ldg(g.off + x);
  }
  const uint32_t mn = __reduce_min_sync(kFull, myd);
  LevelSetup s;
  s.drv_b = __ffs(__ballot_sync(kFull, myd == mn)) - 1;
  s.deg_sum = __reduce_add_sync(kFull, lane < nb ? myd : 0u);
  const uint32_t bd = __shfl_sync(kFull, myd, lb_list);
  const uint64_t bo = __shfl_sync(kFull, myo, lb_list);
  uint32_t bnd = 0;
  if (lane < 2 * nb) {
    if (bd <= 32) bnd = (lane & 1) ? bd : 0u;
    else if (g.loff) bnd = lp.lcls == kNone ? 0u : ibnd;
    else bnd = label_bound(g, M[lp.back[lb_list]], g.adj + bo, bd, lp.lcls, lp.vlo, lp.vhi, lane & 1);
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
                                                 bool& tc_out, bool have_pf = false, uint32_t pf_c = 0,
                                                 uint32_t pf_rw = 0) {
  const DevGraph& g = a.g;
  const uint32_t idx = cur + lane;
  bool ok = idx < end2;
  uint32_t c = 0xffffffffu;
  uint32_t rw = 0;
  if (have_pf) {  // driver entry and its row were prefetched while the previous chunk was weighted
    c = pf_c;
    rw = pf_rw;
  } else {
    if (ok) c = __ldg(g.adj + c_off + idx);
    if (ok) rw = __ldg(a.rows + c);  // candidate bits + batch-endpoint flags
  }
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
    if (g.hub_slot && !g.elab) {  // hub list: one bitmap load instead of a search
      const uint32_t hs = __ldg(g.hub_slot + x);
      if (hs != kNone) {
        if (ok) ok = (__ldg(g.bitmaps + uint64_t(hs) * g.bm_words + (c >> 5)) >> (c & 31)) & 1u;
        continue;
      }
    }
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
    __syncwarp();  // the floor is shared memory read by every lane of the next chunk (racecheck)
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
#ifdef BDSM_TRACE
__device__ uint32_t (*s_dbg)[2];  // per-block shared counters (set by each block; diagnostic builds only)
#endif
struct TailFactor {
  unsigned long long f, v, b, c;
};

// Weight of a leaf level t of T for the level-T candidate x: the number of
// its candidates, i.e. neighbours c of x in label(order[t])'s id range with
// candidate bit order[t], the query edge's label, and — only when x is a
// same-kind batch endpoint — visible under the lowest-order rule.  (c != x
// always; no other position shares the label, EdgeProg::leafmask.)  Warp-
// collective over one x.
__device__ __forceinline__ unsigned long long leaf_count(const PhaseArgs& a, const LevelProg& lp, uint32_t x,
                                                         bool x_touched, uint32_t anchor, uint32_t flag,
                                                         uint32_t lane) {
  const DevGraph& g = a.g;
  // the label-index bounds are loaded in the same round trip as the list
  uint32_t ib = 0;
  if (g.loff && lp.lcls != kNone && lane < 2) ib = __ldg(g.loff + uint64_t(x) * (g.nlab + 1) + lp.lcls + lane);
  const uint64_t xo = __ldg(g.off + x);
  const uint32_t xd = __ldg(g.deg + x);
  uint32_t lo = 0, hi = xd;
  if (xd > 32) {
    uint32_t bnd = 0;
    if (lane < 2)
      bnd = g.loff ? (lp.lcls == kNone ? 0u : ib) : label_bound(g, x, g.adj + xo, xd, lp.lcls, lp.vlo, lp.vhi, lane);
    lo = __shfl_sync(kFull, bnd, 0);
    hi = __shfl_sync(kFull, bnd, 1);
  }
  unsigned long long cnt = 0;
  constexpr uint32_t U = 4;  // chunks in flight
  for (uint32_t cur = lo; cur < hi; cur += 32 * U) {
    uint32_t c[U], rw[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      const uint32_t idx = cur + 32 * k + lane;
      c[k] = idx < hi ? __ldg(g.adj + xo + idx) : kNone;
    }
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) rw[k] = c[k] != kNone ? __ldg(a.rows + c[k]) : 0u;
    uint32_t n = 0;
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      const uint32_t idx = cur + 32 * k + lane;
      bool ok = (rw[k] & lp.qbit) != 0;
      if (ok && g.elab) ok = __ldg(g.elab + xo + idx) == lp.elab[0];
      if (ok && x_touched && (rw[k] & flag)) ok = !hidden_edge(a, x, c[k], anchor);
      n += ok;
    }
    cnt += __reduce_add_sync(kFull, n);
  }
  return cnt;
}

// The same count computed by one lane alone (small neighbour lists: the
// lanes of a warp count their own candidates concurrently).
__device__ __forceinline__ unsigned long long leaf_count_lane(const PhaseArgs& a, const LevelProg& lp, uint32_t x,
                                                              uint64_t xo, uint32_t xd, bool x_touched,
                                                              uint32_t anchor, uint32_t flag) {
  const DevGraph& g = a.g;
  const uint32_t* L = g.adj + xo;
  uint32_t i = label_bound(g, x, L, xd, lp.lcls, lp.vlo, lp.vhi, 0);
  const uint32_t end = label_bound(g, x, L, xd, lp.lcls, lp.vlo, lp.vhi, 1);
  unsigned long long cnt = 0;
  // 8 entries per step: their list loads, then their row loads, are all in
  // flight together (two round trips per step instead of two per entry)
  constexpr uint32_t U = 8;
  for (; i < end; i += U) {
    uint32_t c[U], rw[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) c[k] = i + k < end ? __ldg(L + i + k) : kNone;
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) rw[k] = c[k] != kNone ? __ldg(a.rows + c[k]) : 0u;
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      bool ok = (rw[k] & lp.qbit) != 0;
      if (ok && g.elab) ok = __ldg(g.elab + xo + i + k) == lp.elab[0];
      if (ok && x_touched && (rw[k] & flag)) ok = !hidden_edge(a, x, c[k], anchor);
      cnt += ok;
    }
  }
  return cnt;
}

constexpr uint32_t kLeafLaneMax = 256;  // lists up to this length are counted per lane

// Leaf weights are memoised without the visibility rule; for a level-T
// candidate x that is a same-kind batch endpoint the hidden edges are then
// subtracted: the same-kind updates (x, y) with order < anchor whose y passes
// the leaf's filter (x's segment of the sorted directed batch keys).
__device__ __forceinline__ unsigned long long hidden_count(const PhaseArgs& a, const LevelProg& lp, uint32_t x,
                                                           uint32_t anchor) {
  // x's segment start from the visibility table's (x, kNone) entry
  const unsigned long long hk = (uint64_t(x) << 32) | kNone;
  uint32_t pos = pair_hash(hk) & a.hmask;
  uint32_t i = a.m_keys;
  while (true) {
    const unsigned long long k = __ldg(a.hkeys + pos);
    if (k == hk) {
      i = __ldg(a.hvals + pos);
      break;
    }
    if (k == kEmptyKey) break;
    pos = (pos + 1) & a.hmask;
  }
  unsigned long long n = 0;
  for (; i < a.m_keys; ++i) {
    const unsigned long long k = __ldg(a.skeys + i);
    if ((k >> 32) != x) break;
    const uint32_t val = __ldg(a.svals + i);
    const uint32_t ord = val & 0x7fffffffu;
    if ((val >> 31) != (a.phase == 0 ? 1u : 0u) || ord >= anchor) continue;  // other kind, or not earlier
    const uint32_t y = uint32_t(k);
    if (y < lp.vlo || y >= lp.vhi || !(__ldg(a.rows + y) & lp.qbit)) continue;
    if (a.g.elab) {
      const uint32_t el = a.phase == 0 ? __ldg(a.dlab + ord) : a.ups[ord].elab;
      if (el != lp.elab[0]) continue;
    }
    ++n;
  }
  return n;
}

// Weight memo of this launch's query (common.cuh); persistent across launches
// and batches, invalidated by the merge (store.cu finish_vertex).
__device__ __forceinline__ bool memo_get(const PhaseArgs& a, uint32_t x, uint32_t sig, unsigned long long* w) {
  return ::bdsm_b200::memo_get(a.memo, a.memo_mask, x, a.query, sig, w);
}

__device__ __forceinline__ void memo_put(const PhaseArgs& a, uint32_t x, uint32_t sig, unsigned long long w) {
  if (::bdsm_b200::memo_put(a.memo, a.memo_mask, x, a.query, sig, w)) {
    atomicAdd(a.memo_fill, 1ull);
    if (a.g.memo_bits && !((__ldcg(a.g.memo_bits + (x >> 5)) >> (x & 31)) & 1u))
      atomicOr(a.g.memo_bits + (x >> 5), 1u << (x & 31));
  }
}

// Per-lane leaf weight of level t for the lane's level-T candidate c (lanes
// with `want`): memo hits answer directly, misses are counted one candidate
// at a time by the whole warp and memoised (candidates that are same-kind
// batch endpoints depend on the anchor through the visibility rule and are
// never memoised).
__device__ __forceinline__ unsigned long long leaf_weight(const PhaseArgs& a, const EdgeProg& P, uint32_t t,
                                                          uint32_t c, bool tc, bool want, uint32_t anchor,
                                                          uint32_t flag, uint32_t lane, unsigned long long* stat) {
  const uint32_t sig = P.sig[t];
  const LevelProg& lp = P.lv[t];
  unsigned long long wgt = 0;
  bool hit = false;
  if (want) hit = memo_get(a, c, sig, &wgt);
  // misses on short lists: every lane counts its own candidate
  bool big = false;
  if (want && !hit) {
    const uint32_t xd = __ldg(a.g.deg + c);
    if (xd <= kLeafLaneMax) {
      const uint64_t xo = __ldg(a.g.off + c);
      wgt = leaf_count_lane(a, lp, c, xo, xd, false, anchor, flag);
      memo_put(a, c, sig, wgt);
      atomicAdd(stat + 4, 4ull * xd);  // one GenCandidates call made
    } else {
      big = true;
    }
  }
  // misses on long lists: the whole warp counts one candidate at a time
  uint32_t todo = __ballot_sync(kFull, big);
  while (todo) {
    const uint32_t k = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t ck = __shfl_sync(kFull, c, k);
    const unsigned long long wk = leaf_count(a, lp, ck, false, anchor, flag, lane);
#ifdef BDSM_TRACE
    if (lane == 0) ++s_dbg[threadIdx.x >> 5][1];
#endif
    if (lane == k) wgt = wk;
    if (lane == 0) {
      memo_put(a, ck, sig, wk);
      stat[4] += 4ull * __ldg(a.g.deg + ck);  // one GenCandidates call made
    }
  }
  if (want && tc) wgt -= hidden_count(a, lp, c, anchor);
  return wgt;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Leaf-weight prefill (before each matching launch of a query with leaf
// levels): the weights of every long-list vertex that can be a weighted
// parent of a leaf signature — label(parent), its candidate bit — computed by
// the whole grid up front, so no DFS warp counts a hub's list on its critical
// path.  The candidates come from the engine's hub list (ids with > 256
// neighbours, refreshed every few batches; a stale list only means a lazy
// count later).  Warp per (signature, 32 hubs); qualifying lanes are counted
// one by one by the whole warp.
__global__ void __launch_bounds__(256) k_leaf_prefill(PhaseArgs a, const LeafSig* __restrict__ sigs, uint32_t nsig,
                                                      const uint32_t* __restrict__ hubs,
                                                      const uint32_t* __restrict__ n_hubs) {
  if (batch_aborted(a.st)) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t flag = a.flag;
  // hubs == nullptr: the batch's touched vertices (their weights were
  // invalidated by the merge) instead of the engine's hub list
  const uint32_t nh = hubs ? *n_hubs : a.st->n_touched;
  // a warp takes kPrefillGroup candidates per signature, so the few long
  // lists among them are spread over many warps instead of queueing in one
  constexpr uint32_t kPrefillGroup = 4;
  const uint64_t nblk = (uint64_t(nh) + kPrefillGroup - 1) / kPrefillGroup;
  for (uint64_t gi = warp; gi < nblk * nsig; gi += nwarps) {
    const LeafSig& ls = sigs[gi / nblk];
    const uint64_t hi = (gi % nblk) * kPrefillGroup + lane;
    bool want = false;
    uint32_t x = 0;
    if (lane < kPrefillGroup && hi < nh) {
      x = hubs ? __ldg(hubs + hi) : uint32_t(__ldg(a.skeys + __ldg(a.heads + hi)) >> 32);
      want = x >= ls.plo && x < ls.phi && (__ldg(a.rows + x) & ls.pbit) && __ldg(a.g.deg + x) > kLeafLaneMax;
    }
    uint32_t todo = __ballot_sync(kFull, want);
    while (todo) {
      const uint32_t k = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t xk = __shfl_sync(kFull, x, k);
      const unsigned long long wk = leaf_count(a, ls.leaf, xk, false, 0, flag, lane);
      if (lane == 0) memo_put(a, xk, ls.sig, wk);
    }
  }
}

// Tail counts are cached per warp: level t's count depends only on the images
// of its dependency positions (EdgeProg::lv[t].depmask = backward + same-label
// positions), so it is recomputed only after one of them was reassigned
// (`tvalid` bit t cleared through EdgeProg::inval).  With the greedy order
// most tail levels hang off shallow positions and are counted once per item.
__device__ __forceinline__ void tail_factor(const PhaseArgs& a, const EdgeProg& P, uint32_t T, uint32_t w,
                                            const uint32_t* M, uint32_t (*s_floor)[kMaxQ][kFloorB],
                                            uint32_t (*s_ceil)[kMaxQ][kFloorB], uint32_t touched, uint32_t anchor,
                                            uint32_t flag, uint32_t lane, TailFactor* out,
                                            unsigned long long* stat, unsigned long long* tcnt, uint32_t* tdeg,
                                            uint32_t& tvalid, uint32_t task_id) {
  unsigned long long prod = 1, v = 1, b = 0, c = 0;
  for (uint32_t t = T + 1; t < P.n; ++t) {
    if ((P.leafmask >> t) & 1u) continue;  // leaves of T: weighted per level-T candidate
    unsigned long long cnt;
    uint32_t degsum;
    if ((tvalid >> t) & 1u) {
      cnt = tcnt[t];
      degsum = tdeg[t];
    } else if ((P.singlemask >> t) & 1u) {
      // one backward neighbour x = M[j]: the memoised weight of x, minus the
      // edges the lowest-order rule hides when x is a same-kind batch endpoint
      const LevelProg& lp = P.lv[t];
      const uint32_t j = lp.back[0];
      const uint32_t x = M[j];
      degsum = __ldg(a.g.deg + x);
      unsigned long long wx = 0;
      bool hit = false;
      if (lane == 0) hit = memo_get(a, x, P.sig[t], &wx);
      hit = __shfl_sync(kFull, uint32_t(hit), 0) != 0;
      if (!hit) {
        wx = leaf_count(a, lp, x, false, anchor, flag, lane);
        if (lane == 0) {
          memo_put(a, x, P.sig[t], wx);
          stat[4] += 4ull * degsum;
        }
      }
      if ((touched >> j) & 1u) {
        unsigned long long h = 0;
        if (lane == 0) h = hidden_count(a, lp, x, anchor);
        wx -= h;
      }
      cnt = __shfl_sync(kFull, wx, 0);
      if (lane == 0) {
        tcnt[t] = cnt;
        tdeg[t] = degsum;
      }
      tvalid |= 1u << t;
    } else if (P.atail_slot[t] != 0xff && a.task_tail &&
               __shfl_sync(kFull, lane == 0 ? uint32_t(__ldcg(a.task_tail + uint64_t(task_id) * a.natail_stride +
                                                              P.atail_slot[t]) != kMemoEmpty)
                                            : 0u, 0)) {
      // anchor-only level already counted by another item of this task
      const LevelProg& lp = P.lv[t];
      cnt = __ldcg(a.task_tail + uint64_t(task_id) * a.natail_stride + P.atail_slot[t]);
      degsum = 0;
      for (uint32_t b = 0; b < lp.nback; ++b) degsum += __ldg(a.g.deg + M[lp.back[b]]);
      if (lane == 0) {
        tcnt[t] = cnt;
        tdeg[t] = degsum;
      }
      tvalid |= 1u << t;
    } else {
      const LevelProg& lp = P.lv[t];
      const LevelSetup su = setup_level(lp, a.g, M, lane, s_floor[w][t], s_ceil[w][t]);
      __syncwarp();
#ifdef BDSM_TRACE
      if (lane == 0) {
        atomicAdd((unsigned long long*)&a.st->trace_setups[a.phase][t], 1ull);
        atomicAdd((unsigned long long*)&a.st->trace_chunks[a.phase][t], (unsigned long long)((su.hi - su.lo + 31) / 32));
      }
#endif
      degsum = su.deg_sum;
      if (lane == 0) stat[4] += 4ull * su.deg_sum;
      cnt = 0;
      for (uint32_t cur = su.lo; cur < su.hi; cur += 32) {
        uint32_t cc;
        bool tc;
        cnt += __popc(filter_chunk(a, lp, M, s_floor[w][t], s_ceil[w][t], su.drv_off, cur, su.hi, su.drv_b, touched,
                                   anchor, flag, lane, cc, tc));
#ifdef BDSM_TRACE
        if (lane == 0) ++s_dbg[w][0];
#endif
        __syncwarp();
      }
      if (lane == 0) {
        tcnt[t] = cnt;
        tdeg[t] = degsum;
        if (P.atail_slot[t] != 0xff && a.task_tail)
          a.task_tail[uint64_t(task_id) * a.natail_stride + P.atail_slot[t]] = cnt;
      }
      tvalid |= 1u << t;
    }
    b += prod * 4ull * degsum;  // one call per visit at level t-1
    c += prod;
    prod *= cnt;
    v += prod;
    if (prod == 0) break;  // the reference tree has no deeper nodes either
  }
  if (lane == 0) *out = TailFactor{prod, v, b, c};
  __syncwarp();
}

// Register budget per instantiation: kMinBlocks resident 256-thread CTAs per
// SM.  2 (104 registers, no spills) wins when the launch is bound by its
// longest subtree (C2: +6 % over 4); 4 (64 registers) wins when thousands of
// items keep every warp busy (C5 cycle: +40 %).  The engine picks per launch
// from the previous batch's work-item count (launch_wbm).
// kEmit: bounded match materialisation (the reference's Match vectors,
// src/matcher.cpp:169-217, for --dump-matches): the whole order is
// enumerated (no counted tail) and every complete match is written in query
// vertex order to a.match_out.
// kPairs: 1 for a single phase (the phase arguments are compile-time uniform),
// 2 for the pipelined stream's fused launch.
template <bool kEmit, int kMinBlocks, int kPairs>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kMinBlocks) k_wbm(const __grid_constant__ PhasePair pp) {
  __shared__ uint32_t s_cand[kWarpsPerBlock][kMaxQ][32];
  __shared__ uint32_t s_M[kWarpsPerBlock][kMaxQ];
  __shared__ uint32_t s_floor[kWarpsPerBlock][kMaxQ][kFloorB];
  __shared__ uint32_t s_ceil[kWarpsPerBlock][kMaxQ][kFloorB];
  __shared__ TailFactor s_tail[kWarpsPerBlock];
  __shared__ unsigned long long s_tcnt[kWarpsPerBlock][kMaxQ];  // cached tail-level counts
  __shared__ uint32_t s_tdeg[kWarpsPerBlock][kMaxQ];
#ifdef BDSM_TRACE
  __shared__ uint32_t s_dbg_[kWarpsPerBlock][2];
  s_dbg = s_dbg_;
#endif
  // per-warp counters (lane 0 updates them; kept out of the register budget)
  __shared__ unsigned long long s_stat[kWarpsPerBlock][10];  // per phase: count, visits, bytes, calls, kernel bytes
  __shared__ unsigned long long s_lacc[kWarpsPerBlock][32][4];  // per-lane count/visits/bytes/calls (leaf levels)
  // One launch runs up to two phases (the pipelined stream's positive phase
  // of batch i and negative phase of batch i+1, both on the same graph): the
  // static items of pp.p[0] come first in the shared queue, then pp.p[1]'s;
  // a donated item records its phase.  Queue, donation slots, memo and graph
  // are shared; a phase whose batch was aborted contributes no items.
  const PhaseArgs& a0 = pp.p[0];
  // static items of each phase: all of them, or this rank's contiguous range
  auto phase_items = [](const PhaseArgs& a, uint32_t& lo) -> uint32_t {
    lo = 0;
    if (batch_aborted(a.st)) return 0u;
    if (a.shard_world <= 1) return a.st->n_items[a.phase];
    const uint32_t l = a.st->item_lo[a.phase], h = a.st->item_hi[a.phase];
    lo = l;
    return h > l ? h - l : 0u;
  };
  uint32_t lo0 = 0, lo1 = 0;
  const uint32_t n0 = phase_items(a0, lo0);
  const uint32_t n1 = kPairs < 2 ? 0u : phase_items(pp.p[kPairs - 1], lo1);
  const uint32_t n_items = n0 + n1;
  if (n_items == 0) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  if (lane < 10) s_stat[w][lane] = 0;
  for (int k = 0; k < 4; ++k) s_lacc[w][lane][k] = 0;
  __syncwarp();
  uint32_t dtick = 0;
  unsigned long long tt_pref = 0;  // prefetched donation-demand poll
  uint32_t pf_c = 0, pf_rw = 0, pf_pos = kNone;  // prefetched next chunk of the last DFS level
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

  while (true) {
    // ---- acquire work ----------------------------------------------------
    uint32_t kind = 0, ref = 0;  // 1 static item, 2 donated item, 3 exit, 4 deadline
    QueueState* Q = a0.q;
    if (lane == 0) {
      // Static items first (counted as held before the index is taken, so a
      // waiter never sees holders == 0 while a static item is in flight).
      // the deadline is checked before every work item, as the reference's
      // workers check it before every task (Shared::stopping,
      // src/scheduler.cpp:101-110): an expired budget stops the phase
      if (a0.deadline_ns && globaltimer() > a0.deadline_ns) {
        kind = 4;
        static_done = true;
      }
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
      if (!kind && !(a0.deadline_ns && globaltimer() > a0.deadline_ns)) {
        // Donated work: one ticket per idle period, then wait on that slot.
        if (ticket == kNone) ticket = atomicAdd(&Q->tt.tickets, 1u);
        uint32_t backoff = 128, spins = 0;
        while (true) {
          if (ticket < a0.dyn_cap && ld_volatile(a0.dyn_ready + ticket) == a0.epoch) {
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
            if (a0.deadline_ns && globaltimer() > a0.deadline_ns) {
              kind = 4;
              break;
            }
          }
          __nanosleep(backoff);
          if (backoff < a0.backoff_max) backoff *= 2;
        }
      }
    }
    kind = __shfl_sync(kFull, kind, 0);
    ref = __shfl_sync(kFull, ref, 0);
    if (kind == 4) {  // deadline: counts of this query are dropped
      timed_out = true;
      break;
    }
    if (kind == 3) break;
    // the phase this item belongs to
    uint32_t sel = 0;
    if (kPairs > 1) {
      if (kind == 1 && ref >= n0) {
        sel = 1;
        ref -= n0;
      } else if (kind == 2) {
        __threadfence();
        sel = __ldcg(&a0.dyn[ref].pad[0]);
      }
    }
    const PhaseArgs& a = pp.p[sel];
    BatchState* st = a.st;
    const DevGraph& g = a.g;
    const uint32_t flag = a.flag;
    unsigned long long* stat = s_stat[w] + 5 * sel;
#ifdef BDSM_TRACE
    const uint64_t t_item = globaltimer();
    uint32_t it_chunks = 0, it_don = 0;
    long long cy_don = 0, cy_filter = 0, cy_leaf = 0, cy_setup = 0, cy0 = 0;
    s_dbg[w][0] = s_dbg[w][1] = 0;
#endif
    uint32_t task_id, lstart, rbegin, rend, ncand = 0;
    if (kind == 1) {
      const Item item = a.items[(sel ? lo1 : lo0) + ref];
      task_id = item.task;
      lstart = 2;
      rbegin = item.begin;
      rend = 0;  // set below from the task
    } else {
      __syncwarp();
      __threadfence();
      // L2-coherent loads (.cg): the slot was written by another SM in this launch
      const DynItem* it = a0.dyn + ref;
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
    const uint32_t T = kEmit ? P.n - 1 : P.tail;  // deepest DFS level; deeper levels are counted by tail_factor
    uint32_t tvalid = 0;        // tail levels whose cached count is current
    pf_pos = kNone;
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
      if (lstart == T) tail_factor(a, P, T, w, s_M[w], s_floor, s_ceil, touched, anchor, flag, lane, &s_tail[w], stat,
                                 s_tcnt[w], s_tdeg[w], tvalid, task_id);
    }
    uint32_t l = lstart;
    while (true) {
      if (c_mask == 0) {
        if (c_cur >= c_end) {
          if (l == lstart) break;
          --l;  // backtrack: restore the parked state of level l
          pf_pos = kNone;
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
        {
          if (a.deadline_ns && ((++dtick) & 255u) == 0 &&
              __shfl_sync(kFull, uint32_t(globaltimer() > a.deadline_ns), 0)) {
            timed_out = true;
            break;
          }
          // demand: tickets handed out beyond the slots reserved so far.  The
          // poll is issued one chunk fetch ahead so its L2 round trip overlaps
          // the chunk's filtering.
          const unsigned long long tt = tt_pref;
          tt_pref = *reinterpret_cast<const volatile unsigned long long*>(&a0.q->tt.tickets);
          if (int32_t(uint32_t(tt) - uint32_t(tt >> 32)) > 0) {
            if (lane == l) {  // park the current level: the stack now covers [lstart, l]
              r_cur = c_cur;
              r_end = c_end;
              r_mask = 0;
            }
            bool can_r = lane >= lstart && lane <= l && r_end > r_cur && (r_end - r_cur) >= kSplitMin;
            bool can_m = lane >= lstart && lane < l && __popc(r_mask) >= 2;
            uint32_t cb = __ballot_sync(kFull, can_r || can_m);
            if (cb) {
              uint32_t j = __ffs(cb) - 1;
              bool by_range = (__ballot_sync(kFull, can_r) >> j) & 1u;
#ifdef BDSM_TRACE
              cy0 = clock64();
#endif
              uint32_t slot = 0;
              if (lane == 0) slot = dyn_reserve(a0.q, a0.dyn_cap);
              slot = __shfl_sync(kFull, slot, 0);
              if (slot != kNone) {
                DynItem* it = a0.dyn + slot;
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
                  it->pad[0] = sel;
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                  atomicExch(a0.dyn_ready + slot, a0.epoch);
                  atomicAdd(&st->donations, 1u);
                }
#ifdef BDSM_TRACE
                ++it_don;
#endif
              }
#ifdef BDSM_TRACE
              cy_don += clock64() - cy0;
#endif
              c_end = __shfl_sync(kFull, r_end, l);  // shrinks when j == l
            }
          }
        }
        const uint32_t cur = c_cur;
        c_cur += 32;
#ifdef BDSM_TRACE
        if (lane == 0) atomicAdd((unsigned long long*)&st->trace_chunks[a.phase][l], 1ull);
        ++it_chunks;
#endif
        uint32_t c;
        bool tc;
#ifdef BDSM_TRACE
        cy0 = clock64();
#endif
        const uint32_t m = filter_chunk(a, P.lv[l], s_M[w], s_floor[w][l], s_ceil[w][l], c_off, cur, c_end, c_drv,
                                        touched, anchor, flag, lane, c, tc, pf_pos == cur, pf_c, pf_rw);
        pf_pos = kNone;
        // last DFS level: the next chunk's driver entries are loaded now, their
        // rows after this chunk's weights, so both round trips overlap the work
        const bool prefetch = l == T && c_cur < c_end;
        if (prefetch) pf_c = c_cur + lane < c_end ? __ldg(g.adj + c_off + c_cur + lane) : kNone;
#ifdef BDSM_TRACE
        cy_filter += clock64() - cy0;
        cy0 = clock64();
#endif
        if (kEmit && l == T && m) {  // write every survivor's full match (query vertex order)
          const uint32_t pm = __popc(m);
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(a.match_count, (unsigned long long)pm);
          base = __shfl_sync(kFull, base, 0);
          if ((m >> lane) & 1u) {
            const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
            if (k < a.match_cap) {
              uint32_t* out = a.match_out + k * P.n;
              for (uint32_t j = 0; j < T; ++j) out[P.order[j]] = s_M[w][j];
              out[P.order[T]] = c;
            }
          }
        }
        if (!kEmit && l == T && P.leafmask && m) {
          // last DFS level with leaves of T: per-survivor weights; each lane
          // walks the tail levels for its own reference-tree counters
          const bool ok = (m >> lane) & 1u;
          unsigned long long prod = ok ? 1ull : 0ull, vis = prod, bb = 0, cc = 0;
          const uint32_t degc = ok ? __ldg(g.deg + c) : 0u;
          for (uint32_t t = T + 1; t < P.n; ++t) {
            unsigned long long cnt;
            uint32_t dsum;
            if ((P.leafmask >> t) & 1u) {
              cnt = leaf_weight(a, P, t, c, tc, ok && prod != 0, anchor, flag, lane, stat);
              dsum = degc;
            } else {
              cnt = s_tcnt[w][t];
              dsum = s_tdeg[w][t];
            }
            bb += prod * 4ull * dsum;
            cc += prod;
            prod *= cnt;
            vis += prod;
          }
          // per-lane accumulators, summed across the warp once at the end
          unsigned long long* la = s_lacc[w][lane];
          la[0] += prod * task.mult;
          la[1] += vis;
          la[2] += bb;
          la[3] += cc;
#ifdef BDSM_TRACE
          cy_leaf += clock64() - cy0;
#endif
          if (prefetch) {
            pf_rw = pf_c != kNone ? __ldg(a.rows + pf_c) : 0u;
            pf_pos = c_cur;
          }
          continue;
        }
        if (l == T) {  // last DFS level: every survivor roots the counted tail
          const unsigned long long pm = __popc(m);
          if (pm && lane == 0) {
            const TailFactor tf = s_tail[w];
            stat[0] += pm * tf.f * task.mult;
            stat[1] += pm * tf.v;
            stat[2] += pm * tf.b;
            stat[3] += pm * tf.c;
          }
          if (prefetch) {
            pf_rw = pf_c != kNone ? __ldg(a.rows + pf_c) : 0u;
            pf_pos = c_cur;
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
        pf_pos = kNone;
        const uint32_t c = s_cand[w][l][k];
        __syncwarp();  // every lane's reads of M[] for the previous candidate are done (racecheck)
        if (lane == 0) s_M[w][l] = c;
        tvalid &= ~P.inval[l];
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
#ifdef BDSM_TRACE
        cy0 = clock64();
#endif
        const LevelSetup su = setup_level(P.lv[l], g, s_M[w], lane, s_floor[w][l], s_ceil[w][l]);
        if (lane == 0) {
          stat[2] += 4ull * su.deg_sum;
          stat[3] += 1;
          stat[4] += 4ull * su.deg_sum;
#ifdef BDSM_TRACE
          atomicAdd((unsigned long long*)&st->trace_setups[a.phase][l], 1ull);
#endif
        }
        c_off = su.drv_off;
        c_cur = su.lo;
        c_end = su.hi;
        c_mask = 0;
        c_drv = su.drv_b;
        c_tmask = 0;
        if (l == T) tail_factor(a, P, T, w, s_M[w], s_floor, s_ceil, touched, anchor, flag, lane, &s_tail[w], stat,
                                 s_tcnt[w], s_tdeg[w], tvalid, task_id);
#ifdef BDSM_TRACE
        cy_setup += clock64() - cy0;
#endif
      }
    }
    if (lane == 0) atomicSub(&a0.q->holders.v, 1u);
    {  // fold the per-lane leaf-level accumulators into this phase's counters
      unsigned long long v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = warp_sum_u64(s_lacc[w][lane][k]);
        s_lacc[w][lane][k] = 0;
      }
      if (lane == 0)
        for (int k = 0; k < 4; ++k) stat[k] += v[k];
      __syncwarp();
    }
#ifdef BDSM_TRACE
    if (lane == 0) {
      const uint64_t t1 = globaltimer(), dt = t1 - t_item;
      unsigned long long* tr = (unsigned long long*)st->trace[a.phase];
      atomicAdd(tr + 0, (unsigned long long)dt);
      const unsigned long long prev = atomicMax(tr + 1, (unsigned long long)dt);
      if (dt > prev) {  // racy, diagnostic only
        tr[2] = (kind << 8) | lstart;
        tr[7] = it_chunks;
        tr[8] = s_dbg[w][0];
        tr[9] = s_dbg[w][1];
        tr[10] = it_don;
        tr[12] = cy_don;
        tr[13] = cy_filter;
        tr[14] = cy_leaf;
        tr[15] = cy_setup;
        tr[11] = (uint64_t(__ldg(g.deg + s_M[w][0])) << 32) | __ldg(g.deg + s_M[w][1]);
      }
      atomicAdd(tr + (kind == 1 ? 3 : 4), 1ull);
      atomicMin(tr + 5, (unsigned long long)t_item);
      atomicMax(tr + 6, (unsigned long long)t1);
    }
#endif
    if (timed_out) break;
  }
  __syncwarp();
  if (lane == 0) {
    for (uint32_t sel = 0; sel < uint32_t(kPairs); ++sel) {
      const PhaseArgs& a = pp.p[sel];
      const unsigned long long* stat = s_stat[w] + 5 * sel;
      if (stat[0]) atomicAdd(a.count_out, stat[0]);
      if (stat[1]) atomicAdd((unsigned long long*)&a.st->visits, stat[1]);
      if (stat[2]) atomicAdd((unsigned long long*)&a.st->bytes_phase, stat[2]);
      if (stat[3]) atomicAdd((unsigned long long*)&a.st->gen_calls, stat[3]);
      if (stat[4]) atomicAdd((unsigned long long*)&a.st->bytes_kernel, stat[4]);
    }
    // a deadline stops the launch: the counts of its queries are dropped
    if (timed_out)
      for (uint32_t sel = 0; sel < uint32_t(kPairs); ++sel) atomicExch(pp.p[sel].timed_out, 1u);
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

void launch_leaf_prefill(const PhaseArgs& a, const LeafSig* sigs, uint32_t nsig, const uint32_t* hubs,
                         const uint32_t* n_hubs, int num_sms, cudaStream_t s) {
  if (nsig) k_leaf_prefill<<<unsigned(num_sms * 8), 256, 0, s>>>(a, sigs, nsig, hubs, n_hubs);
}

template <bool kEmit, int kMinBlocks, int kPairs>
void launch_wbm_variant(const PhasePair& pp, int num_sms, cudaStream_t s) {
  // persistent: as many resident CTAs as the SMs hold (queried once per
  // variant; a function-local static is initialised once even when engines on
  // several host threads launch concurrently, e.g. a multi-device group)
  static const int per_sm = [] {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_wbm<kEmit, kMinBlocks, kPairs>, kWarpsPerBlock * 32, 0) !=
            cudaSuccess ||
        n <= 0)
      n = 1;
    return n;
  }();
  k_wbm<kEmit, kMinBlocks, kPairs><<<unsigned(num_sms * per_sm), kWarpsPerBlock * 32, 0, s>>>(pp);
}

void launch_wbm(const PhaseArgs& a, const PhaseArgs* second, int num_sms, int ctas_per_sm, cudaStream_t s) {
  PhasePair pp;
  pp.p[0] = a;
  pp.p[1] = second ? *second : a;
  pp.n = second ? 2u : 1u;
  if (a.match_out) launch_wbm_variant<true, 2, 1>(pp, num_sms, s);
  else if (second && ctas_per_sm >= 4) launch_wbm_variant<false, 4, 2>(pp, num_sms, s);
  else if (second && ctas_per_sm == 3) launch_wbm_variant<false, 3, 2>(pp, num_sms, s);
  else if (second) launch_wbm_variant<false, 2, 2>(pp, num_sms, s);
  else if (ctas_per_sm >= 4) launch_wbm_variant<false, 4, 1>(pp, num_sms, s);
  else if (ctas_per_sm == 3) launch_wbm_variant<false, 3, 1>(pp, num_sms, s);
  else launch_wbm_variant<false, 2, 1>(pp, num_sms, s);
}

}  // namespace bdsm_b200
