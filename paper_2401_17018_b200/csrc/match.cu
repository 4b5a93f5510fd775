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

struct AnchorCounts {
  uint32_t tasks, items;
  uint64_t cost;
};

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
        uint32_t m0 = flip ? up.v : up.u, m1 = flip ? up.u : up.v, pos;
        uint32_t d = a.g.deg[level2_driver(p, m0, m1, a.g, &pos)];
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
        a.tasks[t++] = Task{i, prog, flip, 0};
        c += 1;
        return;
      }
      const EdgeProg& p = a.progs[prog];
      uint32_t m0 = flip ? up.v : up.u, m1 = flip ? up.u : up.v, pos;
      uint32_t d = a.g.deg[level2_driver(p, m0, m1, a.g, &pos)];
      a.tasks[t] = Task{i, prog, flip, d};
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
  uint64_t key = (uint64_t(x) << 32) | c;
  uint32_t p = lb_u64(a.skeys, a.m_keys, key);
  if (p >= a.m_keys || __ldg(a.skeys + p) != key) return false;
  uint32_t val = __ldg(a.svals + p);
  bool is_del = val >> 31;
  return is_del == (a.phase == 0) && (val & 0x7fffffffu) < anchor;
}

__device__ __forceinline__ bool bit_set(const uint32_t* bits, uint32_t v) {
  return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

// K6: persistent warp-per-partial-match DFS counter.
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_wbm(PhaseArgs a) {
  __shared__ uint32_t s_cand[kWarpsPerBlock][kMaxQ][32];
  __shared__ uint32_t s_M[kWarpsPerBlock][kMaxQ];
  if (batch_aborted(a.st)) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t n_items = a.st->n_items[a.phase];
  const DevGraph& g = a.g;
  uint64_t count = 0, visits = 0, bytes = 0, calls = 0;
  uint32_t tick = 0;
  bool timed_out = false;

  // Lane-distributed per-level DFS state: lane l holds level l's.
  uint64_t r_off = 0;   // driver list offset
  uint32_t r_cur = 0;   // next driver index to fetch
  uint32_t r_end = 0;   // end of driver range
  uint32_t r_mask = 0;  // unexplored candidates of the current chunk
  uint32_t r_drv = 0;   // position of the driver among the backward neighbours
  uint32_t r_touch = 0; // lane l: is M[l] a same-kind batch endpoint

  while (true) {
    uint32_t item_idx = 0;
    if (lane == 0) item_idx = atomicAdd(&a.st->next_item, 1u);
    item_idx = __shfl_sync(kFull, item_idx, 0);
    if (item_idx >= n_items) break;
    if (a.deadline_ns) {
      if (globaltimer() > a.deadline_ns) {
        timed_out = true;
        break;
      }
    }
    const Item item = a.items[item_idx];
    if (item.task == kNone) continue;  // another rank's share
    const Task task = a.tasks[item.task];
    const EdgeProg& P = a.progs[task.prog];
    const bdsm_update_dev up = a.ups[task.upd];
    const uint32_t anchor = task.upd;
    const uint32_t n = P.n;
    const uint32_t m0 = task.flip ? up.v : up.u, m1 = task.flip ? up.u : up.v;
    if (lane == 0) {
      s_M[w][0] = m0;
      s_M[w][1] = m1;
    }
    // both anchor endpoints are same-kind batch endpoints by construction
    r_touch = (lane == 0 || lane == 1) ? 1u : 0u;
    {
      uint32_t dpos;
      uint32_t drv = level2_driver(P, m0, m1, g, &dpos);
      if (lane == 2) {
        r_off = g.off[drv];
        r_cur = item.begin;
        r_end = min(item.begin + a.chunk, task.d);
        r_mask = 0;
        r_drv = P.lv[2].backmask == 3u ? dpos : 0u;  // index into the backward list
      }
    }
    __syncwarp();
    uint32_t l = 2;
    while (true) {
      uint32_t mask = __shfl_sync(kFull, r_mask, l);
      if (mask == 0) {
        const uint32_t cur = __shfl_sync(kFull, r_cur, l);
        const uint32_t end = __shfl_sync(kFull, r_end, l);
        if (cur >= end) {
          if (l == 2) break;
          --l;
          continue;
        }
        const uint64_t doff = __shfl_sync(kFull, r_off, l);
        const uint32_t dpos = __shfl_sync(kFull, r_drv, l);
        const uint32_t touched = __ballot_sync(kFull, r_touch) ;
        if (lane == l) r_cur = cur + 32;
        if (a.deadline_ns && ((++tick & 255u) == 0) && globaltimer() > a.deadline_ns) {
          timed_out = true;
          break;
        }
        const LevelProg& lp = P.lv[l];
        const uint32_t idx = cur + lane;
        bool ok = idx < end;
        uint32_t c = 0;
        if (ok) c = __ldg(g.adj + doff + idx);
        if (ok) ok = (__ldg(a.rows + c) & lp.qbit) != 0;
        if (ok && g.elab) ok = __ldg(g.elab + doff + idx) == lp.elab[dpos];
        if (ok) {  // injectivity: only same-label positions can collide
          uint32_t eq = lp.eqmask;
          while (eq) {
            uint32_t j = __ffs(eq) - 1;
            eq &= eq - 1;
            if (s_M[w][j] == c) {
              ok = false;
              break;
            }
          }
        }
        for (uint32_t b = 0; b < lp.nback; ++b) {  // other backward lists
          if (b == dpos) continue;
          const uint32_t x = s_M[w][lp.back[b]];
          const uint64_t xo = __ldg(g.off + x);
          const uint32_t xd = __ldg(g.deg + x);
          if (ok) {
            uint32_t p = lb_u32(g.adj + xo, xd, c);
            ok = p < xd && __ldg(g.adj + xo + p) == c;
            if (ok && g.elab) ok = __ldg(g.elab + xo + p) == lp.elab[b];
          }
        }
        if (ok && (touched & lp.backmask) && bit_set(a.touched_bits, c)) {
          uint32_t tb = touched & lp.backmask;
          while (tb && ok) {
            uint32_t j = __ffs(tb) - 1;
            tb &= tb - 1;
            if (hidden_edge(a, s_M[w][j], c, anchor)) ok = false;
          }
        }
        const uint32_t m = __ballot_sync(kFull, ok);
        visits += __popc(m);
        if (l + 1 == n) {
          count += __popc(m);
          continue;
        }
        s_cand[w][l][lane] = c;
        if (lane == l) r_mask = m;
        __syncwarp();
      } else {
        const uint32_t k = __ffs(mask) - 1;
        if (lane == l) r_mask = mask & (mask - 1);
        const uint32_t c = s_cand[w][l][k];
        const bool tc = bit_set(a.touched_bits, c);
        if (lane == l) r_touch = tc ? 1u : 0u;
        if (lane == 0) s_M[w][l] = c;
        __syncwarp();
        ++l;
        // GenCandidates for level l: driver = smallest backward list
        const LevelProg& lp = P.lv[l];
        uint32_t best_deg = 0xffffffffu, best_b = 0;
        uint64_t sum = 0;
        for (uint32_t b = 0; b < lp.nback; ++b) {
          uint32_t x = s_M[w][lp.back[b]];
          uint32_t d = __ldg(g.deg + x);
          sum += d;
          if (d < best_deg) {
            best_deg = d;
            best_b = b;
          }
        }
        bytes += 4 * sum;
        ++calls;
        if (lane == l) {
          uint32_t x = s_M[w][lp.back[best_b]];
          r_off = __ldg(g.off + x);
          r_cur = 0;
          r_end = best_deg;
          r_mask = 0;
          r_drv = best_b;
        }
        __syncwarp();
      }
    }
    if (timed_out) break;
  }
  if (lane == 0) {
    if (count) atomicAdd((unsigned long long*)&a.st->counts[a.phase][a.query], (unsigned long long)count);
    if (visits) atomicAdd((unsigned long long*)&a.st->visits, (unsigned long long)visits);
    if (bytes) atomicAdd((unsigned long long*)&a.st->bytes_phase, (unsigned long long)bytes);
    if (calls) atomicAdd((unsigned long long*)&a.st->gen_calls, (unsigned long long)calls);
    if (timed_out) atomicOr(&a.st->timed_out, 1u << a.query);
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
