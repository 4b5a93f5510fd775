// Multi-device engine group (SURVEY.md §8(e) inside one process; §8(b)'s
// `devices[]` option): one engine per listed device, every engine holding a
// replica of the graph and applying every batch to it (redundant and
// deterministic, so the replicas never diverge), and counting only its share
// of the work units — engine r of n is shard (r, n) of the canonical,
// cost-balanced work-unit order (bdsm_shard_owners).  The counts of a batch
// are the sums over the engines; the engines run concurrently (asynchronous
// submit on each device, then the waits; the pipelined stream on one host
// thread per device).  A device may be listed more than once (the engines
// then share it), which is how the CPU-less tests check the split on one GPU.
//
// The reference runs one match_batch per graph (src/matcher.cpp:370-389,
// src/bench.cpp:370-564); it has no multi-device mode.  Host code only: the
// engines' own C ABI does all device work.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bdsm_gpu.h"

extern "C" void bdsm_internal_set_last_error(const char* msg);

struct bdsm_group {
  std::vector<bdsm_engine*> engines;
  std::vector<int32_t> devices;
  std::vector<uint32_t> nverts;  // per query: vertices (match rows)
  uint64_t collect_cap = 0;      // per engine (bdsm_group_collect_matches)
  std::vector<uint8_t> timed;    // per query: timed out in some engine during the last batch
};

namespace {

bdsm_status group_fail(bdsm_status s, const std::string& msg) {
  bdsm_internal_set_last_error(msg.c_str());
  return s;
}

// Folds per-engine stats into the group's: times are the slowest engine's,
// work counters (shard-local) are summed, graph-side counters (every engine
// applies the whole batch) are engine 0's.
void fold_stats(bdsm_batch_stats* out, const std::vector<bdsm_batch_stats>& st) {
  if (!out || st.empty()) return;
  *out = st[0];
  for (size_t r = 1; r < st.size(); ++r) {
    const bdsm_batch_stats& s = st[r];
    out->ms_total = std::max(out->ms_total, s.ms_total);
    out->ms_device = std::max(out->ms_device, s.ms_device);
    out->ms_negative = std::max(out->ms_negative, s.ms_negative);
    out->ms_update = std::max(out->ms_update, s.ms_update);
    out->ms_positive = std::max(out->ms_positive, s.ms_positive);
    out->ms_match_kernel = std::max(out->ms_match_kernel, s.ms_match_kernel);
    out->ms_merge_kernel = std::max(out->ms_merge_kernel, s.ms_merge_kernel);
    out->dfs_visits += s.dfs_visits;
    out->work_items += s.work_items;
    out->gen_calls += s.gen_calls;
    out->bytes_phase += s.bytes_phase;
    out->bytes_kernel += s.bytes_kernel;
    out->timed_out |= s.timed_out;
    out->h2d_bytes += s.h2d_bytes;
    out->d2h_bytes += s.d2h_bytes;
    out->kernel_launches += s.kernel_launches;
    out->cub_launches += s.cub_launches;
    out->attempts = std::max(out->attempts, s.attempts);
    out->reruns = std::max(out->reruns, s.reruns);
  }
}

// Sums per-engine counts of one batch; a query whose deadline fired in any
// engine reports 0/0 for that batch (its counts are incomplete).
void fold_counts(bdsm_group* g, const std::vector<std::vector<uint64_t>>& pos,
                 const std::vector<std::vector<uint64_t>>& neg, size_t off, uint64_t* out_pos, uint64_t* out_neg) {
  const size_t nq = g->nverts.size();
  for (size_t q = 0; q < nq; ++q) {
    uint64_t p = 0, n = 0;
    for (size_t r = 0; r < g->engines.size(); ++r) {
      p += pos[r][off + q];
      n += neg[r][off + q];
    }
    if (g->timed[q]) p = n = 0;
    if (out_pos) out_pos[off + q] = p;
    if (out_neg) out_neg[off + q] = n;
  }
}

void note_timeouts(bdsm_group* g) {
  for (size_t q = 0; q < g->nverts.size(); ++q) {
    g->timed[q] = 0;
    for (bdsm_engine* e : g->engines) g->timed[q] |= bdsm_engine_query_timed_out(e, int(q)) == 1;
  }
}

}  // namespace

extern "C" {

bdsm_status bdsm_group_create(const bdsm_graph_desc* graph, const bdsm_options* opts, const int32_t* devices,
                              uint32_t num_devices, bdsm_group** out) {
  if (!out) return group_fail(BDSM_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (!graph || !devices || num_devices == 0) return group_fail(BDSM_INVALID_ARGUMENT, "no devices");
  auto* g = new bdsm_group();
  g->devices.assign(devices, devices + num_devices);
  g->engines.assign(num_devices, nullptr);
  std::vector<bdsm_status> st(num_devices, BDSM_OK);
  std::vector<std::string> msg(num_devices);
  std::vector<std::thread> th;
  for (uint32_t r = 0; r < num_devices; ++r)
    th.emplace_back([&, r] {  // the replicas are built concurrently (graph upload and CSR build per device)
      bdsm_options o{};
      if (opts) o = *opts;
      else {
        o.group_bits = 2;
        o.slack = 0.25f;
        o.pool_reserve = 0.5f;
        o.chunk = 32;
      }
      o.device = devices[r];
      o.shard_rank = r;
      o.shard_world = num_devices;
      st[r] = bdsm_engine_create(graph, &o, &g->engines[r]);
      if (st[r] != BDSM_OK) msg[r] = bdsm_last_error();
    });
  for (auto& t : th) t.join();
  for (uint32_t r = 0; r < num_devices; ++r)
    if (st[r] != BDSM_OK) {
      for (bdsm_engine* e : g->engines)
        if (e) bdsm_engine_destroy(e);
      delete g;
      return group_fail(st[r], "device " + std::to_string(devices[r]) + ": " + msg[r]);
    }
  *out = g;
  return BDSM_OK;
}

void bdsm_group_destroy(bdsm_group* g) {
  if (!g) return;
  for (bdsm_engine* e : g->engines) bdsm_engine_destroy(e);
  delete g;
}

uint32_t bdsm_group_size(bdsm_group* g) { return g ? uint32_t(g->engines.size()) : 0u; }

bdsm_engine* bdsm_group_engine(bdsm_group* g, uint32_t r) {
  return g && r < g->engines.size() ? g->engines[r] : nullptr;
}

int bdsm_group_add_query(bdsm_group* g, const bdsm_query_desc* query) {
  if (!g) return -int(group_fail(BDSM_INVALID_ARGUMENT, "null group"));
  int idx = -1;
  for (bdsm_engine* e : g->engines) {
    const int i = bdsm_engine_add_query(e, query);
    if (i < 0) return i;  // the first engine rejects it (same checks everywhere), nothing added
    if (idx >= 0 && i != idx) return -int(group_fail(BDSM_RUNTIME_ERROR, "engines disagree on the query index"));
    idx = i;
  }
  g->nverts.push_back(query->num_vertices);
  g->timed.push_back(0);
  return idx;
}

bdsm_status bdsm_group_submit_batch(bdsm_group* g, const bdsm_update* updates, size_t n) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  for (size_t r = 0; r < g->engines.size(); ++r) {
    const bdsm_status s = bdsm_engine_submit_batch(g->engines[r], updates, n);
    if (s != BDSM_OK) {
      for (size_t k = 0; k < r; ++k) bdsm_engine_wait(g->engines[k], nullptr, nullptr, nullptr);
      return s;
    }
  }
  return BDSM_OK;
}

bdsm_status bdsm_group_wait(bdsm_group* g, uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  const size_t nq = g->nverts.size(), ne = g->engines.size();
  std::vector<std::vector<uint64_t>> p(ne, std::vector<uint64_t>(nq)), q(ne, std::vector<uint64_t>(nq));
  std::vector<bdsm_batch_stats> st(ne);
  bdsm_status first = BDSM_OK;
  std::string msg;
  for (size_t r = 0; r < ne; ++r) {  // every engine is waited on, also after a failure
    const bdsm_status s = bdsm_engine_wait(g->engines[r], p[r].data(), q[r].data(), &st[r]);
    if (s != BDSM_OK && first == BDSM_OK) {
      first = s;
      msg = bdsm_last_error();
    }
  }
  if (first != BDSM_OK) return group_fail(first, msg);
  note_timeouts(g);
  fold_counts(g, p, q, 0, pos, neg);
  fold_stats(stats, st);
  return BDSM_OK;
}

bdsm_status bdsm_group_apply_batch(bdsm_group* g, const bdsm_update* updates, size_t n, uint64_t* pos,
                                   uint64_t* neg, bdsm_batch_stats* stats) {
  const bdsm_status s = bdsm_group_submit_batch(g, updates, n);
  if (s != BDSM_OK) return s;
  return bdsm_group_wait(g, pos, neg, stats);
}

bdsm_status bdsm_group_apply_stream(bdsm_group* g, const bdsm_update* const* batches, const size_t* sizes,
                                    size_t k, uint64_t* pos, uint64_t* neg, bdsm_batch_stats* stats,
                                    size_t* done) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  const size_t nq = g->nverts.size(), ne = g->engines.size();
  std::vector<std::vector<uint64_t>> p(ne, std::vector<uint64_t>(k * nq)), q(ne, std::vector<uint64_t>(k * nq));
  std::vector<std::vector<bdsm_batch_stats>> st(ne, std::vector<bdsm_batch_stats>(k));
  std::vector<size_t> dn(ne, 0);
  std::vector<bdsm_status> rs(ne, BDSM_OK);
  std::vector<std::string> msg(ne);
  std::vector<std::thread> th;
  for (size_t r = 0; r < ne; ++r)
    th.emplace_back([&, r] {
      rs[r] = bdsm_engine_apply_stream(g->engines[r], batches, sizes, k, 0, p[r].data(), q[r].data(),
                                       st[r].data(), &dn[r]);
      if (rs[r] != BDSM_OK) msg[r] = bdsm_last_error();
    });
  for (auto& t : th) t.join();
  // every replica applies the same batches, so they stop at the same one
  const size_t d = *std::min_element(dn.begin(), dn.end());
  if (done) *done = d;
  std::fill(g->timed.begin(), g->timed.end(), 0);  // streams run without deadlines
  for (size_t i = 0; i < d; ++i) {
    fold_counts(g, p, q, i * nq, pos, neg);
    if (stats) {
      std::vector<bdsm_batch_stats> one(ne);
      for (size_t r = 0; r < ne; ++r) one[r] = st[r][i];
      fold_stats(stats + i, one);
    }
  }
  for (size_t r = 0; r < ne; ++r)
    if (rs[r] != BDSM_OK) return group_fail(rs[r], msg[r]);
  return BDSM_OK;
}

size_t bdsm_group_last_batch_errors(bdsm_group* g, bdsm_update_error* out, size_t cap) {
  return g && !g->engines.empty() ? bdsm_last_batch_errors(g->engines[0], out, cap) : 0;
}

bdsm_status bdsm_group_set_deadline(bdsm_group* g, int query, double seconds_from_now) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  for (bdsm_engine* e : g->engines) {
    const bdsm_status s = bdsm_engine_set_deadline(e, query, seconds_from_now);
    if (s != BDSM_OK) return s;
  }
  return BDSM_OK;
}

bdsm_status bdsm_group_set_query_active(bdsm_group* g, int query, int active) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  for (bdsm_engine* e : g->engines) {
    const bdsm_status s = bdsm_engine_set_query_active(e, query, active);
    if (s != BDSM_OK) return s;
  }
  return BDSM_OK;
}

int bdsm_group_query_timed_out(bdsm_group* g, int query) {
  if (!g || query < 0 || size_t(query) >= g->timed.size()) return -int(BDSM_INVALID_ARGUMENT);
  return g->timed[size_t(query)];
}

bdsm_status bdsm_group_replan(bdsm_group* g, int query) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  for (bdsm_engine* e : g->engines) {
    const bdsm_status s = bdsm_engine_replan(e, query);
    if (s != BDSM_OK) return s;
  }
  return BDSM_OK;
}

bdsm_status bdsm_group_collect_matches(bdsm_group* g, uint64_t cap) {
  if (!g) return group_fail(BDSM_INVALID_ARGUMENT, "null group");
  for (bdsm_engine* e : g->engines) {
    const bdsm_status s = bdsm_engine_collect_matches(e, cap);
    if (s != BDSM_OK) return s;
  }
  g->collect_cap = cap;
  return BDSM_OK;
}

int64_t bdsm_group_matches(bdsm_group* g, int query, int phase, uint32_t* out, size_t cap) {
  if (!g || query < 0 || size_t(query) >= g->nverts.size()) return -int64_t(BDSM_INVALID_ARGUMENT);
  const size_t n = g->nverts[size_t(query)];
  int64_t total = 0;
  std::vector<int64_t> per(g->engines.size());
  for (size_t r = 0; r < g->engines.size(); ++r) {  // counts first: no rows are fetched for a count query
    per[r] = bdsm_engine_matches(g->engines[r], query, phase, nullptr, 0);
    if (per[r] < 0) return per[r];
    total += per[r];
  }
  if (!out) return total;
  std::vector<uint32_t> all;
  for (size_t r = 0; r < g->engines.size(); ++r) {  // each engine holds the matches of its own work units
    // at most the engine's cap of rows exists; rows beyond what it collected stay ~0 and are dropped
    const size_t rows = size_t(std::min<uint64_t>(uint64_t(per[r]), g->collect_cap));
    std::vector<uint32_t> m(rows * n, ~0u);
    const int64_t c2 = bdsm_engine_matches(g->engines[r], query, phase, m.data(), rows);
    if (c2 < 0) return c2;
    for (size_t i = 0; n && i < rows; ++i)
      if (m[i * n] != ~0u) all.insert(all.end(), m.begin() + i * n, m.begin() + (i + 1) * n);
  }
  // one sorted list, as a single engine reports it (src/matcher.cpp:365-366)
  const size_t have = n ? all.size() / n : 0;
  std::vector<size_t> idx(have);
  for (size_t i = 0; i < have; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    return std::lexicographical_compare(all.begin() + a * n, all.begin() + (a + 1) * n, all.begin() + b * n,
                                        all.begin() + (b + 1) * n);
  });
  if (out)
    for (size_t i = 0; i < std::min(have, cap); ++i) std::copy_n(all.begin() + idx[i] * n, n, out + i * n);
  return total;
}

}  // extern "C"
