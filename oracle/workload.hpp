// TEST / BENCH INFRASTRUCTURE ONLY.
//
// Binary workload file shared by bench.py (writer, numpy) and the CPU
// baselines oracle/ref_bench.cpp and oracle/oracle_bench.cpp (readers), so the
// GPU engine and both CPU paths consume bit-identical graphs, queries and
// update streams (SURVEY.md §8(d) "one generator feeds both CPU and GPU").
//
// Layout, little endian:
//   char magic[8] = "BDSMWL01"
//   u64 nv, ne, has_elab, qn, qm, nbatches, total_updates
//   u32 vlabels[nv]
//   u32 eu[ne]; u32 ev[ne]; if has_elab: u32 elab[ne]   (0xffffffff = none)
//   u32 qlabels[qn]; u32 qa[qm]; u32 qb[qm]; u32 qlab[qm]
//   u64 batch_offsets[nbatches + 1]
//   u32 uu[T]; u32 uv[T]; u32 uop[T] (0 insert, 1 delete); u32 ulab[T]
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace wl {

struct Workload {
  std::uint64_t nv = 0, ne = 0, qn = 0, qm = 0, nbatches = 0, total = 0;
  bool has_elab = false;
  std::vector<std::uint32_t> vlabels, eu, ev, elab;
  std::vector<std::uint32_t> qlabels, qa, qb, qlab;
  std::vector<std::uint64_t> boffs;
  std::vector<std::uint32_t> uu, uv, uop, ulab;
};

inline void read_exact(std::FILE* f, void* p, std::size_t bytes) {
  if (bytes && std::fread(p, 1, bytes, f) != bytes) throw std::runtime_error("short workload file");
}

template <typename T>
inline void read_vec(std::FILE* f, std::vector<T>& v, std::uint64_t n) {
  v.resize(n);
  read_exact(f, v.data(), n * sizeof(T));
}

inline Workload load(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open " + path);
  Workload w;
  char magic[8];
  read_exact(f, magic, 8);
  if (std::memcmp(magic, "BDSMWL01", 8) != 0) throw std::runtime_error("bad workload magic");
  std::uint64_t hdr[7];
  read_exact(f, hdr, sizeof(hdr));
  w.nv = hdr[0];
  w.ne = hdr[1];
  w.has_elab = hdr[2] != 0;
  w.qn = hdr[3];
  w.qm = hdr[4];
  w.nbatches = hdr[5];
  w.total = hdr[6];
  read_vec(f, w.vlabels, w.nv);
  read_vec(f, w.eu, w.ne);
  read_vec(f, w.ev, w.ne);
  if (w.has_elab) read_vec(f, w.elab, w.ne);
  read_vec(f, w.qlabels, w.qn);
  read_vec(f, w.qa, w.qm);
  read_vec(f, w.qb, w.qm);
  read_vec(f, w.qlab, w.qm);
  read_vec(f, w.boffs, w.nbatches + 1);
  read_vec(f, w.uu, w.total);
  read_vec(f, w.uv, w.total);
  read_vec(f, w.uop, w.total);
  read_vec(f, w.ulab, w.total);
  std::fclose(f);
  return w;
}

}  // namespace wl
