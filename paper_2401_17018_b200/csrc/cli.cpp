// `bdsm run` — drop-in for the reference CLI (tools/bdsm.cpp:26-156) on the
// B200 engine.  Same flags and the same outputs: the stdout summary line
// (tools/bdsm.cpp:148-150) and the report CSVs latency.csv, deltas.csv,
// stages.csv, utilization.csv (src/bench.cpp:566-591).  Text formats follow
// src/io.cpp:16-148 (graph/query `v id label` / `e u v [label]`, `#`
// comments; stream `+ u v [label]` / `- u v`, blank line ends a batch).
//
// The per-batch loop mirrors run_pipeline (src/bench.cpp:370-564): per query a
// cumulative time budget (--timeout; the first overrun marks the query
// unsolved and drops its counts from that batch on), deltas summed over the
// live queries, drift replanning when the candidate columns moved by more than
// 0.25 (src/bench.cpp:451-453; it changes the matching order only, never the
// counts).  The device graph is the single source of truth, so the
// reference's preprocess replica (src/bench.cpp:388-404) is not needed.
//
// `bdsm generate` (not in the reference) runs only the seeded generators and
// writes query_<i>.txt / stream.txt as `bdsm run` would, without a GPU.
//
// GPU-build differences: --coalesce defaults to off and "on" runs the EXACT
// coalesced search (one search per automorphism orbit of directed query
// edges, counted with the orbit size: the counts equal "off"; the reference's
// coalesced search misses matches);
// --workers/--group-size/--stealing are accepted and ignored (the device
// schedules its own warps); utilization.csv reports the device.
#include <sys/stat.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bdsm_gpu.hpp"
#include "textio.hpp"

namespace {

using bdsm::gpu::Engine;
using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void mkdirs(const std::string& path) {
  std::string cur;
  std::stringstream ss(path);
  std::string part;
  if (!path.empty() && path[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    ::mkdir(cur.c_str(), 0755);
  }
}

std::string join(const std::string& dir, const std::string& name) {
  if (dir.empty()) return name;
  return dir.back() == '/' ? dir + name : dir + "/" + name;
}

struct Args {
  std::string graph, query, gen_queries, stream, gen_stream, stealing = "off", coalesce = "off", out = "out",
                                                                          dump_plan;
  unsigned long workers = 1, group_size = 4;
  double timeout = 1800.0;
  unsigned long long seed = 1;
  unsigned group_bits = 2;
  bool no_pipeline = false, dump_matches = false;
  int device = 0;
  std::vector<std::int32_t> devices;  // --devices a,b,...: a multi-device group (work units split over them)
  bool generate_only = false;
};

[[noreturn]] void usage(const std::string& msg) {
  std::cerr << msg << "\n"
            << "Usage: bdsm run|generate --graph FILE (--query FILE | --gen-queries cat,size,count)\n"
               "                (--stream FILE | --gen-stream rate,mode,batches[,kcore])\n"
               "                [--workers N] [--group-size N] [--stealing off|passive|active]\n"
               "                [--coalesce on|off] [--timeout S] [--seed N] [--out DIR]\n"
               "                [--group-bits N] [--dump-plan FILE] [--no-pipeline] [--dump-matches]\n"
               "                [--device N] [--devices N,N,...]\n";
  std::exit(msg.empty() ? 0 : 109);  // CLI11 parse errors exit non-zero
}

Args parse(int argc, char** argv) {
  if (argc < 2) usage("A subcommand is required");
  std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") usage("");
  if (sub != "run" && sub != "generate") usage("The following argument was not expected: " + sub);
  Args a;
  a.generate_only = sub == "generate";
  std::map<std::string, std::string*> str = {
      {"--graph", &a.graph},       {"--query", &a.query},   {"--gen-queries", &a.gen_queries},
      {"--stream", &a.stream},     {"--gen-stream", &a.gen_stream}, {"--stealing", &a.stealing},
      {"--coalesce", &a.coalesce}, {"--out", &a.out},       {"--dump-plan", &a.dump_plan}};
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i], v;
    auto eq = k.find('=');
    bool has_eq = k.rfind("--", 0) == 0 && eq != std::string::npos;
    if (has_eq) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    }
    if (k == "-h" || k == "--help") usage("");
    if (k == "--no-pipeline") {
      a.no_pipeline = true;
      continue;
    }
    if (k == "--dump-matches") {
      a.dump_matches = true;
      continue;
    }
    if (!has_eq) {
      if (i + 1 >= argc) usage(k + " requires an argument");
      v = argv[++i];
    }
    try {
      if (str.count(k)) *str[k] = v;
      else if (k == "--workers") a.workers = std::stoul(v);
      else if (k == "--group-size") a.group_size = std::stoul(v);
      else if (k == "--timeout") a.timeout = std::stod(v);
      else if (k == "--seed") a.seed = std::stoull(v);
      else if (k == "--group-bits") a.group_bits = unsigned(std::stoul(v));
      else if (k == "--device") a.device = std::stoi(v);
      else if (k == "--devices") {
        std::stringstream ds(v);
        std::string tok;
        while (std::getline(ds, tok, ',')) a.devices.push_back(std::stoi(tok));
        if (a.devices.empty()) throw std::invalid_argument("empty device list");
      }
      else usage("The following argument was not expected: " + k);
    } catch (const std::logic_error&) {
      usage("bad value for " + k + ": " + v);
    }
  }
  if (a.graph.empty()) usage("--graph is required");
  return a;
}

std::vector<std::string> split_csv(const std::string& s) {
  std::vector<std::string> parts;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) parts.push_back(item);
  return parts;
}

struct QueryRun {
  bdsm::text::Query q;
  std::string category;
  std::vector<std::uint64_t> plan_cols;  // column sizes the current order was built from
  double spent = 0;
  bool solved = true;
};

bdsm::text::StreamSpec stream_spec(const Args& args) {
  auto parts = split_csv(args.gen_stream);
  if (parts.size() < 3) throw std::runtime_error("--gen-stream wants <rate,mode,batches[,k]>");
  bdsm::text::StreamSpec spec;
  spec.rate = std::stod(parts[0]);
  spec.mode = parts[1];
  spec.batches = std::stoul(parts[2]);
  if (parts.size() > 3) spec.kcore = std::uint32_t(std::stoul(parts[3]));
  spec.seed = args.seed;
  return spec;
}

int generate(const Args& args, const bdsm::text::Graph& g) {
  mkdirs(args.out);
  if (!args.gen_queries.empty()) {
    auto parts = split_csv(args.gen_queries);
    if (parts.size() != 3) throw std::runtime_error("--gen-queries wants <cat,size,count>");
    auto qs = bdsm::text::generate_queries(g, parts[0], std::stoul(parts[1]), std::stoul(parts[2]), args.seed);
    for (std::size_t i = 0; i < qs.size(); ++i) {
      std::ofstream qf(join(args.out, "query_" + std::to_string(i) + ".txt"));
      bdsm::text::save_query(qf, qs[i]);
    }
  }
  if (!args.gen_stream.empty()) {
    auto stream = bdsm::text::generate_stream(g, stream_spec(args));
    std::ofstream sf(join(args.out, "stream.txt"));
    bdsm::text::save_stream(sf, stream);
  }
  return 0;
}

int run(const Args& args) {
  if (args.stealing != "off" && args.stealing != "passive" && args.stealing != "active")
    throw std::invalid_argument("unknown stealing mode: " + args.stealing);  // src/scheduler.cpp:16
  if (args.coalesce != "on" && args.coalesce != "off") throw std::invalid_argument("--coalesce wants on|off");
  if (!args.dump_plan.empty())
    throw std::runtime_error("--dump-plan is not supported by the GPU build (plan_to_json is a debug dump)");

  bdsm::text::Graph g = bdsm::text::load_graph_file(args.graph);
  if (args.generate_only) return generate(args, g);
  // LabeledGraph::build_from_edges happens at load time in the reference
  // (src/io.cpp:56-59): graph errors surface before any generator runs.
  bdsm_options opts = Engine::defaults();
  opts.group_bits = args.group_bits;
  opts.device = args.device;
  opts.coalesce = args.coalesce == "on" ? 1u : 0u;
  Engine engine(g.vertices, g.edges, opts, args.devices);
  std::vector<QueryRun> queries;
  if (!args.query.empty()) {
    queries.push_back({bdsm::text::load_query_file(args.query), "file", {}, 0, true});
  } else if (!args.gen_queries.empty()) {
    auto parts = split_csv(args.gen_queries);
    if (parts.size() != 3) throw std::runtime_error("--gen-queries wants <cat,size,count>");
    auto qs = bdsm::text::generate_queries(g, parts[0], std::stoul(parts[1]), std::stoul(parts[2]), args.seed);
    mkdirs(args.out);
    for (std::size_t i = 0; i < qs.size(); ++i) {
      std::ofstream qf(join(args.out, "query_" + std::to_string(i) + ".txt"));
      bdsm::text::save_query(qf, qs[i]);
      queries.push_back({std::move(qs[i]), parts[0], {}, 0, true});
    }
  } else {
    throw std::runtime_error("need --query or --gen-queries");
  }

  std::vector<std::vector<bdsm::gpu::EdgeUpdate>> stream;
  if (!args.stream.empty()) {
    stream = bdsm::text::load_stream_file(args.stream);
  } else if (!args.gen_stream.empty()) {
    stream = bdsm::text::generate_stream(g, stream_spec(args));
    mkdirs(args.out);
    std::ofstream sf(join(args.out, "stream.txt"));
    bdsm::text::save_stream(sf, stream);
  } else {
    throw std::runtime_error("need --stream or --gen-stream");
  }

  // --dump-matches: bounded materialisation (BDSM_DUMP_CAP matches per query and phase)
  const char* capenv = std::getenv("BDSM_DUMP_CAP");
  const std::uint64_t dump_cap = capenv ? std::strtoull(capenv, nullptr, 10) : (1ull << 22);
  if (args.dump_matches) engine.collect_matches(dump_cap);
  std::vector<int> qid(queries.size());
  for (std::size_t i = 0; i < queries.size(); ++i) {
    auto t0 = Clock::now();
    qid[i] = engine.add_query(queries[i].q.labels, queries[i].q.edges);
    queries[i].plan_cols = engine.column_sizes(qid[i], std::uint32_t(queries[i].q.labels.size()));
    queries[i].spent = since(t0);
    if (queries[i].spent > args.timeout) queries[i].solved = false;
  }

  struct Delta {
    std::uint64_t pos = 0, neg = 0;
  };
  std::vector<Delta> deltas;
  struct Stage {
    double pre = 0, match = 0;
  };
  std::vector<Stage> stages;
  double busy = 0, total = 0;
  // run_pipeline (src/bench.cpp:370-564): by default the stages overlap —
  // batch i+1 is packed on the host while batch i runs on the device, and
  // batch i's report is written while batch i+1 runs (the reference's
  // preprocess / match / postprocess threads); --no-pipeline runs them in turn.
  const bool pipelined = !args.no_pipeline && stream.size() > 1;
  auto prepare = [&](std::size_t bi) {  // deadlines and the live set of batch bi
    std::size_t live = 0;
    for (std::size_t i = 0; i < queries.size(); ++i) {
      // an unsolved query is no longer matched (src/bench.cpp:463-467); a live
      // one gets the rest of its budget as this batch's deadline
      engine.set_query_active(qid[i], queries[i].solved);
      if (!queries[i].solved) continue;
      ++live;
      engine.set_deadline(qid[i], std::max(args.timeout - queries[i].spent, 1e-9));
    }
    (void)bi;
    return live;
  };
  std::vector<bdsm_update> packed = stream.empty() ? std::vector<bdsm_update>() : Engine::pack(stream[0]);
  std::size_t live = 0;
  Clock::time_point t_submit;
  double host_pre = 0;
  if (!stream.empty()) {
    live = prepare(0);
    t_submit = Clock::now();
    engine.submit_packed(packed);
  }
  for (std::size_t bi = 0; bi < stream.size(); ++bi) {
    // preprocess stage of batch bi+1, overlapped with batch bi on the device
    std::vector<bdsm_update> next;
    auto tp = Clock::now();
    if (pipelined && bi + 1 < stream.size()) next = Engine::pack(stream[bi + 1]);
    host_pre = since(tp);
    bdsm_batch_stats st{};
    std::vector<bdsm::gpu::Counts> c = engine.wait(&st);
    double wall = since(t_submit);
    Delta d;
    for (std::size_t i = 0; i < queries.size(); ++i) {
      QueryRun& q = queries[i];
      if (!q.solved) continue;
      // the whole batch is charged to every live query (the engine runs them in one call)
      q.spent += live ? wall : 0.0;
      if (engine.query_timed_out(qid[i]) || q.spent > args.timeout) {
        q.solved = false;
        continue;
      }
      d.pos += c[i].positive;
      d.neg += c[i].negative;
      // drift replanning (src/bench.cpp:451-453, plan_column_drift src/query_analysis.cpp:449-459)
      std::vector<std::uint64_t> now = engine.column_sizes(qid[i], std::uint32_t(q.q.labels.size()));
      std::uint64_t tot = 0, del = 0;
      for (std::size_t u = 0; u < now.size(); ++u) {
        tot += q.plan_cols[u];
        del += now[u] > q.plan_cols[u] ? now[u] - q.plan_cols[u] : q.plan_cols[u] - now[u];
      }
      if (double(del) / double(std::max<std::uint64_t>(tot, 1)) > 0.25) {
        engine.replan(qid[i]);
        q.plan_cols = now;
      }
    }
    // the materialised matches of batch bi are read before batch bi+1 reuses the buffers
    std::vector<std::string> dump;
    if (args.dump_matches) {  // src/bench.cpp:484-491 (format_match, src/matcher.cpp:391-398)
      for (std::size_t i = 0; i < queries.size(); ++i) {
        if (!queries[i].solved) continue;
        const std::uint32_t n = std::uint32_t(queries[i].q.labels.size());
        for (int phase : {1, 0}) {
          const std::vector<std::uint32_t> m = engine.matches(qid[i], phase, n);
          if (m.size() / std::max<std::uint32_t>(n, 1) > dump_cap)
            throw std::runtime_error("too many matches to dump (raise BDSM_DUMP_CAP)");
          for (std::size_t k = 0; k + n <= m.size(); k += n) {
            std::string line(1, phase ? '+' : '-');
            for (std::uint32_t u = 0; u < n; ++u) line += " u" + std::to_string(u) + ":v" + std::to_string(m[k + u]);
            dump.push_back(std::move(line));
          }
        }
      }
    }
    // submit batch bi+1 before the postprocess stage of batch bi
    if (bi + 1 < stream.size()) {
      live = prepare(bi + 1);
      if (!pipelined) {
        auto tq = Clock::now();
        next = Engine::pack(stream[bi + 1]);
        host_pre = since(tq);
      }
      t_submit = Clock::now();
      engine.submit_packed(next);
    }
    // postprocess stage of batch bi (overlapped with batch bi+1 when pipelined)
    if (args.dump_matches) {
      mkdirs(args.out);
      std::ofstream mf(join(args.out, "matches_batch" + std::to_string(bi) + ".txt"));
      for (const std::string& line : dump) mf << line << '\n';
    }
    deltas.push_back(d);
    // preprocess = the graph update (device merge + refresh) and the host
    // packing of the batch; match = the two matching phases (src/bench.cpp:394-402, :470)
    stages.push_back({st.ms_update * 1e-3 + host_pre, (st.ms_negative + st.ms_positive) * 1e-3});
    busy += (st.ms_match_kernel + st.ms_merge_kernel) * 1e-3;
    total += wall;
  }

  // emit_report (src/bench.cpp:566-591)
  mkdirs(args.out);
  {
    std::ofstream f(join(args.out, "latency.csv"));
    f << "query_id,category,size,seconds,solved\n";
    for (std::size_t i = 0; i < queries.size(); ++i)
      f << i << ',' << queries[i].category << ',' << queries[i].q.labels.size() << ',' << queries[i].spent << ','
        << (queries[i].solved ? 1 : 0) << '\n';
  }
  {
    std::ofstream f(join(args.out, "deltas.csv"));
    f << "batch,positive,negative\n";
    for (std::size_t i = 0; i < deltas.size(); ++i) f << i << ',' << deltas[i].pos << ',' << deltas[i].neg << '\n';
  }
  {
    std::ofstream f(join(args.out, "stages.csv"));
    f << "batch,preprocess_s,match_s,ratio\n";
    for (std::size_t i = 0; i < stages.size(); ++i) {
      double t = stages[i].pre + stages[i].match;
      f << i << ',' << stages[i].pre << ',' << stages[i].match << ',' << (t > 0 ? stages[i].pre / t : 0.0) << '\n';
    }
  }
  {
    std::ofstream f(join(args.out, "utilization.csv"));
    f << "worker,busy_seconds,total_seconds,fraction\n";
    f << 0 << ',' << busy << ',' << total << ',' << (total > 0 ? busy / total : 0.0) << '\n';
  }
  std::uint64_t pos = 0, neg = 0;
  std::size_t unsolved = 0;
  for (const auto& d : deltas) {
    pos += d.pos;
    neg += d.neg;
  }
  for (const auto& q : queries) unsolved += q.solved ? 0 : 1;
  std::cout << "batches=" << deltas.size() << " positive=" << pos << " negative=" << neg
            << " unsolved_queries=" << unsolved << " reports=" << args.out << "/\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args args = parse(argc, argv);
  try {
    return run(args);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
