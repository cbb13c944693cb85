// refdrv — TEST INFRASTRUCTURE (oracle).  A driver over the UNMODIFIED
// reference library (oracle/_ref/libplansim_ref.a, built from
// /root/reference/proj/src by oracle/Makefile).  It stands in for the
// reference CLI (tools/plansim_main.cpp, which needs the absent CLI11): it
// loads the same input files, calls generate_plans + search / simulate_plan
// through the public API, times search(), and dumps every output field so
// tests/ can compare the B200 engine against the reference bit for bit.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs run this binary.
//
// usage:
//   refdrv search   <inputs> [sim flags] [--jobs N] [--repeat R] [--plans a:b]
//                   [--no-search] [--out-result F [--digest]] [--out-plans F] [--out-store F] [--out-trace F]
//   refdrv simulate <inputs> [sim flags] --plan-spec dp,pp,mode:cdp:intra,...
//                   [--out-result F] [--emit-iterations F]
//   refdrv sweep    <inputs> [sim flags] --plan-spec ... --segments N [--subset M]
//                   (prints the SweepTable with hex floats)
//   refdrv synth    --model F --cluster F [--synth-profiles MAXCTX] [--synth-trace ...]
//                   [--out-store F] [--out-trace F]
// inputs:  --model F --cluster F (--profiles F | --synth-profiles MAXCTX)
//          (--trace F | --synth-trace cmean,cstd,gmean,gstd,rate,n,seed)
// sim flags: --objective latency|energy --freqs a,b --batching contiguous|chunked
//          --chunk N --max-batch N --anchor arrival|admission
//          --activation-reserve X --no-embedding --max-combos N
//
// Exit codes follow the reference CLI: 3 InfeasibleError, 4 DataError.

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "json.hpp"
#include "plansim/batching.hpp"
#include "plansim/cluster.hpp"
#include "plansim/common.hpp"
#include "plansim/cost.hpp"
#include "plansim/ir.hpp"
#include "plansim/planner.hpp"
#include "plansim/simulator.hpp"
#include "plansim/traces.hpp"

using namespace plansim;

namespace {

struct Args {
  std::string cmd;
  std::string model, cluster, profiles, trace;
  double synth_max_ctx = 0;
  std::vector<double> synth_trace_params;
  std::string objective = "latency";
  std::vector<double> freqs;
  std::string batching = "contiguous";
  long long chunk = 256, max_batch = 0;
  std::string anchor = "arrival";
  double reserve = 0.10;
  bool no_embedding = false;
  bool digest = false;
  bool no_search = false;
  int max_combos = 65536;
  int jobs = 1, repeat = 1;
  long long plan_lo = 0, plan_hi = -1;
  std::string plan_spec;
  std::string out_result, out_plans, out_store, out_trace, emit_iterations;
  int segments = 4;
  long long subset = 256;
  // the reference CLI's output files, produced with its own recipe
  // (tools/plansim_main.cpp:128-131, :166-172, :184-199)
  std::string out_ranked, out_report, out_summary, out_sweep;
};

std::vector<double> split_doubles(const std::string& s) {
  std::vector<double> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stod(tok));
  return out;
}

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw DataError("usage: refdrv search|simulate|synth ...");
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto v = [&]() -> std::string {
      if (i + 1 >= argc) throw DataError("missing value for " + k);
      return argv[++i];
    };
    if (k == "--model") a.model = v();
    else if (k == "--cluster") a.cluster = v();
    else if (k == "--profiles") a.profiles = v();
    else if (k == "--trace") a.trace = v();
    else if (k == "--synth-profiles") a.synth_max_ctx = std::stod(v());
    else if (k == "--synth-trace") a.synth_trace_params = split_doubles(v());
    else if (k == "--objective") a.objective = v();
    else if (k == "--freqs") a.freqs = split_doubles(v());
    else if (k == "--batching") a.batching = v();
    else if (k == "--chunk") a.chunk = std::stoll(v());
    else if (k == "--max-batch") a.max_batch = std::stoll(v());
    else if (k == "--anchor") a.anchor = v();
    else if (k == "--activation-reserve") a.reserve = std::stod(v());
    else if (k == "--no-embedding") a.no_embedding = true;
    else if (k == "--max-combos") a.max_combos = std::stoi(v());
    else if (k == "--jobs") a.jobs = std::stoi(v());
    else if (k == "--repeat") a.repeat = std::stoi(v());
    else if (k == "--plans") {
      const std::string s = v();
      const auto c = s.find(':');
      a.plan_lo = std::stoll(s.substr(0, c));
      a.plan_hi = std::stoll(s.substr(c + 1));
    } else if (k == "--plan-spec") a.plan_spec = v();
    else if (k == "--out-result") a.out_result = v();
    else if (k == "--digest") a.digest = true;
    else if (k == "--no-search") a.no_search = true;
    else if (k == "--out-plans") a.out_plans = v();
    else if (k == "--out-store") a.out_store = v();
    else if (k == "--out-trace") a.out_trace = v();
    else if (k == "--emit-iterations") a.emit_iterations = v();
    else if (k == "--segments") a.segments = std::stoi(v());
    else if (k == "--out-ranked") a.out_ranked = v();
    else if (k == "--out-report") a.out_report = v();
    else if (k == "--out-summary") a.out_summary = v();
    else if (k == "--out-sweep") a.out_sweep = v();
    else if (k == "--subset") a.subset = std::stoll(v());
    else throw DataError("unknown flag " + k);
  }
  return a;
}

SimConfig sim_config(const Args& a) {
  SimConfig cfg;
  cfg.policy.mode = a.batching == "chunked" ? BatchMode::ChunkedPrefill
                                            : BatchMode::Contiguous;
  cfg.policy.chunk_size = a.chunk;
  cfg.policy.max_batch_size = a.max_batch;
  cfg.ttft_anchor =
      a.anchor == "admission" ? TtftAnchor::Admission : TtftAnchor::Arrival;
  return cfg;
}

PlanOptions plan_options(const Args& a) {
  PlanOptions p;
  p.activation_reserve = a.reserve;
  p.include_embedding = !a.no_embedding;
  p.enumeration.max_cell_combinations = a.max_combos;
  return p;
}

ProfileStore load_store(const Args& a, const ModelSpec& m, const ClusterSpec& c) {
  if (!a.profiles.empty()) return ProfileStore::load_file(a.profiles);
  if (a.synth_max_ctx > 0)
    return synth_profiles(c.device, c, GridSpec::for_model(m, c, a.synth_max_ctx));
  throw DataError("need --profiles or --synth-profiles");
}

Trace load_or_synth_trace(const Args& a) {
  if (!a.trace.empty()) return load_trace_file(a.trace);
  if (a.synth_trace_params.size() == 7) {
    const auto& p = a.synth_trace_params;
    return synth_trace({p[0], p[1]}, {p[2], p[3]}, p[4], int64_t(p[5]),
                       uint64_t(p[6]));
  }
  throw DataError("need --trace or --synth-trace (7 values)");
}

// ---- binary result dump (read by tests/refdump.py) -------------------------
// SHA-256 (FIPS 180-4) of a byte string: the digest form of the result dump
// (--digest) for traces whose per-request arrays are too large to dump.
std::string sha256(const std::string& msg) {
  static const uint32_t K[64] = {
      0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
      0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
      0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
      0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
      0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
      0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
      0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
      0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::string m = msg;
  const uint64_t bits = uint64_t(msg.size()) * 8;
  m.push_back(char(0x80));
  while (m.size() % 64 != 56) m.push_back(char(0));
  for (int i = 7; i >= 0; --i) m.push_back(char((bits >> (8 * i)) & 0xff));
  auto rotr = [](uint32_t x, int n) { return (x >> n) | (x << (32 - n)); };
  for (size_t off = 0; off < m.size(); off += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = uint32_t(uint8_t(m[off + 4 * i])) << 24 | uint32_t(uint8_t(m[off + 4 * i + 1])) << 16 |
             uint32_t(uint8_t(m[off + 4 * i + 2])) << 8 | uint32_t(uint8_t(m[off + 4 * i + 3]));
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
      const uint32_t ch = (e & f) ^ (~e & g);
      const uint32_t t1 = hh + S1 + ch + K[i] + w[i];
      const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
      const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
      const uint32_t t2 = S0 + mj;
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  std::string out;
  for (uint32_t v : h)
    for (int i = 3; i >= 0; --i) out.push_back(char((v >> (8 * i)) & 0xff));
  return out;
}

struct Writer {
  std::string buf;
  void i64(long long v) { buf.append(reinterpret_cast<const char*>(&v), 8); }
  void f64(double v) { buf.append(reinterpret_cast<const char*>(&v), 8); }
  void str(const std::string& s) {
    i64((long long)s.size());
    buf.append(s);
  }
};

void dump_report(Writer& w, long long plan_index, double freq,
                 const SimulationReport& r, bool digest) {
  w.i64(plan_index);
  w.f64(freq);
  w.f64(r.e2e_latency);
  w.f64(r.total_energy);
  w.f64(r.p95_latency);
  w.f64(r.mean_ttft);
  w.f64(r.mean_tpot);
  w.f64(r.mfu);
  w.f64(r.mbu);
  w.i64(r.num_completed);
  w.i64(r.num_rejected);
  w.i64(r.num_iterations);
  w.i64(r.max_batch_observed);
  w.str(r.plan_encoding);
  Writer pr, rj;
  Writer& a = digest ? pr : w;
  Writer& b = digest ? rj : w;
  w.i64((long long)r.per_request.size());
  for (const auto& m : r.per_request) {
    a.i64(m.id);
    a.f64(m.ttft);
    a.f64(m.tpot);
    a.f64(m.e2e);
    a.i64(m.gen_len);
  }
  if (digest) w.buf.append(sha256(pr.buf));
  w.i64((long long)r.rejected_ids.size());
  for (long long id : r.rejected_ids) b.i64(id);
  if (digest) w.buf.append(sha256(rj.buf));
}

void write_result(const std::string& path,
                  const std::vector<std::pair<long long, double>>& keys,
                  const std::vector<const SimulationReport*>& reports,
                  const ProfileStore& store, bool digest = false) {
  Writer w;
  w.buf.append("PSGR", 4);
  w.i64(digest ? 2 : 1);  // 2: per-request / rejected arrays as SHA-256 digests
  w.i64((long long)reports.size());
  for (size_t i = 0; i < reports.size(); ++i)
    dump_report(w, keys[i].first, keys[i].second, *reports[i], digest);
  const auto warns = store.warnings();
  w.i64((long long)warns.size());
  for (const auto& s : warns) w.str(s);
  write_file(path, w.buf);
}

std::string plans_json(const std::vector<ExecutionPlan>& plans) {
  nlohmann::ordered_json arr = nlohmann::ordered_json::array();
  for (const auto& p : plans) {
    nlohmann::ordered_json d;
    d["encoding"] = p.scheme.encoding;
    d["model_dp"] = p.scheme.model_dp;
    d["num_stages"] = p.scheme.num_stages;
    d["stage_devices"] = p.scheme.stage_devices;
    d["stage_repetitions"] = p.scheme.stage_repetitions;
    d["compute_dtype"] = int(p.compute_dtype);
    d["kv_bytes_per_token"] = p.kv_bytes_per_token;
    d["kv_budget_per_replica"] = p.kv_budget_per_replica;
    d["static_bytes_per_device"] = p.static_bytes_per_device;
    d["p2p_payload_per_token"] = p.p2p_payload_per_token;
    d["shape"] = {p.op_shape.model_hidden, p.op_shape.head_dim,
                  p.op_shape.kv_elems_per_task_token};
    d["cells"] = nlohmann::ordered_json::array();
    for (const auto& c : p.scheme.cells)
      d["cells"].push_back({{"kind", int(c.cell.kind)},
                            {"mode", int(c.mode)},
                            {"cell_dp", c.cell_dp},
                            {"intra_degree", c.intra_degree},
                            {"op", int(c.op)},
                            {"query_tasks", c.query_tasks},
                            {"query_width", c.query_width},
                            {"token_scale", c.token_scale},
                            {"weight_bytes_per_device",
                             c.mapping.weight_bytes_per_device}});
    d["collectives"] = nlohmann::ordered_json::array();
    for (const auto& rc : p.block_collectives)
      d["collectives"].push_back({{"kind", int(rc.kind)},
                                  {"payload_bytes_per_token", rc.payload_bytes_per_token},
                                  {"token_share", rc.token_share},
                                  {"num_devices", rc.num_devices},
                                  {"num_nodes", rc.num_nodes},
                                  {"groups_per_stage", rc.groups_per_stage}});
    d["p2p_boundary_nodes"] = p.p2p_boundary_nodes;
    d["assignment"] = p.assignment.phys;
    arr.push_back(d);
  }
  return arr.dump() + "\n";
}

ExecutionPlan plan_from_spec(const std::string& spec, const ModelSpec& m,
                             const BlockSpec& block, const ClusterSpec& c,
                             const PlanOptions& opts) {
  // dp,pp,mode:cdp:intra,mode:cdp:intra,...
  std::vector<std::string> parts;
  std::stringstream ss(spec);
  std::string tok;
  while (std::getline(ss, tok, ',')) parts.push_back(tok);
  if (parts.size() < 3) throw DataError("bad --plan-spec");
  std::vector<CellChoice> cells;
  for (size_t i = 2; i < parts.size(); ++i) {
    CellChoice ch;
    const auto c1 = parts[i].find(':');
    const auto c2 = parts[i].find(':', c1 + 1);
    ch.mode = parts[i].substr(0, c1) == "ep" ? ParallelMode::EP : ParallelMode::TP;
    ch.cell_dp = std::stoi(parts[i].substr(c1 + 1, c2 - c1 - 1));
    ch.intra_degree = std::stoi(parts[i].substr(c2 + 1));
    cells.push_back(ch);
  }
  return build_plan(m, block, c, std::stoi(parts[0]), std::stoi(parts[1]), cells,
                    opts);
}

int run(const Args& a) {
  const ModelSpec model = parse_model_config_file(a.model);
  const BlockSpec block = to_transformer_ir(model);
  const ClusterSpec cluster = parse_cluster_spec_file(a.cluster);

  if (a.cmd == "synth") {
    if (!a.out_store.empty())
      write_file(a.out_store, load_store(a, model, cluster).serialize());
    if (!a.out_trace.empty())
      write_file(a.out_trace, serialize_trace(load_or_synth_trace(a)));
    return 0;
  }

  const ProfileStore store = load_store(a, model, cluster);
  const Trace trace = load_or_synth_trace(a);
  if (!a.out_store.empty()) write_file(a.out_store, store.serialize());
  if (!a.out_trace.empty()) write_file(a.out_trace, serialize_trace(trace));
  const SimConfig cfg = sim_config(a);
  const PlanOptions popt = plan_options(a);

  if (a.cmd == "simulate") {
    const ExecutionPlan plan = plan_from_spec(a.plan_spec, model, block, cluster, popt);
    SimConfig run_cfg = cfg;
    if (!a.freqs.empty()) run_cfg.freq_ghz = a.freqs.front();
    run_cfg.emit_iterations = !a.emit_iterations.empty();
    const auto t0 = std::chrono::steady_clock::now();
    const SimulationReport r =
        simulate_plan(plan, model, cluster, trace, store, run_cfg);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!a.emit_iterations.empty())
      write_file(a.emit_iterations, iterations_to_jsonl(r));
    if (!a.out_report.empty()) {  // cmd_simulate: records live in the JSONL stream
      SimulationReport rr = r;
      rr.iterations.clear();
      write_file(a.out_report, report_to_json(rr));
    }
    if (!a.out_summary.empty()) write_file(a.out_summary, report_summary_line(r) + "\n");
    if (!a.out_result.empty())
      write_result(a.out_result, {{0LL, r.frequency_ghz}}, {&r}, store);
    if (!a.out_plans.empty()) write_file(a.out_plans, plans_json({plan}));
    std::printf("{\"cmd\":\"simulate\",\"iterations\":%lld,\"seconds\":%.9g}\n",
                (long long)r.num_iterations, dt);
    return 0;
  }

  if (a.cmd == "sweep") {
    const ExecutionPlan plan = plan_from_spec(a.plan_spec, model, block, cluster, popt);
    SimConfig run_cfg = cfg;
    if (!a.freqs.empty()) run_cfg.freq_ghz = a.freqs.front();
    const SweepTable t =
        sweep_max_batch(plan, model, cluster, trace, store, run_cfg, a.segments, a.subset);
    if (!a.out_plans.empty()) write_file(a.out_plans, plans_json({plan}));
    if (!a.out_sweep.empty()) {  // cmd_sweep's table
      nlohmann::ordered_json doc;
      doc["observed_max_batch"] = t.observed_max_batch;
      doc["rows"] = nlohmann::ordered_json::array();
      for (const auto& row : t.rows)
        doc["rows"].push_back({{"max_batch_size", row.max_batch_size},
                               {"mean_tpot_s", row.mean_tpot},
                               {"mean_ttft_s", row.mean_ttft},
                               {"e2e_latency_s", row.e2e_latency}});
      write_file(a.out_sweep, doc.dump(2) + "\n");
    }
    std::printf("{\"cmd\":\"sweep\",\"observed_max_batch\":%lld,\"rows\":[",
                (long long)t.observed_max_batch);
    for (size_t i = 0; i < t.rows.size(); ++i)
      std::printf("%s[%lld,\"%a\",\"%a\",\"%a\"]", i ? "," : "",
                  (long long)t.rows[i].max_batch_size, t.rows[i].mean_tpot, t.rows[i].mean_ttft,
                  t.rows[i].e2e_latency);
    std::printf("]}\n");
    return 0;
  }

  if (a.cmd != "search") throw DataError("unknown command " + a.cmd);
  std::vector<ExecutionPlan> plans = generate_plans(model, block, cluster, popt);
  const size_t total_plans = plans.size();
  if (a.plan_hi >= 0) {
    const size_t lo = size_t(std::min<long long>(a.plan_lo, (long long)plans.size()));
    const size_t hi = size_t(std::min<long long>(a.plan_hi, (long long)plans.size()));
    plans = std::vector<ExecutionPlan>(plans.begin() + lo, plans.begin() + hi);
  }
  if (!a.out_plans.empty()) write_file(a.out_plans, plans_json(plans));
  if (a.no_search) {  // generate_plans only (input-parity tests)
    std::printf("{\"cmd\":\"search\",\"plans\":%zu,\"searched\":false}\n", plans.size());
    return 0;
  }
  const Objective obj =
      a.objective == "energy" ? Objective::Energy : Objective::Latency;

  double best = 1e300;
  RankedPlans ranked;
  for (int rep = 0; rep < std::max(1, a.repeat); ++rep) {
    const auto t0 = std::chrono::steady_clock::now();
    ranked = search(plans, model, cluster, trace, store, obj, a.freqs, cfg, a.jobs);
    best = std::min(best, std::chrono::duration<double>(
                              std::chrono::steady_clock::now() - t0).count());
  }
  long long iters = 0;
  for (const auto& e : ranked.entries) iters += e.report.num_iterations;
  double ranked_s = 0.0;
  if (!a.out_ranked.empty()) {  // cmd_search's ranked.json
    const auto t0 = std::chrono::steady_clock::now();
    nlohmann::ordered_json doc = nlohmann::ordered_json::array();
    for (const auto& e : ranked.entries)
      doc.push_back(nlohmann::ordered_json::parse(report_to_json(e.report)));
    write_file(a.out_ranked, doc.dump(2) + "\n");
    ranked_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  if (!a.out_result.empty()) {
    std::vector<std::pair<long long, double>> keys;
    std::vector<const SimulationReport*> reps;
    for (const auto& e : ranked.entries) {
      keys.push_back({(long long)e.plan_index, e.freq_ghz});
      reps.push_back(&e.report);
    }
    write_result(a.out_result, keys, reps, store, a.digest);
  }
  std::printf(
      "{\"cmd\":\"search\",\"plans\":%zu,\"plans_total\":%zu,\"entries\":%zu,"
      "\"requests\":%zu,\"plan_iterations\":%lld,\"jobs\":%d,\"repeat\":%d,"
      "\"search_s_best\":%.9g,\"plan_iter_per_s\":%.9g,\"ranked_s\":%.9g,\"best\":\"%s\"}\n",
      plans.size(), total_plans, ranked.entries.size(), trace.requests.size(), iters,
      a.jobs, a.repeat, best, double(iters) / best, ranked_s,
      ranked.entries.empty() ? "" : ranked.entries.front().report.plan_encoding.c_str());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(parse(argc, argv));
  } catch (const InfeasibleError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  } catch (const DataError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
}
