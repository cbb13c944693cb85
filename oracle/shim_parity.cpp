// shim_parity — TEST INFRASTRUCTURE.  Runs the reference's plansim::search
// (oracle/_ref/libplansim_ref.a) and the drop-in plansim_gpu::search
// (paper_2411_17651_b200/csrc/shim, over libpsg.so) on the SAME in-memory
// reference objects and compares every RankedPlans field: ranked order, all
// SimulationReport scalars (bit-exact, MFU/MBU included), every
// per_request metric, rejected ids, and the store's clamp-warning set.
//
// usage: shim_parity --model F --cluster F (--profiles F | --synth-profiles X)
//        (--trace F | --synth-trace a,b,c,d,rate,n,seed) [--objective energy]
//        [--freqs a,b] [--batching chunked --chunk N] [--max-batch N]
//        [--anchor admission] [--jobs N] [--threads T] [--drop-table OP]
//        [--single K [--sweep-segments S --sweep-subset M]]
// --single K additionally compares simulate_plan(plans[K]) with
// emit_iterations (every IterationRecord) and, with --sweep-segments,
// sweep_max_batch (every SweepRow).
// Prints one JSON line; exit 0 on full parity, 1 on a mismatch, 3/4 when both
// implementations raise the same InfeasibleError / DataError.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "plansim/simulator.hpp"
#include "plansim_gpu.hpp"

using namespace plansim;

namespace {

std::vector<double> doubles(const std::string& s) {
  std::vector<double> v;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) v.push_back(std::stod(t));
  return v;
}

std::string drop_lines(const std::string& text, const std::string& needle) {
  std::istringstream in(text);
  std::ostringstream out;
  std::string line;
  while (std::getline(in, line))
    if (line.find(needle) == std::string::npos) out << line << "\n";
  return out.str();
}

// Mismatches between two rankings (every report field, per-request metrics, rejected ids).
int diff_ranked(const RankedPlans& a, const RankedPlans& b, std::string& first) {
  int bad = 0;
  auto miss = [&](const std::string& what) {
    if (!bad++) first = what;
  };
  if (a.entries.size() != b.entries.size()) miss("entry count");
  for (size_t i = 0; i < a.entries.size() && i < b.entries.size(); ++i) {
    const auto& x = a.entries[i];
    const auto& y = b.entries[i];
    const auto& r = x.report;
    const auto& g = y.report;
    const std::string at = " at rank " + std::to_string(i) + " " + r.plan_encoding;
    if (x.plan_index != y.plan_index || x.freq_ghz != y.freq_ghz) miss("entry identity" + at);
    if (r.plan_encoding != g.plan_encoding || r.frequency_ghz != g.frequency_ghz) miss("encoding" + at);
    if (r.e2e_latency != g.e2e_latency || r.total_energy != g.total_energy ||
        r.p95_latency != g.p95_latency || r.mean_ttft != g.mean_ttft || r.mean_tpot != g.mean_tpot)
      miss("latency/energy/ttft/tpot" + at);
    if (r.mfu != g.mfu || r.mbu != g.mbu) miss("mfu/mbu" + at);
    if (r.num_completed != g.num_completed || r.num_rejected != g.num_rejected ||
        r.num_iterations != g.num_iterations || r.max_batch_observed != g.max_batch_observed)
      miss("counters" + at);
    if (r.rejected_ids != g.rejected_ids) miss("rejected ids" + at);
    if (r.per_request.size() != g.per_request.size()) {
      miss("per_request size" + at);
    } else {
      for (size_t k = 0; k < r.per_request.size(); ++k) {
        const auto& p = r.per_request[k];
        const auto& q = g.per_request[k];
        if (p.id != q.id || p.ttft != q.ttft || p.tpot != q.tpot || p.e2e != q.e2e || p.gen_len != q.gen_len) {
          miss("per_request" + at);
          break;
        }
      }
    }
  }
  return bad;
}

}  // namespace

int main(int argc, char** argv) {
  std::string model_p, cluster_p, prof_p, trace_p, objective = "latency", drop;
  double synth_ctx = 0;
  std::vector<double> synth_tr, freqs;
  SimConfig cfg;
  int jobs = 1, single = -1, sweep_segments = 0, threads = 1;
  long long sweep_subset = 256;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--model") model_p = v;
    else if (k == "--cluster") cluster_p = v;
    else if (k == "--profiles") prof_p = v;
    else if (k == "--trace") trace_p = v;
    else if (k == "--synth-profiles") synth_ctx = std::stod(v);
    else if (k == "--synth-trace") synth_tr = doubles(v);
    else if (k == "--objective") objective = v;
    else if (k == "--freqs") freqs = doubles(v);
    else if (k == "--batching") cfg.policy.mode = v == "chunked" ? BatchMode::ChunkedPrefill : BatchMode::Contiguous;
    else if (k == "--chunk") cfg.policy.chunk_size = std::stoll(v);
    else if (k == "--max-batch") cfg.policy.max_batch_size = std::stoll(v);
    else if (k == "--anchor") cfg.ttft_anchor = v == "admission" ? TtftAnchor::Admission : TtftAnchor::Arrival;
    else if (k == "--jobs") jobs = std::stoi(v);
    else if (k == "--threads") threads = std::stoi(v);
    else if (k == "--drop-table") drop = v;
    else if (k == "--single") single = std::stoi(v);
    else if (k == "--sweep-segments") sweep_segments = std::stoi(v);
    else if (k == "--sweep-subset") sweep_subset = std::stoll(v);
  }
  try {
    const ModelSpec model = parse_model_config_file(model_p);
    const ClusterSpec cluster = parse_cluster_spec_file(cluster_p);
    std::string store_text;
    if (!prof_p.empty()) {
      store_text = read_file(prof_p);
    } else {
      store_text = synth_profiles(cluster.device, cluster, GridSpec::for_model(model, cluster, synth_ctx)).serialize();
    }
    if (!drop.empty()) store_text = drop_lines(store_text, "\"op\":\"" + drop + "\"");
    std::istringstream s1(store_text), s2(store_text);
    const ProfileStore ref_store = ProfileStore::load(s1);
    const ProfileStore gpu_store = ProfileStore::load(s2);
    const Trace trace = !trace_p.empty() ? load_trace_file(trace_p)
                                         : synth_trace({synth_tr[0], synth_tr[1]}, {synth_tr[2], synth_tr[3]},
                                                       synth_tr[4], int64_t(synth_tr[5]), uint64_t(synth_tr[6]));
    const auto plans = generate_plans(model, to_transformer_ir(model), cluster);
    const Objective obj = objective == "energy" ? Objective::Energy : Objective::Latency;

    int ref_code = 0, gpu_code = 0;
    std::string ref_msg, gpu_msg;
    RankedPlans a, b;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      a = search(plans, model, cluster, trace, ref_store, obj, freqs, cfg, jobs);
    } catch (const InfeasibleError& e) { ref_code = 3; ref_msg = e.what(); }
    catch (const DataError& e) { ref_code = 4; ref_msg = e.what(); }
    const auto t1 = std::chrono::steady_clock::now();
    try {
      b = plansim_gpu::search(plans, model, cluster, trace, gpu_store, obj, freqs, cfg, jobs);
    } catch (const InfeasibleError& e) { gpu_code = 3; gpu_msg = e.what(); }
    catch (const DataError& e) { gpu_code = 4; gpu_msg = e.what(); }
    const auto t2 = std::chrono::steady_clock::now();

    if (ref_code || gpu_code) {
      const bool same = ref_code == gpu_code && ref_msg == gpu_msg;
      std::printf("{\"error_parity\":%s,\"ref\":\"%s\",\"gpu\":\"%s\"}\n", same ? "true" : "false",
                  ref_msg.c_str(), gpu_msg.c_str());
      return same ? ref_code : 1;
    }
    int bad = 0;
    std::string first;
    auto miss = [&](const std::string& what) {
      if (!bad++) first = what;
    };
    {
      std::string f;
      if (const int d = diff_ranked(a, b, f)) {
        bad += d - 1;
        miss(f);
      }
    }
    // concurrent callers of the drop-in (each with its own store: clamp
    // replays write its warnings) get the single caller's result
    if (threads > 1) {
      std::vector<RankedPlans> got(static_cast<size_t>(threads));
      std::vector<std::string> errs(static_cast<size_t>(threads));
      std::vector<std::thread> th;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          try {
            std::istringstream st(store_text);
            const ProfileStore own = ProfileStore::load(st);
            got[size_t(t)] = plansim_gpu::search(plans, model, cluster, trace, own, obj, freqs, cfg, jobs);
          } catch (const std::exception& e) {
            errs[size_t(t)] = e.what();
          }
        });
      for (auto& x : th) x.join();
      for (int t = 0; t < threads; ++t) {
        std::string f;
        if (!errs[size_t(t)].empty()) miss("thread " + std::to_string(t) + ": " + errs[size_t(t)]);
        else if (diff_ranked(b, got[size_t(t)], f)) miss("thread " + std::to_string(t) + ": " + f);
      }
    }
    size_t n_iter = 0, n_rows = 0;
    if (single >= 0 && size_t(single) < plans.size()) {
      const ExecutionPlan& plan = plans[size_t(single)];
      SimConfig ec = cfg;
      ec.emit_iterations = true;
      if (!freqs.empty()) ec.freq_ghz = freqs.front();
      const SimulationReport ra = simulate_plan(plan, model, cluster, trace, ref_store, ec);
      const SimulationReport rb = plansim_gpu::simulate_plan(plan, model, cluster, trace, gpu_store, ec);
      n_iter = ra.iterations.size();
      if (ra.e2e_latency != rb.e2e_latency || ra.total_energy != rb.total_energy ||
          ra.num_iterations != rb.num_iterations || ra.per_request.size() != rb.per_request.size())
        miss("simulate_plan report");
      if (ra.iterations.size() != rb.iterations.size()) {
        miss("iteration count");
      } else {
        for (size_t k = 0; k < ra.iterations.size(); ++k) {
          const auto& x = ra.iterations[k];
          const auto& y = rb.iterations[k];
          if (x.clock_start != y.clock_start || x.duration != y.duration || x.energy != y.energy ||
              x.batch_size != y.batch_size || x.stage_seconds != y.stage_seconds ||
              x.stage_joules != y.stage_joules) {
            miss("iteration record " + std::to_string(k));
            break;
          }
        }
      }
      if (sweep_segments > 0) {
        SimConfig sc = cfg;
        if (!freqs.empty()) sc.freq_ghz = freqs.front();
        const SweepTable ta = sweep_max_batch(plan, model, cluster, trace, ref_store, sc,
                                              sweep_segments, sweep_subset);
        const SweepTable tb = plansim_gpu::sweep_max_batch(plan, model, cluster, trace, gpu_store, sc,
                                                           sweep_segments, sweep_subset);
        n_rows = ta.rows.size();
        bool same = ta.observed_max_batch == tb.observed_max_batch && ta.rows.size() == tb.rows.size();
        for (size_t k = 0; same && k < ta.rows.size(); ++k)
          same = ta.rows[k].max_batch_size == tb.rows[k].max_batch_size &&
                 ta.rows[k].mean_tpot == tb.rows[k].mean_tpot &&
                 ta.rows[k].mean_ttft == tb.rows[k].mean_ttft &&
                 ta.rows[k].e2e_latency == tb.rows[k].e2e_latency;
        if (!same) miss("sweep table");
      }
    }
    const auto wa = ref_store.warnings(), wb = gpu_store.warnings();
    const std::set<std::string> sa(wa.begin(), wa.end()), sb(wb.begin(), wb.end());
    if (sa != sb) miss("clamp warnings");
    std::printf("{\"entries\":%zu,\"mismatches\":%d,\"first\":\"%s\",\"warnings\":%zu,"
                "\"iterations\":%zu,\"sweep_rows\":%zu,"
                "\"ref_s\":%.6f,\"gpu_s\":%.6f,\"best\":\"%s\"}\n",
                a.entries.size(), bad, first.c_str(), sa.size(), n_iter, n_rows,
                std::chrono::duration<double>(t1 - t0).count(),
                std::chrono::duration<double>(t2 - t1).count(),
                a.entries.empty() ? "" : a.entries.front().report.plan_encoding.c_str());
    return bad ? 1 : 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
}
