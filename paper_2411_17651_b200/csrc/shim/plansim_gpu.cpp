// plansim_gpu.cpp — flattens the reference's types into the psg C ABI
// (include/psg.h), runs the B200 engine, and rebuilds plansim::RankedPlans.
//
// Compiled inside a plansim build (it includes the reference headers and
// nlohmann/json like the reference sources do); the engine itself is
// libpsg.so.  Inputs are read-only, exactly as plansim::search takes them.
//
// ProfileStore keeps its grids private (include/plansim/cost.hpp:96-128), so
// the shim reads them through the store's own serialize() (cost.cpp:355-382),
// whose shortest-round-trip doubles re-parse exactly.  Clamp warnings the
// engine reports are replayed as one clamped query per (table, axis,
// direction) against the caller's store, so store.warnings() ends up with the
// reference's warn-once messages (cost.cpp:191-212, :273-278).
#include "plansim_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <thread>
#include <tuple>

#include "json.hpp"
#include "psg.h"

namespace plansim_gpu {

namespace {

using namespace plansim;

// A cached engine context.  A psg_context is not thread-shared (psg.h), so
// every use holds its mutex from psg_search until the results are copied out.
struct Ctx {
  psg_context* h = nullptr;
  std::mutex mu;
  ~Ctx() {
    if (h) psg_context_destroy(h);
  }
};

// Context `slot` of `device` (slots > 0 only when several shards share a
// device: PSG_SHIM_CONTEXTS_PER_DEVICE).
Ctx& context_for(int device, int slot = 0) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, std::unique_ptr<Ctx>> ctxs;
  std::lock_guard<std::mutex> lock(mu);
  auto& c = ctxs[{device, slot}];
  if (!c) {
    auto made = std::make_unique<Ctx>();
    if (psg_context_create(device, &made->h) != PSG_OK)
      throw DataError("plansim_gpu: cannot create a CUDA context on device " +
                      std::to_string(device));
    c = std::move(made);
  }
  return *c;
}

struct ResultFree {
  void operator()(psg_result* r) const { psg_result_free(r); }
};
using ResultPtr = std::unique_ptr<psg_result, ResultFree>;

// Flat store tables parsed from ProfileStore::serialize().
struct FlatStore {
  std::vector<int32_t> c_op, c_dt, c_nc, c_nt, c_nw, k_kind, k_dev, k_nodes, k_n;
  std::vector<int64_t> c_fm, c_kb, c_vb, k_b;
  std::vector<double> knots, sec, jou, pay, ksec, kjou;
  psg_store v{};

  explicit FlatStore(const ProfileStore& store) {
    using Grid = std::map<std::array<double, 3>, std::pair<double, double>>;
    std::map<std::tuple<int, int, long long>, Grid> grids;
    std::map<std::tuple<int, int, int>, std::map<double, std::pair<double, double>>> curves;
    std::istringstream in(store.serialize());
    std::string line;
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      const auto r = nlohmann::json::parse(line);
      const auto& ax = r.at("axes");
      const std::pair<double, double> v{r.at("seconds").get<double>(), r.at("joules").get<double>()};
      if (r.at("table").get<std::string>() == "compute") {
        const int op = int(op_kind_from_string(r.at("op").get<std::string>()));
        const int dt = int(DtypeFormat::from_string(r.at("dtype").get<std::string>()).name);
        const long long fm = llround(r.at("freq_ghz").get<double>() * 1e6);
        grids[{op, dt, fm}][{ax.at("context_tokens").get<double>(), ax.at("tasks").get<double>(),
                             ax.at("hidden_dim").get<double>()}] = v;
      } else {
        const int kind = int(collective_kind_from_string(r.at("op").get<std::string>()));
        curves[{kind, ax.at("num_devices").get<int>(), ax.at("num_nodes").get<int>()}]
              [ax.at("payload_bytes").get<double>()] = v;
      }
    }
    for (const auto& [key, g] : grids) {
      std::set<double> a[3];
      for (const auto& kv : g)
        for (int i = 0; i < 3; ++i) a[i].insert(kv.first[size_t(i)]);
      c_op.push_back(std::get<0>(key));
      c_dt.push_back(std::get<1>(key));
      c_fm.push_back(std::get<2>(key));
      c_nc.push_back(int32_t(a[0].size()));
      c_nt.push_back(int32_t(a[1].size()));
      c_nw.push_back(int32_t(a[2].size()));
      c_kb.push_back(int64_t(knots.size()));
      c_vb.push_back(int64_t(sec.size()));
      for (int i = 0; i < 3; ++i) knots.insert(knots.end(), a[i].begin(), a[i].end());
      for (const auto& kv : g) {  // lexicographic keys == row-major grid order
        sec.push_back(kv.second.first);
        jou.push_back(kv.second.second);
      }
    }
    for (const auto& [key, c] : curves) {
      k_kind.push_back(std::get<0>(key));
      k_dev.push_back(std::get<1>(key));
      k_nodes.push_back(std::get<2>(key));
      k_n.push_back(int32_t(c.size()));
      k_b.push_back(int64_t(pay.size()));
      for (const auto& [p, v] : c) {
        pay.push_back(p);
        ksec.push_back(v.first);
        kjou.push_back(v.second);
      }
    }
    auto nz = [](auto& x) { return x.empty() ? nullptr : x.data(); };
    v.n_compute = int32_t(c_op.size());
    v.c_op = nz(c_op);
    v.c_dtype = nz(c_dt);
    v.c_freq_micro = nz(c_fm);
    v.c_n_ctx = nz(c_nc);
    v.c_n_tasks = nz(c_nt);
    v.c_n_width = nz(c_nw);
    v.c_knot_begin = nz(c_kb);
    v.c_value_begin = nz(c_vb);
    v.c_knots = nz(knots);
    v.c_seconds = nz(sec);
    v.c_joules = nz(jou);
    v.n_curves = int32_t(k_kind.size());
    v.k_kind = nz(k_kind);
    v.k_devices = nz(k_dev);
    v.k_nodes = nz(k_nodes);
    v.k_n = nz(k_n);
    v.k_begin = nz(k_b);
    v.k_payload = nz(pay);
    v.k_seconds = nz(ksec);
    v.k_joules = nz(kjou);
  }

  // One clamped query per flagged (table, axis, direction): registers the
  // reference's warn-once message in the caller's store.
  void replay_clamps(const ProfileStore& store, const uint8_t* cb, const uint8_t* kb) const {
    for (size_t t = 0; t < c_op.size(); ++t) {
      const double* k = knots.data() + c_kb[t];
      const int n[3] = {c_nc[t], c_nt[t], c_nw[t]};
      const double* ax[3] = {k, k + n[0], k + n[0] + n[1]};
      for (int b = 0; b < 6; ++b) {
        if (!(cb[t] >> b & 1)) continue;
        double x[3] = {ax[0][0], ax[1][0], ax[2][0]};
        const int a = b / 2;
        x[a] = (b & 1) ? ax[a][n[a] - 1] * 2.0 + 1.0 : ax[a][0] - (std::fabs(ax[a][0]) + 1.0);
        OpQuery q;
        q.op = OpKind(c_op[t]);
        q.dtype = Dtype(c_dt[t]);
        q.freq_ghz = double(c_fm[t]) / 1e6;
        q.context_tokens = x[0];
        q.tasks_on_device = x[1];
        q.width = x[2];
        store.query_time(q);
      }
    }
    for (size_t u = 0; u < k_kind.size(); ++u)
      for (int b = 0; b < 2; ++b) {
        if (!(kb[u] >> b & 1)) continue;
        const double* p = pay.data() + k_b[u];
        CollectiveQuery q;
        q.kind = CollectiveKind(k_kind[u]);
        q.num_devices = k_dev[u];
        q.num_nodes = k_nodes[u];
        q.payload_bytes = b ? p[k_n[u] - 1] * 2.0 + 1.0 : p[0] - (std::fabs(p[0]) + 1.0);
        store.query_time(q);
      }
  }
};

struct FlatPlans {
  std::vector<int32_t> dp, st, sd, reps, dt, enc, cb, cop, kb, kk, kd, kn, kg, pb, pn;
  std::vector<double> kv, bud, p2p, hid, head, kve, ct, cw, cs, kp, ksh;
  psg_plan_set v{};

  explicit FlatPlans(const std::vector<ExecutionPlan>& plans) {
    std::vector<std::string> uniq;
    for (const auto& p : plans) uniq.push_back(p.scheme.encoding);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    cb.push_back(0);
    kb.push_back(0);
    pb.push_back(0);
    for (const auto& p : plans) {
      const auto& s = p.scheme;
      dp.push_back(s.model_dp);
      st.push_back(s.num_stages);
      sd.push_back(s.stage_devices);
      reps.push_back(s.stage_repetitions);
      dt.push_back(int32_t(p.compute_dtype));
      enc.push_back(int32_t(std::lower_bound(uniq.begin(), uniq.end(), s.encoding) - uniq.begin()));
      kv.push_back(p.kv_bytes_per_token);
      bud.push_back(p.kv_budget_per_replica);
      p2p.push_back(p.p2p_payload_per_token);
      hid.push_back(p.op_shape.model_hidden);
      head.push_back(p.op_shape.head_dim);
      kve.push_back(p.op_shape.kv_elems_per_task_token);
      for (const auto& c : s.cells) {
        cop.push_back(int32_t(c.op));
        ct.push_back(c.query_tasks);
        cw.push_back(c.query_width);
        cs.push_back(c.token_scale);
      }
      cb.push_back(int32_t(cop.size()));
      for (const auto& r : p.block_collectives) {
        kk.push_back(int32_t(r.kind));
        kd.push_back(r.num_devices);
        kn.push_back(r.num_nodes);
        kg.push_back(r.groups_per_stage);
        kp.push_back(r.payload_bytes_per_token);
        ksh.push_back(r.token_share);
      }
      kb.push_back(int32_t(kk.size()));
      pn.insert(pn.end(), p.p2p_boundary_nodes.begin(), p.p2p_boundary_nodes.end());
      pb.push_back(int32_t(pn.size()));
    }
    auto nz = [](auto& x) { return x.empty() ? nullptr : x.data(); };
    v = psg_plan_set{int32_t(plans.size()), nz(dp), nz(st), nz(sd), nz(reps), nz(dt), nz(enc),
                     nz(kv), nz(bud), nz(p2p), nz(hid), nz(head), nz(kve), cb.data(), nz(cop),
                     nz(ct), nz(cw), nz(cs), kb.data(), nz(kk), nz(kd), nz(kn), nz(kg), nz(kp),
                     nz(ksh), pb.data(), nz(pn)};
  }
};

}  // namespace

namespace {

struct ShardFailed {};

// SearchEntry k of a psg_result (report scalars, per-request metrics, rejected ids).
void fill_entry(const psg_result& res, int64_t k, const std::vector<plansim::ExecutionPlan>& plans,
                plansim::SearchEntry& se) {
  using namespace plansim;
  const psg_entry& e = res.entries[k];
  se.plan_index = size_t(e.plan_index);
  se.freq_ghz = e.freq_ghz;
  SimulationReport& r = se.report;
  r.plan_encoding = plans[size_t(e.plan_index)].scheme.encoding;
  r.frequency_ghz = e.freq_ghz;
  r.e2e_latency = e.e2e_latency;
  r.total_energy = e.total_energy;
  r.p95_latency = e.p95_latency;
  r.mean_ttft = e.mean_ttft;
  r.mean_tpot = e.mean_tpot;
  r.mfu = e.mfu;
  r.mbu = e.mbu;
  r.num_completed = e.num_completed;
  r.num_rejected = e.num_rejected;
  r.num_iterations = e.num_iterations;
  r.max_batch_observed = e.max_batch_observed;
  static_assert(sizeof(RequestMetrics) == sizeof(psg_request_metrics), "layout");
  r.per_request.resize(size_t(e.num_completed));
  if (e.num_completed)
    std::memcpy(r.per_request.data(), res.per_request + e.per_request_offset,
                sizeof(RequestMetrics) * size_t(e.num_completed));
  r.rejected_ids.assign(res.rejected_ids + e.rejected_offset,
                        res.rejected_ids + e.rejected_offset + e.num_rejected);
}

// A ranked search over `shards` engine contexts (one per device, cycling over
// the visible devices): entries are assigned longest-first (cost = requests
// per DP replica, the length of the entry's serial chain), each shard runs
// unranked on its own thread, and the gathered ranking records are ordered on
// the first context's device with the reference comparator
// (simulator.cpp:283-294; entry index breaks exact ties, as in one search).
// Any shard error re-runs the search on one context, which reports the
// reference's error for the lowest failing entry.
plansim::RankedPlans run_sharded(const std::vector<plansim::ExecutionPlan>& plans,
                                 const FlatPlans& fp, const FlatStore& fs,
                                 const plansim::ProfileStore& store, const psg_cluster& cl,
                                 const psg_trace& tr, const psg_config& base,
                                 plansim::Objective objective, int device, int shards) {
  using namespace plansim;
  int ndev = 0;
  if (psg_device_count(&ndev) != PSG_OK || ndev < 1) ndev = 1;
  const int F = std::max(1, base.n_freqs);
  const int64_t n_entries = int64_t(plans.size()) * F;
  std::vector<std::pair<double, int32_t>> cost;
  for (int64_t e = 0; e < n_entries; ++e)
    cost.push_back({double(tr.n) / double(std::max(1, fp.v.model_dp[e / F])), int32_t(e)});
  std::sort(cost.begin(), cost.end(),
            [](const auto& a, const auto& b) { return a.first != b.first ? a.first > b.first : a.second < b.second; });
  std::vector<double> load(static_cast<size_t>(shards), 0.0);
  std::vector<std::vector<int32_t>> sub(static_cast<size_t>(shards));
  for (const auto& [w, e] : cost) {
    const size_t k = size_t(std::min_element(load.begin(), load.end()) - load.begin());
    load[k] += w;
    sub[k].push_back(e);
  }
  std::vector<ResultPtr> res(static_cast<size_t>(shards));
  std::vector<int> rcs(static_cast<size_t>(shards), PSG_OK);
  std::vector<std::thread> th;
  for (int k = 0; k < shards; ++k) {
    std::sort(sub[size_t(k)].begin(), sub[size_t(k)].end());
    th.emplace_back([&, k] {
      psg_config c = base;
      c.rank = 0;
      c.n_entry_subset = int32_t(sub[size_t(k)].size());
      c.entry_subset = sub[size_t(k)].data();
      try {
        Ctx& cx = context_for((device + k) % ndev, k / ndev);
        std::lock_guard<std::mutex> lock(cx.mu);
        psg_result* raw = nullptr;
        rcs[size_t(k)] = psg_search(cx.h, &fp.v, &cl, &fs.v, &tr, &c, &raw);
        res[size_t(k)].reset(raw);
      } catch (...) {
        rcs[size_t(k)] = PSG_ERR_CUDA;
      }
    });
  }
  for (auto& t : th) t.join();
  for (int k = 0; k < shards; ++k)
    if (rcs[size_t(k)] != PSG_OK) throw ShardFailed{};
  std::vector<psg_rank_key> keys;
  std::vector<std::pair<int, int64_t>> where;
  const bool lat = objective == Objective::Latency;
  for (int k = 0; k < shards; ++k) {
    const psg_result& r = *res[size_t(k)];
    fs.replay_clamps(store, r.compute_clamp, r.curve_clamp);
    for (int64_t i = 0; i < r.n_entries; ++i) {
      const psg_entry& e = r.entries[i];
      psg_rank_key key{};
      key.num_rejected = e.num_rejected;
      key.objective_metric = lat ? e.e2e_latency : e.total_energy;
      key.other_metric = lat ? e.total_energy : e.e2e_latency;
      key.enc_rank = fp.v.enc_rank[e.plan_index];
      key.freq_ghz = e.freq_ghz;
      key.entry_index = e.entry_index;
      keys.push_back(key);
      where.push_back({k, i});
    }
  }
  std::vector<int64_t> order(keys.size());
  {
    Ctx& cx = context_for(device % ndev, 0);
    std::lock_guard<std::mutex> lock(cx.mu);
    if (psg_rank_keys(cx.h, keys.data(), int64_t(keys.size()), order.data()) != PSG_OK)
      throw DataError(psg_last_error(cx.h));
  }
  RankedPlans out;
  out.entries.resize(keys.size());
  for (size_t j = 0; j < order.size(); ++j) {
    const auto& [k, i] = where[size_t(order[j])];
    fill_entry(*res[size_t(k)], i, plans, out.entries[j]);
  }
  return out;
}

// One psg_search call.  subset / caps: optional repeated entry list with
// per-entry max_batch_size (sweeps); emit: IterationRecords into the single
// entry's report.
plansim::RankedPlans run(const std::vector<plansim::ExecutionPlan>& plans,
                         const plansim::ClusterSpec& cluster, const plansim::Trace& trace,
                         const plansim::ProfileStore& store, plansim::Objective objective,
                         const std::vector<double>& frequencies, const plansim::SimConfig& cfg,
                         int device, bool rank, bool detail, bool emit,
                         const std::vector<int32_t>& subset = {},
                         const std::vector<int64_t>& caps = {}, int jobs = 1) {
  using namespace plansim;
  if (plans.empty()) throw InfeasibleError("search: no feasible plan");
  const FlatPlans fp(plans);
  const FlatStore fs(store);
  psg_cluster cl{};
  cl.total_devices = cluster.total_devices();
  cl.peak_mem_bandwidth = cluster.device.peak_mem_bandwidth;
  for (const auto& [d, f] : cluster.device.peak_flops) cl.peak_flops[int(d)] = f;
  cl.max_frequency_ghz = cluster.device.max_frequency();
  std::vector<int64_t> id, ctx, gen;
  std::vector<double> arr;
  for (const auto& r : trace.requests) {
    id.push_back(r.id);
    ctx.push_back(r.context_len);
    gen.push_back(r.gen_len);
    arr.push_back(r.arrival);
  }
  int64_t zi = 0;
  double zd = 0.0;
  const psg_trace tr{int64_t(id.size()), id.empty() ? &zi : id.data(),
                     ctx.empty() ? &zi : ctx.data(), gen.empty() ? &zi : gen.data(),
                     arr.empty() ? &zd : arr.data()};
  psg_config c{};
  c.objective = objective == Objective::Latency ? PSG_OBJ_LATENCY : PSG_OBJ_ENERGY;
  c.batch_mode = cfg.policy.mode == BatchMode::ChunkedPrefill ? PSG_BATCH_CHUNKED : PSG_BATCH_CONTIGUOUS;
  c.chunk_size = cfg.policy.chunk_size;
  c.max_batch_size = cfg.policy.max_batch_size;
  c.ttft_anchor = cfg.ttft_anchor == TtftAnchor::Admission ? PSG_ANCHOR_ADMISSION : PSG_ANCHOR_ARRIVAL;
  c.n_freqs = int32_t(frequencies.size());
  c.freqs = frequencies.empty() ? nullptr : frequencies.data();
  c.detail = detail ? 1 : 0;
  c.rank = rank ? 1 : 0;
  c.n_entry_subset = int32_t(subset.size());
  c.entry_subset = subset.empty() ? nullptr : subset.data();
  c.entry_max_batch_size = caps.empty() ? nullptr : caps.data();
  c.emit_iterations = emit ? 1 : 0;
  // jobs -> devices (simulator.cpp:251-275 maps jobs to worker threads):
  // a ranked search with jobs > 1 shards its entries over the visible devices
  int shards = 1;
  if (rank && !emit && subset.empty() && caps.empty() && jobs > 1) {
    int ndev = 0;
    if (psg_device_count(&ndev) != PSG_OK || ndev < 1) ndev = 1;
    int per = 1;
    if (const char* e = std::getenv("PSG_SHIM_CONTEXTS_PER_DEVICE")) per = std::max(1, std::atoi(e));
    const int64_t F = frequencies.empty() ? 1 : int64_t(frequencies.size());
    shards = int(std::min<int64_t>({int64_t(jobs), int64_t(ndev) * per, int64_t(plans.size()) * F}));
  }
  if (shards > 1) {
    try {
      return run_sharded(plans, fp, fs, store, cl, tr, c, objective, device, shards);
    } catch (const ShardFailed&) {  // the single-context search reports the error
    }
  }
  Ctx& cx = context_for(device);
  std::lock_guard<std::mutex> lock(cx.mu);
  psg_result* raw = nullptr;
  const int rc = psg_search(cx.h, &fp.v, &cl, &fs.v, &tr, &c, &raw);
  ResultPtr res(raw);
  if (rc == PSG_ERR_INFEASIBLE) throw InfeasibleError(psg_last_error(cx.h));
  if (rc != PSG_OK) throw DataError(psg_last_error(cx.h));
  fs.replay_clamps(store, res->compute_clamp, res->curve_clamp);
  RankedPlans out;
  out.entries.resize(size_t(res->n_entries));
  for (int64_t k = 0; k < res->n_entries; ++k)
    fill_entry(*res, k, plans, out.entries[size_t(k)]);
  if (emit && res->n_iterations > 0) {  // simulator.cpp:158-170
    SimulationReport& r = out.entries.front().report;
    const int S = res->n_stages;
    r.iterations.resize(size_t(res->n_iterations));
    for (int64_t i = 0; i < res->n_iterations; ++i) {
      IterationRecord& it = r.iterations[size_t(i)];
      it.clock_start = res->iterations[i].clock_start;
      it.duration = res->iterations[i].duration;
      it.energy = res->iterations[i].energy;
      it.batch_size = res->iterations[i].batch_size;
      it.stage_seconds.assign(res->stage_seconds + i * S, res->stage_seconds + (i + 1) * S);
      it.stage_joules.assign(res->stage_joules + i * S, res->stage_joules + (i + 1) * S);
    }
  }
  return out;
}

}  // namespace

plansim::RankedPlans search(const std::vector<plansim::ExecutionPlan>& plans,
                            const plansim::ModelSpec& /*model*/,
                            const plansim::ClusterSpec& cluster, const plansim::Trace& trace,
                            const plansim::ProfileStore& store, plansim::Objective objective,
                            const std::vector<double>& frequencies,
                            const plansim::SimConfig& cfg, int jobs, int device) {
  return run(plans, cluster, trace, store, objective, frequencies, cfg, device, true, true, false,
             {}, {}, jobs);
}

plansim::SimulationReport simulate_plan(const plansim::ExecutionPlan& plan,
                                        const plansim::ModelSpec& model,
                                        const plansim::ClusterSpec& cluster,
                                        const plansim::Trace& trace,
                                        const plansim::ProfileStore& store,
                                        const plansim::SimConfig& cfg, int device) {
  // simulator.cpp:180-181: cfg.freq_ghz > 0 ? cfg.freq_ghz : device max
  const double f = cfg.freq_ghz > 0 ? cfg.freq_ghz : cluster.device.max_frequency();
  (void)model;
  auto r = run({plan}, cluster, trace, store, plansim::Objective::Latency, {f}, cfg, device, false,
               true, cfg.emit_iterations);
  return std::move(r.entries.front().report);
}

plansim::SweepTable sweep_max_batch(const plansim::ExecutionPlan& plan,
                                    const plansim::ModelSpec& model,
                                    const plansim::ClusterSpec& cluster,
                                    const plansim::Trace& trace,
                                    const plansim::ProfileStore& store,
                                    const plansim::SimConfig& cfg, int segments,
                                    int64_t subset_size, int device) {
  using namespace plansim;
  // simulator.cpp:298-329: uncapped probe on the first subset_size requests,
  // then `segments` capped runs of the whole trace — one launch here.
  if (segments < 1) throw DataError("sweep: segments must be >= 1");
  Trace subset;
  subset.metadata = trace.metadata;
  const size_t take =
      std::min(trace.requests.size(), size_t(std::max<int64_t>(1, subset_size)));
  subset.requests.assign(trace.requests.begin(), trace.requests.begin() + long(take));
  SimConfig probe_cfg = cfg;
  probe_cfg.policy.max_batch_size = 0;
  probe_cfg.emit_iterations = false;
  const SimulationReport probe = simulate_plan(plan, model, cluster, subset, store, probe_cfg, device);
  SweepTable table;
  table.observed_max_batch = std::max<int64_t>(1, probe.max_batch_observed);
  std::vector<int64_t> caps;
  for (int i = 1; i <= segments; ++i)
    caps.push_back(std::max<int64_t>(
        1, llround(double(i) * double(table.observed_max_batch) / segments)));
  const double f = cfg.freq_ghz > 0 ? cfg.freq_ghz : cluster.device.max_frequency();
  SimConfig run_cfg = cfg;
  run_cfg.emit_iterations = false;
  const auto r = run({plan}, cluster, trace, store, Objective::Latency, {f}, run_cfg, device, false,
                     false, false, std::vector<int32_t>(size_t(segments), 0), caps);
  for (int i = 0; i < segments; ++i) {
    const SimulationReport& rep = r.entries[size_t(i)].report;
    table.rows.push_back({caps[size_t(i)], rep.mean_tpot, rep.mean_ttft, rep.e2e_latency});
  }
  return table;
}

}  // namespace plansim_gpu
