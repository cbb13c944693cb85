// psb::search / psb::simulate_plan: the reference-shaped C++ entry points,
// implemented by flattening the inputs to the C ABI (include/psg.h) and
// running the CUDA engine.  Replaces plansim::search
// (/root/reference/proj/src/simulator.cpp:242-296) and simulate_plan
// (:176-240) with the same signatures plus an optional engine handle.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "psb/plansim_b200.hpp"

namespace psb {

PlanSoA::PlanSoA(const std::vector<ExecutionPlan>& plans) {
  std::vector<std::string> enc;
  for (const auto& p : plans) enc.push_back(p.scheme.encoding);
  std::vector<std::string> uniq = enc;
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  cb_.push_back(0);
  kb_.push_back(0);
  pb_.push_back(0);
  for (size_t i = 0; i < plans.size(); ++i) {
    const ExecutionPlan& p = plans[i];
    const ParallelScheme& s = p.scheme;
    dp_.push_back(s.model_dp);
    st_.push_back(s.num_stages);
    sd_.push_back(s.stage_devices);
    reps_.push_back(s.stage_repetitions);
    dt_.push_back(int32_t(p.compute_dtype));
    enc_.push_back(int32_t(std::lower_bound(uniq.begin(), uniq.end(), enc[i]) - uniq.begin()));
    kv_.push_back(p.kv_bytes_per_token);
    bud_.push_back(p.kv_budget_per_replica);
    p2p_.push_back(p.p2p_payload_per_token);
    hid_.push_back(p.op_shape.model_hidden);
    head_.push_back(p.op_shape.head_dim);
    kve_.push_back(p.op_shape.kv_elems_per_task_token);
    for (const auto& c : s.cells) {
      cop_.push_back(int32_t(c.op));
      ct_.push_back(c.query_tasks);
      cw_.push_back(c.query_width);
      cs_.push_back(c.token_scale);
    }
    cb_.push_back(int32_t(cop_.size()));
    for (const auto& rc : p.block_collectives) {
      kk_.push_back(int32_t(rc.kind));
      kd_.push_back(rc.num_devices);
      kn_.push_back(rc.num_nodes);
      kg_.push_back(rc.groups_per_stage);
      kp_.push_back(rc.payload_bytes_per_token);
      ksh_.push_back(rc.token_share);
    }
    kb_.push_back(int32_t(kk_.size()));
    for (int b : p.p2p_boundary_nodes) pn_.push_back(b);
    pb_.push_back(int32_t(pn_.size()));
  }
  auto nz = [](auto& v) { return v.empty() ? nullptr : v.data(); };
  view_.n_plans = int32_t(plans.size());
  view_.model_dp = nz(dp_);
  view_.num_stages = nz(st_);
  view_.stage_devices = nz(sd_);
  view_.stage_repetitions = nz(reps_);
  view_.compute_dtype = nz(dt_);
  view_.enc_rank = nz(enc_);
  view_.kv_bytes_per_token = nz(kv_);
  view_.kv_budget_per_replica = nz(bud_);
  view_.p2p_payload_per_token = nz(p2p_);
  view_.shape_hidden = nz(hid_);
  view_.shape_head_dim = nz(head_);
  view_.shape_kv_elems = nz(kve_);
  view_.cell_begin = cb_.data();
  view_.cell_op = nz(cop_);
  view_.cell_tasks = nz(ct_);
  view_.cell_width = nz(cw_);
  view_.cell_token_scale = nz(cs_);
  view_.coll_begin = kb_.data();
  view_.coll_kind = nz(kk_);
  view_.coll_devices = nz(kd_);
  view_.coll_nodes = nz(kn_);
  view_.coll_groups = nz(kg_);
  view_.coll_ppt = nz(kp_);
  view_.coll_share = nz(ksh_);
  view_.p2p_begin = pb_.data();
  view_.p2p_nodes = nz(pn_);
}

psg_cluster cluster_view(const ClusterSpec& c) {
  psg_cluster v{};
  v.total_devices = c.total_devices();
  v.peak_mem_bandwidth = c.device.peak_mem_bandwidth;
  for (const auto& [dt, f] : c.device.peak_flops) v.peak_flops[int(dt)] = f;
  v.max_frequency_ghz = c.device.max_frequency();
  return v;
}

Engine::Engine(int device) {
  const int rc = psg_context_create(device, &ctx_);
  if (rc != PSG_OK) throw DeviceError("psg_context_create failed on device " + std::to_string(device));
}

Engine::~Engine() { psg_context_destroy(ctx_); }

namespace {

void raise(int rc, const char* msg) {
  if (rc == PSG_ERR_INFEASIBLE) throw InfeasibleError(msg);
  if (rc == PSG_ERR_DATA) throw DataError(msg);
  throw DeviceError(msg);
}

// Trace as SoA (caller keeps `t` alive during the call).
struct TraceSoA {
  std::vector<int64_t> id, ctx, gen;
  std::vector<double> arr;
  psg_trace view{};
  explicit TraceSoA(const Trace& t) {
    for (const auto& r : t.requests) {
      id.push_back(r.id);
      ctx.push_back(r.context_len);
      gen.push_back(r.gen_len);
      arr.push_back(r.arrival);
    }
    view.n = int64_t(t.requests.size());
    static int64_t zi = 0;
    static double zd = 0.0;
    view.id = id.empty() ? &zi : id.data();
    view.context_len = ctx.empty() ? &zi : ctx.data();
    view.gen_len = gen.empty() ? &zi : gen.data();
    view.arrival = arr.empty() ? &zd : arr.data();
  }
};

}  // namespace

namespace {

struct RunOpts {
  bool rank = true, detail = true, emit = false;
  std::vector<int32_t> subset;
  std::vector<int64_t> caps;
};

RankedPlans run(const std::vector<ExecutionPlan>& plans, const ClusterSpec& cluster,
                const Trace& trace, const ProfileStore& store, Objective objective,
                const std::vector<double>& frequencies, const SimConfig& cfg, Engine* engine,
                const RunOpts& o) {
  if (plans.empty()) throw InfeasibleError("search: no feasible plan");
  std::unique_ptr<Engine> own;
  if (!engine) {
    own = std::make_unique<Engine>(0);
    engine = own.get();
  }
  const PlanSoA soa(plans);
  const psg_cluster cl = cluster_view(cluster);
  const TraceSoA tr(trace);
  psg_config c{};
  c.objective = objective == Objective::Latency ? PSG_OBJ_LATENCY : PSG_OBJ_ENERGY;
  c.batch_mode = cfg.policy.mode == BatchMode::ChunkedPrefill ? PSG_BATCH_CHUNKED : PSG_BATCH_CONTIGUOUS;
  c.chunk_size = cfg.policy.chunk_size;
  c.max_batch_size = cfg.policy.max_batch_size;
  c.ttft_anchor = cfg.ttft_anchor == TtftAnchor::Admission ? PSG_ANCHOR_ADMISSION : PSG_ANCHOR_ARRIVAL;
  c.n_freqs = int32_t(frequencies.size());
  c.freqs = frequencies.empty() ? nullptr : frequencies.data();
  c.detail = o.detail ? 1 : 0;
  c.rank = o.rank ? 1 : 0;
  c.n_entry_subset = int32_t(o.subset.size());
  c.entry_subset = o.subset.empty() ? nullptr : o.subset.data();
  c.entry_max_batch_size = o.caps.empty() ? nullptr : o.caps.data();
  c.emit_iterations = o.emit ? 1 : 0;
  c.ttft_slo = cfg.ttft_slo;
  c.slo_quantile = cfg.slo_quantile;
  psg_result* res = nullptr;
  const int rc = psg_search(engine->handle(), &soa.view(), &cl, &store.view(), &tr.view, &c, &res);
  if (rc != PSG_OK) raise(rc, psg_last_error(engine->handle()));
  store.record_clamps(res->compute_clamp, res->curve_clamp);
  RankedPlans out;
  out.entries.resize(size_t(res->n_entries));
  for (int64_t k = 0; k < res->n_entries; ++k) {
    const psg_entry& e = res->entries[k];
    SearchEntry& se = out.entries[size_t(k)];
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
    r.p50_ttft = e.p50_ttft;
    r.p99_ttft = e.p99_ttft;
    r.p50_tpot = e.p50_tpot;
    r.p99_tpot = e.p99_tpot;
    r.slo_ttft = e.slo_ttft;
    r.slo_met = e.slo_met != 0;
    r.per_request.resize(size_t(e.num_completed));
    if (e.num_completed)
      std::memcpy(r.per_request.data(), res->per_request + e.per_request_offset,
                  sizeof(RequestMetrics) * size_t(e.num_completed));
    r.rejected_ids.assign(res->rejected_ids + e.rejected_offset,
                          res->rejected_ids + e.rejected_offset + e.num_rejected);
  }
  if (o.emit && res->n_iterations > 0) {  // simulator.cpp:158-170, replicas in order
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
  psg_result_free(res);
  return out;
}

}  // namespace

RankedPlans search(const std::vector<ExecutionPlan>& plans, const ModelSpec& /*model*/,
                   const ClusterSpec& cluster, const Trace& trace, const ProfileStore& store,
                   Objective objective, const std::vector<double>& frequencies,
                   const SimConfig& cfg, int /*jobs*/, Engine* engine) {
  return run(plans, cluster, trace, store, objective, frequencies, cfg, engine, RunOpts{});
}

SimulationReport simulate_plan(const ExecutionPlan& plan, const ModelSpec& /*model*/,
                               const ClusterSpec& cluster, const Trace& trace,
                               const ProfileStore& store, const SimConfig& cfg, Engine* engine) {
  // simulator.cpp:179-180: cfg.freq_ghz > 0 ? cfg.freq_ghz : device max
  const double f = cfg.freq_ghz > 0 ? cfg.freq_ghz : cluster.device.max_frequency();
  RunOpts o;
  o.rank = false;
  o.emit = cfg.emit_iterations;
  RankedPlans r = run({plan}, cluster, trace, store, Objective::Latency, {f}, cfg, engine, o);
  return std::move(r.entries.front().report);
}

SweepTable sweep_max_batch(const ExecutionPlan& plan, const ModelSpec& model,
                           const ClusterSpec& cluster, const Trace& trace,
                           const ProfileStore& store, const SimConfig& cfg, int segments,
                           int64_t subset_size, Engine* engine) {
  // simulator.cpp:298-329
  if (segments < 1) throw DataError("sweep: segments must be >= 1");
  std::unique_ptr<Engine> own;
  if (!engine) {
    own = std::make_unique<Engine>(0);
    engine = own.get();
  }
  Trace subset;
  const size_t take = std::min(trace.requests.size(), size_t(std::max<int64_t>(1, subset_size)));
  subset.requests.assign(trace.requests.begin(), trace.requests.begin() + long(take));
  SimConfig probe_cfg = cfg;
  probe_cfg.policy.max_batch_size = 0;
  probe_cfg.emit_iterations = false;
  const SimulationReport probe = simulate_plan(plan, model, cluster, subset, store, probe_cfg, engine);
  SweepTable table;
  table.observed_max_batch = std::max<int64_t>(1, probe.max_batch_observed);
  RunOpts o;
  o.rank = false;
  o.detail = false;
  for (int i = 1; i <= segments; ++i) {
    o.caps.push_back(std::max<int64_t>(
        1, llround(double(i) * double(table.observed_max_batch) / segments)));
    o.subset.push_back(0);
  }
  const double f = cfg.freq_ghz > 0 ? cfg.freq_ghz : cluster.device.max_frequency();
  SimConfig run_cfg = cfg;
  run_cfg.emit_iterations = false;
  const RankedPlans r = run({plan}, cluster, trace, store, Objective::Latency, {f}, run_cfg, engine, o);
  for (int i = 0; i < segments; ++i) {
    const SimulationReport& rep = r.entries[size_t(i)].report;
    table.rows.push_back({o.caps[size_t(i)], rep.mean_tpot, rep.mean_ttft, rep.e2e_latency});
  }
  return table;
}

}  // namespace psb
