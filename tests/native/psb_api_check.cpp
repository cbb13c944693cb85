// Exercises the native C++ host API (include/psb/plansim_b200.hpp) end to
// end: model / cluster JSON -> synth_profiles + synth_trace ->
// generate_plans -> psb::search, psb::simulate_plan(emit_iterations),
// psb::sweep_max_batch.  Prints one JSON line with exact (hex) values that
// tests/test_gpu_psb_api.py compares with the Python engine (itself checked
// against the reference).
//
// usage: psb_api_check model.json cluster.json max_ctx cm,cs,gm,gs,rate,n,seed plan segments subset
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "psb/plansim_b200.hpp"

static std::string slurp(const char* p) {
  std::ifstream f(p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

static uint64_t mix(uint64_t h, double v) {
  uint64_t b;
  std::memcpy(&b, &v, sizeof b);
  return (h ^ b) * 1099511628211ull;
}

int main(int argc, char** argv) {
  if (argc < 8) return 2;
  const psb::ModelSpec model = psb::parse_model_config(slurp(argv[1]));
  const psb::ClusterSpec cluster = psb::parse_cluster_spec(slurp(argv[2]));
  double t[7];
  std::sscanf(argv[4], "%lf,%lf,%lf,%lf,%lf,%lf,%lf", &t[0], &t[1], &t[2], &t[3], &t[4], &t[5], &t[6]);
  const int plan_k = std::atoi(argv[5]), segments = std::atoi(argv[6]);
  const int64_t subset = std::atoll(argv[7]);
  const psb::ProfileStore store = psb::synth_profiles(
      cluster.device, cluster, psb::GridSpec::for_model(model, cluster, std::atof(argv[3])));
  const psb::Trace trace =
      psb::synth_trace({t[0], t[1]}, {t[2], t[3]}, t[4], int64_t(t[5]), uint64_t(t[6]));
  const auto plans = psb::generate_plans(model, psb::to_transformer_ir(model), cluster, {});
  psb::Engine engine(0);
  psb::SimConfig cfg;
  const psb::RankedPlans ranked = psb::search(plans, model, cluster, trace, store,
                                              psb::Objective::Latency, {}, cfg, 1, &engine);
  psb::SimConfig ec = cfg;
  ec.emit_iterations = true;
  const psb::SimulationReport rep =
      psb::simulate_plan(plans[size_t(plan_k)], model, cluster, trace, store, ec, &engine);
  uint64_t h = 1469598103934665603ull;
  for (const auto& it : rep.iterations) {
    h = mix(h, it.clock_start);
    h = mix(h, it.duration);
    h = mix(h, it.energy);
    h = mix(h, double(it.batch_size));
    for (double v : it.stage_seconds) h = mix(h, v);
    for (double v : it.stage_joules) h = mix(h, v);
  }
  const psb::SweepTable sw = psb::sweep_max_batch(plans[size_t(plan_k)], model, cluster, trace,
                                                  store, cfg, segments, subset, &engine);
  std::printf("{\"entries\":%zu,\"best_plan\":%zu,\"best_e2e\":\"%a\",\"sim_e2e\":\"%a\","
              "\"sim_iterations\":%" PRId64 ",\"records\":%zu,\"records_hash\":\"%016" PRIx64 "\","
              "\"observed\":%" PRId64 ",\"rows\":[",
              ranked.entries.size(), ranked.entries.front().plan_index,
              ranked.entries.front().report.e2e_latency, rep.e2e_latency, rep.num_iterations,
              rep.iterations.size(), h, sw.observed_max_batch);
  for (size_t i = 0; i < sw.rows.size(); ++i)
    std::printf("%s[%" PRId64 ",\"%a\",\"%a\",\"%a\"]", i ? "," : "", sw.rows[i].max_batch_size,
                sw.rows[i].mean_tpot, sw.rows[i].mean_ttft, sw.rows[i].e2e_latency);
  std::printf("]}\n");
  return 0;
}
