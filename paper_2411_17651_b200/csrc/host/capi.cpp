// C ABI over the native host library (include/psg_host.h).
#include <cstring>
#include <memory>

#include "psb/plansim_b200.hpp"
#include "psg_host.h"

struct psgh_problem {
  psb::ModelSpec model;
  psb::BlockSpec block;
  psb::ClusterSpec cluster;
  psb::PlanOptions opts;
  psb::ProfileStore store;
  psb::Trace trace;
  std::vector<psb::ExecutionPlan> plans;
  std::unique_ptr<psb::PlanSoA> soa;
  std::unique_ptr<psb::DevicePlanSet> direct;  // generate_plans_direct: SoA only, no ExecutionPlans
  psg_cluster cl{};
  // trace SoA
  std::vector<int64_t> t_id, t_ctx, t_gen;
  std::vector<double> t_arr;
  psg_trace tv{};
  bool trace_dirty = true;

  void refresh_trace() {
    if (!trace_dirty) return;
    t_id.clear();
    t_ctx.clear();
    t_gen.clear();
    t_arr.clear();
    for (const auto& r : trace.requests) {
      t_id.push_back(r.id);
      t_ctx.push_back(r.context_len);
      t_gen.push_back(r.gen_len);
      t_arr.push_back(r.arrival);
    }
    static int64_t zi = 0;
    static double zd = 0.0;
    tv.n = int64_t(t_id.size());
    tv.id = t_id.empty() ? &zi : t_id.data();
    tv.context_len = t_ctx.empty() ? &zi : t_ctx.data();
    tv.gen_len = t_gen.empty() ? &zi : t_gen.data();
    tv.arrival = t_arr.empty() ? &zd : t_arr.data();
    trace_dirty = false;
  }
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const psb::InfeasibleError& e) {
    g_err = e.what();
    return PSG_ERR_INFEASIBLE;
  } catch (const psb::DataError& e) {
    g_err = e.what();
    return PSG_ERR_DATA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PSG_ERR_DATA;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

const char* psgh_last_error(void) { return g_err.c_str(); }

int psgh_problem_create(const char* model_json, const char* cluster_json,
                        const psgh_plan_options* opts, psgh_problem** out) {
  if (!model_json || !cluster_json || !out) return PSG_ERR_USAGE;
  *out = nullptr;
  auto p = std::make_unique<psgh_problem>();
  const int rc = guarded([&] {
    p->model = psb::parse_model_config(model_json);
    p->block = psb::to_transformer_ir(p->model);
    p->cluster = psb::parse_cluster_spec(cluster_json);
    if (opts) {
      p->opts.activation_reserve = opts->activation_reserve;
      p->opts.include_embedding = opts->include_embedding != 0;
      p->opts.max_cell_combinations = opts->max_cell_combinations;
    }
    p->cl = psb::cluster_view(p->cluster);
  });
  if (rc == PSG_OK) *out = p.release();
  return rc;
}

void psgh_problem_destroy(psgh_problem* p) { delete p; }

int psgh_store_synth(psgh_problem* p, double max_context) {
  return guarded([&] {
    p->store = psb::synth_profiles(p->cluster.device, p->cluster,
                                   psb::GridSpec::for_model(p->model, p->cluster, max_context));
  });
}

int psgh_store_synth_device(psgh_problem* p, double max_context) {
  return guarded([&] {
    p->store = psb::synth_profiles_device(p->cluster.device, p->cluster,
                                          psb::GridSpec::for_model(p->model, p->cluster, max_context));
  });
}

int psgh_store_load(psgh_problem* p, const char* jsonl) {
  return guarded([&] { p->store = psb::ProfileStore::load(jsonl ? jsonl : ""); });
}

int psgh_trace_synth(psgh_problem* p, double cm, double cs, double gm, double gs, double rate,
                     int64_t n, uint64_t seed) {
  return guarded([&] {
    p->trace = psb::synth_trace({cm, cs}, {gm, gs}, rate, n, seed);
    p->trace_dirty = true;
  });
}

int psgh_trace_load(psgh_problem* p, const char* jsonl) {
  return guarded([&] {
    p->trace = psb::load_trace(jsonl ? jsonl : "");
    p->trace_dirty = true;
  });
}

int psgh_plans_generate(psgh_problem* p) {
  return guarded([&] {
    p->plans = psb::generate_plans(p->model, p->block, p->cluster, p->opts);
    p->soa.reset();
    p->direct.reset();
  });
}

int psgh_plans_generate_device(psgh_problem* p) {
  return guarded([&] {
    p->plans = psb::generate_plans_device(p->model, p->block, p->cluster, p->opts);
    p->soa.reset();
    p->direct.reset();
  });
}

int psgh_plans_generate_direct(psgh_problem* p) {
  return guarded([&] {
    p->direct = psb::generate_plans_direct(p->model, p->block, p->cluster, p->opts);
    p->plans.clear();
    p->soa.reset();
  });
}

int psgh_plan_build(psgh_problem* p, int dp, int stages, int n_cells, const int32_t* modes,
                    const int32_t* cell_dp, const int32_t* intra) {
  return guarded([&] {
    std::vector<psb::CellChoice> ch(static_cast<size_t>(n_cells));
    for (int i = 0; i < n_cells; ++i)
      ch[size_t(i)] = {modes[i] ? psb::ParallelMode::EP : psb::ParallelMode::TP, cell_dp[i], intra[i]};
    if (p->direct) throw psb::DataError("build_plan: the problem holds a device-emitted plan set");
    p->plans.push_back(psb::build_plan(p->model, p->block, p->cluster, dp, stages, ch, p->opts));
    p->soa.reset();
  });
}

int psgh_plans_count(const psgh_problem* p) {
  return int(p->direct ? p->direct->size() : p->plans.size());
}

const char* psgh_plan_encoding(const psgh_problem* p, int i) {
  return p->direct ? p->direct->encodings[size_t(i)].c_str() : p->plans[size_t(i)].scheme.encoding.c_str();
}

const psg_plan_set* psgh_plans_view(psgh_problem* p) {
  if (p->direct) return &p->direct->view();
  if (!p->soa) p->soa = std::make_unique<psb::PlanSoA>(p->plans);
  return &p->soa->view();
}

const psg_store* psgh_store_view(const psgh_problem* p) { return &p->store.view(); }

const psg_trace* psgh_trace_view(psgh_problem* p) {
  p->refresh_trace();
  return &p->tv;
}

const psg_cluster* psgh_cluster_view(const psgh_problem* p) { return &p->cl; }

char* psgh_plans_json(const psgh_problem* p) {
  if (p->direct) {
    g_err = "plans_json: a device-emitted plan set has no ExecutionPlans";
    return nullptr;
  }
  return dup(psb::plans_to_json(p->plans));
}
char* psgh_store_serialize(const psgh_problem* p) { return dup(p->store.serialize()); }
char* psgh_trace_serialize(const psgh_problem* p) { return dup(psb::serialize_trace(p->trace)); }
void psgh_string_free(char* s) { std::free(s); }

}  // extern "C"
