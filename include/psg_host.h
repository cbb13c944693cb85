/*
 * psg_host.h — C ABI of the native host side (psb::, include/psb/plansim_b200.hpp).
 *
 * A "problem" bundles the inputs of one evaluate-all-plans call, built with
 * the reference's own input formats and host algorithms:
 *   model / cluster JSON       parse_model_config, parse_cluster_spec
 *                              (/root/reference/proj/src/ir.cpp:91-150, cluster.cpp:34-99)
 *   plans                      generate_plans / build_plan (planner.cpp:371-418)
 *   profile tables             ProfileStore::load, GridSpec::for_model + synth_profiles
 *                              (cost.cpp:307-348, :384-509)
 *   trace                      load_trace / synth_trace (traces.cpp:48-139)
 * and exposes them as the psg_* SoA views that psg_search() consumes.
 * Strings returned by *_json / *_serialize are released with psgh_string_free.
 */
#ifndef PSG_HOST_H_
#define PSG_HOST_H_

#include <stdint.h>

#include "psg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psgh_problem psgh_problem;

typedef struct psgh_plan_options {
  double activation_reserve;      /* PlanOptions::activation_reserve (default 0.10) */
  int32_t include_embedding;      /* PlanOptions::include_embedding (default 1) */
  int32_t max_cell_combinations;  /* EnumOptions::max_cell_combinations (default 65536) */
} psgh_plan_options;

/* Message of the last failed psgh_* call on this thread. */
const char* psgh_last_error(void);

int psgh_problem_create(const char* model_json, const char* cluster_json,
                        const psgh_plan_options* opts, psgh_problem** out);
void psgh_problem_destroy(psgh_problem* p);

int psgh_store_synth(psgh_problem* p, double max_context);
/* synth_profiles with the compute tables computed on the GPU (device 0). */
int psgh_store_synth_device(psgh_problem* p, double max_context);
int psgh_store_load(psgh_problem* p, const char* jsonl);
int psgh_trace_synth(psgh_problem* p, double ctx_mean, double ctx_std, double gen_mean,
                     double gen_std, double rate, int64_t n, uint64_t seed);
int psgh_trace_load(psgh_problem* p, const char* jsonl);
/* generate_plans(): replaces the problem's plan list. */
int psgh_plans_generate(psgh_problem* p);
/* The same plans with the candidates mapped and finalized on the GPU. */
int psgh_plans_generate_device(psgh_problem* p);
/* The same plans emitted by the device straight into the engine's plan SoA
   (psg_plan_emit): no ExecutionPlans on the host; plans_view / count /
   encoding serve it, plans_json and plan_build refuse it. */
int psgh_plans_generate_direct(psgh_problem* p);
/* build_plan(): appends one plan; modes[i] is 0 (TP) or 1 (EP). */
int psgh_plan_build(psgh_problem* p, int model_dp, int num_stages, int n_cells,
                    const int32_t* modes, const int32_t* cell_dp, const int32_t* intra);

int psgh_plans_count(const psgh_problem* p);
const char* psgh_plan_encoding(const psgh_problem* p, int i);
const psg_plan_set* psgh_plans_view(psgh_problem* p);
const psg_store* psgh_store_view(const psgh_problem* p);
const psg_trace* psgh_trace_view(psgh_problem* p);
const psg_cluster* psgh_cluster_view(const psgh_problem* p);

char* psgh_plans_json(const psgh_problem* p);
char* psgh_store_serialize(const psgh_problem* p);
char* psgh_trace_serialize(const psgh_problem* p);
void psgh_string_free(char* s);

/* Report materialization over psg_search results: streams the reference
   CLI's ranked.json (tools/plansim_main.cpp:128-131: the array of
   report_to_json objects, simulator.cpp:331-369, dumped with indent 2)
   byte for byte, without building a JSON document.  entries in output order
   (ranked), per_request / rejected_ids addressed by the entries' offsets,
   plan_encodings indexed by psg_entry.plan_index. */
int psgh_write_ranked_json(const psg_entry* entries, int64_t n_entries,
                           const psg_request_metrics* per_request, const int64_t* rejected_ids,
                           const char* const* plan_encodings, int32_t n_plans, const char* path);
/* The CLI's simulate --out report (report_to_json of one entry; iterations go
   to the JSONL stream, tools/plansim_main.cpp:166-171). */
int psgh_write_report_json(const psg_entry* entry, const psg_request_metrics* per_request,
                           const int64_t* rejected_ids, const char* plan_encoding,
                           const char* path);
/* iterations_to_jsonl (simulator.cpp:371-385) over psg_result.iterations. */
int psgh_write_iterations_jsonl(const psg_iteration* iterations, int64_t n,
                                const double* stage_seconds, const double* stage_joules,
                                int32_t n_stages, const char* path);
/* The CLI's sweep --out table (tools/plansim_main.cpp:184-199). */
int psgh_write_sweep_json(int64_t observed_max_batch, const int64_t* caps, const double* mean_tpot,
                          const double* mean_ttft, const double* e2e_latency, int32_t n_rows,
                          const char* path);

#ifdef __cplusplus
}
#endif

#endif /* PSG_HOST_H_ */
