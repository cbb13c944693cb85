/*
 * psg.h — C ABI of the B200 plan-search engine ("psg" = plan search on GPU).
 *
 * This is the drop-in boundary for the reference's evaluate-all-plans call
 *
 *     RankedPlans plansim::search(const std::vector<ExecutionPlan>& plans,
 *                                 const ModelSpec&, const ClusterSpec&,
 *                                 const Trace&, const ProfileStore&, Objective,
 *                                 const std::vector<double>& frequencies,
 *                                 const SimConfig& cfg, int jobs);
 *   (/root/reference/proj/include/plansim/simulator.hpp:99-103,
 *    implementation /root/reference/proj/src/simulator.cpp:242-296)
 *
 * and, with a one-plan / one-frequency set, of
 *
 *     SimulationReport plansim::simulate_plan(...)   (simulator.hpp:80-82).
 *
 * Everything crossing this boundary is plain C: structure-of-arrays views
 * over caller-owned memory, sizes, and library-owned results released with
 * psg_result_free().  No C++ or torch types appear here.  Each struct field
 * names the reference field it flattens.
 *
 * Error behaviour mirrors the reference's exceptions: PSG_ERR_INFEASIBLE for
 * InfeasibleError (empty plan list, simulator.cpp:247), PSG_ERR_DATA for
 * DataError (missing profile table when an iteration queries it,
 * cost.cpp:178-189 / :262-270; chunk_size < 1 in chunked mode,
 * batching.cpp:63-64).  The message is available from psg_last_error().
 */
#ifndef PSG_H_
#define PSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_ABI_VERSION 1

/* Return codes (the reference CLI's exit codes, tools/plansim_main.cpp:28-31). */
enum {
  PSG_OK = 0,
  PSG_ERR_USAGE = 2,      /* malformed arguments to this ABI */
  PSG_ERR_INFEASIBLE = 3, /* plansim::InfeasibleError */
  PSG_ERR_DATA = 4,       /* plansim::DataError */
  PSG_ERR_CUDA = 5        /* device / driver failure (no reference analogue) */
};

/* plansim::OpKind (cost.hpp:20). */
enum { PSG_OP_ATTENTION = 0, PSG_OP_GEMM = 1, PSG_OP_MOE_GEMM = 2 };
/* plansim::CollectiveKind (cost.hpp:21). */
enum {
  PSG_COLL_ALLREDUCE = 0,
  PSG_COLL_ALLGATHER = 1,
  PSG_COLL_REDUCE_SCATTER = 2,
  PSG_COLL_ALL_TO_ALL = 3,
  PSG_COLL_P2P = 4
};
/* plansim::Dtype (ir.hpp:13). */
enum { PSG_DTYPE_FP16 = 0, PSG_DTYPE_FP8 = 1, PSG_DTYPE_INT4 = 2 };
/* plansim::Objective (simulator.hpp:84). */
enum { PSG_OBJ_LATENCY = 0, PSG_OBJ_ENERGY = 1 };
/* plansim::BatchMode (batching.hpp:15). */
enum { PSG_BATCH_CONTIGUOUS = 0, PSG_BATCH_CHUNKED = 1 };
/* plansim::TtftAnchor (simulator.hpp:71). */
enum { PSG_ANCHOR_ARRIVAL = 0, PSG_ANCHOR_ADMISSION = 1 };

/*
 * Flattened std::vector<ExecutionPlan> (planner.hpp:92-106).  Per-plan
 * scalars are arrays of length n_plans; the variable-length lists (cells,
 * block_collectives, p2p_boundary_nodes) are CSR arrays whose *_begin index
 * arrays have n_plans + 1 entries.
 */
typedef struct psg_plan_set {
  int32_t n_plans;
  const int32_t* model_dp;            /* scheme.model_dp */
  const int32_t* num_stages;          /* scheme.num_stages */
  const int32_t* stage_devices;       /* scheme.stage_devices */
  const int32_t* stage_repetitions;   /* scheme.stage_repetitions */
  const int32_t* compute_dtype;       /* compute_dtype (PSG_DTYPE_*) */
  const int32_t* enc_rank;            /* rank of scheme.encoding under std::string operator<
                                         (equal strings share a rank) */
  const double* kv_bytes_per_token;   /* kv_bytes_per_token */
  const double* kv_budget_per_replica;/* kv_budget_per_replica */
  const double* p2p_payload_per_token;/* p2p_payload_per_token */
  const double* shape_hidden;         /* op_shape.model_hidden */
  const double* shape_head_dim;       /* op_shape.head_dim */
  const double* shape_kv_elems;       /* op_shape.kv_elems_per_task_token */
  /* scheme.cells[] (CellScheme, planner.hpp:27-41) */
  const int32_t* cell_begin;          /* [n_plans + 1] */
  const int32_t* cell_op;             /* CellScheme::op (PSG_OP_*) */
  const double* cell_tasks;           /* CellScheme::query_tasks */
  const double* cell_width;           /* CellScheme::query_width */
  const double* cell_token_scale;     /* CellScheme::token_scale */
  /* block_collectives[] (ResolvedCollective, planner.hpp:83-90) */
  const int32_t* coll_begin;          /* [n_plans + 1] */
  const int32_t* coll_kind;           /* PSG_COLL_* */
  const int32_t* coll_devices;        /* num_devices */
  const int32_t* coll_nodes;          /* num_nodes */
  const int32_t* coll_groups;         /* groups_per_stage */
  const double* coll_ppt;             /* payload_bytes_per_token */
  const double* coll_share;           /* token_share */
  /* p2p_boundary_nodes[] (one per stage boundary) */
  const int32_t* p2p_begin;           /* [n_plans + 1] */
  const int32_t* p2p_nodes;
} psg_plan_set;

/* The parts of ClusterSpec (cluster.hpp:22-46) the evaluation reads. */
typedef struct psg_cluster {
  int32_t total_devices;              /* ClusterSpec::total_devices() */
  double peak_mem_bandwidth;          /* device.peak_mem_bandwidth */
  double peak_flops[3];               /* device.peak_flops by PSG_DTYPE_*; <= 0: absent */
  double max_frequency_ghz;           /* device.max_frequency() */
} psg_cluster;

/*
 * Flattened, finalized ProfileStore (cost.hpp:63-129).  Compute grid t has
 * knots[knot_begin[t] ...] laid out as ctx[n_ctx], tasks[n_tasks],
 * width[n_width] (each strictly ascending), and values
 * seconds/joules[value_begin[t] ...] row-major over (ctx, tasks, width).
 * Collective curve u has payload/seconds/joules[curve_begin[u] ...][n].
 */
typedef struct psg_store {
  int32_t n_compute;
  const int32_t* c_op;
  const int32_t* c_dtype;
  const int64_t* c_freq_micro;        /* llround(freq_ghz * 1e6), cost.cpp:77 */
  const int32_t* c_n_ctx;
  const int32_t* c_n_tasks;
  const int32_t* c_n_width;
  const int64_t* c_knot_begin;
  const int64_t* c_value_begin;
  const double* c_knots;
  const double* c_seconds;
  const double* c_joules;
  int32_t n_curves;
  const int32_t* k_kind;
  const int32_t* k_devices;
  const int32_t* k_nodes;
  const int32_t* k_n;
  const int64_t* k_begin;
  const double* k_payload;
  const double* k_seconds;
  const double* k_joules;
} psg_store;

/* plansim::Trace (traces.hpp:14-31): requests in trace order. */
typedef struct psg_trace {
  int64_t n;
  const int64_t* id;
  const int64_t* context_len;
  const int64_t* gen_len;
  const double* arrival;
} psg_trace;

/* SimConfig (simulator.hpp:73-78) + the other search() arguments. */
typedef struct psg_config {
  int32_t objective;                  /* PSG_OBJ_* */
  int32_t batch_mode;                 /* PSG_BATCH_* (BatchPolicy::mode) */
  int64_t chunk_size;                 /* BatchPolicy::chunk_size */
  int64_t max_batch_size;             /* BatchPolicy::max_batch_size, 0 = unlimited */
  int32_t ttft_anchor;                /* PSG_ANCHOR_* */
  int32_t n_freqs;                    /* frequencies; 0 => {max_frequency_ghz} */
  const double* freqs;
  int32_t detail;                     /* 1: return per-request metrics + rejected ids
                                         (drop-in); 0: summaries only */
  int32_t rank;                       /* 1: sort entries (search); 0: entry order */
  int32_t n_entry_subset;             /* >0: simulate only these entry indices (sharding) */
  const int32_t* entry_subset;
  /* per-entry override of max_batch_size (one value per simulated entry:
     per entry_subset element, else per global entry; NULL = none).  With a
     repeated entry_subset this runs several BatchPolicy caps of one plan in
     one launch (sweep_max_batch, simulator.cpp:298-329). */
  const int64_t* entry_max_batch_size;
  /* SimConfig::emit_iterations (simulator.hpp:77): one IterationRecord per
     iteration (simulator.cpp:158-170); requires exactly one entry */
  int32_t emit_iterations;
  /* TTFT-SLO-constrained ranking (BASELINE configs[2]; the reference ranks
     without an SLO, simulator.cpp:277-294, and the paper's SLO use case is
     PAPER.md:607-615).  ttft_slo > 0: an entry meets the SLO iff it completed
     requests and the nearest-rank slo_quantile of its per-request TTFT
     (the p95 rule of simulator.cpp:223-225; slo_quantile 0 => 0.99) is
     <= ttft_slo.  Entries meeting it rank first, each group in the
     reference's order.  0 => off (the reference's ranking). */
  double ttft_slo;
  double slo_quantile;
} psg_config;

/* plansim::IterationRecord (simulator.hpp:35-42) without the stage vectors,
   which are returned as psg_result.stage_seconds / stage_joules with stride
   psg_result.n_stages. */
typedef struct psg_iteration {
  double clock_start;
  double duration;                    /* max over stages */
  double energy;                      /* sum over stages */
  int64_t batch_size;
} psg_iteration;

/* plansim::RequestMetrics (simulator.hpp:44-50); identical layout (40 B). */
typedef struct psg_request_metrics {
  int64_t id;
  double ttft;
  double tpot;
  double e2e;
  int64_t gen_len;
} psg_request_metrics;

/* One SearchEntry + SimulationReport scalars (simulator.hpp:52-69, :86-90). */
typedef struct psg_entry {
  int64_t entry_index;                /* i: plan i / F, freq i % F (simulator.cpp:255-258) */
  int64_t plan_index;
  double freq_ghz;
  double e2e_latency;
  double total_energy;
  double p95_latency;
  double mean_ttft;
  double mean_tpot;
  double mfu;
  double mbu;
  int64_t num_completed;
  int64_t num_rejected;
  int64_t num_iterations;
  int64_t max_batch_observed;
  /* additive outputs the reference does not compute (nearest-rank rule of
     simulator.cpp:223-225 applied at 0.50 / 0.99) */
  double p50_ttft, p99_ttft, p50_tpot, p99_tpot;
  /* TTFT at config.slo_quantile (nearest rank) and whether the entry meets
     config.ttft_slo (1), misses it (0); both 0 when the SLO is off */
  double slo_ttft;
  int64_t slo_met;
  int64_t per_request_offset;         /* into psg_result.per_request */
  int64_t rejected_offset;            /* into psg_result.rejected_ids */
} psg_entry;

/* Ranking record exchanged between ranks for the multi-GPU merge. */
typedef struct psg_rank_key {
  int64_t num_rejected;
  double objective_metric;
  double other_metric;
  int32_t enc_rank;
  int32_t slo_miss;                   /* 1: misses config.ttft_slo (ranks after every entry that meets it) */
  double freq_ghz;
  int64_t entry_index;
} psg_rank_key;

typedef struct psg_result {
  int64_t n_entries;
  psg_entry* entries;                 /* ranked best-first when config.rank, else entry order */
  int64_t n_per_request;
  psg_request_metrics* per_request;   /* per entry sorted by id (simulator.cpp:205-206) */
  int64_t n_rejected;
  int64_t* rejected_ids;              /* per entry sorted (simulator.cpp:207) */
  int32_t n_compute;
  uint8_t* compute_clamp;             /* per store compute grid: bit 2*axis + (above) */
  int32_t n_curves;
  uint8_t* curve_clamp;               /* per collective curve: bit 0 below, bit 1 above */
  /* instrumentation */
  int64_t gpu_launches;               /* kernels launched by this call */
  int64_t total_iterations;           /* sum of num_iterations over entries */
  double ms_total;                    /* host wall time of the call */
  double ms_h2d;                      /* CUDA-event time: input H2D + output clears */
  double ms_sim;                      /* CUDA-event time: simulation kernel */
  double ms_reduce;                   /* CUDA-event time: reduce + rank + compaction kernels */
  double ms_d2h;                      /* CUDA-event time: result D2H copies */
  int64_t h2d_bytes, d2h_bytes;       /* bytes copied host<->device by this call */
  /* work counters behind the algorithmic-bytes roofline */
  int64_t sum_batch;                  /* sum over all iterations of the batch size */
  int64_t admissions;                 /* admissions, re-admissions included */
  int64_t finishes;                   /* completed requests */
  /* emit_iterations: records of all replicas in replica order (run_replica
     appends replica by replica, simulator.cpp:196-199) */
  int64_t n_iterations;
  psg_iteration* iterations;
  int32_t n_stages;
  double* stage_seconds;              /* [n_iterations][n_stages] */
  double* stage_joules;               /* [n_iterations][n_stages] */
} psg_result;

/* Device synthesis of the analytical roofline compute tables (synth_profiles,
   cost.cpp:454-487): values for every (variant, op, ctx, tasks, width) in the
   reference's loop order, variant = (dtype, frequency) in loop order, op in
   {attention, gemm, moe_gemm}. */
typedef struct psg_synth_grid {
  int32_t n_ctx, n_tasks, n_width, n_variants;
  const double* ctx;                  /* GridSpec::context_knots */
  const double* tasks;                /* GridSpec::task_knots */
  const double* width;                /* GridSpec::width_knots */
  const double* peak_scaled;          /* per variant: peak_flops_for(dtype) * (f / f_max) */
  const double* elem_bytes;           /* per variant: 2 (fp16), 1 (fp8), 0.5 */
  const double* power;                /* per variant: tdp * scale * scale * scale */
  double mem_bw;                      /* DeviceSpec::peak_mem_bandwidth */
  double hidden, head_dim, kv_elems;  /* GridSpec::shape */
} psg_synth_grid;

/* Plan enumeration / device mapping on the device (generate_plans,
   planner.cpp:188-389): the host lists the candidate groups (model_dp,
   stages) with their per-cell scheme choices (enumerate_schemes order); the
   device maps each group onto the cluster (map_devices, cluster.cpp:118-198),
   and for every candidate (one per choice combination, last cell fastest)
   resolves the reshard collectives against that mapping (worst group span)
   and computes the memory ledger (finalize_plan, planner.cpp:307-370). */
#define PSG_PLAN_MAX_CELLS 8
#define PSG_PLAN_MAX_COLLS (2 * PSG_PLAN_MAX_CELLS)
typedef struct psg_plan_space {
  int32_t n_devices, per_node, n_levels;
  const int32_t* subtree_cap;         /* [n_levels + 1] devices per subtree of each level */
  double memory_capacity, activation_reserve, emb_bytes, kv_elem_bytes;
  int32_t include_embedding, num_layers, n_cells;
  const int32_t* cell_is_attention;   /* [n_cells] */
  const double* cell_kv_heads;        /* [n_cells] */
  const double* cell_head_dim;        /* [n_cells] */
  int32_t n_groups;
  const int32_t* group_dp;            /* [n_groups] */
  const int32_t* group_stages;
  const int32_t* group_sdev;          /* devices per stage */
  const int32_t* group_reps;          /* stage repetitions */
  const int64_t* group_first;         /* [n_groups + 1] candidate ranges */
  const int32_t* choice_begin;        /* [n_groups * n_cells + 1] */
  const int32_t* ch_mode;             /* per choice: CellScheme mode (0 TP, 1 EP), cell_dp, intra */
  const int32_t* ch_cdp;
  const int32_t* ch_intra;
  const double* ch_weight;            /* weight_bytes_per_device */
} psg_plan_space;

typedef struct psg_plan_record {
  int32_t feasible;                   /* static_bytes_per_device <= memory capacity */
  int32_t n_colls;
  double static_bytes_per_device, kv_budget_per_replica, kv_bytes_per_token;
  int32_t coll_kind[PSG_PLAN_MAX_COLLS];   /* PSG_COLL_* */
  int32_t coll_devices[PSG_PLAN_MAX_COLLS];
  int32_t coll_nodes[PSG_PLAN_MAX_COLLS];
  int32_t coll_groups[PSG_PLAN_MAX_COLLS];
  double coll_share[PSG_PLAN_MAX_COLLS];
} psg_plan_record;

/* Device-emitted plan set (generate_plans without host ExecutionPlans):
   the plan kernels' feasible candidates, first occurrence of each encoding,
   compacted on the device straight into the psg_plan_set SoA psg_search
   consumes.  The host lists the candidate space (psg_plan_space) and per
   candidate / choice the few values that are strings or CellScheme
   constants on the host side. */
typedef struct psg_plan_emit_in {
  const uint8_t* keep;                /* [candidates] 1: first occurrence of its encoding */
  const int32_t* enc_rank;            /* [candidates] rank of its encoding (std::string order) */
  const int32_t* ch_op;               /* [choices] CellScheme::op (PSG_OP_*) */
  const double* ch_tasks;             /* [choices] CellScheme::query_tasks */
  const double* ch_width;             /* [choices] CellScheme::query_width */
  const double* ch_scale;             /* [choices] CellScheme::token_scale */
  int32_t compute_dtype;              /* ExecutionPlan::compute_dtype */
  double payload_per_token;           /* p2p_payload_per_token == every collective's */
  double shape_hidden, shape_head_dim, shape_kv_elems;  /* ExecutionPlan::op_shape */
} psg_plan_emit_in;

typedef struct psg_plan_soa {
  psg_plan_set set;                   /* views into library-owned arrays */
  const int64_t* candidate;           /* per plan: its candidate index (group_first order) */
} psg_plan_soa;

typedef struct psg_context psg_context;

const char* psg_version(void);

/* Visible CUDA devices (0 and PSG_OK when there are none). */
int psg_device_count(int* count);

/* One context per device; a context is not thread-shared. */
int psg_context_create(int device, psg_context** out);
void psg_context_destroy(psg_context* ctx);
const char* psg_last_error(const psg_context* ctx);

/* seconds / joules: n_variants * 3 * n_ctx * n_tasks * n_width values each. */
int psg_synth_compute(psg_context* ctx, const psg_synth_grid* grid, double* seconds,
                      double* joules);

/* records: group_first[n_groups] entries; phys: [n_groups * n_devices]
   assignment ((r * stages + s) * stage_devices + slot); p2p: per group
   stages - 1 boundary node counts at p2p_offset[g] ([n_groups + 1]). */
int psg_plan_compute(psg_context* ctx, const psg_plan_space* space, psg_plan_record* records,
                     int32_t* phys, const int64_t* p2p_offset, int32_t* p2p);

/* Maps, finalizes and compacts the candidate space on the device (the
   kernels of psg_plan_compute plus plan_emit_kernel); *out is freed with
   psg_plan_soa_free.  InfeasibleError (3) when no candidate is kept. */
int psg_plan_emit(psg_context* ctx, const psg_plan_space* space, const psg_plan_emit_in* in,
                  psg_plan_soa** out);
void psg_plan_soa_free(psg_plan_soa* soa);

/* Evaluate-all-plans: plansim::search semantics (see header comment).
   Device memory grows with the search and stays cached in the context; a
   contiguous-batching search may add mixed-iteration cost tables for its
   longest entries, at most a quarter of the free device memory (PSG_MIXTAB=0
   disables them; results do not depend on them). */
int psg_search(psg_context* ctx, const psg_plan_set* plans,
               const psg_cluster* cluster, const psg_store* store,
               const psg_trace* trace, const psg_config* config,
               psg_result** out);

/* n independent searches (e.g. the design spaces of several quantization
   formats) run concurrently on one device, one context (stream, buffers,
   result) each; shared memory is sized for all of them at once.  outs[i] as
   from psg_search(ctxs[i], ...).  Returns the first failing search's code
   (psg_last_error(ctxs[i]) says which); on failure outs of the successful
   searches are still valid and must be freed.  kernel_span_ms (optional):
   device time from the first search's kernels starting to the last one's
   finishing (inputs resident, transfers excluded). */
int psg_search_many(psg_context* const* ctxs, int n, const psg_plan_set* const* plans,
                    const psg_cluster* const* clusters, const psg_store* const* stores,
                    const psg_trace* const* traces, const psg_config* const* configs,
                    psg_result** outs, double* kernel_span_ms);

/* Device ranking of gathered keys (multi-GPU merge): order[k] = index into
   keys of the k-th best entry under the comparator of simulator.cpp:283-294. */
int psg_rank_keys(psg_context* ctx, const psg_rank_key* keys, int64_t n,
                  int64_t* order);

void psg_result_free(psg_result* result);

#ifdef __cplusplus
}
#endif

#endif /* PSG_H_ */
