// psg_reduce.cuh — shared declarations of the engine's kernels.
#pragma once

#include <cstddef>
#include <cstdint>

#include "psg.h"
#include "psg_device.cuh"

namespace psg {

struct EntryOut {
  double e2e, energy, flops, bytes, mean_ttft, mean_tpot, mfu, mbu, p95;
  double p50_ttft, p99_ttft, p50_tpot, p99_tpot, slo_ttft;
  int64_t iterations, max_batch, completed, rejected, sum_batch, admissions;
  int32_t err, pad;
};

struct ReduceParams {
  int64_t n_slots;
  int32_t cand_cap;          // radix-select candidates per statistic in dynamic shared memory (0: off)
  const uint8_t* slot_status;
  const double *slot_ttft, *slot_e2e;
  double* slot_tpot;  // numerators from the simulation; divided in place by entry_reduce_kernel
  const int64_t* slot_gen;   // gen_len by slot (id order)
  const int64_t* slot_id;    // id by slot
  const UnitOut* uout;
  const int32_t* entry_unit_begin;  // [entries + 1]
  const int32_t* entry_units;       // unit ids, replica order
  const double* entry_peak;         // peak_flops_for(dtype) * total_devices
  const int32_t* entry_enc_rank;
  const double* entry_freq;
  const int64_t* entry_global;      // global entry index
  double mem_bw;
  int32_t total_devices;
  int32_t objective;
  int32_t extras;
  int32_t chain_replicas;  // uout flops/bytes are running tallies: take the last replica's
  double ttft_slo;         // > 0: TTFT-SLO-constrained ranking (psg_config.ttft_slo)
  double slo_quantile;
  EntryOut* eout;
  psg_rank_key* keys;
};

__global__ void synth_compute_kernel(const psg_synth_grid g, double* sec, double* jou);
int synth_compute(psg_context* ctx, const psg_synth_grid* g, double* seconds, double* joules);
__global__ void plan_map_kernel(const psg_plan_space s, int32_t* phys_out, const int64_t* p2p_off,
                                int32_t* p2p_out, int32_t* span_nodes, int32_t* span_level);
__global__ void plan_candidate_kernel(const psg_plan_space s, const int32_t* span_nodes,
                                      psg_plan_record* out);
// plan_emit_kernel arguments: host per-candidate / per-choice values (device
// copies) and the psg_plan_set arrays it fills (device, sized for every
// candidate kept); counts = {plans, collectives, p2p boundaries}.
struct PlanEmitArgs {
  const uint8_t* keep;
  const int32_t* enc_rank;
  const int32_t* ch_op;
  const double *ch_tasks, *ch_width, *ch_scale;
  const int64_t* p2p_off;  // [groups + 1] into p2p (group boundary node counts)
  const int32_t* p2p;
  int32_t compute_dtype;
  double payload_per_token, shape_hidden, shape_head_dim, shape_kv_elems;
};
struct PlanEmitOut {
  int32_t *model_dp, *num_stages, *stage_devices, *stage_reps, *dtype, *enc_rank;
  double *kv, *budget, *p2p_ppt, *sh_hidden, *sh_head, *sh_kv;
  int32_t *cell_begin, *cell_op;
  double *cell_tasks, *cell_width, *cell_scale;
  int32_t *coll_begin, *coll_kind, *coll_devices, *coll_nodes, *coll_groups;
  double *coll_ppt, *coll_share;
  int32_t *p2p_begin, *p2p_nodes;
  int64_t* candidate;
  int32_t* counts;
};
constexpr int kEmitThreads = 1024;
__global__ void plan_emit_kernel(const psg_plan_space s, const psg_plan_record* rec,
                                 const PlanEmitArgs a, PlanEmitOut o);
int plan_emit(psg_context* ctx, const psg_plan_space* s, const psg_plan_emit_in* in,
              psg_plan_soa** out);
void plan_soa_free(psg_plan_soa* soa);
int plan_compute(psg_context* ctx, const psg_plan_space* s, psg_plan_record* records,
                 int32_t* phys, const int64_t* p2p_offset, int32_t* p2p);
__global__ void sim_kernel(const SimParams p);       // one warp per block
__global__ void sim_kernel_spec(const SimParams p);  // + a speculation warp per block
__global__ void sim_kernel_lane(const SimParams p);  // lane-resident slots, no speculation warp
__global__ void sim_kernel_emit(const SimParams p);  // iteration-record pass
__global__ void sim_kernel_chunked(const SimParams p);       // chunked-prefill variants
__global__ void sim_kernel_spec_chunked(const SimParams p);
// One CTA per entry, four resident per SM (a C5 search's 301 entries fit one
// wave): warp 0 runs the ordered means chain, warps 1..7 the radix select,
// each thread with kSweepU independent slot loads in flight.
constexpr int kReduceThreads = 256;
constexpr int kReduceStats = 6;       // p95 e2e, p50/p99 TTFT, p50/p99 TPOT, TTFT at the SLO quantile
constexpr int kReduceCandCap = 512;  // radix-select candidates kept per statistic (24 KB)
constexpr int kSweepU = 4;           // slots per thread per sweep iteration (loads in flight)
__global__ void entry_reduce_kernel(const ReduceParams r);
__global__ void offsets_kernel(const EntryOut* eout, int n_entries, int64_t* pr_off,
                               int64_t* rj_off, int64_t* totals);
__global__ void compact_kernel(const ReduceParams r, const int64_t* pr_off,
                               const int64_t* rj_off, psg_request_metrics* out_pr,
                               int64_t* out_rj);
__global__ void rank_kernel(const psg_rank_key* keys, int64_t n, int64_t* order);

size_t sim_smem_bytes(int smem_cap, int memo_cap, int tab_smem, int cm2_cap);
__global__ void qtab_kernel(const TabParams p);
__global__ void dectab_kernel(const TabParams p);
__global__ void mixtab_kernel(const TabParams p);
__global__ void colltab_kernel(const TabParams p);
__global__ void mixsel_kernel(const TabParams p);
constexpr int kScratchI32 = 7, kScratchF64 = 4;  // per-unit global fallback arrays

}  // namespace psg
