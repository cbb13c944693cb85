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
int plan_compute(psg_context* ctx, const psg_plan_space* s, psg_plan_record* records,
                 int32_t* phys, const int64_t* p2p_offset, int32_t* p2p);
__global__ void sim_kernel(const SimParams p);       // one warp per block
__global__ void sim_kernel_spec(const SimParams p);  // + a speculation warp per block
__global__ void sim_kernel_emit(const SimParams p);  // iteration-record pass
__global__ void sim_kernel_chunked(const SimParams p);       // chunked-prefill variants
__global__ void sim_kernel_spec_chunked(const SimParams p);
// One CTA per entry; 32 warps hide the slot arrays' load latency in the
// radix-select sweeps.
constexpr int kReduceThreads = 1024;
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
constexpr int kScratchI32 = 7, kScratchF64 = 4;  // per-unit global fallback arrays

}  // namespace psg
