// psg_device.cuh — device-side data views and the bit-exact FP64 cost
// evaluator of the plan-search engine.
//
// Every floating-point expression here reproduces the reference's operation
// sequence with explicit round-to-nearest intrinsics
// (__dadd_rn / __dmul_rn / __ddiv_rn / __dsub_rn), so neither FMA
// contraction nor reassociation can change a bit; the file is also compiled
// with -fmad=false as a second guard.
#pragma once

#include <cstdint>

#include "psg.h"

namespace psg {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxCells = 8;      // cells per block (the reference IR emits 2)
constexpr int kMaxClampSlots = 64;

// ---------------------------------------------------------------------------
// Device views of the ABI inputs (all pointers are device pointers).
struct DPlans {
  int n_plans;
  const int32_t *model_dp, *num_stages, *stage_devices, *stage_reps, *dtype, *enc_rank;
  const double *kv, *budget, *p2p_ppt, *sh_hidden, *sh_head, *sh_kv;
  const int32_t *cell_begin, *cell_op;
  const double *cell_tasks, *cell_width, *cell_scale;
  const int32_t *coll_begin, *coll_kind, *coll_devices, *coll_nodes, *coll_groups;
  const double *coll_ppt, *coll_share;
  const int32_t *p2p_begin, *p2p_nodes;
};

struct DStore {
  const int32_t *c_n_ctx, *c_n_tasks, *c_n_width;
  const int64_t *c_knot_begin, *c_value_begin;
  const double *c_knots, *c_seconds, *c_joules;
  const int32_t* k_n;
  const int64_t* k_begin;
  const double *k_payload, *k_seconds, *k_joules;
};

struct DTrace {
  int64_t n;
  const int64_t *ctx, *gen;
  const double* arrival;
  const int32_t* slot;       // trace index -> output slot (rank in id order)
  const int32_t* seq;        // optional explicit per-replica order (unsorted traces)
};

// One simulation unit = (plan, frequency, DP replica): run_replica()
// (simulator.cpp:98-172) for one replica's share of the trace.
struct Unit {
  int32_t entry;       // local entry slot
  int32_t plan;
  int32_t fslot;       // frequency slot
  int32_t replica;
  int32_t replicas;    // model_dp
  int32_t n_req;       // requests in this replica
  int64_t seq_base;    // offset into DTrace::seq (if used)
  int64_t scratch;     // offset (elements) into the per-unit global scratch
};

struct UnitOut {
  double clock, energy, flops, bytes;
  int64_t iterations, max_batch, completed, rejected;
  int64_t sum_batch, admissions;  // work counters (algorithmic bytes)
  int32_t err;         // 0 ok, 1 chunk_size < 1, 2 missing table
  int32_t pad;
};

struct SimParams {
  DPlans P;
  DStore S;
  DTrace T;
  const double* freqs;
  const int32_t* cell_tab;   // [n_freq_slots * n_cells_total]
  const int32_t* coll_tab;   // [n_colls_total]
  const int32_t* p2p_tab;    // [n_p2p_total]
  const int32_t* entry_missing;  // per local entry: 1 if any table it queries is absent
  int32_t n_cells_total;
  const Unit* units;
  int32_t n_units;
  int32_t batch_mode;
  int64_t chunk_size;
  int64_t max_batch_size;
  int32_t anchor;
  int32_t smem_cap;          // active-list capacity held in shared memory
  int32_t memo_cap;          // decode-cost memo entries in shared memory
  int64_t n_slots;           // requests per entry (== trace length)
  // outputs
  UnitOut* uout;
  double* slot_ttft;         // [entries * n_slots]
  double* slot_tpot;
  double* slot_e2e;
  uint8_t* slot_status;      // 0 untouched, 1 completed, 2 rejected
  uint32_t* clamp_compute;   // per compute grid, bit 2*axis + above
  uint32_t* clamp_curve;     // per curve, bit 0 below / bit 1 above
  // scratch (global fallback for large batches)
  int32_t* g_i32;            // 6 int32 arrays per unit, stride n_req
  double* g_f64;             // 2 double arrays per unit, stride n_req
};

// ---------------------------------------------------------------------------
// Interpolation primitives (cost.cpp:85-102, :214-234, :279).

struct AxisPos {
  int lo, hi;
  double t;
  int clamp;  // -1 below, +1 above
};

// locate(): x <= first -> (0,0,t=0); x >= last -> (n-1,n-1,t=0);
// else hi = upper_bound(x), lo = hi-1, t = (x-k[lo])/(k[hi]-k[lo]).
__device__ __forceinline__ AxisPos locate(const double* __restrict__ k, int n, double x) {
  AxisPos p;
  p.t = 0.0;
  p.clamp = 0;
  const double first = __ldg(k);
  if (x <= first) {
    p.lo = p.hi = 0;
    p.clamp = x < first ? -1 : 0;
    return p;
  }
  const double last = __ldg(k + n - 1);
  if (x >= last) {
    p.lo = p.hi = n - 1;
    p.clamp = x > last ? 1 : 0;
    return p;
  }
  // upper_bound over (0, n-1): first index with k[i] > x; k[0] <= x < k[n-1].
  int lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(k + mid) > x) hi = mid; else lo = mid;
  }
  p.lo = lo;
  p.hi = hi;
  const double klo = __ldg(k + lo);
  p.t = __ddiv_rn(__dsub_rn(x, klo), __dsub_rn(__ldg(k + hi), klo));
  return p;
}

// Per-cell constant coordinates: the (tasks, width) positions are fixed for a
// (plan, cell), so they are located once per unit.
struct CellConst {
  int table;          // compute grid index
  int op;
  int n_ctx, n_tasks, n_width;
  int64_t knot_begin, value_begin;
  AxisPos pj, pk;
  double tasks, width, scale;
};

// Trilinear sample with the reference's skip-zero-weight loop order:
// acc += ((wi*wj)*wk)*v for ci, cj, ck in {0,1}.
__device__ __forceinline__ void sample_grid(const DStore& S, const CellConst& c,
                                            const AxisPos& pi, double& sec,
                                            double& joule) {
  const double* __restrict__ vs = S.c_seconds + c.value_begin;
  const double* __restrict__ vj = S.c_joules + c.value_begin;
  double as = 0.0, aj = 0.0;
#pragma unroll
  for (int ci = 0; ci < 2; ++ci) {
    const double wi = ci ? pi.t : __dsub_rn(1.0, pi.t);
    if (wi == 0.0) continue;
    const int i = ci ? pi.hi : pi.lo;
#pragma unroll
    for (int cj = 0; cj < 2; ++cj) {
      const double wj = cj ? c.pj.t : __dsub_rn(1.0, c.pj.t);
      if (wj == 0.0) continue;
      const int j = cj ? c.pj.hi : c.pj.lo;
#pragma unroll
      for (int ck = 0; ck < 2; ++ck) {
        const double wk = ck ? c.pk.t : __dsub_rn(1.0, c.pk.t);
        if (wk == 0.0) continue;
        const int k = ck ? c.pk.hi : c.pk.lo;
        const int64_t idx = (int64_t(i) * c.n_tasks + j) * c.n_width + k;
        const double w = __dmul_rn(__dmul_rn(wi, wj), wk);
        as = __dadd_rn(as, __dmul_rn(w, __ldg(vs + idx)));
        aj = __dadd_rn(aj, __dmul_rn(w, __ldg(vj + idx)));
      }
    }
  }
  sec = as;
  joule = aj;
}

// op_flops / op_bytes (cost.cpp:51-68), written in the reference's order.
__device__ __forceinline__ double op_flops(int op, double t, double k, double w,
                                           double hidden, double head_dim) {
  double f = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, t), k), hidden), w);
  if (op == PSG_OP_ATTENTION)
    f = __dadd_rn(f, __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(4.0, t), t), k), head_dim));
  return f;
}

__device__ __forceinline__ double op_bytes(int op, double t, double k, double w,
                                           double hidden, double kv_elems) {
  const double e = 2.0;  // simulator.cpp:43-44 always tallies 2-byte elements
  double b = __dmul_rn(__dmul_rn(__dmul_rn(k, hidden), w), e);
  b = __dadd_rn(b, __dmul_rn(__dmul_rn(__dmul_rn(2.0, t), hidden), e));
  if (op == PSG_OP_ATTENTION)
    b = __dadd_rn(b, __dmul_rn(__dmul_rn(__dmul_rn(t, k), kv_elems), e));
  return b;
}

// Collective curve: (1-t)*s[lo] + t*s[hi] (cost.cpp:279, :290).
__device__ __forceinline__ void sample_curve(const DStore& S, int curve, double x,
                                             double& sec, double& joule, int& clamp) {
  const int64_t b = __ldg(S.k_begin + curve);
  const int n = __ldg(S.k_n + curve);
  const AxisPos p = locate(S.k_payload + b, n, x);
  clamp = p.clamp;
  const double u = __dsub_rn(1.0, p.t);
  sec = __dadd_rn(__dmul_rn(u, __ldg(S.k_seconds + b + p.lo)),
                  __dmul_rn(p.t, __ldg(S.k_seconds + b + p.hi)));
  joule = __dadd_rn(__dmul_rn(u, __ldg(S.k_joules + b + p.lo)),
                    __dmul_rn(p.t, __ldg(S.k_joules + b + p.hi)));
}

}  // namespace psg
