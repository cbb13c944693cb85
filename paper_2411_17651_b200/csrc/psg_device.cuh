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
constexpr int kMaxClampSlots = 64;  // collectives + distinct p2p curves of a plan
constexpr int kWindow = 32;         // prefetched upcoming requests per unit
constexpr int kProfSlots = 32;      // phase-profile counters per unit (dev builds)

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
  int64_t gtab;        // staged curves in SimParams::g_tab at this offset (doubles), or -1:
                       // shared memory (they fit the launch's per-unit budget)
  int64_t log_off;     // chain_replicas == 2, replica >= 1: tally log at SimParams::rlog + log_off
  int32_t log_cap;     // ... holding at most this many records
  int32_t pad;
};

struct UnitOut {
  double clock, energy, flops, bytes;
  int64_t iterations, max_batch, completed, rejected;
  int64_t sum_batch, admissions;  // work counters (algorithmic bytes)
  int32_t err;         // 0 ok, 1 chunk_size < 1, 2 missing table, 9 tally log overflow (internal)
  int32_t nlog;        // tally records logged (chain_replicas == 2, replica >= 1)
};

struct SimParams {
  DPlans P;
  DStore S;
  DTrace T;
  const double* freqs;
  const int32_t* cell_tab;   // [n_freq_slots * n_cells_total]
  const int32_t* coll_tab;   // [n_colls_total]
  const int32_t* p2p_tab;    // [n_p2p_total]
  const uint8_t* p2p_bslot;  // [n_p2p_total] boundary -> distinct p2p curve of its plan
  double* g_tab;             // global curve staging of units whose curves exceed tab_smem
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
  int32_t serial_run;        // decode runs longer than this take the closed form
  int32_t chain_replicas;    // 1: grid = entries, replicas run in order with one tally;
                             // 2: grid = replica groups (block_k0/k1), each group's replicas
                             // in order on one warp, groups concurrently, the last group to
                             // finish replays the tally from the later groups' logs;
                             // 0: grid = units, per-replica tallies (dev)
  int32_t speculate;         // 1: blockDim 64, a second warp prices the next mixed iteration
  int32_t spec_sleep_ns;     // the speculation warp's polling interval
  const int32_t* entry_unit_begin;  // [E+1] units of entry e (replica order) ...
  const int32_t* entry_units;       // ... as unit indices
  int32_t tab_smem;          // doubles of per-unit curve staging in shared memory
  int32_t cm2_cap;           // finish-summary groups (1024 slots each) in shared memory
  // precomputed cost tables (psg_tables.cu)
  const int32_t* cell_sig;   // [n_freq_slots * n_cells_total] -> cell signature
  const double* qtab;        // per signature, per token count: {t, e_raw, flops, bytes}
  const int64_t* qoff;       // [n_sig] first row of the signature
  const double* dectab;      // per local entry, per batch B >= 1: {dur, energy, flops, bytes}
  const int64_t* doff;       // [entries] first row of the entry
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
  unsigned long long* prof;  // PSG_PHASE_PROFILE builds: kProfSlots counters per unit
  const int64_t* entry_max_bs;  // per-entry max_batch_size override, or null
  // emit_iterations: one record + emit_S stage seconds / joules per iteration
  // at emit_off[unit] + n; null when off (macro-stepping on)
  psg_iteration* emit_it;
  double *emit_sec, *emit_jou;
  const int64_t* emit_off;
  int32_t emit_S;
  int32_t* g_i32;            // kGI32 int32 arrays per unit, stride n_req
  double* g_f64;             // kGF64 8-byte arrays per unit, stride n_req
  int64_t* g_cm;             // per-unit chunk minima once the active slots live in global memory
  double2* rlog;             // chain_replicas == 2: tally logs (Unit::log_off)
  int32_t* entry_done;       // chain_replicas == 2: groups finished per entry (zeroed per launch)
  const int32_t* block_k0;   // chain_replicas == 2: block b runs entry_units[block_k0[b] .. block_k1[b])
  const int32_t* block_k1;
  const int32_t* entry_groups;  // chain_replicas == 2: groups of entry e
  // Streamed results (config.detail): the warp that completes an entry writes
  // its per-request metrics (id order) and rejected ids straight into the
  // caller's pinned result arrays at offsets fixed before the launch (the
  // host derives every entry's completed count from the trace and the KV
  // budget), so the copy overlaps the entries still simulating.  null: off.
  psg_request_metrics* out_pr;  // device view of the pinned per_request array
  int64_t* out_rj;              // ... and of rejected_ids
  const int64_t* out_pr_off;    // [entries] first record of entry e
  const int64_t* out_rj_off;
  const int64_t* out_n_pr;      // [entries] expected completed requests
  int32_t* out_ok;              // [entries] 1: written (counts matched); else the host compacts
  const int64_t* slot_id;       // id by slot
  const int64_t* slot_gen;      // gen_len by slot
  // Mixed-iteration table (psg_tables.cu mixtab_kernel; contiguous batching,
  // search passes): per tabulated entry, per distinct context length r and
  // decode count B < mt_w, the whole cost {duration, energy, flops, bytes}
  // of the iteration {one prefill item of ctx_r tokens, decode = B}.
  const double* mixtab;         // null: off
  const int64_t* moff;          // [entries] first row of the entry, or -1
  const int32_t* t_crank;       // trace index -> rank of its context length
  int32_t mt_w;                 // decode counts 0 .. mt_w-1 per rank
};

// Parameters of the cost-table kernels (psg_tables.cu).
struct TabParams {
  DPlans P;
  DStore S;
  // cell signatures: (compute grid, token_scale, tasks, width, op, shape)
  int32_t n_sig;
  const int32_t* sig_table;
  const int32_t* sig_op;
  const double *sig_scale, *sig_tasks, *sig_width, *sig_hidden, *sig_head, *sig_kv;
  const int64_t* sig_rows;   // rows (token counts 0..rows-1) per signature
  const int64_t* qoff;
  double* qtab;
  // decode tables per local entry
  int32_t n_entries;
  const int32_t* ent_plan;
  const int32_t* ent_fslot;
  const int64_t* ent_rows;   // Dmax per entry (B = 1..Dmax)
  const int64_t* doff;
  const int32_t* cell_sig;   // [n_freq_slots * n_cells_total]
  int32_t n_cells_total;
  const int32_t* coll_tab;
  const int32_t* p2p_tab;
  const int32_t* entry_missing;
  double* dectab;
  // mixed-iteration table (SimParams::mixtab): entries mt_ent[0 .. n_mt)
  int32_t n_mt;
  int32_t mt_w;                // decode counts per rank
  int64_t mt_R;                // distinct context lengths
  const int32_t* mt_ent;
  const int64_t* mt_ctx;       // the distinct context lengths, ascending
  const int64_t* moff;
  double* mixtab;
  int64_t mt_T;                // iteration totals 0 .. mt_T-1 of the curve-value table
  int32_t mt_nq;               // curve slots per total (collectives + <= 2 distinct p2p)
  double* ctab;                // [n_mt][mt_nq][mt_T] double2
  // load test (mixsel_kernel): per tabulated entry the arrival rate of its
  // longest unit; the mean generation length of the trace
  const double* mt_lam;
  double mt_gen;
  int64_t* moff_rw;            // the same array as moff: -1 drops an entry
};

// ---------------------------------------------------------------------------
// Interpolation primitives (cost.cpp:85-102, :214-234, :279).  All table
// pointers are generic: the simulation kernel stages each unit's tables in
// shared memory (global memory only if they do not fit).

struct AxisPos {
  int lo, hi;
  double t;
  int clamp;  // -1 below, +1 above
};

// locate(): x <= first -> (0,0,t=0); x >= last -> (n-1,n-1,t=0);
// else hi = upper_bound(x), lo = hi-1, t = (x-k[lo])/(k[hi]-k[lo]).
__device__ __forceinline__ AxisPos locate(const double* k, int n, double x) {
  AxisPos p;
  p.t = 0.0;
  p.clamp = 0;
  const double first = k[0];
  if (x <= first) {
    p.lo = p.hi = 0;
    p.clamp = x < first ? -1 : 0;
    return p;
  }
  const double last = k[n - 1];
  if (x >= last) {
    p.lo = p.hi = n - 1;
    p.clamp = x > last ? 1 : 0;
    return p;
  }
  // upper_bound: first index with k[i] > x, knowing k[0] <= x < k[n-1]
  int lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] > x) hi = mid; else lo = mid;
  }
  p.lo = lo;
  p.hi = hi;
  const double klo = k[lo];
  p.t = __ddiv_rn(__dsub_rn(x, klo), __dsub_rn(k[hi], klo));
  return p;
}

// locate() with a segment hint (the segment of the table's previous query):
// consecutive queries of one table mostly land in the same knot interval
// (decode counts move by +-1 between events, payload knots are far apart), so
// two loads and compares replace the binary search.  The hinted interval
// k[h] <= x < k[h+1] gives exactly locate()'s (lo, hi, t), except x == k[0],
// where it yields (0, 1, t = 0) instead of (0, 0, 0) — the same sample, as the
// t-weighted corner then contributes an exact +0 (see sample()).
__device__ __forceinline__ AxisPos locate_hint(const double* k, int n, double x, int h) {
  if (h >= 0 && h + 1 < n) {
    const double klo = k[h], khi = k[h + 1];
    if (klo <= x && x < khi) {
      AxisPos p;
      p.lo = h;
      p.hi = h + 1;
      p.t = __ddiv_rn(__dsub_rn(x, klo), __dsub_rn(khi, klo));
      p.clamp = 0;
      return p;
    }
  }
  return locate(k, n, x);
}

constexpr int kMaxCombos = 4;  // nonzero (tasks, width) corner pairs of a cell

// One cost table as the evaluator sees it, in shared memory: knots[n] on the
// queried axis and vals[n][ncombo][2] (seconds, joules interleaved).
//  * compute grid of a cell: the (tasks, width) coordinates are fixed per
//    (plan, cell), so the grid is collapsed to the context axis; the nonzero
//    (cj, ck) corners are kept in the reference's loop order with weights
//    wj, wk (cost.cpp:214-234);
//  * collective curve: ncombo = 1, wj = wk = 1.  The generic sample
//    0 + ((w*1)*1)*s_lo + ((t*1)*1)*s_hi then equals the reference's
//    (1-t)*s[lo] + t*s[hi] (cost.cpp:279) bit for bit, including the t == 0
//    case where the reference adds +0.
struct QDesc {
  int kn_off, n, val_off, ncombo;
  int table;          // store table index (-1: missing)
  int is_cell, op;
  uint32_t clamp_tw;  // cells: tasks/width clamp bits (2..5), reported per query
  double wj[kMaxCombos], wk[kMaxCombos];
  double scale;       // cells: token_scale; curves: payload_bytes_per_token
  double share;       // curves: token_share (p2p: 1.0, exact)
  double emul;        // energy multiplier: stage_devices / groups_per_stage / 1 (p2p)
  double tasks, width;
};

// Trilinear sample with the reference's skip-zero-weight loop order:
// acc += ((wi*wj)*wk)*v over ci, then the (cj, ck) corners.
// The reference skips zero-weight corners; adding them instead is bit-
// identical because every table value is finite and >= 0 (loaders reject
// negatives), so a skipped term is an exact +0 and acc + (+0) == acc for the
// non-negative accumulator.  Dropping the skip removes two data-dependent
// branches (~20 cycles each on B200) from every query.
__device__ __forceinline__ void sample(const QDesc& d, const double* vals, const AxisPos& pi,
                                       double& sec, double& joule) {
  double as = 0.0, aj = 0.0;
#pragma unroll
  for (int ci = 0; ci < 2; ++ci) {
    const double wi = ci ? pi.t : __dsub_rn(1.0, pi.t);
    const double* v = vals + (ci ? pi.hi : pi.lo) * d.ncombo * 2;
#pragma unroll
    for (int k = 0; k < kMaxCombos; ++k) {
      if (k < d.ncombo) {
        const double w = __dmul_rn(__dmul_rn(wi, d.wj[k]), d.wk[k]);
        as = __dadd_rn(as, __dmul_rn(w, v[2 * k]));
        aj = __dadd_rn(aj, __dmul_rn(w, v[2 * k + 1]));
      }
    }
  }
  sec = as;
  joule = aj;
}

// The reference's query_time + query_energy of one compute grid, literally
// (cost.cpp:196-260: locate per axis, skip-zero-weight trilinear sum), reading
// the store from global memory.  Used by the table kernels.
__device__ __forceinline__ void cell_query_ref(const DStore& S, int table, double x, double tasks,
                                               double width, double& sec, double& joule,
                                               uint32_t& clamp) {
  const int nc = S.c_n_ctx[table], nt = S.c_n_tasks[table], nw = S.c_n_width[table];
  const double* kn = S.c_knots + S.c_knot_begin[table];
  const double* vs = S.c_seconds + S.c_value_begin[table];
  const double* vj = S.c_joules + S.c_value_begin[table];
  const AxisPos pi = locate(kn, nc, x);
  const AxisPos pj = locate(kn + nc, nt, tasks);
  const AxisPos pk = locate(kn + nc + nt, nw, width);
  clamp = uint32_t(pi.clamp < 0) | uint32_t(pi.clamp > 0) << 1 | uint32_t(pj.clamp < 0) << 2 |
          uint32_t(pj.clamp > 0) << 3 | uint32_t(pk.clamp < 0) << 4 | uint32_t(pk.clamp > 0) << 5;
  double as = 0.0, aj = 0.0;
  for (int ci = 0; ci < 2; ++ci) {
    const double wi = ci ? pi.t : __dsub_rn(1.0, pi.t);
    if (wi == 0.0) continue;
    for (int cj = 0; cj < 2; ++cj) {
      const double wj = cj ? pj.t : __dsub_rn(1.0, pj.t);
      if (wj == 0.0) continue;
      for (int ck = 0; ck < 2; ++ck) {
        const double wk = ck ? pk.t : __dsub_rn(1.0, pk.t);
        if (wk == 0.0) continue;
        const int64_t idx = (int64_t(ci ? pi.hi : pi.lo) * nt + (cj ? pj.hi : pj.lo)) * nw +
                            (ck ? pk.hi : pk.lo);
        const double w = __dmul_rn(__dmul_rn(wi, wj), wk);
        as = __dadd_rn(as, __dmul_rn(w, vs[idx]));
        aj = __dadd_rn(aj, __dmul_rn(w, vj[idx]));
      }
    }
  }
  sec = as;
  joule = aj;
}

// The reference's collective query (cost.cpp:262-291): (1-t)*s[lo] + t*s[hi].
__device__ __forceinline__ void curve_query_ref(const DStore& S, int curve, double x, double& sec,
                                                double& joule) {
  const int64_t b = S.k_begin[curve];
  const AxisPos p = locate(S.k_payload + b, S.k_n[curve], x);
  const double u = __dsub_rn(1.0, p.t);
  sec = __dadd_rn(__dmul_rn(u, S.k_seconds[b + p.lo]), __dmul_rn(p.t, S.k_seconds[b + p.hi]));
  joule = __dadd_rn(__dmul_rn(u, S.k_joules[b + p.lo]), __dmul_rn(p.t, S.k_joules[b + p.hi]));
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

}  // namespace psg
