// psg_sim.cu — the simulation kernel: one warp per (plan, frequency,
// DP-replica) unit runs the reference's continuous-batching event loop
// (run_replica, /root/reference/proj/src/simulator.cpp:98-172, over
// BatchState, batching.cpp:11-125) and prices iterations with the profiled
// tables (iteration_time, simulator.cpp:17-87).
//
// B200 design:
//  * Scalar state is warp-uniform (every lane holds the same clock/energy),
//    so there is no broadcast; batch scans are lane-parallel over the active
//    slots with ballot/popc and REDUX reductions.
//  * Cell queries are table lookups: psg_tables.cu tabulates every cell
//    signature over token counts and every entry's decode-only iteration cost
//    over batch sizes in parallel before this kernel runs.  The serial path
//    only prices collectives (curves staged in shared memory) and performs
//    the reference-ordered adds.
//  * Shared memory holds everything an event touches: the active slots
//    (SoA, tombstoned, migrating to a global region only if the batch
//    outgrows them), a 32-request prefetch window of the replica's arrivals,
//    a decode-cost memo with the cached binade segments, and the unit's
//    collective curves.  In the speculation kernel a batch of at most one
//    warp lives in registers instead (lane i = slot i).
//  * The KV ledger is an exact integer: cap_tok = max{T : double(T)*kv <= cap}
//    turns every admission / overflow / admissibility test into an integer
//    compare.
//  * Exact event-driven macro-stepping: a decode-only iteration's workload is
//    {decode_count = B}, so its (seconds, joules, flops, bytes) are bit-
//    identical until the batch changes.  Between events (arrival of an
//    admissible/rejectable head, first finish, first KV overflow) the unit
//    runs the reference's sequential FP64 adds (software-pipelined), or for
//    long runs their exact closed form (psg_fastsum.cuh).
//  * Clamp warnings (cost.cpp:204-212, :273-278) are monotone in the token
//    count, so the unit tracks the extreme token counts / totals it queried
//    and derives the per-table flags once at the end.
#include <climits>

#include "psg_device.cuh"
#include "psg_fastsum.cuh"

namespace psg {

namespace {

constexpr int64_t kNoFin = INT64_MAX;  // prefill phase
constexpr int64_t kDead = INT64_MIN;   // tombstone (finished / evicted slot)
constexpr unsigned kNoRel = 0xffffffffu;
constexpr int kQvStride = kWarp + 1;  // query-value rows; +1 keeps lanes 0..3 on distinct banks
constexpr int kGI32 = 7;  // global fallback arrays: stack, tidx, ctx, gen, done, slot, items
constexpr int kGF64 = 4;  // adm, ft, arr, fin

// Phase profiler (dev builds only: -DPSG_PHASE_PROFILE; zero code otherwise).
// slots: 0 admit, 1 mixed scan, 2 cost eval, 3 mixed advance, 4 decode cost,
// 5 run setup, 6 tight loop, 7 finish, 8 evict, 9 head refill, 10 #mixed,
// 11 #decode runs, 12 #decode table reads, 13 #finish events, 14 #speculation hits, 15 total,
// 16 cycles waited for speculation results, 17 eval cycles of misses,
// speculation misses by cause: 18 no job, 19 not one item, 20 other decode
// count, 21 other tokens, 22 job not started; own evaluations: 23 query
// values (loads + curves), 24 the four chains, 25 stage pass; slot-array
// mode: 26 finish cycles, 27 #finish events, 28 #admissions, 29 #mixed,
// 30 cycles of admit passes that admitted, 31 cycles of outer passes that
// started in slot-array mode.
#ifdef PSG_PHASE_PROFILE
#define PROF_T0(v) const long long v = clock64()
#define PROF_ADD(slot, v) (prof_acc[slot] += (unsigned long long)(clock64() - (v)))
#define PROF_CNT(slot) (prof_acc[slot] += 1ull)
#else
#define PROF_T0(v)
#define PROF_ADD(slot, v)
#define PROF_CNT(slot)
#endif

// Warp sum of 32-bit lane values without 32-bit overflow (two REDUX).
__device__ __forceinline__ int64_t warp_sum_wide(unsigned v) {
  return int64_t(__reduce_add_sync(kFull, v & 0xffffu)) +
         (int64_t(__reduce_add_sync(kFull, v >> 16)) << 16);
}

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;  // std::max(a, b)
}

struct ActiveList {
  int32_t *tidx, *ctx, *gen, *done, *slot, *items;
  int64_t* fin;  // iteration index of the finishing decode step; kNoFin while prefilling
  double *adm, *ft, *arr;
};

// A collective / p2p curve staged in shared memory (cost.cpp:262-291).
struct CurveDesc {
  int kn_off, n, table, hint;  // hint: last interior interval (knot index) queried
  double ppt, share, emul;  // payload = (ppt * tokens) * share; energy * emul
};

__host__ __device__ constexpr size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Compile-time tuning knobs (defaults are the measured best; A/B variants are
// built with tools/variant_build.sh):
//   PSG_REG_ALL   1: lane-resident slots in sim_kernel too (default: only the
//                 speculation kernel)
//   PSG_PIPE_MIN  shortest decode run stepped by the software-pipelined loop
//   PSG_FILL_B    live slots at or below which a finish returns the batch to
//                 lane-resident slots
//   PSG_SHORT_COLS  short slot-array mode: while at most 32 x this many slots
//                 are in use, lane l mirrors the finish iteration of slots
//                 l, 32+l, ... in registers and the finish summary is not kept
#ifndef PSG_REG_ALL
#define PSG_REG_ALL 0
#endif
#ifndef PSG_PIPE_MIN
#define PSG_PIPE_MIN 8
#endif
#ifndef PSG_FILL_B
#define PSG_FILL_B 32
#endif
#ifndef PSG_SHORT_COLS  // slot-array batches of <= 32x this many slots keep their finish iterations in registers
#define PSG_SHORT_COLS 4
#endif
constexpr int kMemoCap = 256;  // decode-cost memo entries (SimParams::memo_cap must match)

// Fixed-size per-unit state lives in static shared memory: constant addresses,
// so the hot loops index it without recomputing a dynamic-shared base.
__shared__ __align__(16) double s_qv[4 * kQvStride];              // query values (4 chains)
__shared__ __align__(16) CurveDesc s_cdesc[kMaxClampSlots];       // staged curves
__shared__ __align__(16) int64_t s_cellq[kMaxCells];              // qtab row 0 per cell
__shared__ __align__(16) double s_p2p_val[2 * kMaxClampSlots];    // p2p (seconds, joules)
__shared__ __align__(16) double s_w_arr[kWindow];                 // prefetch window: arrival
__shared__ __align__(16) int32_t s_w_i32[5 * kWindow];            // tidx, ctx, gen, slot, ctx rank
__shared__ __align__(16) double s_memo[4 * kMemoCap];             // decode-only cost per B
// closed-form decode runs: per (B, accumulator) the binade segment key
// (exponent field << 53 | tie << 52 | R; 0 = none), psg_fastsum.cuh segment_key
__shared__ __align__(16) unsigned long long s_rkey[4 * kMemoCap];

struct SmemLayout {
  size_t qv, cdesc, cellq, p2p_val, win_arr, win_i32, memo, act_f64, act_fin, act_i32,
      cm1, cm2, tab, total;
};

__host__ __device__ SmemLayout smem_layout(int smem_cap, int memo_cap, int tab_smem, int cm2_cap) {
  SmemLayout L;
  size_t o = 0;
  (void)memo_cap;  // the fixed-size state is static shared memory (above)
  L.qv = L.cdesc = L.cellq = L.p2p_val = L.win_arr = L.win_i32 = L.memo = 0;
  L.act_f64 = o;   o = al16(o + sizeof(double) * 3 * size_t(smem_cap));
  L.act_fin = o;   o = al16(o + sizeof(int64_t) * size_t(smem_cap));
  L.act_i32 = o;   o = al16(o + sizeof(int32_t) * 6 * size_t(smem_cap));
  L.cm1 = o;       o = al16(o + sizeof(int64_t) * size_t(smem_cap / kWarp + 1));
  L.cm2 = o;       o = al16(o + sizeof(int64_t) * size_t(cm2_cap));
  L.tab = o;       o = al16(o + sizeof(double) * size_t(tab_smem));
  L.total = o;
  return L;
}

// Unit constants the cost evaluation reads (the main warp's registers; a
// copy in shared memory for the speculation warp).
struct EvalCtx {
  const double* qtab;
  const double* tab;      // the unit's staged curves (shared memory, or global if too large)
  const uint8_t* bslot;   // boundary -> distinct p2p curve (global, first-appearance order)
  uint64_t p2p_mask;      // the same for boundaries 0..63 when ND <= 2
  double sdd, reps, Sd;
  int C, K, NQ, ND, NB, n_curve_knots;
};

struct EvalOut {
  double cd, ce, cf, cb, srep, jrep;
};

// iteration_time (simulator.cpp:17-87) of {items, decode}: one lane per query
// (cell lanes read their qtab row, curve lanes interpolate their staged
// curve), lanes 0..3 run the four reference-ordered FP64 chains, then the
// stage pass.  `item(i)` is the i-th prefill item's token count.  qv / p2p_val
// are the calling warp's scratch.
// kPlain (the plain kernel, C5's): the knot search on a missed interval hint
// follows std::upper_bound's probes (log2 steps instead of a scan) and the
// stage-energy chain of up to 16 boundaries runs as predicated straight-line
// adds (deep pipelines, e.g. C5's pp16): C5 352 -> 344 ms.  The speculation
// kernel keeps the compact forms: there the larger code costs more than it
// saves (C2 +1-3%, measured).
template <bool kPlain = false, typename Item>
__device__ __forceinline__ EvalOut eval_iteration(const EvalCtx& E, const int lane, Item item,
                                                  const int n_items, const int64_t decode,
                                                  const int64_t total, const int64_t* cellq,
                                                  CurveDesc* cdesc, const double* tab,
                                                  const uint8_t* p2p_slot, double* qv,
                                                  double* p2p_val,
                                                  unsigned long long* prof = nullptr) {
#ifdef PSG_PHASE_PROFILE
  long long pt = clock64();
  auto pmark = [&](int slot) {
    const long long t = clock64();
    if (prof) prof[slot] += (unsigned long long)(t - pt);
    pt = t;
  };
#else
  auto pmark = [](int) {};
#endif
  const int nq_c = n_items + (decode > 0 ? 1 : 0);
  const int Qc = E.C * nq_c;
  const int Q = Qc + E.NQ;
  const double total_d = double(total);
  // lanes 0..3 run the four reference-ordered chains (seconds, joules,
  // flops, bytes); lanes 2, 3 stop at the cells (collectives add none)
  double chain = 0.0;
  const double* qrow = qv + (lane < 4 ? lane : 0) * kQvStride;
  const float inv_nq = __frcp_rn(float(nq_c));
  for (int base = 0; base < Q; base += kWarp) {
    const int q = base + lane;
    // cell query = one precomputed row {t, e_raw, flops, bytes}: issue the
    // loads first so their latency overlaps the curve lanes' work
    const bool cell_lane = q < Qc;
    double2 te = make_double2(0.0, 0.0), fb = make_double2(0.0, 0.0);
    if (cell_lane) {
      const int c = int((float(q) + 0.5f) * inv_nq);  // q / nq_c (q, nq_c < 2^16)
      const int i = q - c * nq_c;
      const int64_t tok = i < n_items ? int64_t(item(i)) : decode;
      const double2* row = reinterpret_cast<const double2*>(E.qtab + (cellq[c] + tok) * 4);
      te = __ldg(row);
      fb = __ldg(row + 1);
    }
    if (!cell_lane && q < Q) {
      // collective / p2p curve query on the staged curve
      const int k = q - Qc;
      CurveDesc& d = cdesc[k];
      const double x = __dmul_rn(__dmul_rn(d.ppt, total_d), d.share);
      const double* kn = tab + d.kn_off;
      const int cn = d.n;
      // cnt = #knots <= x; the last interval usually still holds
      const int h = d.hint;
      int cnt;
      if (h + 1 < cn && kn[h] <= x && x < kn[h + 1]) {
        cnt = h + 1;
      } else if (kPlain) {
        // std::upper_bound's probe sequence (locate, cost.cpp:97): ~log2(cn)
        // dependent steps instead of a scan of every knot
        int first = 0, len = cn;
        while (len > 0) {
          const int half = len >> 1;
          if (x < kn[first + half]) {
            len = half;
          } else {
            first += half + 1;
            len -= half + 1;
          }
        }
        cnt = first;
        if (cnt >= 1 && cnt < cn) d.hint = cnt - 1;
      } else {  // (the speculation kernel keeps the compact scan: C2 +1% otherwise)
        cnt = 0;
        for (int j = 0; j < E.n_curve_knots; ++j)
          cnt += (j < cn && kn[j < cn ? j : cn - 1] <= x) ? 1 : 0;
        if (cnt >= 1 && cnt < cn) d.hint = cnt - 1;
      }
      const bool lo_c = x <= kn[0], hi_c = x >= kn[cn - 1];
      const int lo = lo_c ? 0 : (hi_c ? cn - 1 : cnt - 1);
      const int hi = lo_c ? 0 : (hi_c ? cn - 1 : cnt);
      const bool interior = !(lo_c || hi_c);
      const double t = __ddiv_rn(interior ? __dsub_rn(x, kn[lo]) : 0.0,
                                 interior ? __dsub_rn(kn[hi], kn[lo]) : 1.0);
      const double u = __dsub_rn(1.0, t);
      const double* v = kn + cn;
      const double sec = __dadd_rn(__dmul_rn(u, v[2 * lo]), __dmul_rn(t, v[2 * hi]));
      const double jou = __dadd_rn(__dmul_rn(u, v[2 * lo + 1]), __dmul_rn(t, v[2 * hi + 1]));
      const double en = __dmul_rn(jou, d.emul);
      if (k >= E.K) {
        p2p_val[k - E.K] = sec;
        p2p_val[kMaxClampSlots + k - E.K] = en;
      } else {
        te = make_double2(sec, en);  // a collective adds seconds and energy only
      }
    }
    // Every lane writes its column — p2p and idle lanes zeros — so the four
    // chains run one uniform, 4-aligned trip count: the accumulators are sums
    // of non-negative values starting at +0, where adding +0.0 is exact.
    qv[lane] = te.x;
    qv[kQvStride + lane] = cell_lane ? __dmul_rn(te.y, E.sdd) : te.y;  // cells: x stage_devices
    qv[2 * kQvStride + lane] = fb.x;
    qv[3 * kQvStride + lane] = fb.y;
    __syncwarp();
    pmark(23);
    const int coll_end = min(kWarp, max(0, Qc + E.K - base));
    for (int l = 0; l < coll_end; l += 4) {
      const double v0 = qrow[l], v1 = qrow[l + 1], v2 = qrow[l + 2], v3 = qrow[l + 3];
      chain = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(chain, v0), v1), v2), v3);
    }
    __syncwarp();
    pmark(24);
  }
  const double bs = __shfl_sync(kFull, chain, 0);
  const double bj = __shfl_sync(kFull, chain, 1);
  const double bf = __shfl_sync(kFull, chain, 2);
  const double bb = __shfl_sync(kFull, chain, 3);
  // stages (simulator.cpp:64-78, :125-130): every stage prices the same
  // block * reps; boundary b adds its p2p to stage b+1
  EvalOut o;
  o.srep = __dmul_rn(bs, E.reps);
  o.jrep = __dmul_rn(bj, E.reps);
  double cd = dmax_ref(0.0, o.srep);
  double ce = __dadd_rn(0.0, o.jrep);
  if (E.ND <= 2 && E.NB <= 64) {
    const double s0 = __dadd_rn(o.srep, p2p_val[0]), s1 = __dadd_rn(o.srep, p2p_val[1]);
    const double j0 = __dadd_rn(o.jrep, p2p_val[kMaxClampSlots]);
    const double j1 = __dadd_rn(o.jrep, p2p_val[kMaxClampSlots + 1]);
    if (E.NB > 0) cd = dmax_ref(cd, s0);
    if (E.ND == 2) cd = dmax_ref(cd, s1);
    if (kPlain && E.NB > 0 && E.NB <= 16) {
      const unsigned mk = unsigned(E.p2p_mask);
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (b < E.NB) ce = __dadd_rn(ce, ((mk >> b) & 1u) ? j1 : j0);
    } else {
      for (int b = 0; b < E.NB; ++b) ce = __dadd_rn(ce, ((E.p2p_mask >> b) & 1) ? j1 : j0);
    }
  } else {
    for (int b = 0; b < E.NB; ++b) {
      const int s = __ldg(p2p_slot + b);
      cd = dmax_ref(cd, __dadd_rn(o.srep, p2p_val[s]));
      ce = __dadd_rn(ce, __dadd_rn(o.jrep, p2p_val[kMaxClampSlots + s]));
    }
  }
  o.cd = cd;
  o.ce = ce;
  o.cf = __dmul_rn(__dmul_rn(__dmul_rn(bf, E.sdd), E.reps), E.Sd);
  o.cb = __dmul_rn(__dmul_rn(__dmul_rn(bb, E.sdd), E.reps), E.Sd);
  pmark(25);
  return o;
}

// Speculative evaluation (block = 2 warps).  While the simulation warp runs a
// decode run, the speculation warp prices the mixed iteration the queue head
// will most likely trigger — items {head's first chunk}, decode = the current
// batch — with the same eval_iteration; if the real iteration matches, the
// simulation warp takes the result instead of pricing it.  Job hand-off is a
// seqlock in shared memory (posted is odd while a job is being written).
struct SpecSlot {
  EvalCtx ctx;           // the running unit's constants (written while the helper is idle)
  unsigned long long job;  // seq:20 | tok:22 | decode:22 — one store, no seqlock needed
  int started;           // seq the helper is pricing
  int done;              // seq of the results below
  int quit;
  int pad;
  double cd, ce, cf, cb;
};
constexpr int kSpecField = 22;  // tok, decode < 2^22 to be speculated
constexpr unsigned kSeqMask = (1u << 20) - 1u;
__shared__ __align__(16) SpecSlot s_spec;
__shared__ __align__(16) double s_qv2[4 * kQvStride];            // speculation warp scratch
__shared__ __align__(16) double s_p2p_val2[2 * kMaxClampSlots];

__device__ __forceinline__ int vload(const int& x) { return *reinterpret_cast<const volatile int*>(&x); }
__device__ __forceinline__ void vstore(int& x, int v) { *reinterpret_cast<volatile int*>(&x) = v; }
__device__ __forceinline__ unsigned long long vload64(const unsigned long long& x) {
  return *reinterpret_cast<const volatile unsigned long long*>(&x);
}
__device__ __forceinline__ void vstore64(unsigned long long& x, unsigned long long v) {
  *reinterpret_cast<volatile unsigned long long*>(&x) = v;
}

// max{T >= -1 : double(T) * kv <= cap} with the reference's exact product
// (kv is integral and every ledger value < 2^53, checked on the host).
__device__ int64_t ledger_cap_tokens(double kv, double cap) {
  if (!(kv > 0.0)) return (0.0 <= cap) ? (int64_t(1) << 60) : -1;
  if (!(0.0 <= cap)) return -1;
  const double q = floor(cap / kv);
  if (q >= 9007199254740992.0) return int64_t(1) << 53;  // beyond any ledger value
  int64_t t = int64_t(q);
  while (t >= 0 && __dmul_rn(double(t), kv) > cap) --t;
  while (!(__dmul_rn(double(t + 1), kv) > cap)) ++t;
  return t;
}


}  // namespace

// One DP replica (run_replica, simulator.cpp:98-172).  tally_flops / _bytes
// carry WorkTally across the entry's replicas (simulator.cpp:195-201).
// Refills the 32-request prefetch window from request w_base (rare: once per
// 32 admissions; out of line so the admit path stays compact).
__device__ __noinline__ void refill_window(const int32_t* seq, const double* arrival,
                                           const int64_t* ctx, const int64_t* gen,
                                           const int32_t* slot, const int32_t* crank,
                                           int64_t seq_base, int replica,
                                           int replicas, int n_req, int w_base, bool chunked,
                                           int64_t chunk, int C, const double* qtab,
                                           const int64_t* cellq) {
  const int lane = threadIdx.x & (kWarp - 1);
  const int j = w_base + lane;
  if (j < n_req) {
    const int t = seq ? seq[seq_base + j] : int(int64_t(replica) + int64_t(j) * replicas);
    s_w_arr[lane] = arrival[t];
    s_w_i32[lane] = t;
    s_w_i32[kWindow + lane] = int(ctx[t]);
    s_w_i32[2 * kWindow + lane] = int(gen[t]);
    s_w_i32[3 * kWindow + lane] = slot[t];
    s_w_i32[4 * kWindow + lane] = crank ? crank[t] : -1;
    // warm L1 with the cell rows this request's prefill will read
    int64_t first = ctx[t];
    if (chunked && chunk >= 1 && first > chunk) first = chunk;
    for (int c = 0; c < C; ++c)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(qtab + (cellq[c] + first) * 4));
  }
  __syncwarp();
}

// kMode: batching mode fixed at compile time (1 contiguous, 2 chunked) or
// read from the parameters (0).
template <bool kSpec, bool kEmit, int kMode, bool kLane = false>
__device__ __forceinline__ void sim_unit(const SimParams& p, const int unit_idx,
                                         double& tally_flops, double& tally_bytes,
                                         unsigned char* smem_raw) {
  const int lane = threadIdx.x;
  const unsigned lt_mask = (1u << lane) - 1u;
  const Unit U = p.units[unit_idx];
#ifdef PSG_PHASE_PROFILE
  unsigned long long prof_acc[kProfSlots] = {};
  const long long prof_start = clock64();
#endif

  const SmemLayout L = smem_layout(p.smem_cap, p.memo_cap, p.tab_smem, p.cm2_cap);
  double* qv = s_qv;
  CurveDesc* cdesc = s_cdesc;
  int64_t* cellq = s_cellq;
  const uint8_t* p2p_slot = p.p2p_bslot;  // advanced to the plan's boundaries below
  double* p2p_val = s_p2p_val;
  double* w_arr = s_w_arr;
  int32_t* w_i32 = s_w_i32;
  double* memo = s_memo;
  // curves too large for the shared-memory budget stage into the unit's
  // global region (host: Unit::gtab)
  double* tab = U.gtab >= 0 ? p.g_tab + U.gtab : reinterpret_cast<double*>(smem_raw + L.tab);

  // ---- plan constants (warp-uniform) ----
  const int pl = U.plan;
  const double kv = p.P.kv[pl], cap = p.P.budget[pl];
  const int S = p.P.num_stages[pl];
  const double reps = double(p.P.stage_reps[pl]);
  const double sdd = double(p.P.stage_devices[pl]);
  const double Sd = double(S);
  const double p2p_ppt = p.P.p2p_ppt[pl];
  const int c0 = p.P.cell_begin[pl], C = p.P.cell_begin[pl + 1] - c0;
  const int k0 = p.P.coll_begin[pl], K = p.P.coll_begin[pl + 1] - k0;
  const int b0 = p.P.p2p_begin[pl], NB = p.P.p2p_begin[pl + 1] - b0;
  const int64_t cap_tok = ledger_cap_tokens(kv, cap);
  const double* qtab = p.qtab;
  const double* dtab = p.dectab + p.doff[U.entry] * 4;  // row B-1 = decode-only cost of B
  // mixed iterations {one item of a context length, decode B < mt_w}: one
  // table row (psg_tables.cu mixtab_kernel) instead of pricing them here
  const double* mtab = nullptr;
  if (!kEmit && p.mixtab) {
    const int64_t mo = p.moff[U.entry];
    if (mo >= 0) mtab = p.mixtab + mo * 4;
  }

  // the speculation warp reads the unit's staged state: let it go idle first
  // 2: helper idles (dev); concurrent replicas (chain_replicas == 2) are short
  // and leave the helper to the DP=1 units
  const bool spec_on = kSpec && !kEmit && p.speculate == 1;
  if (spec_on)
    while (unsigned(vload(s_spec.done)) != unsigned(vload64(s_spec.job) >> 44)) {
    }
  __syncwarp();

  // distinct p2p tables in first-appearance order (the host's bslot uses
  // the same rule): boundaries only span 1 or 2 nodes in practice
  p2p_slot += b0;
  int ND = 0;
  uint64_t p2p_mask = 0;  // ND <= 2: bit b = distinct-curve slot of boundary b < 64
  for (int b = 0; b < NB; ++b) {
    const int t = p.p2p_tab[b0 + b];
    int s = 0;
    for (; s < ND; ++s)
      if (cdesc[K + s].table == t) break;
    if (s == ND) {
      if (lane == 0) cdesc[K + ND].table = t;
      ++ND;
      __syncwarp();
    }
    if (s == 1 && b < 64) p2p_mask |= uint64_t(1) << b;
  }
  const int NQ = K + ND;  // curves: collectives, then distinct p2p
  __syncwarp();
  for (int i = lane; i < 4 * kMemoCap; i += kWarp) {
    memo[i] = -1.0;
    s_rkey[i] = 0ull;
  }
  if (lane < C) {
    const int sig = p.cell_sig[size_t(U.fslot) * p.n_cells_total + c0 + lane];
    cellq[lane] = p.qoff[sig];
  }
  for (int q = lane; q < NQ; q += kWarp) {
    CurveDesc d;
    if (q < K) {
      const int g = k0 + q;
      d.table = p.coll_tab[g];
      d.ppt = p.P.coll_ppt[g];
      d.share = p.P.coll_share[g];
      d.emul = double(p.P.coll_groups[g]);  // query_energy * groups_per_stage
    } else {
      d.table = cdesc[q].table;
      d.ppt = p2p_ppt;  // payload = p2p_ppt * tokens; x * 1.0 is exact
      d.share = 1.0;
      d.emul = 1.0;
    }
    d.n = d.table >= 0 ? p.S.k_n[d.table] : 1;
    d.hint = 0;
    cdesc[q] = d;
  }
  __syncwarp();
  {  // stage the curves: knots[n] then (seconds, joules)[n] interleaved
    int off = 0;
    for (int q = 0; q < NQ; ++q) {
      const int n = cdesc[q].n, t = cdesc[q].table;
      double* kd = tab + off;
      if (t >= 0) {
        const int64_t b = p.S.k_begin[t];
        for (int i = lane; i < n; i += kWarp) {
          kd[i] = p.S.k_payload[b + i];
          kd[n + 2 * i] = p.S.k_seconds[b + i];
          kd[n + 2 * i + 1] = p.S.k_joules[b + i];
        }
      }
      if (lane == 0) cdesc[q].kn_off = off;
      off += 3 * n;
    }
  }
  int n_curve_knots = 1;  // longest payload axis among the unit's curves
  for (int q = 0; q < NQ; ++q) n_curve_knots = max(n_curve_knots, cdesc[q].n);
  __syncwarp();
  EvalCtx ectx;
  ectx.qtab = qtab;
  ectx.tab = tab;
  ectx.bslot = p2p_slot;
  ectx.p2p_mask = p2p_mask;
  ectx.sdd = sdd;
  ectx.reps = reps;
  ectx.Sd = Sd;
  ectx.C = C;
  ectx.K = K;
  ectx.NQ = NQ;
  ectx.ND = ND;
  ectx.NB = NB;
  ectx.n_curve_knots = n_curve_knots;
  unsigned spec_seq = unsigned(vload64(s_spec.job) >> 44);  // last posted job (warp-uniform)
  int spec_tok = -1;
  int64_t spec_dec = -1;
  if (spec_on && lane == 0) {
    s_spec.ctx = ectx;
    __threadfence_block();  // before any job of this unit
  }
  __syncwarp();
  auto spec_post = [&](int tok, int64_t dec) {
    spec_seq = (spec_seq + 1) & kSeqMask;
    if (lane == 0)
      vstore64(s_spec.job, (static_cast<unsigned long long>(spec_seq) << 44) |
                               (static_cast<unsigned long long>(tok) << kSpecField) |
                               static_cast<unsigned long long>(dec));
    spec_tok = tok;
    spec_dec = dec;
  };

  // ---- active slots ----
  int cap_now = p.smem_cap;
  ActiveList a;
  {
    double* af = reinterpret_cast<double*>(smem_raw + L.act_f64);
    int32_t* ai = reinterpret_cast<int32_t*>(smem_raw + L.act_i32);
    const int sc = p.smem_cap;
    a.adm = af;
    a.ft = af + sc;
    a.arr = af + 2 * sc;
    a.fin = reinterpret_cast<int64_t*>(smem_raw + L.act_fin);
    a.tidx = ai;
    a.ctx = ai + sc;
    a.gen = ai + 2 * sc;
    a.done = ai + 3 * sc;
    a.slot = ai + 4 * sc;
    a.items = ai + 5 * sc;
  }
  const size_t nr = size_t(U.n_req);
  int32_t* g_i = p.g_i32 + size_t(U.scratch) * kGI32;  // [stack | tidx ctx gen done slot items]
  double* g_f = p.g_f64 + size_t(U.scratch) * kGF64;   // [adm | ft | arr | fin]
  int32_t* g_stack = g_i;
  // Finish summary: cm1[c] = min decode fin of slots [32c, 32c+32), cm2[g] =
  // min of cm1 over chunks [32g, 32g+32) (kNoFin if none).  A finish event
  // visits only the groups / chunks whose minimum is due.
  int64_t* cm1 = reinterpret_cast<int64_t*>(smem_raw + L.cm1);
  int64_t* cm2 = reinterpret_cast<int64_t*>(smem_raw + L.cm2);
  int64_t* g_cm = p.g_cm + (U.scratch >> 5) + 2 * int64_t(unit_idx);

  auto req_tidx = [&](int j) -> int {
    return p.T.seq ? p.T.seq[U.seq_base + j]
                   : int(int64_t(U.replica) + int64_t(j) * U.replicas);
  };
  const size_t slot_base = size_t(U.entry) * size_t(p.n_slots);
  const bool chunked = kMode == 2 || (kMode == 0 && p.batch_mode == PSG_BATCH_CHUNKED);
  const int64_t chunk = p.chunk_size;
  const int64_t max_bs = p.entry_max_bs ? p.entry_max_bs[U.entry] : p.max_batch_size;
  constexpr bool stepwise = kEmit;  // iteration records (second pass): no macro-stepping
  const bool chunk_err = chunked && chunk < 1;
  const bool missing = p.entry_missing[U.entry] != 0;

  double clock = 0.0, energy = 0.0, flops = tally_flops, bytes = tally_bytes;
  // Replica groups (chain_replicas == 2): the replicas of groups >= 1 log
  // their tally increments (Unit::log_off >= 0) so the entry's last group to
  // finish can replay the one running WorkTally (simulator.cpp:195-201) in
  // replica order.  Records:
  // {cf, cb} of a mixed iteration, or {-B tag, j} of a j-iteration decode run
  // at batch B (its increments are the entry's decode-table row).
  const bool logging = !kEmit && p.chain_replicas == 2 && U.log_off >= 0;
  double2* const rlog = logging ? p.rlog + U.log_off : nullptr;
  int nlog = 0;
  int64_t n = 0, max_batch = 0, completed = 0, rejected = 0, sum_batch = 0, admissions = 0;
  int pend = 0, stack_top = 0, w_base = -kWindow;
  // Active slots in admission order with tombstones: B live of len used;
  // live slots below first_pre are all decode-phase (prefill frontier).
  int B = 0, len = 0, first_pre = 0, n_pre = 0;
  int64_t used = 0;  // KV ledger in tokens: sum(ctx + generated) <= cap_tok
  int64_t next_fin = kNoFin;
  int err = 0;
  int mix_r = -1;  // context-length rank of the last admission (-1: re-admitted from the stack)
  // the table row of the mixed iteration the last admission triggers, loaded
  // at admission (lane l < 4 holds value l) so its latency overlaps the scan
  double mt_pre = 0.0;
  int mt_pre_b = -1;  // ... for decode count mt_pre_b
  // Lane-resident mode: while the slots fit one warp (the common case), lane i
  // holds slot i in registers and the slot arrays / finish summary are not
  // maintained; spill() switches to the arrays when a 33rd slot is needed and
  // fill() switches back once the batch is small again.
  constexpr bool kReg = kSpec || kLane || PSG_REG_ALL;
  bool regm = kReg;
  // Short slot-array mode (!regm, len <= kShortCap): a.fin stays the source
  // of truth, lane l mirrors positions l, 32+l, ... in sf[] so a finish is a
  // register compare + ballot instead of a summary walk; cm1 / cm2 are not
  // maintained (rebuilt on leaving the mode).
  constexpr int kSC = PSG_SHORT_COLS > 0 ? PSG_SHORT_COLS : 1;
  constexpr int kShortCap = PSG_SHORT_COLS > 0 ? kSC * kWarp : 0;
  bool shm = !kReg && kShortCap > 0;
  int64_t sf[kSC];
#pragma unroll
  for (int h = 0; h < kSC; ++h) sf[h] = kDead;
  int32_t r_tidx = 0, r_ctx = 0, r_gen = 0, r_done = 0, r_slot = 0;
  int64_t r_fin = kDead;
  double r_adm = 0.0, r_ft = 0.0, r_arr = 0.0;
  // extreme cell-query token counts and iteration totals (clamp reporting)
  int tok_lo = INT_MAX, tok_hi = -1;          // cell token counts (< 2^31)
  int64_t tot_lo = INT64_MAX, tot_hi = -1;     // iteration totals
  int run_lo = INT_MAX, run_hi = -1;           // decode-run batch sizes (both of the above)

  // pending head (batching.hpp:93 pending_.front()), warp-uniform registers
  bool hd_valid = false, hd_stack = false;
  double hd_arr = 0.0;
  int hd_tidx = 0, hd_ctx = 0, hd_gen = 0, hd_slot = 0;
  auto load_head = [&]() {
    if (stack_top > 0) {  // evicted requests re-enter at the queue head
      hd_tidx = g_stack[stack_top - 1];
      hd_arr = p.T.arrival[hd_tidx];
      hd_ctx = int(p.T.ctx[hd_tidx]);
      hd_gen = int(p.T.gen[hd_tidx]);
      hd_slot = p.T.slot[hd_tidx];
      hd_valid = hd_stack = true;
      return;
    }
    hd_stack = false;
    hd_valid = pend < U.n_req;
    if (!hd_valid) return;
    if (pend >= w_base + kWindow) {  // refill the prefetch window
      PROF_T0(t_ref);
      w_base = pend;
      if (kReg) {  // out of line: the lane-resident kernels' admit path stays compact
        refill_window(p.T.seq, p.T.arrival, p.T.ctx, p.T.gen, p.T.slot, p.t_crank, U.seq_base, U.replica,
                      U.replicas, U.n_req, w_base, chunked, chunk, C, qtab, cellq);
      } else {
        const int j = w_base + lane;
        if (j < U.n_req) {
          const int t = req_tidx(j);
          w_arr[lane] = p.T.arrival[t];
          w_i32[lane] = t;
          w_i32[kWindow + lane] = int(p.T.ctx[t]);
          w_i32[2 * kWindow + lane] = int(p.T.gen[t]);
          w_i32[3 * kWindow + lane] = p.T.slot[t];
          w_i32[4 * kWindow + lane] = p.t_crank ? p.t_crank[t] : -1;
          // warm L1 with the cell rows this request's prefill will read
          int64_t first = p.T.ctx[t];
          if (chunked && chunk >= 1 && first > chunk) first = chunk;
          for (int c = 0; c < C; ++c)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(qtab + (cellq[c] + first) * 4));
        }
        __syncwarp();
      }
      PROF_ADD(9, t_ref);
    }
    const int w = pend - w_base;
    hd_arr = w_arr[w];
    hd_tidx = w_i32[w];
    hd_ctx = w_i32[kWindow + w];
    hd_gen = w_i32[2 * kWindow + w];
    hd_slot = w_i32[3 * kWindow + w];
  };
  auto reject_slot = [&](int slot) {
    if (lane == 0) p.slot_status[slot_base + slot] = 2;
    ++rejected;
  };
  auto min_rel = [&](int64_t fin, int64_t base) -> unsigned {  // decode slots only
    return (fin == kNoFin || fin == kDead) ? kNoRel : unsigned(fin - base);
  };
  auto rel_of = [&](int64_t v) -> unsigned {  // v: kNoFin or a fin >= n
    return v == kNoFin ? kNoRel : unsigned(v - n);
  };
  auto abs_of = [&](unsigned r) -> int64_t { return r == kNoRel ? kNoFin : n + int64_t(r); };
  // cm2[g] from the chunk minima of group g
  auto fix_group = [&](int g) {
    __syncwarp();
    const int nch = (len + kWarp - 1) / kWarp;
    const int c = g * kWarp + lane;
    const unsigned r = __reduce_min_sync(kFull, c < nch ? rel_of(cm1[c]) : kNoRel);
    if (lane == 0) cm2[g] = abs_of(r);
    __syncwarp();
  };
  // cm1[c] from the slots of chunk c
  auto fix_chunk = [&](int c) {
    __syncwarp();
    const int i = c * kWarp + lane;
    const unsigned r = __reduce_min_sync(kFull, i < len ? min_rel(a.fin[i], n) : kNoRel);
    if (lane == 0) cm1[c] = abs_of(r);
    __syncwarp();
  };
  auto rebuild_summary = [&]() {
    const int nch = (len + kWarp - 1) / kWarp;
    for (int c = 0; c < nch; ++c) fix_chunk(c);
    for (int g = 0; g * kWarp < nch; ++g) fix_group(g);
  };
  // short slot-array mode: mirror a.fin of positions < len into sf[]
  auto sf_load = [&]() {
    __syncwarp();
#pragma unroll
    for (int h = 0; h < kSC; ++h) sf[h] = h * kWarp + lane < len ? a.fin[h * kWarp + lane] : kDead;
  };
  auto sf_set = [&](int pos, int64_t v) {  // the owner lane of position pos
#pragma unroll
    for (int h = 0; h < kSC; ++h)
      if (h * kWarp + lane == pos) sf[h] = v;
  };
  // Order-preserving in-place compaction of the live slots.
  auto compact = [&]() {
    __syncwarp();
    int w = 0, below = 0;
    for (int base = 0; base < len; base += kWarp) {
      const int i = base + lane;
      const int64_t fin = i < len ? a.fin[i] : kDead;
      const bool live = fin != kDead;
      int32_t tidx = 0, ctx = 0, gen = 0, done = 0, slot = 0;
      double adm = 0.0, ft = 0.0, arr = 0.0;
      if (live) {
        tidx = a.tidx[i];
        ctx = a.ctx[i];
        gen = a.gen[i];
        done = a.done[i];
        slot = a.slot[i];
        adm = a.adm[i];
        ft = a.ft[i];
        arr = a.arr[i];
      }
      const unsigned km = __ballot_sync(kFull, live);
      const int pos = w + __popc(km & lt_mask);
      below += __popc(__ballot_sync(kFull, live && i < first_pre));
      __syncwarp();
      if (live) {
        a.tidx[pos] = tidx;
        a.ctx[pos] = ctx;
        a.gen[pos] = gen;
        a.done[pos] = done;
        a.slot[pos] = slot;
        a.fin[pos] = fin;
        a.adm[pos] = adm;
        a.ft[pos] = ft;
        a.arr[pos] = arr;
      }
      w += __popc(km);
      __syncwarp();
    }
    len = w;
    first_pre = below;
    if (shm) sf_load(); else rebuild_summary();
  };
  auto migrate = [&]() {
    // Move the (compacted) active slots to the unit's global region: capacity n_req.
    __syncwarp();
    int32_t* gi = g_i + nr;
    int64_t* gfin = reinterpret_cast<int64_t*>(g_f + 3 * nr);
    for (int i = lane; i < len; i += kWarp) {
      gi[i] = a.tidx[i];
      gi[nr + i] = a.ctx[i];
      gi[2 * nr + i] = a.gen[i];
      gi[3 * nr + i] = a.done[i];
      gi[4 * nr + i] = a.slot[i];
      g_f[i] = a.adm[i];
      g_f[nr + i] = a.ft[i];
      g_f[2 * nr + i] = a.arr[i];
      gfin[i] = a.fin[i];
    }
    __syncwarp();
    a.tidx = gi;
    a.ctx = gi + nr;
    a.gen = gi + 2 * nr;
    a.done = gi + 3 * nr;
    a.slot = gi + 4 * nr;
    a.items = gi + 5 * nr;
    a.adm = g_f;
    a.ft = g_f + nr;
    a.arr = g_f + 2 * nr;
    a.fin = gfin;
    for (int c = lane; c <= p.smem_cap / kWarp; c += kWarp) g_cm[c] = cm1[c];
    __syncwarp();
    cm1 = g_cm;
    cap_now = int(nr);
  };
  // Drops trailing tombstones so slot len-1 is the newest live request.
  auto trim = [&]() {
    __syncwarp();
    while (len > 0) {
      const int base = len > kWarp ? len - kWarp : 0;
      const int i = base + lane;
      const unsigned lm = __ballot_sync(kFull, i < len && a.fin[i] != kDead);
      if (lm) {
        len = base + kWarp - __clz(lm);
        break;
      }
      len = base;
    }
    first_pre = first_pre < len ? first_pre : len;
  };
  auto recompute_next_fin = [&]() {
    if (shm) {
      unsigned m = kNoRel;
#pragma unroll
      for (int h = 0; h < kSC; ++h) m = min(m, min_rel(sf[h], n));
      next_fin = abs_of(__reduce_min_sync(kFull, m));
      return;
    }
    const int ng = ((len + kWarp - 1) / kWarp + kWarp - 1) / kWarp;
    unsigned m = kNoRel;
    for (int base = 0; base < ng; base += kWarp) {
      const int g = base + lane;
      m = min(m, __reduce_min_sync(kFull, g < ng ? rel_of(cm2[g]) : kNoRel));
    }
    next_fin = abs_of(m);
  };
  // lane-resident slots -> slot arrays + finish summary
  auto spill = [&]() {
    if (lane < len) {
      a.tidx[lane] = r_tidx;
      a.ctx[lane] = r_ctx;
      a.gen[lane] = r_gen;
      a.done[lane] = r_done;
      a.slot[lane] = r_slot;
      a.fin[lane] = r_fin;
      a.adm[lane] = r_adm;
      a.ft[lane] = r_ft;
      a.arr[lane] = r_arr;
    }
    const unsigned pm = __ballot_sync(kFull, lane < len && r_fin == kNoFin);
    first_pre = pm ? __ffs(pm) - 1 : len;
    if (kShortCap > 0) {  // into the short slot-array mode
      sf[0] = lane < len ? r_fin : kDead;
#pragma unroll
      for (int h = 1; h < kSC; ++h) sf[h] = kDead;
      shm = true;
      __syncwarp();
    } else {
      rebuild_summary();
    }
    regm = false;
  };
  // slot arrays -> lane-resident slots (len <= kWarp)
  auto fill = [&]() {
    __syncwarp();
    r_fin = kDead;
    if (lane < len) {
      r_tidx = a.tidx[lane];
      r_ctx = a.ctx[lane];
      r_gen = a.gen[lane];
      r_done = a.done[lane];
      r_slot = a.slot[lane];
      r_fin = a.fin[lane];
      r_adm = a.adm[lane];
      r_ft = a.ft[lane];
      r_arr = a.arr[lane];
    }
    __syncwarp();
    regm = kReg;
    shm = false;
  };
  // order-preserving compaction of the lane-resident slots (staged through
  // the otherwise unused slot arrays)
  auto reg_compact = [&]() {
    const bool live = lane < len && r_fin != kDead;
    const unsigned km = __ballot_sync(kFull, live);
    const int pos = __popc(km & lt_mask);
    if (live) {
      a.tidx[pos] = r_tidx;
      a.ctx[pos] = r_ctx;
      a.gen[pos] = r_gen;
      a.done[pos] = r_done;
      a.slot[pos] = r_slot;
      a.fin[pos] = r_fin;
      a.adm[pos] = r_adm;
      a.ft[pos] = r_ft;
      a.arr[pos] = r_arr;
    }
    len = __popc(km);
    fill();
  };
  auto reg_trim = [&]() {
    const unsigned lm = __ballot_sync(kFull, lane < len && r_fin != kDead);
    len = lm ? kWarp - __clz(lm) : 0;
  };

  // the queue head changed: reload it (the lane-resident variant keeps one
  // call site of load_head for a smaller loop body)
  bool head_dirty = kReg;
  if (!kReg) load_head();
#ifdef PSG_PHASE_PROFILE
  long long pass_t = clock64();
  bool pass_arr = false;
#endif
  while (true) {
#ifdef PSG_PHASE_PROFILE
    {
      const long long now = clock64();
      if (pass_arr) prof_acc[31] += (unsigned long long)(now - pass_t);
      pass_t = now;
      pass_arr = !regm;
    }
    const int64_t adm0 = admissions;
#endif
    // ---- admit (batching.cpp:35-60) ----
    PROF_T0(t_adm);
    while (true) {
      if (kReg && head_dirty) {
        load_head();
        head_dirty = false;
      }
      if (!(hd_valid && hd_arr <= clock)) break;
      if (hd_ctx <= cap_tok) {  // context alone fits; else rejected below
        if (max_bs > 0 && int64_t(B) >= max_bs) break;
        if (used + hd_ctx > cap_tok) break;  // head blocks, FIFO
        if (regm && len == kWarp) {
          if (B < kWarp) reg_compact();
          if (len == kWarp) spill();
        }
        if (regm) {
          if (lane == len) {
            r_tidx = hd_tidx;
            r_ctx = hd_ctx;
            r_gen = hd_gen;
            r_done = 0;
            r_slot = hd_slot;
            r_fin = kNoFin;
            r_adm = clock;
            r_ft = 0.0;
            r_arr = hd_arr;
          }
        } else {
          if (shm && len == kShortCap) {  // the short mode is full
            if (B < len) compact();
            if (len == kShortCap) {
              rebuild_summary();
              shm = false;
            }
          }
          if (len >= cap_now) {
            if (len > B) compact();
            if (len >= cap_now) migrate();
          }
          if (shm) sf_set(len, kNoFin);
          if (lane == 0) {
            if (!shm) {
              if ((len & (kWarp - 1)) == 0) cm1[len / kWarp] = kNoFin;  // fresh chunk / group
              if ((len & (kWarp * kWarp - 1)) == 0) cm2[len / (kWarp * kWarp)] = kNoFin;
            }
            a.tidx[len] = hd_tidx;
            a.ctx[len] = hd_ctx;
            a.gen[len] = hd_gen;
            a.done[len] = 0;
            a.slot[len] = hd_slot;
            a.fin[len] = kNoFin;
            a.adm[len] = clock;
            a.ft[len] = 0.0;
            a.arr[len] = hd_arr;
          }
        }
        ++len;
        ++B;
        ++n_pre;
        ++admissions;
        used += hd_ctx;
        mix_r = hd_stack ? -1 : w_i32[4 * kWindow + (pend - w_base)];
        // (slot-array kernel only: the lane-resident loop measured slower with it)
        if (!kReg && mtab && mix_r >= 0 && B - 1 < p.mt_w) {  // the rest of the batch decodes
          mt_pre = __ldg(mtab + (int64_t(mix_r) * p.mt_w + (B - 1)) * 4 + (lane & 3));
          mt_pre_b = B - 1;
        }
      } else {
        reject_slot(hd_slot);
      }
      if (hd_stack) --stack_top; else ++pend;
      if (kReg) head_dirty = true; else load_head();
    }
    __syncwarp();
    PROF_ADD(0, t_adm);
#ifdef PSG_PHASE_PROFILE
    if (admissions != adm0) {
      prof_acc[30] += (unsigned long long)(clock64() - t_adm);
      if (!regm) prof_acc[28] += (unsigned long long)(admissions - adm0);
    }
#endif

    if (B == 0) {  // idle (simulator.cpp:116-120)
      if (!hd_valid) break;
      clock = dmax_ref(clock, hd_arr);
      continue;
    }
    if (chunk_err) { err = 1; break; }
    if (missing) { err = 2; break; }

    bool settle = true;
    if (n_pre > 0 || stepwise) {
      // ---- mixed iteration (batching.cpp:62-108): prefill items from the
      // prefill frontier, decode count = the rest ----
      PROF_CNT(10);
#ifdef PSG_PHASE_PROFILE
      if (!regm) prof_acc[29] += 1ull;
#endif
      PROF_T0(t_m1);
      int n_items = 0;
      int64_t pre_tok = 0;
      unsigned it_lo = 0xffffffffu, it_hi = 0;
      if (regm) {
        const bool pre = lane < len && r_fin == kNoFin;
        int tok = 0;
        if (pre) {
          int64_t t = int64_t(r_ctx) - r_done;
          if (chunked) t = t < chunk ? t : chunk;
          tok = int(t);
        }
        const unsigned pm = __ballot_sync(kFull, pre);
        if (pre) a.items[__popc(pm & lt_mask)] = tok;
        n_items = __popc(pm);
        pre_tok = __reduce_add_sync(kFull, unsigned(tok));
        it_lo = __reduce_min_sync(kFull, pre ? unsigned(tok) : 0xffffffffu);
        it_hi = __reduce_max_sync(kFull, pre ? unsigned(tok) : 0u);
      } else {
      for (int base = first_pre; base < len; base += kWarp) {
        const int i = base + lane;
        const bool pre = i < len && a.fin[i] == kNoFin;
        int tok = 0;
        if (pre) {
          int64_t t = int64_t(a.ctx[i]) - a.done[i];
          if (chunked) t = t < chunk ? t : chunk;
          tok = int(t);
        }
        const unsigned pm = __ballot_sync(kFull, pre);
        if (pre) a.items[n_items + __popc(pm & lt_mask)] = tok;
        n_items += __popc(pm);
        pre_tok += __reduce_add_sync(kFull, unsigned(tok));
        it_lo = min(it_lo, __reduce_min_sync(kFull, pre ? unsigned(tok) : 0xffffffffu));
        it_hi = max(it_hi, __reduce_max_sync(kFull, pre ? unsigned(tok) : 0u));
      }
      }
      __syncwarp();
      const int64_t decode = int64_t(B) - n_items;
      const int64_t total = decode + pre_tok;
      if (n_items > 0) {
        tok_lo = min(tok_lo, int(it_lo));
        tok_hi = max(tok_hi, int(it_hi));
      }
      if (decode > 0) {
        tok_lo = min(tok_lo, int(decode));
        tok_hi = max(tok_hi, int(decode));
      }
      tot_lo = min(tot_lo, total);
      tot_hi = max(tot_hi, total);
      PROF_ADD(1, t_m1);

      // ---- iteration_time (simulator.cpp:17-87) ----
      PROF_T0(t_ev);
      EvalOut ev;
      bool use_spec = false;
      // contiguous batching: a single prefill item is the request admitted in
      // this pass (every earlier one completed its prefill)
      const bool use_mt = mtab && n_items == 1 && decode < p.mt_w && mix_r >= 0;
      if (spec_on && !use_mt && n_items == 1 && decode == spec_dec && a.items[0] == spec_tok) {
        // the speculation warp prices exactly this iteration: wait for it if
        // it has started (it is ahead of us), else price it here
        const unsigned st = unsigned(__shfl_sync(kFull, vload(s_spec.started), 0));
        use_spec = st == spec_seq;
      }
#ifdef PSG_PHASE_PROFILE
      if (spec_on && !use_spec && !use_mt) {  // speculation miss: why
        const int why = spec_tok < 0 ? 18 : n_items != 1 ? 19 : decode != spec_dec ? 20
                        : a.items[0] != spec_tok ? 21 : 22;
        prof_acc[why] += 1ull;
      }
#endif
      if (use_mt) {
        PROF_T0(t_mt);
        if (!kReg && decode == mt_pre_b) {
          ev.cd = __shfl_sync(kFull, mt_pre, 0);
          ev.ce = __shfl_sync(kFull, mt_pre, 1);
          ev.cf = __shfl_sync(kFull, mt_pre, 2);
          ev.cb = __shfl_sync(kFull, mt_pre, 3);
        } else {
          const double2* row = reinterpret_cast<const double2*>(mtab + (int64_t(mix_r) * p.mt_w + decode) * 4);
          const double2 x = __ldg(row), y = __ldg(row + 1);
          ev.cd = x.x;
          ev.ce = x.y;
          ev.cf = y.x;
          ev.cb = y.y;
        }
        ev.srep = ev.jrep = 0.0;
        PROF_ADD(17, t_mt);
      } else if (use_spec) {
        PROF_CNT(14);
        PROF_T0(t_wait);
        while (unsigned(vload(s_spec.done)) != spec_seq) {
        }
        PROF_ADD(16, t_wait);
        __threadfence_block();
        ev.cd = s_spec.cd;
        ev.ce = s_spec.ce;
        ev.cf = s_spec.cf;
        ev.cb = s_spec.cb;
        ev.srep = ev.jrep = 0.0;  // stage values only matter when emitting (no speculation)
        spec_tok = -1;
        __syncwarp();
      } else {
        PROF_T0(t_own);
        ev = eval_iteration<!kSpec && !kEmit>(
            ectx, lane, [&](int i) { return a.items[i]; }, n_items, decode, total, cellq, cdesc,
            tab, p2p_slot, qv, p2p_val
#ifdef PSG_PHASE_PROFILE
            , prof_acc
#endif
        );
        PROF_ADD(17, t_own);
      }
      const double srep = ev.srep, jrep = ev.jrep;
      const double cd = ev.cd, ce = ev.ce, cf = ev.cf, cb = ev.cb;
      if (stepwise) {  // IterationRecord (simulator.cpp:158-170)
        const int64_t r = p.emit_off[unit_idx] + n;
        if (lane == 0) {
          psg_iteration it;
          it.clock_start = clock;
          it.duration = cd;
          it.energy = ce;
          it.batch_size = B;
          p.emit_it[r] = it;
        }
        double* sv = p.emit_sec + r * int64_t(p.emit_S);
        double* jv = p.emit_jou + r * int64_t(p.emit_S);
        for (int st = lane; st < S; st += kWarp) {
          double sec = srep, jou = jrep;  // stage s: block * reps, + p2p of boundary s-1
          if (st > 0 && st - 1 < NB) {
            const int sl = __ldg(p2p_slot + st - 1);
            sec = __dadd_rn(srep, p2p_val[sl]);
            jou = __dadd_rn(jrep, p2p_val[kMaxClampSlots + sl]);
          }
          sv[st] = sec;
          jv[st] = jou;
        }
      }
      PROF_ADD(2, t_ev);

      // ---- advance (batching.cpp:78-93) over the prefill frontier ----
      PROF_T0(t_m3);
      clock = __dadd_rn(clock, cd);
      energy = __dadd_rn(energy, ce);
      flops = __dadd_rn(flops, cf);
      bytes = __dadd_rn(bytes, cb);
      if (logging) {
        if (lane == 0 && nlog < U.log_cap) rlog[nlog] = make_double2(cf, cb);
        ++nlog;
      }
      max_batch = max_batch > B ? max_batch : int64_t(B);
      sum_batch += B;
      const int64_t n_new = n + 1;
      unsigned ncompl = 0, m = min_rel(next_fin, n_new);
      int new_fp = -1;
      if (regm) {
        bool compl_now = false;
        unsigned rel = kNoRel;
        if (lane < len && r_fin == kNoFin) {
          int64_t tok = int64_t(r_ctx) - r_done;
          if (chunked) tok = tok < chunk ? tok : chunk;
          const int64_t done = r_done + tok;
          r_done = int32_t(done);
          if (done == r_ctx) {  // the prefill iteration samples the first token
            const int64_t fin = n_new + (r_gen > 1 ? r_gen - 1 : 0);
            r_fin = fin;
            r_ft = clock;
            compl_now = true;
            rel = unsigned(fin - n_new);
          }
        }
        ncompl = __popc(__ballot_sync(kFull, compl_now));
        m = min(m, __reduce_min_sync(kFull, rel));
      } else {
      for (int base = first_pre & ~(kWarp - 1); base < len; base += kWarp) {  // whole chunks
        const int i = base + lane;
        bool compl_now = false, still = false;
        unsigned rel = kNoRel;
        int64_t fin = kDead;
        if (i < len && a.fin[i] == kNoFin) {
          const int32_t ctx = a.ctx[i];
          int64_t tok = int64_t(ctx) - a.done[i];
          if (chunked) tok = tok < chunk ? tok : chunk;
          const int64_t done = a.done[i] + tok;
          a.done[i] = int32_t(done);
          if (done == ctx) {  // the prefill iteration samples the first token
            const int32_t gen = a.gen[i];
            fin = n_new + (gen > 1 ? gen - 1 : 0);
            a.fin[i] = fin;
            a.ft[i] = clock;
            compl_now = true;
            rel = unsigned(fin - n_new);
          } else {
            still = true;
          }
        }
        if (shm) {  // mirror the new decode slots
          const int c = base / kWarp;
#pragma unroll
          for (int h = 0; h < kSC; ++h)
            if (compl_now && h == c) sf[h] = fin;
        }
        ncompl += __popc(__ballot_sync(kFull, compl_now));
        const unsigned cr = __reduce_min_sync(kFull, rel);
        m = min(m, cr);
        if (!shm && cr != kNoRel && lane == 0) {  // new decode slots in this chunk
          const int64_t v = n_new + int64_t(cr);
          const int c = base / kWarp;
          cm1[c] = min(cm1[c], v);
          cm2[c / kWarp] = min(cm2[c / kWarp], v);
        }
        const unsigned sm = __ballot_sync(kFull, still);
        if (new_fp < 0 && sm) new_fp = base + __ffs(sm) - 1;
      }
      first_pre = new_fp < 0 ? len : new_fp;
      }
      __syncwarp();
      used += decode + int64_t(ncompl);
      n_pre -= int(ncompl);
      n = n_new;
      next_fin = m == kNoRel ? kNoFin : n + m;
      PROF_ADD(3, t_m3);
    } else {
      // ---- decode-only run: exact macro-stepping ----
      PROF_CNT(11);
      PROF_T0(t_d1);
      // decode-only cost of B: the memo row (two 16-byte loads issued
      // together), else the entry's decode table (first run at this B)
      double d = -1.0, e = 0.0, f = 0.0, b = 0.0;
      if (B <= kMemoCap) {
        const double2* mrow = reinterpret_cast<const double2*>(memo + 4 * (B - 1));
        const double2 de = mrow[0], fb = mrow[1];
        d = de.x;
        e = de.y;
        f = fb.x;
        b = fb.y;
      }
      if (!(d >= 0.0)) {
        PROF_CNT(12);
        const double2* row = reinterpret_cast<const double2*>(dtab + int64_t(B - 1) * 4);
        const double2 de = __ldg(row), fb = __ldg(row + 1);
        d = de.x;
        e = de.y;
        f = fb.x;
        b = fb.y;
        if (B <= kMemoCap) {
          if (lane == 0) {
            memo[4 * (B - 1) + 1] = e;
            memo[4 * (B - 1) + 2] = f;
            memo[4 * (B - 1) + 3] = b;
            memo[4 * (B - 1)] = d;
          }
          __syncwarp();
        }
        // decode-run batch extremes for the clamp report: every batch size
        // passes here on its first run
        run_lo = min(run_lo, B);
        run_hi = max(run_hi, B);
      }
      PROF_ADD(4, t_d1);
      PROF_T0(t_d2);
      // iterations until the first finish (inclusive), cut at the first KV
      // overflow (batching.cpp:112): used + k*B > cap_tok
      int64_t kmax = next_fin - n;
      if (used + kmax * int64_t(B) > cap_tok) {
        // (cap_tok - used) / B + 1 without a 64-bit integer division: both
        // are < 2^53, so the float quotient is within one of the exact one
        const int64_t num = cap_tok - used;
        int64_t q = int64_t(__ddiv_rz(double(num), double(B)));
        if (q * int64_t(B) > num) --q;
        if ((q + 1) * int64_t(B) <= num) ++q;
        kmax = q + 1;
      }
      // Arrival event: only a not-yet-arrived head can change the batch; an
      // arrived head that admit() left in place stays blocked for the whole
      // run (used only grows, B is fixed).
      bool check = false, rej_h = false;
      if (hd_valid && !hd_stack && hd_arr > clock) {
        rej_h = hd_ctx > cap_tok;
        if (rej_h) {
          check = true;
        } else if (!(max_bs > 0 && int64_t(B) >= max_bs) && used + hd_ctx <= cap_tok) {
          check = true;  // admissible at iteration start j while used + j*B + ctx fits
        }
      }
      // speculate only when the head arrives before the next finish (the batch
      // it joins is then exactly this one); the estimate only picks jobs,
      // correctness comes from the exact match at use
      if (spec_on && n_pre == 0 && hd_valid && !hd_stack && hd_arr > clock && !rej_h &&
          hd_arr < clock + double(next_fin - n) * d && !(mtab && B < p.mt_w)) {
        int64_t first = hd_ctx;  // the head's first prefill chunk
        if (chunked && first > chunk) first = chunk;
        if ((int(first) != spec_tok || int64_t(B) != spec_dec) && first < (1 << kSpecField) &&
            B < (1 << kSpecField))
          spec_post(int(first), int64_t(B));
      }
      bool stop = false;
      PROF_ADD(5, t_d2);
      PROF_T0(t_d3);
      int64_t j = 0;
      bool cf = false;
      if (kmax > p.serial_run) {
        // Closed-form run (psg_fastsum.cuh): lanes 1..3 carry energy / flops /
        // bytes, the others the clock.  Each accumulator's binade segment
        // (per-step mantissa increment R) depends only on its increment —
        // fixed for this B — and its exponent, so it is cached per (B,
        // accumulator) and the whole run is integer arithmetic when every
        // accumulator's segment is cached and the run stays in its binade.
        const int al = (lane >= 1 && lane <= 3) ? lane : 0;
        const double acc = al == 1 ? energy : al == 2 ? flops : al == 3 ? bytes : clock;
        const double inc = al == 1 ? e : al == 2 ? f : al == 3 ? b : d;
        const uint64_t abits = uint64_t(__double_as_longlong(acc));
        unsigned long long key = B <= kMemoCap ? s_rkey[4 * (B - 1) + al] : 0ull;
        if ((key >> 53) != (abits >> 52)) {  // new batch size or binade: derive it
          int64_t keb = 0, R = 0;
          bool tie = false;
          key = 0ull;
          if (fastsum::segment_key(acc, inc, keb, R, tie) && R < (int64_t(1) << 52))
            key = (uint64_t(keb) << 53) | (uint64_t(tie) << 52) | uint64_t(R);
          if (B <= kMemoCap && lane < 4) s_rkey[4 * (B - 1) + lane] = key;
        }
        const int64_t m = int64_t(abits & uint64_t(fastsum::kHidden - 1)) | fastsum::kHidden;
        const int64_t R = int64_t(key & ((uint64_t(1) << 52) - 1));
        const bool ok = key != 0ull && !(((key >> 52) & 1) && (m & 1)) &&
                        (R == 0 || fastsum::fits(kmax, R, fastsum::kTop - 2 - m));
        if (__all_sync(kFull, ok)) {
          const int64_t Rc = __shfl_sync(kFull, R, 0);  // the clock's segment
          const int64_t mc = __shfl_sync(kFull, m, 0);
          const int64_t ec = int64_t(__double_as_longlong(clock) >> 52);
          double a = check ? hd_arr : __longlong_as_double(0x7ff0000000000000ll);
          while (true) {
            int64_t t = kmax - j;  // iterations from j whose start clock is below a
            if (j == 0 && check) {
              if (!(clock < a)) {
                t = 0;
              } else if (Rc > 0) {
                const int64_t ab = __double_as_longlong(a);
                if ((ab >> 52) == ec) {  // a in the clock's binade: a = M * ulp
                  const int64_t gap = ((ab & (fastsum::kHidden - 1)) | fastsum::kHidden) - mc;
                  const int64_t ta = fastsum::floor_div(gap - 1, Rc) + 1;
                  t = ta < t ? ta : t;
                }  // else a lies above the binade: every step starts below it
              }
            }
            j += t;
            if (j < kmax && !(rej_h || used + j * int64_t(B) + hd_ctx <= cap_tok)) continue;
            break;
          }
          const double r = R > 0 ? fastsum::compose(m + j * R, int64_t(abits >> 52)) : acc;
          clock = __shfl_sync(kFull, r, 0);
          energy = __shfl_sync(kFull, r, 1);
          flops = __shfl_sync(kFull, r, 2);
          bytes = __shfl_sync(kFull, r, 3);
          stop = j < kmax;
          cf = true;
        }
      }
      if (!cf) {
        // serial stepping (short runs, and runs the closed form cannot take:
        // a binade crossing, a tie from an odd mantissa)
        double a_h = check ? hd_arr : __longlong_as_double(0x7ff0000000000000ll);
        // 32-bit counters: a run is bounded by one request's remaining decode steps
        const int km = int(kmax);
        int jj = 0;
        while (true) {
          if (km - jj >= PSG_PIPE_MIN) {
            // software-pipelined by one group of 4: the arrival test of a group
            // reads start clocks computed in the previous one, so the branch is
            // off the clock's DADD dependency chain
            double n1 = __dadd_rn(clock, d), n2 = __dadd_rn(n1, d), n3 = __dadd_rn(n2, d);
            double n4 = __dadd_rn(n3, d);
            while (jj + 8 <= km) {
              if (!(n3 < a_h)) break;  // start clocks never decrease (d >= 0 or NaN)
              const double m1 = __dadd_rn(n4, d), m2 = __dadd_rn(m1, d), m3 = __dadd_rn(m2, d);
              const double m4 = __dadd_rn(m3, d);
              clock = n4;
              energy = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(energy, e), e), e), e);
              flops = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(flops, f), f), f), f);
              bytes = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(bytes, b), b), b), b);
              jj += 4;
              n1 = m1;
              n2 = m2;
              n3 = m3;
              n4 = m4;
            }
          }
          while (jj + 4 <= km) {
            const double c1 = __dadd_rn(clock, d);
            const double c2 = __dadd_rn(c1, d);
            const double c3 = __dadd_rn(c2, d);
            if (!(c3 < a_h)) break;
            clock = __dadd_rn(c3, d);
            energy = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(energy, e), e), e), e);
            flops = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(flops, f), f), f), f);
            bytes = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(bytes, b), b), b), b);
            jj += 4;
          }
          while (jj < km && clock < a_h) {
            clock = __dadd_rn(clock, d);
            energy = __dadd_rn(energy, e);
            flops = __dadd_rn(flops, f);
            bytes = __dadd_rn(bytes, b);
            ++jj;
          }
          // the head arrived at iteration j; one that cannot join lets the run go on
          if (jj < km && !(rej_h || used + int64_t(jj) * B + hd_ctx <= cap_tok)) {
            a_h = __longlong_as_double(0x7ff0000000000000ll);
            continue;
          }
          break;
        }
        j = jj;
        stop = j < kmax;
      }
      PROF_ADD(6, t_d3);
      n += j;
      if (logging && j > 0) {
        if (lane == 0 && nlog < U.log_cap)
          rlog[nlog] = make_double2(__longlong_as_double(int64_t(B) | INT64_MIN),
                                    __longlong_as_double(j));
        ++nlog;
      }
      used += j * int64_t(B);
      sum_batch += j * int64_t(B);
      if (j > 0) max_batch = max_batch > B ? max_batch : int64_t(B);
      settle = !stop;
    }
    if (!settle) continue;

    // ---- finish removal (batching.cpp:95-102) + metrics
    // (simulator.cpp:143-156) at iteration n; finished slots become
    // tombstones ----
    PROF_T0(t_fin);
#ifdef PSG_PHASE_PROFILE
    const bool regm_fin = regm || next_fin != n;
#endif
    if (next_fin == n) {  // finishes at this iteration
      if (regm) {
        PROF_CNT(13);
        const bool fnow = lane < len && r_fin == n;
        unsigned tok = 0;
        if (fnow) {
          const double anchor = p.anchor == PSG_ANCHOR_ARRIVAL ? r_arr : r_adm;
          const size_t s = slot_base + r_slot;
          p.slot_e2e[s] = __dsub_rn(clock, r_arr);
          p.slot_ttft[s] = __dsub_rn(r_ft, anchor);
          p.slot_tpot[s] = __dsub_rn(clock, r_ft);  // / (gen - 1) in entry_reduce_kernel
          p.slot_status[s] = 1;
          r_fin = kDead;
          tok = unsigned(r_ctx + (r_gen > 1 ? r_gen : 1));  // the ledger holds ctx + max(gen, 1)
        }
        const int64_t freed = int64_t(__reduce_add_sync(kFull, tok));
        const int nfin = __popc(__ballot_sync(kFull, fnow));
        const unsigned m = __reduce_min_sync(kFull, lane < len ? min_rel(r_fin, n) : kNoRel);
        B -= nfin;
        completed += nfin;
        used -= freed;
        next_fin = abs_of(m);
        reg_trim();
      } else if (shm) {
        // short slot-array mode: this lane's finishing positions as a bit
        // set (positions >= len mirror kDead, which never equals n)
        PROF_CNT(13);
        unsigned fb = 0, lm = kNoRel;
#pragma unroll
        for (int h = 0; h < kSC; ++h) {
          const bool f = sf[h] == n;
          fb |= unsigned(f) << h;
          lm = min(lm, f ? kNoRel : min_rel(sf[h], n));
          sf[h] = f ? kDead : sf[h];
        }
        unsigned tok = 0, nf = 0;  // <= kSC slots of < 2^27 tokens per lane (< 2^32)
        while (__any_sync(kFull, fb != 0)) {  // usually one pass: one finish per lane
          if (fb) {
            const int i = (__ffs(fb) - 1) * kWarp + lane;
            fb &= fb - 1;
            const int32_t gen = a.gen[i];
            const double arr = a.arr[i], ft = a.ft[i];
            const double anchor = p.anchor == PSG_ANCHOR_ARRIVAL ? arr : a.adm[i];
            const size_t s = slot_base + a.slot[i];
            p.slot_e2e[s] = __dsub_rn(clock, arr);
            p.slot_ttft[s] = __dsub_rn(ft, anchor);
            p.slot_tpot[s] = __dsub_rn(clock, ft);  // / (gen - 1) in entry_reduce_kernel
            p.slot_status[s] = 1;
            a.fin[i] = kDead;
            tok += unsigned(a.ctx[i] + (gen > 1 ? gen : 1));  // the ledger holds ctx + max(gen, 1)
            ++nf;
          }
        }
        const int64_t freed = warp_sum_wide(tok);
        const int nfin = int(__reduce_add_sync(kFull, nf));
        B -= nfin;
        completed += nfin;
        used -= freed;
        next_fin = abs_of(__reduce_min_sync(kFull, lm));
        int nl = 0;  // trim: 1 + the newest live position
#pragma unroll
        for (int h = kSC - 1; h >= 0; --h) {
          const unsigned lv = __ballot_sync(kFull, sf[h] != kDead);
          if (nl == 0 && lv) nl = h * kWarp + kWarp - __clz(lv);
        }
        len = nl;
        first_pre = first_pre < len ? first_pre : len;
        const bool small = kReg && B <= PSG_FILL_B;  // small again: back to lane-resident slots
        if (small && len > B) compact();
        if (small) fill();
      } else {
        PROF_CNT(13);
        int64_t freed = 0;
        unsigned m = kNoRel, nfin = 0;
        const int nch = (len + kWarp - 1) / kWarp;
        // finishes of chunk ch (metrics, tombstones); returns its new min rel fin
        auto finish_chunk = [&](int ch) -> unsigned {
          const int i = ch * kWarp + lane;
          const int64_t fin = i < len ? a.fin[i] : kDead;
          const bool fnow = fin == n;
          unsigned tok = 0;
          if (fnow) {
            const int32_t gen = a.gen[i];
            const double arr = a.arr[i], ft = a.ft[i];
            const double anchor = p.anchor == PSG_ANCHOR_ARRIVAL ? arr : a.adm[i];
            const size_t s = slot_base + a.slot[i];
            p.slot_e2e[s] = __dsub_rn(clock, arr);
            p.slot_ttft[s] = __dsub_rn(ft, anchor);
            p.slot_tpot[s] = __dsub_rn(clock, ft);  // / (gen - 1) in entry_reduce_kernel
            p.slot_status[s] = 1;
            a.fin[i] = kDead;
            tok = unsigned(a.ctx[i] + (gen > 1 ? gen : 1));  // the ledger holds ctx + max(gen, 1)
          }
          freed += int64_t(__reduce_add_sync(kFull, tok));
          nfin += __popc(__ballot_sync(kFull, fnow));
          return __reduce_min_sync(kFull, fnow ? kNoRel : min_rel(fin, n));
        };
        if (!kReg && nch == 1) {  // one chunk (small batches): no summary walk
          m = finish_chunk(0);
          if (lane == 0) cm1[0] = cm2[0] = abs_of(m);
        }
        const int ng = !kReg && nch == 1 ? 0 : (nch + kWarp - 1) / kWarp;
        for (int gb = 0; gb < ng; gb += kWarp) {
          const int g = gb + lane;
          const int64_t v2 = g < ng ? cm2[g] : kNoFin;
          unsigned gm = __ballot_sync(kFull, v2 == n);
          m = min(m, __reduce_min_sync(kFull, v2 == n ? kNoRel : rel_of(v2)));
          while (gm) {
            const int grp = gb + __ffs(gm) - 1;
            gm &= gm - 1;
            const int c = grp * kWarp + lane;
            int64_t v1 = c < nch ? cm1[c] : kNoFin;
            unsigned cmask = __ballot_sync(kFull, v1 == n);
            while (cmask) {
              const int cl = __ffs(cmask) - 1;
              cmask &= cmask - 1;
              const unsigned cr = finish_chunk(grp * kWarp + cl);
              if (lane == cl) v1 = abs_of(cr);
              if (lane == 0) cm1[grp * kWarp + cl] = abs_of(cr);
            }
            const unsigned gr = __reduce_min_sync(kFull, rel_of(v1));
            if (lane == 0) cm2[grp] = abs_of(gr);
            m = min(m, gr);
          }
        }
        __syncwarp();
        B -= int(nfin);
        completed += nfin;
        used -= freed;
        next_fin = abs_of(m);
        trim();
        const bool small = kReg && B <= PSG_FILL_B;  // small again: back to lane-resident slots
        if (len > 2 * B + 2 * kWarp || (small && len > B)) compact();
        if (small) {
          fill();
        } else if (len <= kShortCap && cap_now == p.smem_cap) {  // into the short mode
          sf_load();
          shm = true;
        }
      }
    }
    PROF_ADD(7, t_fin);
#ifdef PSG_PHASE_PROFILE
    if (!regm_fin) {
      prof_acc[26] += (unsigned long long)(clock64() - t_fin);
      prof_acc[27] += 1ull;
    }
#endif
    // ---- LIFO eviction on overflow (batching.cpp:110-125) ----
    PROF_T0(t_evi);
    if (used > cap_tok) {  // KV overflow (rare): the block below
      bool evicted = false;
      while (regm && B > 1 && used > cap_tok) {
        const int i = len - 1;  // newest live request (trim invariant)
        const int64_t fin = __shfl_sync(kFull, r_fin, i);
        const int32_t gen = __shfl_sync(kFull, r_gen, i), ctx = __shfl_sync(kFull, r_ctx, i);
        const int32_t tidx = __shfl_sync(kFull, r_tidx, i);
        const int64_t tok = fin == kNoFin ? 0 : int64_t(gen) - (fin - n);
        used -= int64_t(ctx) + tok;
        if (fin == kNoFin) --n_pre;
        if (lane == 0) g_stack[stack_top] = tidx;  // push_front of pending
        if (lane == i) r_fin = kDead;
        ++stack_top;
        --B;
        evicted = true;
        reg_trim();
      }
      while (!regm && B > 1 && used > cap_tok) {
        const int i = len - 1;  // newest live request (trim invariant)
        const int64_t fin = a.fin[i];
        const int64_t tok = fin == kNoFin ? 0 : int64_t(a.gen[i]) - (fin - n);
        used -= int64_t(a.ctx[i]) + tok;
        if (fin == kNoFin) --n_pre;
        if (lane == 0) {
          g_stack[stack_top] = a.tidx[i];  // push_front of pending
          a.fin[i] = kDead;
        }
        if (shm) sf_set(i, kDead);
        ++stack_top;
        --B;
        evicted = true;
        trim();
        if (!shm && fin != kNoFin) {  // a decode slot left the summary
          fix_chunk(i / kWarp);
          fix_group(i / (kWarp * kWarp));
        }
      }
      if (B == 1 && used > cap_tok) {  // a lone outgrowing request is rejected
        reject_slot(regm ? __shfl_sync(kFull, r_slot, len - 1) : a.slot[len - 1]);
        B = len = first_pre = n_pre = 0;
        used = 0;
        next_fin = kNoFin;
        regm = kReg;  // empty: lane-resident
        shm = !kReg && kShortCap > 0;
#pragma unroll
        for (int h = 0; h < kSC; ++h) sf[h] = kDead;
      }
      __syncwarp();
      if (evicted) {  // the evicted requests wait at the queue head (batching.cpp:114-118)
        if (kReg) head_dirty = true; else load_head();
        if (regm)
          next_fin = abs_of(__reduce_min_sync(kFull, lane < len ? min_rel(r_fin, n) : kNoRel));
        else
          recompute_next_fin();
      }
    }
    PROF_ADD(8, t_evi);
  }

  // ---- unit outputs ----
  __syncwarp();
  tally_flops = flops;
  tally_bytes = bytes;
#ifdef PSG_PHASE_PROFILE
  prof_acc[15] = (unsigned long long)(clock64() - prof_start);
  if (lane == 0 && p.prof)
    for (int k = 0; k < kProfSlots; ++k) p.prof[size_t(unit_idx) * kProfSlots + k] = prof_acc[k];
#endif
  if (lane == 0) {
    UnitOut o;
    o.clock = clock;
    o.energy = energy;
    o.flops = flops;
    o.bytes = bytes;
    o.iterations = n;
    o.max_batch = max_batch;
    o.completed = completed;
    o.rejected = rejected;
    o.sum_batch = sum_batch;
    o.admissions = admissions;
    o.err = logging && nlog > U.log_cap ? 9 : err;
    o.nlog = nlog;
    p.uout[unit_idx] = o;
  }
  // clamp flags from the extreme queried token counts / totals: every
  // query's x is monotone in its token count (cost.cpp:85-102 locate)
  if (run_hi >= 0) {
    tok_lo = min(tok_lo, run_lo);
    tok_hi = max(tok_hi, run_hi);
    tot_lo = min(tot_lo, int64_t(run_lo));
    tot_hi = max(tot_hi, int64_t(run_hi));
  }
  if (tok_hi >= 0 && lane < C) {
    const int g = c0 + lane;
    const int t = p.cell_tab[size_t(U.fslot) * p.n_cells_total + g];
    if (t >= 0) {
      const int nc = p.S.c_n_ctx[t], nt = p.S.c_n_tasks[t], nw = p.S.c_n_width[t];
      const double* kn = p.S.c_knots + p.S.c_knot_begin[t];
      const double scale = p.P.cell_scale[g];
      const double xlo = __dmul_rn(double(tok_lo), scale), xhi = __dmul_rn(double(tok_hi), scale);
      const AxisPos pj = locate(kn + nc, nt, p.P.cell_tasks[g]);
      const AxisPos pk = locate(kn + nc + nt, nw, p.P.cell_width[g]);
      const uint32_t bits = uint32_t(xlo < kn[0]) | uint32_t(xhi > kn[nc - 1]) << 1 |
                            uint32_t(pj.clamp < 0) << 2 | uint32_t(pj.clamp > 0) << 3 |
                            uint32_t(pk.clamp < 0) << 4 | uint32_t(pk.clamp > 0) << 5;
      if (bits) atomicOr(p.clamp_compute + t, bits);
    }
  }
  for (int q = lane; tot_hi >= 0 && q < NQ; q += kWarp) {
    const CurveDesc& d = cdesc[q];
    if (d.table >= 0) {
      const double xlo = __dmul_rn(__dmul_rn(d.ppt, double(tot_lo)), d.share);
      const double xhi = __dmul_rn(__dmul_rn(d.ppt, double(tot_hi)), d.share);
      const double* kn = tab + d.kn_off;
      const uint32_t bits = uint32_t(xlo < kn[0]) | uint32_t(xhi > kn[d.n - 1]) << 1;
      if (bits) atomicOr(p.clamp_curve + d.table, bits);
    }
  }
}

// The speculation warp: prices posted jobs until the simulation warp quits.
__device__ __noinline__ void spec_helper(const unsigned sleep_ns) {
  const int lane = threadIdx.x - kWarp;
  unsigned last = 0;
  while (true) {
    unsigned long long job;
    while (true) {
      job = __shfl_sync(kFull, vload64(s_spec.job), 0);
      if (unsigned(job >> 44) != last) break;
      if (__shfl_sync(kFull, vload(s_spec.quit), 0)) return;
      __nanosleep(sleep_ns);
    }
    const unsigned sq = unsigned(job >> 44);
    const int tok = int((job >> kSpecField) & ((1ull << kSpecField) - 1));
    const int64_t dec = int64_t(job & ((1ull << kSpecField) - 1));
    if (lane == 0) vstore(s_spec.started, int(sq));
    __threadfence_block();
    const EvalCtx E = s_spec.ctx;
    const EvalOut o = eval_iteration(
        E, lane, [&](int) { return tok; }, 1, dec, dec + tok, s_cellq, s_cdesc, E.tab, E.bslot,
        s_qv2, s_p2p_val2);
    if (lane == 0) {
      s_spec.cd = o.cd;
      s_spec.ce = o.ce;
      s_spec.cf = o.cf;
      s_spec.cb = o.cb;
      __threadfence_block();
      vstore(s_spec.done, int(sq));
    }
    __syncwarp();
    last = sq;
  }
}

// The entry's WorkTally (simulator.cpp:195-201) from concurrently simulated
// replica groups (chain_replicas == 2): group 0's chained tally, then every
// later replica's logged increments in replica order, in the reference's
// addition order — lane 0 carries flops, lane 1 bytes.  A decode run of j
// identical additions takes the exact closed form (psg_fastsum.cuh add_n).
// Runs on the warp of the entry's last group to finish.
// (Plain pointer arguments: a reference to the kernel's parameter struct
// would force a local-memory copy of it.)
__device__ __noinline__ void replay_tally(const int32_t* entry_units, const int kb, const int R,
                                          const Unit* units, UnitOut* uout, const double2* rlog,
                                          const double* dt) {
  const int lane = threadIdx.x & (kWarp - 1);
  int r1 = 1;  // the first logging replica (group 1)
  while (r1 < R && units[entry_units[kb + r1]].log_off < 0) ++r1;
  const UnitOut& o0 = uout[entry_units[kb + r1 - 1]];  // group 0's chained tally
  double acc = lane == 1 ? __ldcg(&o0.bytes) : __ldcg(&o0.flops);
  int err = 0;
  for (int r = r1; r < R && !err; ++r) {
    const int u = entry_units[kb + r];
    const int n = __ldcg(&uout[u].nlog);
    if (n > units[u].log_cap) {
      err = 9;
      break;
    }
    const double2* rec = rlog + units[u].log_off;
    for (int base = 0; base < n; base += kWarp) {
      // a warp of records at a time: lane i loads record base + i (and a
      // run's increments), then the chains walk them in order
      const int i = base + lane;
      double f = 0.0, b = 0.0;
      long long cnt = 1;
      if (i < n) {
        const double2 rc = __ldcg(rec + i);
        const long long xb = __double_as_longlong(rc.x);
        if (xb < 0) {  // decode run: {B tag, j}
          const long long B = xb & 0x7fffffffffffffffll;
          const double2 fb = __ldg(reinterpret_cast<const double2*>(dt + (B - 1) * 4) + 1);
          f = fb.x;
          b = fb.y;
          cnt = __double_as_longlong(rc.y);
        } else {
          f = rc.x;
          b = rc.y;
        }
      }
      const int m = min(kWarp, n - base);
      for (int q = 0; q < m; ++q) {
        const double fi = __shfl_sync(kFull, f, q), bi = __shfl_sync(kFull, b, q);
        const long long cq = __shfl_sync(kFull, cnt, q);
        const double inc = lane == 1 ? bi : fi;
        if (cq <= 8) {
          for (long long t = 0; t < cq; ++t) acc = __dadd_rn(acc, inc);
        } else {
          acc = fastsum::add_n(acc, inc, cq);
        }
      }
    }
  }
  UnitOut& ol = uout[entry_units[kb + R - 1]];  // the reduction reads the last replica's tally
  if (lane == 0) {
    ol.flops = acc;
    if (err) ol.err = err;
  }
  if (lane == 1) ol.bytes = acc;
}

// Streamed results (SimParams::out_pr): entry e's per-request metrics in id
// order (simulator.cpp:205-206; TPOT's division, :150-152) and its rejected
// ids (:207), written by the warp that completes the entry into the caller's
// pinned arrays at the offsets the host fixed.  One pass, four slot groups
// per step so the loads overlap; writes stay inside the entry's own ranges,
// and *ok is set only if the entry completed exactly as many requests as
// the host derived (else the host compacts after the kernels).  Plain
// pointer arguments (no parameter-struct copy).
__device__ __noinline__ void stream_entry_results(const uint8_t* st, const double* ttft,
                                                  const double* tpot_raw, const double* e2e,
                                                  const int64_t* sid, const int64_t* sgen,
                                                  const int64_t n, psg_request_metrics* pr,
                                                  int64_t* rj, const int64_t expect, int32_t* ok) {
  const int lane = threadIdx.x & (kWarp - 1);
  const unsigned lt = (1u << lane) - 1u;
  constexpr int kU = 4;
  int64_t wc = 0, wr = 0;
  for (int64_t b = 0; b < n; b += kU * kWarp) {
    uint8_t v[kU];
    double t[kU], q[kU], l[kU];
    int64_t id[kU], g[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // issue every load of the step first
      const int64_t i = b + u * kWarp + lane;
      v[u] = i < n ? __ldcg(st + i) : 0;
      const bool c = v[u] == 1;
      t[u] = c ? __ldcg(ttft + i) : 0.0;
      q[u] = c ? __ldcg(tpot_raw + i) : 0.0;
      l[u] = c ? __ldcg(e2e + i) : 0.0;
      id[u] = v[u] ? sid[i] : 0;
      g[u] = c ? sgen[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned cm = __ballot_sync(kFull, v[u] == 1), rm = __ballot_sync(kFull, v[u] == 2);
      const int64_t pc = wc + __popc(cm & lt), pj = wr + __popc(rm & lt);
      if (v[u] == 1 && pc < expect) {
        psg_request_metrics m;
        m.id = id[u];
        m.ttft = t[u];
        m.tpot = g[u] >= 2 ? __ddiv_rn(q[u], double(g[u] - 1)) : 0.0;
        m.e2e = l[u];
        m.gen_len = g[u];
        pr[pc] = m;
      }
      if (v[u] == 2 && pj < n - expect) rj[pj] = id[u];
      wc += __popc(cm);
      wr += __popc(rm);
    }
  }
  __syncwarp();
  if (lane == 0 && wc == expect) *ok = 1;
}

// One warp per entry (or unit); with kSpec a second warp per block speculates.
template <bool kSpec, bool kEmit, int kMode, bool kLane = false>
__device__ __forceinline__ void sim_block(const SimParams& p, unsigned char* smem_raw) {
  double tf = 0.0, tb = 0.0;
  // chained (1): one warp per entry runs its replicas in order with one
  // running tally (the reference's WorkTally, so MFU / MBU are bit-exact for
  // DP > 1); concurrent (2): one warp per unit, the tally replayed below;
  // 0: one warp per unit.  One call site keeps one copy of the loop's code.
  const int chain = kEmit ? (p.chain_replicas ? 1 : 0) : p.chain_replicas;
  const int e = blockIdx.x;
  const int k0 = chain == 1 ? p.entry_unit_begin[e] : chain == 2 ? p.block_k0[e] : e;
  const int k1 = chain == 1 ? p.entry_unit_begin[e + 1] : chain == 2 ? p.block_k1[e] : e + 1;
  for (int k = k0; k < k1; ++k) {
    sim_unit<kSpec, kEmit, kMode, kLane>(p, chain == 0 ? k : p.entry_units[k], tf, tb, smem_raw);
    __syncwarp();
  }
  const int ent = chain == 2 ? p.units[p.entry_units[k0]].entry : e;
  bool last = chain != 0;  // this block completes the entry
  if (chain == 2 && p.entry_groups[ent] > 1) {
    __threadfence();  // this group's outputs and logs before the count
    __syncwarp();
    int l = 0;
    if ((threadIdx.x & (kWarp - 1)) == 0)
      l = atomicAdd(p.entry_done + ent, 1) == p.entry_groups[ent] - 1;
    last = __shfl_sync(kFull, l, 0) != 0;
    if (last) {
      __threadfence();
      const int kb = p.entry_unit_begin[ent];
      replay_tally(p.entry_units, kb, p.entry_unit_begin[ent + 1] - kb, p.units, p.uout, p.rlog,
                   p.dectab + p.doff[ent] * 4);
    }
  }
  if (!kEmit && last && p.out_pr) {
    const size_t base = size_t(ent) * size_t(p.n_slots);
    stream_entry_results(p.slot_status + base, p.slot_ttft + base, p.slot_tpot + base,
                         p.slot_e2e + base, p.slot_id, p.slot_gen, p.n_slots,
                         p.out_pr + p.out_pr_off[ent], p.out_rj + p.out_rj_off[ent],
                         p.out_n_pr[ent], p.out_ok + ent);
  }
}

template <int kMode>
__device__ __forceinline__ void spec_block(const SimParams& p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (threadIdx.x == 0) {
    s_spec.job = 0;
    s_spec.started = 0;
    s_spec.done = 0;
    s_spec.quit = 0;
  }
  __syncthreads();
  if (threadIdx.x >= kWarp) {  // the speculation warp
    spec_helper(unsigned(p.spec_sleep_ns));
    return;
  }
  sim_block<true, false, kMode>(p, smem_raw);
  if (threadIdx.x == 0) vstore(s_spec.quit, 1);
}

__global__ void __launch_bounds__(64, 4) sim_kernel_spec(const SimParams p) { spec_block<1>(p); }
__global__ void __launch_bounds__(64, 4) sim_kernel_spec_chunked(const SimParams p) { spec_block<2>(p); }

__global__ void __launch_bounds__(32, 8) sim_kernel(const SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sim_block<false, false, 1>(p, smem_raw);
}

// Lane-resident slots without a speculation warp: contiguous batching with
// mixed-iteration tables, where the table answers what the speculation warp
// would have priced.
__global__ void __launch_bounds__(32, 8) sim_kernel_lane(const SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sim_block<false, false, 1, true>(p, smem_raw);
}

__global__ void __launch_bounds__(32, 8) sim_kernel_chunked(const SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sim_block<false, false, 2>(p, smem_raw);
}

// The iteration-record pass (psg_config::emit_iterations): every iteration
// stepped and recorded, no speculation.
__global__ void __launch_bounds__(32, 8) sim_kernel_emit(const SimParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sim_block<false, true, 0>(p, smem_raw);
}

size_t sim_smem_bytes(int smem_cap, int memo_cap, int tab_smem, int cm2_cap) {
  return smem_layout(smem_cap, memo_cap, tab_smem, cm2_cap).total;
}

}  // namespace psg
