// psg_sim.cu — the simulation kernel: one warp per (plan, frequency,
// DP-replica) unit runs the reference's continuous-batching event loop
// (run_replica, /root/reference/proj/src/simulator.cpp:98-172, over
// BatchState, batching.cpp:11-125) and prices iterations with the profiled
// tables (iteration_time, simulator.cpp:17-87).
//
// B200 design:
//  * Scalar state is warp-uniform (every lane holds the same clock/energy),
//    so there is no broadcast; batch scans (finish compaction, prefill
//    advance, min-finish) are lane-parallel over the active list with
//    ballot/popc prefix compaction that keeps admission order.
//  * The active list lives in shared memory (SoA, conflict-free lane access)
//    and migrates to a per-unit global region if the batch outgrows it.
//  * Exact event-driven macro-stepping: a decode-only iteration's workload is
//    {decode_count = B}, so its (seconds, joules, flops, bytes) are bit-
//    identical until the batch changes.  Between events (arrival of an
//    admissible/rejectable head, first finish, first KV overflow) the unit
//    runs a tight loop of the reference's sequential FP64 adds only.
//  * Costs: per-query locate/interpolate is lane-parallel; accumulation is
//    serial in the reference's order (cells → items in admission order →
//    decode, then collectives, then per-stage p2p), never a tree reduction.
//  * A shared-memory memo caches decode-only costs per batch size.
#include <climits>

#include "psg_device.cuh"

namespace psg {

namespace {

constexpr int64_t kNoFin = INT64_MAX;

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;  // std::max(a, b)
}

// Active list: SoA over generic pointers (shared memory, or global after
// migration).
struct ActiveList {
  int32_t *tidx, *ctx, *gen, *done, *items;
  int64_t* fin;  // iteration index of the finishing decode step; kNoFin while prefilling
  double *adm, *ft;
};

struct PlanConst {
  double kv, cap, reps, sdd, Sd, p2p_ppt, hidden, head_dim, kv_elems;
  int S, C, K, NB, c0, k0, b0;
};

// Lane-parallel query evaluation + reference-ordered serial accumulation.
// Returns the iteration's duration (max over stages), energy (sum over
// stages, in stage order) and the tally increments.
__device__ void eval_iteration(const SimParams& p, const PlanConst& pc,
                               const CellConst* __restrict__ cc,
                               const int32_t* items, int n_items, int64_t decode,
                               int64_t total, double* qv, uint32_t* clampbits,
                               double& dur, double& energy, double& dflops,
                               double& dbytes) {
  const int lane = threadIdx.x;
  const int nq_c = n_items + (decode > 0 ? 1 : 0);
  const int Qc = pc.C * nq_c;
  const int Q = Qc + pc.K + pc.NB;
  const double total_d = double(total);

  double bs = 0.0, bj = 0.0, bf = 0.0, bb = 0.0;
  double srep = 0.0, jrep = 0.0, d = 0.0, e = 0.0;
  bool staged = false;

  for (int base = 0; base < Q; base += kWarp) {
    const int q = base + lane;
    if (q < Q) {
      double t, en, fl = 0.0, by = 0.0;
      if (q < Qc) {
        const int c = q / nq_c;
        const int i = q - c * nq_c;
        const int64_t tok = i < n_items ? int64_t(items[i]) : decode;
        const CellConst& cell = cc[c];
        const double x = __dmul_rn(double(tok), cell.scale);
        const AxisPos pi =
            locate(p.S.c_knots + cell.knot_begin, cell.n_ctx, x);
        sample_grid(p.S, cell, pi, t, en);
        en = __dmul_rn(en, pc.sdd);  // query_energy * stage_devices
        fl = op_flops(cell.op, x, cell.tasks, cell.width, pc.hidden, pc.head_dim);
        by = op_bytes(cell.op, x, cell.tasks, cell.width, pc.hidden, pc.kv_elems);
        const uint32_t bits = (pi.clamp < 0 ? 1u : 0u) | (pi.clamp > 0 ? 2u : 0u) |
                              uint32_t(cell.pj.clamp < 0) << 2 |
                              uint32_t(cell.pj.clamp > 0) << 3 |
                              uint32_t(cell.pk.clamp < 0) << 4 |
                              uint32_t(cell.pk.clamp > 0) << 5;
        if (bits) atomicOr(&clampbits[c], bits);
      } else if (q < Qc + pc.K) {
        const int k = q - Qc;
        const int g = pc.k0 + k;
        const double payload =
            __dmul_rn(__dmul_rn(__ldg(p.P.coll_ppt + g), total_d), __ldg(p.P.coll_share + g));
        int clamp;
        sample_curve(p.S, __ldg(p.coll_tab + g), payload, t, en, clamp);
        en = __dmul_rn(en, double(__ldg(p.P.coll_groups + g)));
        if (clamp) atomicOr(&clampbits[pc.C + k], clamp < 0 ? 1u : 2u);
      } else {
        const int b = q - Qc - pc.K;
        const double payload = __dmul_rn(pc.p2p_ppt, total_d);
        int clamp;
        sample_curve(p.S, __ldg(p.p2p_tab + pc.b0 + b), payload, t, en, clamp);
        if (clamp) atomicOr(&clampbits[pc.C + pc.K + b], clamp < 0 ? 1u : 2u);
      }
      qv[lane] = t;
      qv[kWarp + lane] = en;
      qv[2 * kWarp + lane] = fl;
      qv[3 * kWarp + lane] = by;
    }
    __syncwarp();
    const int here = min(kWarp, Q - base);
    for (int l = 0; l < here; ++l) {
      const int q2 = base + l;
      const double t = qv[l], en = qv[kWarp + l];
      if (q2 < Qc) {
        bs = __dadd_rn(bs, t);
        bj = __dadd_rn(bj, en);
        bf = __dadd_rn(bf, qv[2 * kWarp + l]);
        bb = __dadd_rn(bb, qv[3 * kWarp + l]);
      } else if (q2 < Qc + pc.K) {
        bs = __dadd_rn(bs, t);
        bj = __dadd_rn(bj, en);
      } else {
        if (!staged) {
          srep = __dmul_rn(bs, pc.reps);
          jrep = __dmul_rn(bj, pc.reps);
          d = dmax_ref(0.0, srep);
          e = __dadd_rn(0.0, jrep);
          staged = true;
        }
        d = dmax_ref(d, __dadd_rn(srep, t));
        e = __dadd_rn(e, __dadd_rn(jrep, en));
      }
    }
    __syncwarp();
  }
  if (!staged) {
    srep = __dmul_rn(bs, pc.reps);
    jrep = __dmul_rn(bj, pc.reps);
    d = dmax_ref(0.0, srep);
    e = __dadd_rn(0.0, jrep);
  }
  dur = d;
  energy = e;
  dflops = __dmul_rn(__dmul_rn(__dmul_rn(bf, pc.sdd), pc.reps), pc.Sd);
  dbytes = __dmul_rn(__dmul_rn(__dmul_rn(bb, pc.sdd), pc.reps), pc.Sd);
}

}  // namespace

__global__ void __launch_bounds__(32, 8) sim_kernel(const SimParams p) {
  const int lane = threadIdx.x;
  const unsigned lt_mask = (1u << lane) - 1u;
  const Unit U = p.units[blockIdx.x];

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* qv = reinterpret_cast<double*>(smem_raw);                  // 4 x 32
  CellConst* cc = reinterpret_cast<CellConst*>(qv + 4 * kWarp);       // kMaxCells
  uint32_t* clampbits = reinterpret_cast<uint32_t*>(cc + kMaxCells);  // kMaxClampSlots
  double* memo = reinterpret_cast<double*>(clampbits + kMaxClampSlots);  // memo_cap x 4
  double* s_adm = memo + 4 * p.memo_cap;
  double* s_ft = s_adm + p.smem_cap;
  int64_t* s_fin = reinterpret_cast<int64_t*>(s_ft + p.smem_cap);
  int32_t* s_i32 = reinterpret_cast<int32_t*>(s_fin + p.smem_cap);   // 5 x smem_cap

  // ---- plan constants (warp-uniform) ----
  const int pl = U.plan;
  PlanConst pc;
  pc.kv = p.P.kv[pl];
  pc.cap = p.P.budget[pl];
  pc.S = p.P.num_stages[pl];
  pc.reps = double(p.P.stage_reps[pl]);
  pc.sdd = double(p.P.stage_devices[pl]);
  pc.Sd = double(pc.S);
  pc.p2p_ppt = p.P.p2p_ppt[pl];
  pc.hidden = p.P.sh_hidden[pl];
  pc.head_dim = p.P.sh_head[pl];
  pc.kv_elems = p.P.sh_kv[pl];
  pc.c0 = p.P.cell_begin[pl];
  pc.C = p.P.cell_begin[pl + 1] - pc.c0;
  pc.k0 = p.P.coll_begin[pl];
  pc.K = p.P.coll_begin[pl + 1] - pc.k0;
  pc.b0 = p.P.p2p_begin[pl];
  pc.NB = p.P.p2p_begin[pl + 1] - pc.b0;

  for (int s = lane; s < kMaxClampSlots; s += kWarp) clampbits[s] = 0;
  for (int i = lane; i < 4 * p.memo_cap; i += kWarp) memo[i] = -1.0;
  if (lane < pc.C) {
    CellConst c;
    const int g = pc.c0 + lane;
    c.table = p.cell_tab[size_t(U.fslot) * p.n_cells_total + g];
    c.op = p.P.cell_op[g];
    c.tasks = p.P.cell_tasks[g];
    c.width = p.P.cell_width[g];
    c.scale = p.P.cell_scale[g];
    if (c.table >= 0) {
      c.n_ctx = p.S.c_n_ctx[c.table];
      c.n_tasks = p.S.c_n_tasks[c.table];
      c.n_width = p.S.c_n_width[c.table];
      c.knot_begin = p.S.c_knot_begin[c.table];
      c.value_begin = p.S.c_value_begin[c.table];
      c.pj = locate(p.S.c_knots + c.knot_begin + c.n_ctx, c.n_tasks, c.tasks);
      c.pk = locate(p.S.c_knots + c.knot_begin + c.n_ctx + c.n_tasks, c.n_width, c.width);
    } else {
      c.n_ctx = c.n_tasks = c.n_width = 1;
      c.knot_begin = c.value_begin = 0;
      c.pj = c.pk = AxisPos{0, 0, 0.0, 0};
    }
    cc[lane] = c;
  }
  __syncwarp();

  // ---- active list storage ----
  int cap_now = p.smem_cap;
  ActiveList a;
  a.adm = s_adm;
  a.ft = s_ft;
  a.fin = s_fin;
  a.tidx = s_i32;
  a.ctx = s_i32 + p.smem_cap;
  a.gen = s_i32 + 2 * p.smem_cap;
  a.done = s_i32 + 3 * p.smem_cap;
  a.items = s_i32 + 4 * p.smem_cap;
  const size_t nr = size_t(U.n_req);
  int32_t* g_stack = p.g_i32 + size_t(U.scratch) * 6;  // 6 int32 arrays of n_req
  double* g_f = p.g_f64 + size_t(U.scratch) * 3;      // adm, ft, fin(int64)

  // ---- replica request sequence (round-robin split, simulator.cpp:187-193) ----
  auto req_tidx = [&](int j) -> int {
    return p.T.seq ? p.T.seq[U.seq_base + j]
                   : int(int64_t(U.replica) + int64_t(j) * U.replicas);
  };
  const size_t slot_base = size_t(U.entry) * size_t(p.n_slots);

  const double kv = pc.kv, cap = pc.cap;
  const bool chunked = p.batch_mode == PSG_BATCH_CHUNKED;
  const int64_t chunk = p.chunk_size;
  const int64_t max_bs = p.max_batch_size;
  const bool chunk_err = chunked && chunk < 1;
  const bool missing = p.entry_missing[U.entry] != 0;

  double clock = 0.0, energy = 0.0, flops = 0.0, bytes = 0.0;
  int64_t n = 0, max_batch = 0, completed = 0, rejected = 0, sum_batch = 0, admissions = 0;
  int B = 0, n_pre = 0, pend = 0, stack_top = 0;
  int64_t used = 0;          // KV ledger in tokens: sum(ctx + generated)
  int64_t next_fin = kNoFin;
  int err = 0;

  auto fits = [&](int64_t tokens) -> bool {  // double(tokens) * kv <= cap, exact
    return !(__dmul_rn(double(tokens), kv) > cap);
  };
  auto reject_slot = [&](int tidx) {
    if (lane == 0) p.slot_status[slot_base + p.T.slot[tidx]] = 2;
    ++rejected;
  };
  auto migrate = [&]() {
    // Move the active list (and prefill-item scratch) to the unit's global
    // region; capacity becomes n_req, the largest possible batch.
    int32_t* gi = g_stack + nr;
    int64_t* gfin = reinterpret_cast<int64_t*>(g_f + 2 * nr);
    for (int i = lane; i < B; i += kWarp) {
      gi[i] = a.tidx[i];
      gi[nr + i] = a.ctx[i];
      gi[2 * nr + i] = a.gen[i];
      gi[3 * nr + i] = a.done[i];
      g_f[i] = a.adm[i];
      g_f[nr + i] = a.ft[i];
      gfin[i] = a.fin[i];
    }
    __syncwarp();
    a.tidx = gi;
    a.ctx = gi + nr;
    a.gen = gi + 2 * nr;
    a.done = gi + 3 * nr;
    a.items = gi + 4 * nr;
    a.adm = g_f;
    a.ft = g_f + nr;
    a.fin = gfin;
    cap_now = int(nr);
  };
  auto recompute_next_fin = [&]() {
    int64_t m = kNoFin;
    for (int base = 0; base < B; base += kWarp) {
      const int i = base + lane;
      const int64_t f = i < B ? a.fin[i] : kNoFin;
      m = f < m ? f : m;
    }
    next_fin = warp_min_i64(m);
  };
  // Finish removal (batching.cpp:95-102) + metrics (simulator.cpp:143-156),
  // then LIFO eviction (batching.cpp:110-125).  Runs at iteration n, after
  // the clock has advanced.
  auto finish_and_evict = [&]() {
    if (next_fin == n) {
      int w = 0;
      int64_t freed = 0, m = kNoFin, nfin = 0;
      for (int base = 0; base < B; base += kWarp) {
        const int i = base + lane;
        const bool valid = i < B;
        int32_t tidx = 0, ctx = 0, gen = 0, done = 0;
        int64_t fin = kNoFin;
        double adm = 0.0, ft = 0.0;
        if (valid) {
          tidx = a.tidx[i];
          ctx = a.ctx[i];
          gen = a.gen[i];
          done = a.done[i];
          fin = a.fin[i];
          adm = a.adm[i];
          ft = a.ft[i];
        }
        const bool fnow = valid && fin == n;
        if (fnow) {
          const double arr = p.T.arrival[tidx];
          const double anchor = p.anchor == PSG_ANCHOR_ARRIVAL ? arr : adm;
          const size_t s = slot_base + p.T.slot[tidx];
          p.slot_e2e[s] = __dsub_rn(clock, arr);
          p.slot_ttft[s] = __dsub_rn(ft, anchor);
          p.slot_tpot[s] =
              gen >= 2 ? __ddiv_rn(__dsub_rn(clock, ft), double(gen - 1)) : 0.0;
          p.slot_status[s] = 1;
        }
        const bool keep = valid && !fnow;
        const unsigned km = __ballot_sync(kFull, keep);
        const int pos = w + __popc(km & lt_mask);
        __syncwarp();
        if (keep) {
          a.tidx[pos] = tidx;
          a.ctx[pos] = ctx;
          a.gen[pos] = gen;
          a.done[pos] = done;
          a.fin[pos] = fin;
          a.adm[pos] = adm;
          a.ft[pos] = ft;
        }
        w += __popc(km);
        freed += warp_sum_i64(fnow ? int64_t(ctx) + gen : 0);
        nfin += __popc(__ballot_sync(kFull, fnow));
        const int64_t fk = keep ? fin : kNoFin;
        m = fk < m ? fk : m;
        __syncwarp();
      }
      B = w;
      used -= freed;
      completed += nfin;
      next_fin = warp_min_i64(m);
    }
    bool evicted = false;
    while (B > 1 && !fits(used)) {
      const int i = B - 1;
      const int64_t fin = a.fin[i];
      const int32_t ctx = a.ctx[i], gen = a.gen[i];
      const int64_t tok = fin == kNoFin ? 0 : int64_t(gen) - (fin - n);
      used -= int64_t(ctx) + tok;
      if (fin == kNoFin) --n_pre;
      if (lane == 0) g_stack[stack_top] = a.tidx[i];  // push_front of pending
      ++stack_top;
      --B;
      evicted = true;
    }
    if (B == 1 && !fits(used)) {
      reject_slot(a.tidx[0]);
      B = 0;
      n_pre = 0;
      used = 0;
      next_fin = kNoFin;
      evicted = false;
    }
    __syncwarp();
    if (evicted) recompute_next_fin();
  };

  while (true) {
    // ---- admit (batching.cpp:35-60) ----
    while (true) {
      int h;
      if (stack_top > 0) h = g_stack[stack_top - 1];
      else if (pend < U.n_req) h = req_tidx(pend);
      else break;
      if (!(p.T.arrival[h] <= clock)) break;
      const int64_t ctx = p.T.ctx[h];
      if (__dmul_rn(double(ctx), kv) > cap) {
        reject_slot(h);
        if (stack_top > 0) --stack_top; else ++pend;
        continue;
      }
      if (max_bs > 0 && int64_t(B) >= max_bs) break;
      if (!fits(used + ctx)) break;
      if (B >= cap_now) migrate();
      if (lane == 0) {
        a.tidx[B] = h;
        a.ctx[B] = int32_t(ctx);
        a.gen[B] = int32_t(p.T.gen[h]);
        a.done[B] = 0;
        a.fin[B] = kNoFin;
        a.adm[B] = clock;
        a.ft[B] = 0.0;
      }
      ++B;
      ++n_pre;
      ++admissions;
      used += ctx;
      if (stack_top > 0) --stack_top; else ++pend;
    }
    __syncwarp();

    if (B == 0) {  // idle (simulator.cpp:116-120)
      int h;
      if (stack_top > 0) h = g_stack[stack_top - 1];
      else if (pend < U.n_req) h = req_tidx(pend);
      else break;
      clock = dmax_ref(clock, p.T.arrival[h]);
      continue;
    }
    if (chunk_err) { err = 1; break; }
    if (missing) { err = 2; break; }

    if (n_pre > 0) {
      // ---- mixed iteration: literal step (batching.cpp:62-108) ----
      int n_items = 0;
      int64_t pre_tok = 0;
      for (int base = 0; base < B; base += kWarp) {
        const int i = base + lane;
        bool pre = false;
        int64_t tok = 0;
        if (i < B && a.fin[i] == kNoFin) {
          pre = true;
          tok = int64_t(a.ctx[i]) - a.done[i];
          if (chunked) tok = tok < chunk ? tok : chunk;
        }
        const unsigned pm = __ballot_sync(kFull, pre);
        if (pre) a.items[n_items + __popc(pm & lt_mask)] = int32_t(tok);
        n_items += __popc(pm);
        pre_tok += warp_sum_i64(tok);
      }
      __syncwarp();
      const int64_t decode = int64_t(B) - n_items;
      double d, e, f, b;
      eval_iteration(p, pc, cc, a.items, n_items, decode, decode + pre_tok, qv,
                     clampbits, d, e, f, b);
      clock = __dadd_rn(clock, d);
      energy = __dadd_rn(energy, e);
      flops = __dadd_rn(flops, f);
      bytes = __dadd_rn(bytes, b);
      max_batch = max_batch > B ? max_batch : int64_t(B);
      sum_batch += B;
      const int64_t n_new = n + 1;
      int64_t ncompl = 0, m = next_fin;
      for (int base = 0; base < B; base += kWarp) {
        const int i = base + lane;
        bool compl_now = false;
        int64_t fin = kNoFin;
        if (i < B && a.fin[i] == kNoFin) {
          const int32_t ctx = a.ctx[i];
          int64_t tok = int64_t(ctx) - a.done[i];
          if (chunked) tok = tok < chunk ? tok : chunk;
          const int64_t done = a.done[i] + tok;
          a.done[i] = int32_t(done);
          if (done == ctx) {  // prefill iteration samples the first token
            const int32_t gen = a.gen[i];
            fin = n_new + (gen > 1 ? gen - 1 : 0);
            a.fin[i] = fin;
            a.ft[i] = clock;
            compl_now = true;
          }
        }
        ncompl += __popc(__ballot_sync(kFull, compl_now));
        const int64_t wm = warp_min_i64(fin);
        m = wm < m ? wm : m;
      }
      __syncwarp();
      used += decode + ncompl;
      n_pre -= int(ncompl);
      n = n_new;
      next_fin = m;
      finish_and_evict();
      continue;
    }

    // ---- decode-only run: exact macro-stepping ----
    double d, e, f, b;
    if (B <= p.memo_cap && memo[4 * (B - 1)] >= 0.0) {
      d = memo[4 * (B - 1)];
      e = memo[4 * (B - 1) + 1];
      f = memo[4 * (B - 1) + 2];
      b = memo[4 * (B - 1) + 3];
    } else {
      eval_iteration(p, pc, cc, a.items, 0, B, B, qv, clampbits, d, e, f, b);
      if (B <= p.memo_cap) {
        __syncwarp();
        if (lane == 0) {
          memo[4 * (B - 1) + 1] = e;
          memo[4 * (B - 1) + 2] = f;
          memo[4 * (B - 1) + 3] = b;
          memo[4 * (B - 1)] = d;
        }
        __syncwarp();
      }
    }
    // k_fin: iterations until the first finish (inclusive).
    int64_t kmax = next_fin - n;
    // k_ovf: first k with (used + k*B)*kv > cap.
    if (!fits(used + kmax * int64_t(B))) {
      const double r = (cap / kv - double(used)) / double(B);
      int64_t k0 = r >= double(kmax) ? kmax - 1 : (r < 0.0 ? 0 : int64_t(floor(r)));
      while (k0 > 0 && !fits(used + k0 * int64_t(B))) --k0;
      while (k0 + 1 < kmax && fits(used + (k0 + 1) * int64_t(B))) ++k0;
      kmax = k0 + 1;
    }
    // Arrival event: only a not-yet-arrived head can change the batch; an
    // arrived head that the admit loop left in place is blocked for the
    // whole run (used only grows, B is fixed).
    bool check = false, rej_h = false;
    double a_h = 0.0;
    int64_t j_adm = -1;
    if (stack_top == 0 && pend < U.n_req) {
      const int h = req_tidx(pend);
      a_h = p.T.arrival[h];
      if (a_h > clock) {
        const int64_t ctx_h = p.T.ctx[h];
        rej_h = __dmul_rn(double(ctx_h), kv) > cap;
        if (rej_h) {
          check = true;
        } else if (!(max_bs > 0 && int64_t(B) >= max_bs) && fits(used + ctx_h)) {
          check = true;
          // largest j in [0, kmax] with used + j*B + ctx_h fitting
          if (fits(used + kmax * int64_t(B) + ctx_h)) {
            j_adm = kmax;
          } else {
            const double r = (cap / kv - double(used + ctx_h)) / double(B);
            int64_t j0 = r >= double(kmax) ? kmax - 1 : (r < 0.0 ? 0 : int64_t(floor(r)));
            while (j0 > 0 && !fits(used + j0 * int64_t(B) + ctx_h)) --j0;
            while (j0 + 1 < kmax && fits(used + (j0 + 1) * int64_t(B) + ctx_h)) ++j0;
            j_adm = j0;
          }
        }
      }
    }
    int64_t j = 0;
    bool stop = false;
    if (check) {
      while (j + 4 <= kmax) {
        const double c1 = __dadd_rn(clock, d);
        const double c2 = __dadd_rn(c1, d);
        const double c3 = __dadd_rn(c2, d);
        if (!(clock < a_h && c1 < a_h && c2 < a_h && c3 < a_h)) break;
        clock = __dadd_rn(c3, d);
        energy = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(energy, e), e), e), e);
        flops = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(flops, f), f), f), f);
        bytes = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(bytes, b), b), b), b);
        j += 4;
      }
      while (j < kmax && clock < a_h) {
        clock = __dadd_rn(clock, d);
        energy = __dadd_rn(energy, e);
        flops = __dadd_rn(flops, f);
        bytes = __dadd_rn(bytes, b);
        ++j;
      }
      if (j < kmax && (rej_h || j <= j_adm)) stop = true;
    }
    if (!stop) {
      for (; j + 4 <= kmax; j += 4) {
        clock = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(clock, d), d), d), d);
        energy = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(energy, e), e), e), e);
        flops = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(flops, f), f), f), f);
        bytes = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(bytes, b), b), b), b);
      }
      for (; j < kmax; ++j) {
        clock = __dadd_rn(clock, d);
        energy = __dadd_rn(energy, e);
        flops = __dadd_rn(flops, f);
        bytes = __dadd_rn(bytes, b);
      }
    }
    n += j;
    used += j * int64_t(B);
    sum_batch += j * int64_t(B);
    if (j > 0) max_batch = max_batch > B ? max_batch : int64_t(B);
    if (!stop) finish_and_evict();
  }

  // ---- unit outputs ----
  __syncwarp();
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
    o.err = err;
    o.pad = 0;
    p.uout[blockIdx.x] = o;
  }
  const int nslots = pc.C + pc.K + pc.NB;
  for (int s = lane; s < nslots && s < kMaxClampSlots; s += kWarp) {
    const uint32_t bits = clampbits[s];
    if (!bits) continue;
    if (s < pc.C) {
      if (cc[s].table >= 0) atomicOr(p.clamp_compute + cc[s].table, bits);
    } else if (s < pc.C + pc.K) {
      atomicOr(p.clamp_curve + p.coll_tab[pc.k0 + s - pc.C], bits);
    } else {
      atomicOr(p.clamp_curve + p.p2p_tab[pc.b0 + s - pc.C - pc.K], bits);
    }
  }
}

size_t sim_smem_bytes(int smem_cap, int memo_cap) {
  return sizeof(double) * 4 * kWarp + sizeof(CellConst) * kMaxCells +
         sizeof(uint32_t) * kMaxClampSlots + sizeof(double) * 4 * size_t(memo_cap) +
         size_t(smem_cap) * (2 * sizeof(double) + sizeof(int64_t) + 5 * sizeof(int32_t));
}

}  // namespace psg
