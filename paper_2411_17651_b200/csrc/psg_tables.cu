// psg_tables.cu — cost tables computed in parallel before the simulation.
//
// Every cell query of iteration_time (simulator.cpp:29-52) is a pure function
// of (compute grid, token_scale, tasks, width, op, op shape) — a "cell
// signature" — and of the integer token count, and a decode-only iteration's
// whole cost is a pure function of (plan, frequency) and the batch size B.
// Both are tabulated here, one thread per value (work that fills the GPU),
// so the simulation kernel's serial path only prices collectives and adds:
//
//   qtab_kernel    per signature, per token count t: {seconds, joules (raw,
//                  before * stage_devices), op_flops, op_bytes}
//                  (cost.cpp:196-260, :51-68);
//   dectab_kernel  per (plan, frequency) entry, per B: the full iteration cost
//                  {duration, energy, flops, bytes} of workload {decode = B},
//                  accumulated in the reference's order (simulator.cpp:17-87,
//                  :125-133) from qtab rows and collective curve queries;
//   mixtab_kernel  per selected entry, per distinct context length t and
//                  decode count B: the full cost of the mixed iteration
//                  {prefill_items = {t}, decode_count = B} — the iteration
//                  that admits one request under contiguous batching — in
//                  the order of iteration_time (cells: the item's query,
//                  then the decode query; collectives and p2p at t + B,
//                  read from colltab_kernel's per-total curve values).
#include "psg_device.cuh"

namespace psg {

__device__ __forceinline__ void qtab_row(const TabParams& p, const int sig, const int64_t tok) {
  double* row = p.qtab + (p.qoff[sig] + tok) * 4;
  const int table = p.sig_table[sig];
  if (table < 0) {  // missing grid: never read (the entry fails at its first step)
    row[0] = row[1] = row[2] = row[3] = 0.0;
    return;
  }
  const double x = __dmul_rn(double(tok), p.sig_scale[sig]);  // tokens * token_scale
  const double tasks = p.sig_tasks[sig], width = p.sig_width[sig];
  double sec, joule;
  uint32_t clamp;
  cell_query_ref(p.S, table, x, tasks, width, sec, joule, clamp);
  const int op = p.sig_op[sig];
  row[0] = sec;
  row[1] = joule;
  row[2] = op_flops(op, x, tasks, width, p.sig_hidden[sig], p.sig_head[sig]);
  row[3] = op_bytes(op, x, tasks, width, p.sig_hidden[sig], p.sig_kv[sig]);
}

__device__ __forceinline__ void dectab_row(const TabParams& p, const int e, const int64_t B) {
  double* out = p.dectab + (p.doff[e] + B - 1) * 4;
  if (p.entry_missing[e]) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    return;
  }
  const int pl = p.ent_plan[e], fs = p.ent_fslot[e];
  const double sdd = double(p.P.stage_devices[pl]);
  const double reps = double(p.P.stage_reps[pl]);
  const double Sd = double(p.P.num_stages[pl]);
  const double total = double(B);
  double bs = 0.0, bj = 0.0, bf = 0.0, bb = 0.0;
  for (int c = p.P.cell_begin[pl]; c < p.P.cell_begin[pl + 1]; ++c) {
    const int sig = p.cell_sig[size_t(fs) * p.n_cells_total + c];
    const double* q = p.qtab + (p.qoff[sig] + B) * 4;
    bs = __dadd_rn(bs, q[0]);
    bj = __dadd_rn(bj, __dmul_rn(q[1], sdd));  // query_energy * stage_devices
    bf = __dadd_rn(bf, q[2]);
    bb = __dadd_rn(bb, q[3]);
  }
  for (int k = p.P.coll_begin[pl]; k < p.P.coll_begin[pl + 1]; ++k) {
    const double payload = __dmul_rn(__dmul_rn(p.P.coll_ppt[k], total), p.P.coll_share[k]);
    double t, en;
    curve_query_ref(p.S, p.coll_tab[k], payload, t, en);
    bs = __dadd_rn(bs, t);
    bj = __dadd_rn(bj, __dmul_rn(en, double(p.P.coll_groups[k])));
  }
  const double srep = __dmul_rn(bs, reps), jrep = __dmul_rn(bj, reps);
  double d = srep > 0.0 ? srep : 0.0;  // std::max(0.0, stage 0)
  double E = __dadd_rn(0.0, jrep);
  const double p2p_payload = __dmul_rn(p.P.p2p_ppt[pl], total);
  for (int b = p.P.p2p_begin[pl]; b < p.P.p2p_begin[pl + 1]; ++b) {
    double t, en;
    curve_query_ref(p.S, p.p2p_tab[b], p2p_payload, t, en);
    const double s = __dadd_rn(srep, t);
    d = d < s ? s : d;
    E = __dadd_rn(E, __dadd_rn(jrep, en));
  }
  out[0] = d;
  out[1] = E;
  out[2] = __dmul_rn(__dmul_rn(__dmul_rn(bf, sdd), reps), Sd);
  out[3] = __dmul_rn(__dmul_rn(__dmul_rn(bb, sdd), reps), Sd);
}

// Load test of the tabulated entries (after dectab_kernel): a table only
// pays if the entry's batches stay below mt_w.  With decode-only iteration
// time d(B), a batch of B completes requests at B / (G * d(B)) per second
// (G: mean generation length); if no B <= 0.8 mt_w keeps up with 1.25x the
// unit's arrival rate, its queue (and batch) outgrows the table — the entry
// is dropped (moff = -1): no rows are computed and its simulation prices
// mixed iterations itself.  Only a cost decision: results do not depend on it.
__global__ void mixsel_kernel(const TabParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_mt) return;
  const int e = p.mt_ent[i];
  const int64_t bt = min(int64_t(0.8 * p.mt_w), p.ent_rows[e]);
  const double need = 1.25 * p.mt_lam[i];
  bool ok = false;
  for (int64_t B = 1; B <= bt && !ok; ++B) {
    const double d = p.dectab[(p.doff[e] + B - 1) * 4];
    ok = double(B) >= need * p.mt_gen * d;
  }
  if (!ok) p.moff_rw[e] = -1;
}

// Collective and distinct p2p curve values of a tabulated entry per
// iteration total T (cost.cpp:262-291): {seconds, joules * groups_per_stage}
// for collective q < K, {seconds, joules} for the distinct p2p curves (first
// appearance order) in slots K, K+1.  Every mixed-iteration row of the entry
// reads them at T = t + B instead of interpolating the curves itself.
__global__ void __launch_bounds__(256) colltab_kernel(const TabParams p) {
  const int i = blockIdx.x;
  const int e = p.mt_ent[i], pl = p.ent_plan[e];
  if (p.moff[e] < 0) return;  // dropped by mixsel_kernel
  const int k0 = p.P.coll_begin[pl], K = p.P.coll_begin[pl + 1] - k0;
  const int b0 = p.P.p2p_begin[pl], b1 = p.P.p2p_begin[pl + 1];
  int d0 = -1, d1 = -1;  // distinct p2p curves
  for (int b = b0; b < b1; ++b) {
    const int t = p.p2p_tab[b];
    if (d0 < 0 || t == d0) {
      d0 = t;
    } else if (d1 < 0) {
      d1 = t;
    }
  }
  const double p2p_ppt = p.P.p2p_ppt[pl];
  for (int64_t T = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; T < p.mt_T;
       T += int64_t(gridDim.y) * blockDim.x) {
    // slot-major [entry][slot][T]: the mixed-iteration rows of a block read
    // consecutive totals
    double2* out = reinterpret_cast<double2*>(p.ctab) + int64_t(i) * p.mt_nq * p.mt_T + T;
    const double total = double(T);
    for (int q = 0; q < K; ++q) {
      const int k = k0 + q;
      const double payload = __dmul_rn(__dmul_rn(p.P.coll_ppt[k], total), p.P.coll_share[k]);
      double s, en;
      curve_query_ref(p.S, p.coll_tab[k], payload, s, en);
      out[int64_t(q) * p.mt_T] = make_double2(s, __dmul_rn(en, double(p.P.coll_groups[k])));
    }
    const double payload = __dmul_rn(p2p_ppt, total);
    if (d0 >= 0) {
      double s, en;
      curve_query_ref(p.S, d0, payload, s, en);
      out[int64_t(K) * p.mt_T] = make_double2(s, en);
    }
    if (d1 >= 0) {
      double s, en;
      curve_query_ref(p.S, d1, payload, s, en);
      out[int64_t(K + 1) * p.mt_T] = make_double2(s, en);
    }
  }
}

// The mixed-iteration table: one block per (tabulated entry, context-length
// rank r), a thread per decode count B.  Each value is computed with the
// same operations, in the same order, as the simulation kernel's
// eval_iteration for n_items = 1 (iteration_time, simulator.cpp:17-87):
// cells in order, each the item's query then the decode query; then the
// collectives; then the stage fold.  The block stages the entry's constants
// once; the item's qtab rows are block-uniform, the decode rows and the
// curve values at t + B contiguous across threads, and the block's rows
// leave through shared memory as contiguous 16-byte stores.
// Constants of one tabulated entry, staged per block.
struct MixEntry {
  int C, K, NB, b0, d0, ND;
  uint64_t mask;  // boundary b (< 64) uses the second distinct p2p curve
  double sdd, reps, Sd;
  const double2* ct;  // the entry's curve values, slot-major
};

// {duration, energy}, {flops, bytes} of {prefill_items = {t}, decode = B}.
// qrow[c]: the cell's signature table; qt[c]: its row for the item (block-uniform).
__device__ __forceinline__ void mixtab_value(const TabParams& p, const MixEntry& m,
                                             const double2* const* qrow, const double2* qt,
                                             const int64_t t, const int B,
                                             double2& o0, double2& o1) {
  double bs = 0.0, bj = 0.0, bf = 0.0, bb = 0.0;
  for (int c = 0; c < m.C; ++c) {
    const double2 te = qt[2 * c], fb = qt[2 * c + 1];
    bs = __dadd_rn(bs, te.x);
    bj = __dadd_rn(bj, __dmul_rn(te.y, m.sdd));  // query_energy * stage_devices
    bf = __dadd_rn(bf, fb.x);
    bb = __dadd_rn(bb, fb.y);
    if (B > 0) {  // the decode requests' batched query (simulator.cpp:50)
      const double2* qd = qrow[c] + 2 * B;
      const double2 te2 = __ldg(qd), fb2 = __ldg(qd + 1);
      bs = __dadd_rn(bs, te2.x);
      bj = __dadd_rn(bj, __dmul_rn(te2.y, m.sdd));
      bf = __dadd_rn(bf, fb2.x);
      bb = __dadd_rn(bb, fb2.y);
    }
  }
  const int64_t T = p.mt_T;
  const double2* cv = m.ct + (t + B);
  for (int q = 0; q < m.K; ++q) {
    const double2 v = __ldg(cv + q * T);
    bs = __dadd_rn(bs, v.x);
    bj = __dadd_rn(bj, v.y);
  }
  const double srep = __dmul_rn(bs, m.reps), jrep = __dmul_rn(bj, m.reps);
  double d = srep > 0.0 ? srep : 0.0;  // std::max(0.0, stage 0)
  double E = __dadd_rn(0.0, jrep);
  if (m.NB > 0) {
    // stage b+1 adds boundary b's p2p (simulator.cpp:69-78); the duration
    // is the max over the (at most two) distinct stage values, in the
    // simulation kernel's order (eval_iteration)
    const double2 v0 = __ldg(cv + m.K * T);
    const double2 v1 = m.ND == 2 ? __ldg(cv + (m.K + 1) * T) : v0;
    const double s0 = __dadd_rn(srep, v0.x), s1 = __dadd_rn(srep, v1.x);
    d = d < s0 ? s0 : d;
    if (m.ND == 2) d = d < s1 ? s1 : d;
    const double a0 = __dadd_rn(jrep, v0.y), a1 = __dadd_rn(jrep, v1.y);
    const int nb = m.NB < 64 ? m.NB : 64;
    for (int b = 0; b < nb; ++b) E = __dadd_rn(E, ((m.mask >> b) & 1) ? a1 : a0);
    for (int b = 64; b < m.NB; ++b) E = __dadd_rn(E, p.p2p_tab[m.b0 + b] != m.d0 ? a1 : a0);
  }
  o0 = make_double2(d, E);
  o1 = make_double2(__dmul_rn(__dmul_rn(__dmul_rn(bf, m.sdd), m.reps), m.Sd),
                    __dmul_rn(__dmul_rn(__dmul_rn(bb, m.sdd), m.reps), m.Sd));
}

__global__ void __launch_bounds__(256) mixtab_kernel(const TabParams p) {
  __shared__ const double2* s_q[kMaxCells];  // each cell's signature table
  __shared__ double2 s_t[2 * kMaxCells];       // ... and its row for the item
  __shared__ double2 s_row[2 * 256];           // the block's rows {duration, energy}, {flops, bytes}
  const int i = blockIdx.y;
  const int e = p.mt_ent[i], pl = p.ent_plan[e], fs = p.ent_fslot[e];
  if (p.moff[e] < 0) return;  // dropped by mixsel_kernel
  MixEntry m;
  const int c0 = p.P.cell_begin[pl];
  m.C = p.P.cell_begin[pl + 1] - c0;
  for (int c = threadIdx.x; c < m.C; c += blockDim.x)
    s_q[c] = reinterpret_cast<const double2*>(
        p.qtab + p.qoff[p.cell_sig[size_t(fs) * p.n_cells_total + c0 + c]] * 4);
  __syncthreads();
  m.K = p.P.coll_begin[pl + 1] - p.P.coll_begin[pl];
  m.b0 = p.P.p2p_begin[pl];
  m.NB = p.P.p2p_begin[pl + 1] - m.b0;
  m.d0 = m.NB > 0 ? p.p2p_tab[m.b0] : -1;
  m.mask = 0;
  m.ND = m.NB > 0 ? 1 : 0;
  for (int b = 1; b < m.NB; ++b)
    if (p.p2p_tab[m.b0 + b] != m.d0) {
      m.ND = 2;
      if (b < 64) m.mask |= uint64_t(1) << b;
    }
  m.sdd = double(p.P.stage_devices[pl]);
  m.reps = double(p.P.stage_reps[pl]);
  m.Sd = double(p.P.num_stages[pl]);
  m.ct = reinterpret_cast<const double2*>(p.ctab) + int64_t(i) * p.mt_nq * p.mt_T;
  const int64_t brows = p.ent_rows[e];
  for (int64_t r = blockIdx.x; r < p.mt_R; r += gridDim.x) {
    const int64_t t = p.mt_ctx[r];
    for (int k = threadIdx.x; k < 2 * m.C; k += blockDim.x) s_t[k] = __ldg(s_q[k >> 1] + 2 * t + (k & 1));
    __syncthreads();
    for (int B0 = 0; B0 < p.mt_w; B0 += blockDim.x) {
      const int B = B0 + int(threadIdx.x);
      const int n = min(int(blockDim.x), p.mt_w - B0);
      double2 o0 = make_double2(0.0, 0.0), o1 = o0;  // rows beyond any batch: never read
      if (B < p.mt_w && B <= brows) mixtab_value(p, m, s_q, s_t, t, B, o0, o1);
      s_row[2 * threadIdx.x] = o0;
      s_row[2 * threadIdx.x + 1] = o1;
      __syncthreads();
      double2* dst = reinterpret_cast<double2*>(p.mixtab + (p.moff[e] + r * p.mt_w + B0) * 4);
      for (int k = threadIdx.x; k < 2 * n; k += blockDim.x) dst[k] = s_row[k];
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256) qtab_kernel(const TabParams p) {
  const int sig = blockIdx.x;
  for (int64_t tok = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; tok < p.sig_rows[sig];
       tok += int64_t(gridDim.y) * blockDim.x)
    qtab_row(p, sig, tok);
}

__global__ void __launch_bounds__(256) dectab_kernel(const TabParams p) {
  const int e = blockIdx.x;
  for (int64_t B = int64_t(blockIdx.y) * blockDim.x + threadIdx.x + 1; B <= p.ent_rows[e];
       B += int64_t(gridDim.y) * blockDim.x)
    dectab_row(p, e, B);
}

}  // namespace psg
