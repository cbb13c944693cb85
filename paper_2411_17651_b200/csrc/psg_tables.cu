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
//                  :125-133) from qtab rows and collective curve queries.
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
