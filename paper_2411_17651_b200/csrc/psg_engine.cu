// psg_engine.cu — host orchestration behind the C ABI (include/psg.h).
//
// One psg_search() call = the reference's search() (simulator.cpp:242-296):
//   1. resolve every (plan, frequency) entry's profile tables once on the
//      host (the reference does a std::map lookup per query, cost.cpp:178-189
//      / :262-270), canonicalize the trace (id-order slots, replica order);
//   2. one H2D of a packed, 16-byte-aligned input image from pinned memory;
//   3. sim_kernel over all (plan, freq, replica) units, LPT-ordered;
//   4. entry_reduce_kernel + offsets + rank_kernel;
//   5. one D2H of entry records, then compact_kernel + one D2H of the dense
//      per-request / rejected arrays (sorted by id, simulator.cpp:205-207).
// Device and pinned buffers are cached in the context and only grow.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <new>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "psg.h"
#include "psg_device.cuh"
#include "psg_reduce.cuh"

using namespace psg;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n, 1024);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n + n / 4, 4096);
    // portable + mapped: the result arrays are written by the kernels of the
    // context's device directly (streamed results), whatever device is current
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// Builds the packed input image: arrays appended at 16-byte alignment.
struct Packer {
  std::vector<std::tuple<size_t, const void*, size_t>> parts;  // offset, src, bytes
  size_t size = 0;
  template <typename T>
  size_t add(const T* src, size_t count) {
    size = (size + 15) & ~size_t(15);
    const size_t off = size;
    const size_t bytes = sizeof(T) * count;
    parts.emplace_back(off, src, bytes);
    size += bytes;
    return off;
  }
  void write(unsigned char* dst) const {
    for (const auto& [off, src, bytes] : parts)
      if (bytes) std::memcpy(dst + off, src, bytes);
  }
};

const char* op_name(int op) {
  switch (op) {
    case PSG_OP_ATTENTION: return "attention";
    case PSG_OP_GEMM: return "gemm";
    case PSG_OP_MOE_GEMM: return "moe_gemm";
  }
  return "?";
}
const char* coll_name(int k) {
  switch (k) {
    case PSG_COLL_ALLREDUCE: return "allreduce";
    case PSG_COLL_ALLGATHER: return "allgather";
    case PSG_COLL_REDUCE_SCATTER: return "reduce_scatter";
    case PSG_COLL_ALL_TO_ALL: return "all_to_all";
    case PSG_COLL_P2P: return "p2p";
  }
  return "?";
}
const char* dtype_name(int d) {
  switch (d) {
    case PSG_DTYPE_FP16: return "fp16";
    case PSG_DTYPE_FP8: return "fp8";
    case PSG_DTYPE_INT4: return "int4";
  }
  return "?";
}

}  // namespace

// Start gate of concurrent searches (psg_search_many): every search enqueues
// its inputs, then all launch their kernels together, so the device span is
// not stretched by one search's host-side preparation.  A search that fails
// before the gate still arrives (on exit), so the others never wait for it.
struct StartGate {
  std::mutex m;
  std::condition_variable cv;
  int expected = 0, arrived = 0;
  void arrive(bool wait) {
    std::unique_lock<std::mutex> lk(m);
    if (++arrived >= expected) cv.notify_all();
    if (wait) cv.wait(lk, [&] { return arrived >= expected; });
  }
};

struct psg_context {
  StartGate* gate = nullptr;       // psg_search_many: launch together
  bool gate_passed = false;
  int device = 0;
  int n_sm = 148;                  // device properties used to size the simulation launch
  int64_t smem_sm = 228 * 1024, smem_block_max = 227 * 1024;
  int concurrent_blocks = 0;       // psg_search_many: simulation blocks sharing the device
  int concurrent_groups = 0;       // ... as replica-group blocks (SimParams::chain_replicas 2)
  bool chain_fallback = false;     // rerun with chained replicas (a tally log overflowed)
  int64_t sim_static_smem = 0;     // sim_kernel's static shared memory
  int64_t mt_cap_bytes = 0;        // mixed-iteration table memory cap (0: not yet queried)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  std::string err;
  DevBuf d_in, d_slot_f64, d_slot_u8, d_scratch_i32, d_scratch_f64, d_scratch_cm, d_work, d_pr, d_rj, d_qtab, d_dtab, d_prof, d_mtab, d_ctab;
  HostBuf h_in, h_out, h_pr, h_rj, h_it, h_isec, h_ijou;
  DevBuf d_it, d_isec, d_ijou, d_ioff, d_synth, d_plan, d_gtab, d_rlog, d_edone;
  // storage for results handed out (valid until the next call)
  std::vector<psg_entry> entries;
  std::vector<uint8_t> compute_clamp, curve_clamp;
};

namespace {

// max{T >= -1 : double(T) * kv <= cap}: the host twin of the simulation's
// integer KV ledger bound (psg_sim.cu ledger_cap_tokens), same operations.
int64_t host_cap_tokens(double kv, double cap) {
  if (!(kv > 0.0)) return (0.0 <= cap) ? (int64_t(1) << 60) : -1;
  if (!(0.0 <= cap)) return -1;
  const double q = std::floor(cap / kv);
  if (q >= 9007199254740992.0) return int64_t(1) << 53;
  int64_t t = int64_t(q);
  while (t >= 0 && double(t) * kv > cap) --t;
  while (!(double(t + 1) * kv > cap)) ++t;
  return t;
}

// Replica groups per DP>1 entry (SimParams::chain_replicas 2).
int replica_groups() {
  if (const char* v = std::getenv("PSG_REPLICA_GROUPS")) return std::max(1, std::atoi(v));  // dev knob
  return 2;
}

void launch_sim(int blocks, size_t smem, cudaStream_t st, const SimParams& sp) {
  const bool chunked = sp.batch_mode == PSG_BATCH_CHUNKED;
  if (const char* v = std::getenv("PSG_CARVEOUT"))  // dev knob: shared-memory carve-out, percent
    for (const void* k : {(const void*)sim_kernel, (const void*)sim_kernel_spec, (const void*)sim_kernel_lane, (const void*)sim_kernel_emit,
                          (const void*)sim_kernel_chunked, (const void*)sim_kernel_spec_chunked})
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(v));
  // with mixed-iteration tables the table answers the speculation warp's
  // jobs: the lane-resident kernel without it (C2 -2%)
  const char* lk = std::getenv("PSG_LANE_KERNEL");  // dev knob
  const bool lane_kernel = !lk || std::atoi(lk) != 0;
  if (sp.emit_it)
    sim_kernel_emit<<<blocks, kWarp, smem, st>>>(sp);
  else if (sp.speculate == 1 && sp.mixtab && !chunked && lane_kernel)
    sim_kernel_lane<<<blocks, kWarp, smem, st>>>(sp);
  else if (sp.speculate)
    (chunked ? sim_kernel_spec_chunked : sim_kernel_spec)<<<blocks, 2 * kWarp, smem, st>>>(sp);
  else
    (chunked ? sim_kernel_chunked : sim_kernel)<<<blocks, kWarp, smem, st>>>(sp);
}

int fail(psg_context* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// No C++ exception may cross the C ABI: host-side failures (allocation,
// threads) become error codes with a message.
template <typename F>
int guarded(psg_context* ctx, F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return fail(ctx, PSG_ERR_CUDA, "host memory allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, PSG_ERR_CUDA, std::string("host failure: ") + e.what());
  } catch (...) {
    return fail(ctx, PSG_ERR_CUDA, "host failure");
  }
}

#define PSG_CUDA(call)                                                           \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(ctx, PSG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

namespace psg {

static int synth_compute_impl(psg_context* ctx, const psg_synth_grid* g, double* seconds,
                              double* joules);

int synth_compute(psg_context* ctx, const psg_synth_grid* g, double* seconds, double* joules) {
  return guarded(ctx, [&] { return synth_compute_impl(ctx, g, seconds, joules); });
}

static int synth_compute_impl(psg_context* ctx, const psg_synth_grid* g, double* seconds,
                              double* joules) {
  if (!ctx || !g || !seconds || !joules) return PSG_ERR_USAGE;
  if (g->n_ctx < 1 || g->n_tasks < 1 || g->n_width < 1 || g->n_variants < 0)
    return fail(ctx, PSG_ERR_USAGE, "synth: empty grid axis");
  const int64_t total = int64_t(g->n_variants) * 3 * g->n_ctx * g->n_tasks * g->n_width;
  if (total == 0) return PSG_OK;
  PSG_CUDA(cudaSetDevice(ctx->device));
  Packer pk;
  const size_t oc = pk.add(g->ctx, size_t(g->n_ctx)), ot = pk.add(g->tasks, size_t(g->n_tasks)),
               ow = pk.add(g->width, size_t(g->n_width)),
               op = pk.add(g->peak_scaled, size_t(g->n_variants)),
               oe = pk.add(g->elem_bytes, size_t(g->n_variants)),
               ob = pk.add(g->power, size_t(g->n_variants));
  const size_t in_bytes = (pk.size + 15) & ~size_t(15);
  PSG_CUDA(ctx->d_synth.ensure(in_bytes + 2 * size_t(total) * sizeof(double)));
  PSG_CUDA(ctx->h_in.ensure(in_bytes));
  pk.write(static_cast<unsigned char*>(ctx->h_in.p));
  auto* d = static_cast<unsigned char*>(ctx->d_synth.p);
  PSG_CUDA(cudaMemcpyAsync(d, ctx->h_in.p, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  psg_synth_grid dg = *g;
  dg.ctx = reinterpret_cast<const double*>(d + oc);
  dg.tasks = reinterpret_cast<const double*>(d + ot);
  dg.width = reinterpret_cast<const double*>(d + ow);
  dg.peak_scaled = reinterpret_cast<const double*>(d + op);
  dg.elem_bytes = reinterpret_cast<const double*>(d + oe);
  dg.power = reinterpret_cast<const double*>(d + ob);
  double* dsec = reinterpret_cast<double*>(d + in_bytes);
  double* djou = dsec + total;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, int64_t(ctx->n_sm) * 8);
  synth_compute_kernel<<<unsigned(blocks), 256, 0, ctx->stream>>>(dg, dsec, djou);
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cudaMemcpyAsync(seconds, dsec, size_t(total) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(joules, djou, size_t(total) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  return PSG_OK;
}

static int plan_compute_impl(psg_context* ctx, const psg_plan_space* s, psg_plan_record* records,
                             int32_t* phys, const int64_t* p2p_offset, int32_t* p2p);

int plan_compute(psg_context* ctx, const psg_plan_space* s, psg_plan_record* records,
                 int32_t* phys, const int64_t* p2p_offset, int32_t* p2p) {
  return guarded(ctx, [&] { return plan_compute_impl(ctx, s, records, phys, p2p_offset, p2p); });
}

// Uploads the plan space and runs plan_map_kernel + plan_candidate_kernel;
// the records / assignments / boundary node counts stay on the device.
struct PlanDev {
  psg_plan_space ds;
  psg_plan_record* rec;
  int32_t *phys, *p2p;
  const int64_t* p2p_off;
  size_t end;  // first free byte of ctx->d_plan after the plan buffers
};

static int plan_device(psg_context* ctx, const psg_plan_space* s, const int64_t* p2p_offset,
                       size_t extra, PlanDev& pd) {
  const int n = s->n_devices, G = s->n_groups, nc = s->n_cells;
  if (n < 1 || G < 0 || nc < 1 || nc > PSG_PLAN_MAX_CELLS || s->n_levels < 1)
    return fail(ctx, PSG_ERR_USAGE, "plan space: bad sizes");
  const int64_t total = s->group_first[G];
  const int64_t n_choice = s->choice_begin[int64_t(G) * nc];
  const int64_t n_p2p = p2p_offset[G];
  const size_t map_smem = size_t(n) * (sizeof(int32_t) + 1);
  if (map_smem > size_t(ctx->smem_block_max)) return fail(ctx, PSG_ERR_USAGE, "plan space: too many devices");
  PSG_CUDA(cudaSetDevice(ctx->device));
  Packer pk;
  const size_t o_cap = pk.add(s->subtree_cap, size_t(s->n_levels) + 1),
               o_att = pk.add(s->cell_is_attention, size_t(nc)), o_kvh = pk.add(s->cell_kv_heads, size_t(nc)),
               o_hd = pk.add(s->cell_head_dim, size_t(nc)), o_gdp = pk.add(s->group_dp, size_t(G)),
               o_gst = pk.add(s->group_stages, size_t(G)), o_gsd = pk.add(s->group_sdev, size_t(G)),
               o_grp = pk.add(s->group_reps, size_t(G)), o_gfi = pk.add(s->group_first, size_t(G) + 1),
               o_cb = pk.add(s->choice_begin, size_t(G) * nc + 1), o_cm = pk.add(s->ch_mode, size_t(n_choice)),
               o_cd = pk.add(s->ch_cdp, size_t(n_choice)), o_ci = pk.add(s->ch_intra, size_t(n_choice)),
               o_cw = pk.add(s->ch_weight, size_t(n_choice)), o_p2o = pk.add(p2p_offset, size_t(G) + 1);
  const size_t in_bytes = (pk.size + 15) & ~size_t(15);
  const size_t rec_bytes = sizeof(psg_plan_record) * size_t(std::max<int64_t>(total, 1));
  const size_t phys_bytes = sizeof(int32_t) * size_t(std::max(G, 1)) * n;
  const size_t p2p_bytes = sizeof(int32_t) * size_t(std::max<int64_t>(n_p2p, 1));
  const size_t span_bytes = sizeof(int32_t) * size_t(std::max(G, 1)) * (n + 1);
  const size_t o_rec = in_bytes, o_phys = o_rec + ((rec_bytes + 15) & ~size_t(15)),
               o_p2p = o_phys + ((phys_bytes + 15) & ~size_t(15)),
               o_sn = o_p2p + ((p2p_bytes + 15) & ~size_t(15)),
               o_sl = o_sn + ((span_bytes + 15) & ~size_t(15)), tot = o_sl + ((span_bytes + 15) & ~size_t(15));
  PSG_CUDA(ctx->d_plan.ensure(tot + extra));
  PSG_CUDA(ctx->h_in.ensure(in_bytes));
  pk.write(static_cast<unsigned char*>(ctx->h_in.p));
  auto* d = static_cast<unsigned char*>(ctx->d_plan.p);
  PSG_CUDA(cudaMemcpyAsync(d, ctx->h_in.p, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  psg_plan_space& ds = pd.ds;
  ds = *s;
  ds.subtree_cap = reinterpret_cast<const int32_t*>(d + o_cap);
  ds.cell_is_attention = reinterpret_cast<const int32_t*>(d + o_att);
  ds.cell_kv_heads = reinterpret_cast<const double*>(d + o_kvh);
  ds.cell_head_dim = reinterpret_cast<const double*>(d + o_hd);
  ds.group_dp = reinterpret_cast<const int32_t*>(d + o_gdp);
  ds.group_stages = reinterpret_cast<const int32_t*>(d + o_gst);
  ds.group_sdev = reinterpret_cast<const int32_t*>(d + o_gsd);
  ds.group_reps = reinterpret_cast<const int32_t*>(d + o_grp);
  ds.group_first = reinterpret_cast<const int64_t*>(d + o_gfi);
  ds.choice_begin = reinterpret_cast<const int32_t*>(d + o_cb);
  ds.ch_mode = reinterpret_cast<const int32_t*>(d + o_cm);
  ds.ch_cdp = reinterpret_cast<const int32_t*>(d + o_cd);
  ds.ch_intra = reinterpret_cast<const int32_t*>(d + o_ci);
  ds.ch_weight = reinterpret_cast<const double*>(d + o_cw);
  pd.rec = reinterpret_cast<psg_plan_record*>(d + o_rec);
  pd.phys = reinterpret_cast<int32_t*>(d + o_phys);
  pd.p2p = reinterpret_cast<int32_t*>(d + o_p2p);
  pd.p2p_off = reinterpret_cast<const int64_t*>(d + o_p2o);
  pd.end = tot;
  if (G == 0) return PSG_OK;
  auto* d_sn = reinterpret_cast<int32_t*>(d + o_sn);
  auto* d_sl = reinterpret_cast<int32_t*>(d + o_sl);
  if (map_smem > 48 * 1024)
    PSG_CUDA(cudaFuncSetAttribute(plan_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(map_smem)));
  plan_map_kernel<<<G, 128, map_smem, ctx->stream>>>(ds, pd.phys, pd.p2p_off, pd.p2p, d_sn, d_sl);
  PSG_CUDA(cudaGetLastError());
  if (total > 0) {
    plan_candidate_kernel<<<unsigned((total + 127) / 128), 128, 0, ctx->stream>>>(ds, d_sn, pd.rec);
    PSG_CUDA(cudaGetLastError());
  }
  return PSG_OK;
}

static int plan_compute_impl(psg_context* ctx, const psg_plan_space* s, psg_plan_record* records,
                             int32_t* phys, const int64_t* p2p_offset, int32_t* p2p) {
  if (!ctx || !s || !records || !phys || !p2p_offset || !p2p) return PSG_ERR_USAGE;
  if (s->n_groups == 0) return PSG_OK;
  PlanDev pd{};
  if (const int rc = plan_device(ctx, s, p2p_offset, 0, pd)) return rc;
  const int G = s->n_groups;
  const int64_t total = s->group_first[G], n_p2p = p2p_offset[G];
  if (total > 0)
    PSG_CUDA(cudaMemcpyAsync(records, pd.rec, sizeof(psg_plan_record) * size_t(total), cudaMemcpyDeviceToHost,
                             ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(phys, pd.phys, sizeof(int32_t) * size_t(G) * s->n_devices, cudaMemcpyDeviceToHost,
                           ctx->stream));
  if (n_p2p > 0)
    PSG_CUDA(cudaMemcpyAsync(p2p, pd.p2p, sizeof(int32_t) * size_t(n_p2p), cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  return PSG_OK;
}

// The owned arrays behind a psg_plan_soa.
struct PlanSoaOwned : psg_plan_soa {
  std::vector<int32_t> dp, st, sd, reps, dt, enc, cb, cop, kb, kk, kd, kn, kg, pb, pn;
  std::vector<double> kv, bud, ppt, hid, head, kve, ct, cw, cs, kp, ksh;
  std::vector<int64_t> cand;
};

static int plan_emit_impl(psg_context* ctx, const psg_plan_space* s, const psg_plan_emit_in* in,
                          psg_plan_soa** out) {
  if (!ctx || !s || !in || !out) return PSG_ERR_USAGE;
  *out = nullptr;
  const int G = s->n_groups, nc = s->n_cells;
  if (G < 1) return fail(ctx, PSG_ERR_INFEASIBLE, "no parallel execution plan fits the model on this cluster");
  const int64_t total = s->group_first[G];
  const int64_t n_choice = s->choice_begin[int64_t(G) * nc];
  std::vector<int64_t> p2p_off(size_t(G) + 1, 0);
  int64_t max_p2p = 0;  // boundaries of every candidate (upper bound of the kept ones)
  for (int g = 0; g < G; ++g) {
    p2p_off[size_t(g) + 1] = p2p_off[size_t(g)] + (s->group_stages[g] - 1);
    max_p2p += (s->group_first[g + 1] - s->group_first[g]) * (s->group_stages[g] - 1);
  }
  // host inputs of the emission, then the output arrays (one region)
  Packer pk;
  const size_t o_keep = pk.add(in->keep, size_t(total)), o_enc = pk.add(in->enc_rank, size_t(total)),
               o_op = pk.add(in->ch_op, size_t(n_choice)), o_t = pk.add(in->ch_tasks, size_t(n_choice)),
               o_w = pk.add(in->ch_width, size_t(n_choice)), o_sc = pk.add(in->ch_scale, size_t(n_choice));
  const size_t in_bytes = (pk.size + 15) & ~size_t(15);
  Packer ok;  // offsets only
  const size_t T = size_t(std::max<int64_t>(total, 1)), TC = T * size_t(nc),
               TK = T * PSG_PLAN_MAX_COLLS, TP = size_t(std::max<int64_t>(max_p2p, 1));
  const size_t w_dp = ok.add<int32_t>(nullptr, T), w_st = ok.add<int32_t>(nullptr, T),
               w_sd = ok.add<int32_t>(nullptr, T), w_rp = ok.add<int32_t>(nullptr, T),
               w_dt = ok.add<int32_t>(nullptr, T), w_en = ok.add<int32_t>(nullptr, T),
               w_kv = ok.add<double>(nullptr, T), w_bu = ok.add<double>(nullptr, T),
               w_pp = ok.add<double>(nullptr, T), w_hi = ok.add<double>(nullptr, T),
               w_he = ok.add<double>(nullptr, T), w_ke = ok.add<double>(nullptr, T),
               w_cb = ok.add<int32_t>(nullptr, T + 1), w_co = ok.add<int32_t>(nullptr, TC),
               w_ct = ok.add<double>(nullptr, TC), w_cw = ok.add<double>(nullptr, TC),
               w_cs = ok.add<double>(nullptr, TC), w_kb = ok.add<int32_t>(nullptr, T + 1),
               w_kk = ok.add<int32_t>(nullptr, TK), w_kd = ok.add<int32_t>(nullptr, TK),
               w_kn = ok.add<int32_t>(nullptr, TK), w_kg = ok.add<int32_t>(nullptr, TK),
               w_kp = ok.add<double>(nullptr, TK), w_ks = ok.add<double>(nullptr, TK),
               w_pb = ok.add<int32_t>(nullptr, T + 1), w_pn = ok.add<int32_t>(nullptr, TP),
               w_ca = ok.add<int64_t>(nullptr, T), w_cnt = ok.add<int32_t>(nullptr, 4);
  PlanDev pd{};
  if (const int rc = plan_device(ctx, s, p2p_off.data(), in_bytes + ok.size + 64, pd)) return rc;
  auto* base = static_cast<unsigned char*>(ctx->d_plan.p) + ((pd.end + 15) & ~size_t(15));
  PSG_CUDA(ctx->h_in.ensure(in_bytes));
  pk.write(static_cast<unsigned char*>(ctx->h_in.p));
  PSG_CUDA(cudaMemcpyAsync(base, ctx->h_in.p, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  unsigned char* w = base + in_bytes;
  auto W = [&](size_t o) { return static_cast<void*>(w + o); };
  PlanEmitArgs a{};
  a.keep = reinterpret_cast<const uint8_t*>(base + o_keep);
  a.enc_rank = reinterpret_cast<const int32_t*>(base + o_enc);
  a.ch_op = reinterpret_cast<const int32_t*>(base + o_op);
  a.ch_tasks = reinterpret_cast<const double*>(base + o_t);
  a.ch_width = reinterpret_cast<const double*>(base + o_w);
  a.ch_scale = reinterpret_cast<const double*>(base + o_sc);
  a.p2p_off = pd.p2p_off;
  a.p2p = pd.p2p;
  a.compute_dtype = in->compute_dtype;
  a.payload_per_token = in->payload_per_token;
  a.shape_hidden = in->shape_hidden;
  a.shape_head_dim = in->shape_head_dim;
  a.shape_kv_elems = in->shape_kv_elems;
  PlanEmitOut o{(int32_t*)W(w_dp), (int32_t*)W(w_st), (int32_t*)W(w_sd), (int32_t*)W(w_rp),
                (int32_t*)W(w_dt), (int32_t*)W(w_en), (double*)W(w_kv), (double*)W(w_bu),
                (double*)W(w_pp), (double*)W(w_hi), (double*)W(w_he), (double*)W(w_ke),
                (int32_t*)W(w_cb), (int32_t*)W(w_co), (double*)W(w_ct), (double*)W(w_cw),
                (double*)W(w_cs), (int32_t*)W(w_kb), (int32_t*)W(w_kk), (int32_t*)W(w_kd),
                (int32_t*)W(w_kn), (int32_t*)W(w_kg), (double*)W(w_kp), (double*)W(w_ks),
                (int32_t*)W(w_pb), (int32_t*)W(w_pn), (int64_t*)W(w_ca), (int32_t*)W(w_cnt)};
  plan_emit_kernel<<<1, kEmitThreads, 0, ctx->stream>>>(pd.ds, pd.rec, a, o);
  PSG_CUDA(cudaGetLastError());
  // one D2H of the emitted region (sized for every candidate), then trim
  PSG_CUDA(ctx->h_out.ensure(ok.size + 64));
  PSG_CUDA(cudaMemcpyAsync(ctx->h_out.p, w, ok.size, cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  const unsigned char* h = static_cast<const unsigned char*>(ctx->h_out.p);
  auto Hi = [&](size_t off) { return reinterpret_cast<const int32_t*>(h + off); };
  auto Hd = [&](size_t off) { return reinterpret_cast<const double*>(h + off); };
  const int np = Hi(w_cnt)[0], nk = Hi(w_cnt)[1], nb = Hi(w_cnt)[2];
  if (np == 0) return fail(ctx, PSG_ERR_INFEASIBLE, "no parallel execution plan fits the model on this cluster");
  auto* so = new PlanSoaOwned();
  auto take_i = [&](std::vector<int32_t>& v, size_t off, size_t n) { v.assign(Hi(off), Hi(off) + n); };
  auto take_d = [&](std::vector<double>& v, size_t off, size_t n) { v.assign(Hd(off), Hd(off) + n); };
  take_i(so->dp, w_dp, np); take_i(so->st, w_st, np); take_i(so->sd, w_sd, np);
  take_i(so->reps, w_rp, np); take_i(so->dt, w_dt, np); take_i(so->enc, w_en, np);
  take_d(so->kv, w_kv, np); take_d(so->bud, w_bu, np); take_d(so->ppt, w_pp, np);
  take_d(so->hid, w_hi, np); take_d(so->head, w_he, np); take_d(so->kve, w_ke, np);
  take_i(so->cb, w_cb, size_t(np) + 1); take_i(so->cop, w_co, size_t(np) * nc);
  take_d(so->ct, w_ct, size_t(np) * nc); take_d(so->cw, w_cw, size_t(np) * nc);
  take_d(so->cs, w_cs, size_t(np) * nc); take_i(so->kb, w_kb, size_t(np) + 1);
  take_i(so->kk, w_kk, nk); take_i(so->kd, w_kd, nk); take_i(so->kn, w_kn, nk); take_i(so->kg, w_kg, nk);
  take_d(so->kp, w_kp, nk); take_d(so->ksh, w_ks, nk);
  take_i(so->pb, w_pb, size_t(np) + 1); take_i(so->pn, w_pn, nb);
  so->cand.assign(reinterpret_cast<const int64_t*>(h + w_ca), reinterpret_cast<const int64_t*>(h + w_ca) + np);
  auto nz = [](auto& v) { return v.empty() ? nullptr : v.data(); };
  psg_plan_set& v = so->set;
  v = psg_plan_set{np, nz(so->dp), nz(so->st), nz(so->sd), nz(so->reps), nz(so->dt), nz(so->enc),
                   nz(so->kv), nz(so->bud), nz(so->ppt), nz(so->hid), nz(so->head), nz(so->kve),
                   so->cb.data(), nz(so->cop), nz(so->ct), nz(so->cw), nz(so->cs), so->kb.data(),
                   nz(so->kk), nz(so->kd), nz(so->kn), nz(so->kg), nz(so->kp), nz(so->ksh),
                   so->pb.data(), nz(so->pn)};
  so->candidate = so->cand.data();
  *out = so;
  return PSG_OK;
}

int plan_emit(psg_context* ctx, const psg_plan_space* s, const psg_plan_emit_in* in, psg_plan_soa** out) {
  return guarded(ctx, [&] { return plan_emit_impl(ctx, s, in, out); });
}

void plan_soa_free(psg_plan_soa* soa) { delete static_cast<PlanSoaOwned*>(soa); }

}  // namespace psg

extern "C" {

const char* psg_version(void) { return "psg-b200 1 (sm_100a)"; }

int psg_device_count(int* count) {
  if (!count) return PSG_ERR_USAGE;
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  *count = c;
  return PSG_OK;
}

int psg_context_create(int device, psg_context** out) {
  if (!out) return PSG_ERR_USAGE;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return PSG_ERR_CUDA;
  if (device < 0 || device >= count) return PSG_ERR_USAGE;
  if (cudaSetDevice(device) != cudaSuccess) return PSG_ERR_CUDA;
  auto* ctx = new (std::nothrow) psg_context();
  if (!ctx) return PSG_ERR_CUDA;
  ctx->device = device;
  {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && v > 0) ctx->n_sm = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device) == cudaSuccess && v > 0)
      ctx->smem_sm = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) == cudaSuccess && v > 0)
      ctx->smem_block_max = v;
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PSG_ERR_CUDA;
  }
  // the cap only; each launch asks for what it needs (set once: contexts may
  // launch concurrently from several threads)
  for (const void* k : {(const void*)sim_kernel, (const void*)sim_kernel_spec, (const void*)sim_kernel_lane, (const void*)sim_kernel_emit,
                        (const void*)sim_kernel_chunked, (const void*)sim_kernel_spec_chunked}) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) == cudaSuccess)
      ctx->sim_static_smem = std::max<int64_t>(ctx->sim_static_smem, int64_t(fa.sharedSizeBytes));
  }
  for (const void* k : {(const void*)sim_kernel, (const void*)sim_kernel_spec, (const void*)sim_kernel_lane, (const void*)sim_kernel_emit,
                        (const void*)sim_kernel_chunked, (const void*)sim_kernel_spec_chunked})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(ctx->smem_block_max - ctx->sim_static_smem));
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  cudaFuncSetAttribute((const void*)entry_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(kReduceCandCap * kReduceStats * sizeof(uint64_t)));
  *out = ctx;
  return PSG_OK;
}

void psg_context_destroy(psg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->d_in, &ctx->d_slot_f64, &ctx->d_slot_u8, &ctx->d_scratch_i32,
                    &ctx->d_scratch_f64, &ctx->d_scratch_cm, &ctx->d_work, &ctx->d_pr, &ctx->d_rj, &ctx->d_qtab, &ctx->d_dtab, &ctx->d_prof, &ctx->d_mtab, &ctx->d_ctab,
                    &ctx->d_it, &ctx->d_isec, &ctx->d_ijou, &ctx->d_ioff, &ctx->d_synth, &ctx->d_plan, &ctx->d_gtab,
                    &ctx->d_rlog, &ctx->d_edone})
    b->release();
  for (HostBuf* b : {&ctx->h_in, &ctx->h_out, &ctx->h_pr, &ctx->h_rj, &ctx->h_it, &ctx->h_isec, &ctx->h_ijou})
    b->release();
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* psg_last_error(const psg_context* ctx) { return ctx ? ctx->err.c_str() : ""; }

void psg_result_free(psg_result* r) { delete r; }

int psg_rank_keys(psg_context* ctx, const psg_rank_key* keys, int64_t n, int64_t* order) {
  if (!ctx || (n > 0 && (!keys || !order))) return PSG_ERR_USAGE;
  if (n == 0) return PSG_OK;
  PSG_CUDA(cudaSetDevice(ctx->device));
  const size_t kb = sizeof(psg_rank_key) * size_t(n), ob = sizeof(int64_t) * size_t(n);
  PSG_CUDA(ctx->d_work.ensure(kb + ob + 64));
  PSG_CUDA(ctx->h_out.ensure(kb + ob));
  auto* dk = static_cast<psg_rank_key*>(ctx->d_work.p);
  auto* dord = reinterpret_cast<int64_t*>(static_cast<unsigned char*>(ctx->d_work.p) + ((kb + 15) & ~size_t(15)));
  std::memcpy(ctx->h_out.p, keys, kb);
  PSG_CUDA(cudaMemcpyAsync(dk, ctx->h_out.p, kb, cudaMemcpyHostToDevice, ctx->stream));
  rank_kernel<<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(dk, n, dord);
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(ctx->h_out.p) + kb, dord, ob,
                           cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(order, static_cast<unsigned char*>(ctx->h_out.p) + kb, ob);
  return PSG_OK;
}

static int search_impl(psg_context* ctx, const psg_plan_set* P, const psg_cluster* cl,
                       const psg_store* S, const psg_trace* T, const psg_config* cfg,
                       psg_result** out);

int psg_search(psg_context* ctx, const psg_plan_set* P, const psg_cluster* cl,
               const psg_store* S, const psg_trace* T, const psg_config* cfg,
               psg_result** out) {
  if (out) *out = nullptr;
  return guarded(ctx, [&] { return search_impl(ctx, P, cl, S, T, cfg, out); });
}

static int search_impl(psg_context* ctx, const psg_plan_set* P, const psg_cluster* cl,
                       const psg_store* S, const psg_trace* T, const psg_config* cfg,
                       psg_result** out) {
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  // dev: PSG_HOST_TIMING=1 prints the host phases of the call (ms since entry)
  static const bool host_timing = std::getenv("PSG_HOST_TIMING") != nullptr;
  double host_t[16] = {};
  auto host_mark = [&](int k) {
    if (host_timing) host_t[k] = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
  };
  if (!ctx || !P || !cl || !S || !T || !cfg || !out) return PSG_ERR_USAGE;
  *out = nullptr;
  ctx->err.clear();
  if (P->n_plans <= 0) return fail(ctx, PSG_ERR_INFEASIBLE, "search: no feasible plan");
  PSG_CUDA(cudaSetDevice(ctx->device));

  // ---- frequencies and entries (simulator.cpp:248-258) ----
  std::vector<double> freqs(cfg->freqs, cfg->freqs + std::max(0, cfg->n_freqs));
  if (freqs.empty()) freqs.push_back(cl->max_frequency_ghz);
  const int F = int(freqs.size());
  const int64_t n_total_entries = int64_t(P->n_plans) * F;
  std::vector<int64_t> ent;  // local entry -> global entry index
  if (cfg->n_entry_subset > 0) {
    for (int i = 0; i < cfg->n_entry_subset; ++i) {
      const int64_t g = cfg->entry_subset[i];
      if (g < 0 || g >= n_total_entries) return fail(ctx, PSG_ERR_USAGE, "entry_subset out of range");
      ent.push_back(g);
    }
  } else {
    ent.resize(size_t(n_total_entries));
    std::iota(ent.begin(), ent.end(), 0);
  }
  const int E = int(ent.size());
  if (cfg->emit_iterations && E != 1)
    return fail(ctx, PSG_ERR_USAGE, "emit_iterations requires exactly one (plan, frequency) entry");
  if (!(cfg->ttft_slo >= 0.0) || !(cfg->slo_quantile >= 0.0 && cfg->slo_quantile <= 1.0))
    return fail(ctx, PSG_ERR_USAGE, "ttft_slo must be >= 0 and slo_quantile in [0, 1]");

  // ---- validate plans ----
  const int np = P->n_plans;
  const int n_cells = P->cell_begin[np], n_colls = P->coll_begin[np], n_p2p = P->p2p_begin[np];
  for (int p = 0; p < np; ++p) {
    const int C = P->cell_begin[p + 1] - P->cell_begin[p];
    const int K = P->coll_begin[p + 1] - P->coll_begin[p];
    const int NB = P->p2p_begin[p + 1] - P->p2p_begin[p];
    if (C < 0 || K < 0 || NB < 0 || C > kMaxCells || K > kMaxClampSlots)
      return fail(ctx, PSG_ERR_USAGE, "plan " + std::to_string(p) + ": unsupported cell/collective count");
    if (P->model_dp[p] < 1 || P->num_stages[p] < 1)
      return fail(ctx, PSG_ERR_USAGE, "plan " + std::to_string(p) + ": bad degrees");
    if (NB != P->num_stages[p] - 1)
      return fail(ctx, PSG_ERR_USAGE, "plan " + std::to_string(p) + ": p2p boundaries != stages-1");
  }

  host_mark(0);
  // ---- resolve tables (ProfileStore keys, cost.hpp:105-116) ----
  std::map<std::tuple<int, int, long long>, int> cmap;
  for (int t = 0; t < S->n_compute; ++t) {
    if (S->c_n_ctx[t] < 1 || S->c_n_tasks[t] < 1 || S->c_n_width[t] < 1)
      return fail(ctx, PSG_ERR_DATA, "profile: empty compute grid");
    cmap[{S->c_op[t], S->c_dtype[t], (long long)S->c_freq_micro[t]}] = t;
  }
  std::map<std::tuple<int, int, int>, int> kmap;
  for (int u = 0; u < S->n_curves; ++u) {
    if (S->k_n[u] < 1) return fail(ctx, PSG_ERR_DATA, "profile: empty collective curve");
    kmap[{S->k_kind[u], S->k_devices[u], S->k_nodes[u]}] = u;
  }
  std::vector<int32_t> cell_tab(size_t(F) * n_cells, -1), coll_tab(n_colls, -1), p2p_tab(n_p2p, -1);
  for (int f = 0; f < F; ++f) {
    const long long fk = llround(freqs[f] * 1e6);
    for (int p = 0; p < np; ++p)
      for (int c = P->cell_begin[p]; c < P->cell_begin[p + 1]; ++c) {
        auto it = cmap.find({P->cell_op[c], P->compute_dtype[p], fk});
        cell_tab[size_t(f) * n_cells + c] = it == cmap.end() ? -1 : it->second;
      }
  }
  for (int k = 0; k < n_colls; ++k) {
    auto it = kmap.find({P->coll_kind[k], P->coll_devices[k], P->coll_nodes[k]});
    coll_tab[k] = it == kmap.end() ? -1 : it->second;
  }
  for (int b = 0; b < n_p2p; ++b) {
    auto it = kmap.find({int(PSG_COLL_P2P), 2, P->p2p_nodes[b]});
    p2p_tab[b] = it == kmap.end() ? -1 : it->second;
  }
  // Stage boundaries share a handful of distinct p2p curves (one per node
  // span, planner.cpp:344): boundary -> distinct curve in first-appearance
  // order (the simulation kernel's rule), and per plan the doubles its staged
  // curves take (knots + seconds/joules of the collectives and distinct p2p).
  std::vector<uint8_t> bslot(std::max(n_p2p, 1), 0);
  std::vector<int64_t> plan_tab_need(np, 0);
  for (int p = 0; p < np; ++p) {
    std::vector<int32_t> distinct;
    for (int b = P->p2p_begin[p]; b < P->p2p_begin[p + 1]; ++b) {
      size_t s = 0;
      while (s < distinct.size() && distinct[s] != p2p_tab[b]) ++s;
      if (s == distinct.size()) distinct.push_back(p2p_tab[b]);
      bslot[b] = uint8_t(std::min<size_t>(s, 255));
    }
    const int K = P->coll_begin[p + 1] - P->coll_begin[p];
    if (K + int(distinct.size()) > kMaxClampSlots)
      return fail(ctx, PSG_ERR_USAGE, "plan " + std::to_string(p) + ": more than " +
                                          std::to_string(kMaxClampSlots) + " distinct curves");
    int64_t need = 0;
    for (int k = P->coll_begin[p]; k < P->coll_begin[p + 1]; ++k)
      need += 3 * int64_t(coll_tab[k] >= 0 ? S->k_n[coll_tab[k]] : 1);
    for (int32_t t : distinct) need += 3 * int64_t(t >= 0 ? S->k_n[t] : 1);
    plan_tab_need[p] = need;
  }
  std::vector<int32_t> entry_missing(E, 0);
  std::vector<std::string> missing_msg(E);
  for (int e = 0; e < E; ++e) {
    const int p = int(ent[e] / F), f = int(ent[e] % F);
    for (int c = P->cell_begin[p]; c < P->cell_begin[p + 1] && !entry_missing[e]; ++c)
      if (cell_tab[size_t(f) * n_cells + c] < 0) {
        entry_missing[e] = 1;
        char buf[256];
        std::snprintf(buf, sizeof buf, "profile: no compute table for op=%s dtype=%s freq=%g GHz",
                      op_name(P->cell_op[c]), dtype_name(P->compute_dtype[p]), freqs[f]);
        missing_msg[e] = buf;
      }
    for (int k = P->coll_begin[p]; k < P->coll_begin[p + 1] && !entry_missing[e]; ++k)
      if (coll_tab[k] < 0) {
        entry_missing[e] = 1;
        char buf[256];
        std::snprintf(buf, sizeof buf, "profile: no collective table for op=%s devices=%d nodes=%d",
                      coll_name(P->coll_kind[k]), P->coll_devices[k], P->coll_nodes[k]);
        missing_msg[e] = buf;
      }
    for (int b = P->p2p_begin[p]; b < P->p2p_begin[p + 1] && !entry_missing[e]; ++b)
      if (p2p_tab[b] < 0) {
        entry_missing[e] = 1;
        char buf[256];
        std::snprintf(buf, sizeof buf, "profile: no collective table for op=p2p devices=2 nodes=%d",
                      P->p2p_nodes[b]);
        missing_msg[e] = buf;
      }
  }

  host_mark(1);
  // ---- trace canonicalization ----
  const int64_t N = T->n;
  if (N < 0 || N >= INT32_MAX) return fail(ctx, PSG_ERR_USAGE, "trace too large");
  int64_t tok_total = 0;
  bool sorted = true;
  for (int64_t i = 0; i < N; ++i) {
    // 2^26-token bound keeps every per-warp token reduction inside 32 bits
    if (T->context_len[i] < 0 || T->context_len[i] >= (int64_t(1) << 26) ||
        T->gen_len[i] >= (int64_t(1) << 26))
      return fail(ctx, PSG_ERR_USAGE, "trace lengths outside the supported range [0, 2^26)");
    // a non-finite arrival has no place in the clock order (the decode-run
    // horizon compares it against finite clocks)
    if (!std::isfinite(T->arrival[i]))
      return fail(ctx, PSG_ERR_USAGE, "trace arrivals must be finite");
    tok_total += T->context_len[i] + std::max<int64_t>(T->gen_len[i], 1);
    if (i && T->arrival[i] < T->arrival[i - 1]) sorted = false;
  }
  // Exact ledger: the reference recomputes sum(double(ctx+gen)*kv); with an
  // integral kv every partial sum below 2^53 is exact, so token counts times
  // kv reproduce it bit for bit.
  for (int p = 0; p < np; ++p) {
    const double kv = P->kv_bytes_per_token[p];
    if (!(kv >= 0) || kv != std::floor(kv) || double(tok_total) * kv >= 9007199254740992.0)
      return fail(ctx, PSG_ERR_USAGE,
                  "kv_bytes_per_token must be a non-negative integer with an exactly "
                  "representable ledger");
  }
  std::vector<int32_t> slot(N), slot_order(N);
  std::iota(slot_order.begin(), slot_order.end(), 0);
  bool ids_sorted = true;  // (the common case: the id order is the trace order)
  for (int64_t i = 1; i < N && ids_sorted; ++i) ids_sorted = T->id[i - 1] <= T->id[i];
  if (!ids_sorted)
    std::stable_sort(slot_order.begin(), slot_order.end(),
                     [&](int32_t a, int32_t b) { return T->id[a] < T->id[b]; });
  std::vector<int64_t> slot_id(N), slot_gen(N);
  for (int64_t s = 0; s < N; ++s) {
    slot[slot_order[s]] = int32_t(s);
    slot_id[s] = T->id[slot_order[s]];
    slot_gen[s] = T->gen_len[slot_order[s]];
    // the reference keys per-request state by id (simulator.cpp:103-110):
    // repeated ids blend metrics and leave the per-request order unspecified
    if (s && slot_id[s] == slot_id[s - 1])
      return fail(ctx, PSG_ERR_USAGE, "trace: request ids must be unique (id " +
                                          std::to_string(slot_id[s]) + " repeats)");
  }

  host_mark(2);
  // ---- units: (entry, replica), longest-first ----
  std::vector<Unit> units;
  std::vector<int32_t> seq;
  std::map<int, int64_t> seq_base_of;  // replicas -> base (unsorted traces only)
  for (int e = 0; e < E; ++e) {
    const int p = int(ent[e] / F);
    const int R = P->model_dp[p];
    if (!sorted && !seq_base_of.count(R)) {
      // split round-robin in trace order, then stable-sort each replica by
      // arrival (BatchState's constructor, batching.cpp:16-17)
      seq_base_of[R] = int64_t(seq.size());
      for (int r = 0; r < R; ++r) {
        std::vector<int32_t> idx;
        for (int64_t i = r; i < N; i += R) idx.push_back(int32_t(i));
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int32_t a, int32_t b) { return T->arrival[a] < T->arrival[b]; });
        seq.insert(seq.end(), idx.begin(), idx.end());
      }
    }
    int64_t off = 0;
    for (int r = 0; r < R; ++r) {
      Unit u;
      u.entry = e;
      u.plan = p;
      u.fslot = int(ent[e] % F);
      u.replica = r;
      u.replicas = R;
      u.n_req = int32_t(N > r ? (N - r + R - 1) / R : 0);
      u.seq_base = sorted ? 0 : seq_base_of[R] + off;
      off += u.n_req;
      u.scratch = 0;
      u.gtab = -1;
      u.log_off = -1;
      u.log_cap = 0;
      u.pad = 0;
      units.push_back(u);
    }
  }
  std::vector<int32_t> entry_unit_begin(E + 1, 0), entry_units(units.size());
  {
    std::vector<int32_t> perm(units.size());
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(),
                     [&](int32_t a, int32_t b) { return units[a].n_req > units[b].n_req; });
    std::vector<Unit> sorted_units(units.size());
    std::vector<int32_t> pos_of(units.size());
    int64_t scratch = 0;
    for (size_t k = 0; k < perm.size(); ++k) {
      sorted_units[k] = units[perm[k]];
      sorted_units[k].scratch = scratch;
      scratch += sorted_units[k].n_req;
      pos_of[perm[k]] = int32_t(k);
    }
    // units were generated entry-major, replica order
    for (size_t k = 0; k < units.size(); ++k) {
      entry_units[k] = pos_of[k];
      entry_unit_begin[units[k].entry + 1]++;
    }
    for (int e = 0; e < E; ++e) entry_unit_begin[e + 1] += entry_unit_begin[e];
    units.swap(sorted_units);
  }
  int64_t scratch_total = 0;
  for (const auto& u : units) scratch_total += u.n_req;
  const int n_units = int(units.size());

  // ---- replica mode (SimParams::chain_replicas) ----
  // 2 (default): an entry's DP replicas split into up to `groups` contiguous
  // groups; a group's replicas run in order on one warp carrying the tally,
  // groups run concurrently, and the entry's last group to finish replays
  // the WorkTally from the later groups' logs (the longest DP>1 entries then
  // stop bounding the search); 1: one group per entry (iteration-record
  // pass, and the fallback when a log overflows); 0: one warp per replica
  // with per-replica tallies (dev).
  int chain = (cfg->emit_iterations || ctx->chain_fallback) ? 1 : 2;
  if (const char* v = std::getenv("PSG_CHAIN_REPLICAS"))  // dev knob
    if (!ctx->chain_fallback) chain = std::max(0, std::min(2, std::atoi(v)));
  const int groups = replica_groups();
  int64_t rlog_total = 0;
  std::vector<int32_t> block_k0, block_k1, entry_groups(E, 1);
  std::vector<int64_t> entry_work(E, 0);  // the entry's longest serial chain, in requests
  if (chain == 2) {
    struct Blk { int32_t k0, k1; int64_t work; };
    std::vector<Blk> blks;
    for (int e = 0; e < E; ++e) {
      const int k0 = entry_unit_begin[e], R = entry_unit_begin[e + 1] - k0;
      const int G = std::max(1, std::min(R, groups));
      entry_groups[e] = G;
      for (int g = 0; g < G; ++g) {
        const int a = k0 + int(int64_t(g) * R / G), b = k0 + int(int64_t(g + 1) * R / G);
        int64_t w = 0;
        for (int k = a; k < b; ++k) w += units[entry_units[k]].n_req;
        blks.push_back({a, b, w});
        entry_work[e] = std::max(entry_work[e], w);
      }
    }
    std::stable_sort(blks.begin(), blks.end(), [](const Blk& x, const Blk& y) { return x.work > y.work; });
    for (const Blk& b : blks) {
      block_k0.push_back(b.k0);
      block_k1.push_back(b.k1);
    }
    // records: one per mixed iteration or decode run; a request causes at
    // most ~4 of them plus its prefill chunks (evictions can add more: the
    // kernel flags an overflow and the search reruns chained)
    int64_t ctx_max = 1;
    for (int64_t i = 0; i < N; ++i) ctx_max = std::max<int64_t>(ctx_max, T->context_len[i]);
    const int64_t chunks = (cfg->batch_mode == PSG_BATCH_CHUNKED && cfg->chunk_size >= 1)
                               ? (ctx_max + cfg->chunk_size - 1) / cfg->chunk_size : 1;
    int64_t per_req = 4 + chunks;
    if (const char* v = std::getenv("PSG_RLOG_PER_REQ")) per_req = std::max(0, std::atoi(v));  // dev / tests
    for (int e = 0; e < E; ++e) {  // the replicas of groups >= 1 log
      const int k0 = entry_unit_begin[e], R = entry_unit_begin[e + 1] - k0, G = entry_groups[e];
      for (int k = k0 + (G > 1 ? R / G : R); k < k0 + R; ++k) {
        Unit& u = units[entry_units[k]];
        u.log_off = rlog_total;
        u.log_cap = int32_t(std::min<int64_t>(int64_t(u.n_req) * per_req + 64, INT32_MAX));
        rlog_total += u.log_cap;
      }
    }
  }
  const int sim_blocks = chain == 1 ? E : chain == 2 ? int(block_k0.size()) : n_units;
  if (chain != 2)
    for (const auto& u : units)
      entry_work[u.entry] = chain == 1 ? entry_work[u.entry] + u.n_req
                                       : std::max<int64_t>(entry_work[u.entry], u.n_req);

  host_mark(3);
  // ---- streamed per-request results (SimParams::out_pr) ----
  // A request completes iff its ledger never has to exceed the KV budget
  // while it is active: ctx + max(gen - 1, 0) <= cap_tok (admission needs
  // ctx <= cap_tok, batching.cpp:41-45; an outgrowing request is evicted or,
  // alone, rejected, :110-125; a request leaves at the step that generates
  // its last token, before the overflow check).  So every entry's completed
  // count — and its offset in the result arrays — is known before the
  // launch, and the warp that completes an entry writes its records straight
  // into the pinned result arrays while the others still simulate.  The
  // kernel checks the count; a mismatch falls back to compaction.
  bool stream = cfg->detail && chain != 0 && !cfg->emit_iterations;
  if (const char* v = std::getenv("PSG_STREAM_RESULTS")) stream = stream && std::atoi(v) != 0;  // dev knob
  std::vector<int64_t> exp_pr(stream ? E : 0), pr_off0(stream ? E : 0), rj_off0(stream ? E : 0);
  int64_t tot_pr0 = 0, tot_rj0 = 0;
  if (stream) {
    // counts of requests with need <= cap for every distinct cap: one pass
    // over the trace, a binary search among the (few) distinct caps each
    std::vector<int64_t> caps(static_cast<size_t>(E));
    for (int e = 0; e < E; ++e) {
      const int p = int(ent[e] / F);
      caps[size_t(e)] = host_cap_tokens(P->kv_bytes_per_token[p], P->kv_budget_per_replica[p]);
    }
    std::vector<int64_t> ucap(caps);
    std::sort(ucap.begin(), ucap.end());
    ucap.erase(std::unique(ucap.begin(), ucap.end()), ucap.end());
    std::vector<int64_t> fit(ucap.size() + 1, 0);  // fit[k]: needs in (ucap[k-1], ucap[k]]
    for (int64_t i = 0; i < N; ++i) {
      const int64_t need = T->context_len[i] + std::max<int64_t>(T->gen_len[i] - 1, 0);
      ++fit[size_t(std::lower_bound(ucap.begin(), ucap.end(), need) - ucap.begin())];
    }
    for (size_t k = 1; k < fit.size(); ++k) fit[k] += fit[k - 1];  // fit[k]: needs <= ucap[k]
    for (int e = 0; e < E; ++e) {
      const int64_t c = fit[size_t(std::lower_bound(ucap.begin(), ucap.end(), caps[size_t(e)]) - ucap.begin())];
      exp_pr[e] = c;
      if (e == 0 && std::getenv("PSG_STREAM_SKEW")) exp_pr[e] += 1;  // dev / tests: force the fallback
      pr_off0[e] = tot_pr0;
      rj_off0[e] = tot_rj0;
      tot_pr0 += exp_pr[e];
      tot_rj0 += N - exp_pr[e];
    }
  }

  std::vector<double> entry_peak(E), entry_freq(E);
  std::vector<int32_t> entry_enc(E);
  for (int e = 0; e < E; ++e) {
    const int p = int(ent[e] / F);
    const int dt = P->compute_dtype[p];
    const double pf = (dt >= 0 && dt < 3) ? cl->peak_flops[dt] : 0.0;
    entry_peak[e] = pf > 0 ? pf * double(cl->total_devices) : 0.0;
    entry_freq[e] = freqs[ent[e] % F];
    entry_enc[e] = P->enc_rank[p];
  }

  host_mark(4);
  // ---- cell signatures and cost-table sizes (psg_tables.cu) ----
  // A cell query depends only on (grid, token_scale, tasks, width, op, op
  // shape) and the token count; plans sharing those share one table.
  int64_t item_max = 0;
  for (int64_t i = 0; i < N; ++i) item_max = std::max<int64_t>(item_max, T->context_len[i]);
  if (cfg->batch_mode == PSG_BATCH_CHUNKED && cfg->chunk_size >= 1)
    item_max = std::min<int64_t>(item_max, cfg->chunk_size);
  std::vector<int64_t> ent_rows(E, 1);  // decode tables cover B = 1..max replica size
  for (const auto& u : units) ent_rows[u.entry] = std::max<int64_t>(ent_rows[u.entry], u.n_req);
  auto fbits = [](double v) {
    uint64_t b;
    std::memcpy(&b, &v, sizeof b);
    return b;
  };
  std::map<std::tuple<int, int, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t>, int> sig_of;
  std::vector<int32_t> sig_table, sig_op, cell_sig(std::max<size_t>(size_t(F) * n_cells, 1), 0);
  std::vector<double> sig_scale, sig_tasks, sig_width, sig_hidden, sig_head, sig_kv;
  std::vector<int64_t> sig_rows;
  for (int e = 0; e < E; ++e) {
    const int p = int(ent[e] / F), f = int(ent[e] % F);
    for (int c = P->cell_begin[p]; c < P->cell_begin[p + 1]; ++c) {
      const int t = cell_tab[size_t(f) * n_cells + c];
      const auto key = std::make_tuple(t, P->cell_op[c], fbits(P->cell_token_scale[c]),
                                       fbits(P->cell_tasks[c]), fbits(P->cell_width[c]),
                                       fbits(P->shape_hidden[p]), fbits(P->shape_head_dim[p]),
                                       fbits(P->shape_kv_elems[p]));
      auto it = sig_of.find(key);
      int sg;
      if (it == sig_of.end()) {
        sg = int(sig_table.size());
        sig_of.emplace(key, sg);
        sig_table.push_back(t);
        sig_op.push_back(P->cell_op[c]);
        sig_scale.push_back(P->cell_token_scale[c]);
        sig_tasks.push_back(P->cell_tasks[c]);
        sig_width.push_back(P->cell_width[c]);
        sig_hidden.push_back(P->shape_hidden[p]);
        sig_head.push_back(P->shape_head_dim[p]);
        sig_kv.push_back(P->shape_kv_elems[p]);
        sig_rows.push_back(1);
      } else {
        sg = it->second;
      }
      cell_sig[size_t(f) * n_cells + c] = sg;
      sig_rows[sg] = std::max<int64_t>(sig_rows[sg], std::max(item_max, ent_rows[e]) + 1);
    }
  }
  const int n_sig = int(sig_table.size());
  std::vector<int64_t> qoff(std::max(n_sig, 1), 0), doff(std::max(E, 1), 0);
  int64_t qrows = 0, drows = 0, max_qrows = 1, max_drows = 1;
  for (int g = 0; g < n_sig; ++g) {
    qoff[g] = qrows;
    qrows += sig_rows[g];
    max_qrows = std::max(max_qrows, sig_rows[g]);
  }
  std::vector<int32_t> ent_plan(std::max(E, 1)), ent_fslot(std::max(E, 1));
  for (int e = 0; e < E; ++e) {
    doff[e] = drows;
    drows += ent_rows[e];
    max_drows = std::max(max_drows, ent_rows[e]);
    ent_plan[e] = int32_t(ent[e] / F);
    ent_fslot[e] = int32_t(ent[e] % F);
  }
  int speculate;
  {
    // The speculation warps pay off while they get SM sub-partitions of their
    // own: with more than ~2 simulation blocks per SM they share them with
    // other blocks' simulation warps and slow those down (C5: 437 blocks).
    const int blocks = std::max(sim_blocks, chain == 2 ? ctx->concurrent_groups : ctx->concurrent_blocks);
    double per_sm = 2.0;  // (C2 + C2-fp8 bench: 278 group blocks, on; C5: 437, off)
    if (const char* v = std::getenv("PSG_SPEC_PER_SM")) per_sm = std::atof(v);  // dev knob
    speculate = double(blocks) <= per_sm * double(ctx->n_sm) ? 1 : 0;
  }
  if (const char* v = std::getenv("PSG_SPECULATE")) speculate = std::atoi(v);  // dev knob: 0 off, 2 idle helper

  // ---- mixed-iteration table (psg_tables.cu mixtab_kernel) ----
  // Under contiguous batching a request is admitted by a mixed iteration
  // {its whole context, decode = B}.  For the entries whose serial chains
  // bound the search (longest replica groups), its cost is tabulated per
  // distinct context length and B < mt_w by a throughput kernel, so their
  // simulation warps read one row instead of pricing the iteration.
  std::vector<int64_t> mt_ctx, moff(std::max(E, 1), -1);
  std::vector<int32_t> t_crank, mt_ent;
  std::vector<double> mt_lam;
  double mt_gen = 0.0;
  int mt_w = 256;
  int64_t mt_bytes = 0, mt_T = 0, ct_bytes = 0;
  int mt_nq = 1;
  {
    int mode = 1;  // 0 off, 1 the entries within mt_frac of the longest chain, 2 every entry
    if (const char* v = std::getenv("PSG_MIXTAB")) mode = std::atoi(v);  // dev knob
    double frac = 0.75;
    if (const char* v = std::getenv("PSG_MIXTAB_FRAC")) frac = std::atof(v);  // dev knob
    if (const char* v = std::getenv("PSG_MIXTAB_W")) mt_w = std::max(1, std::atoi(v));  // dev knob
    // table memory: at most a quarter of the device memory free when the
    // context first tabulated (32 GB at most); queried once per context — a
    // driver query on every call stalls behind other driver clients
    if (ctx->mt_cap_bytes == 0) {
      size_t free_b = 0, total_b = 0;
      ctx->mt_cap_bytes = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess
                              ? std::min<int64_t>(int64_t(free_b / 4), int64_t(32) << 30)
                              : int64_t(8) << 30;
    }
    const int64_t cap_bytes = ctx->mt_cap_bytes;
    if (mode != 0 && cfg->batch_mode != PSG_BATCH_CHUNKED && !cfg->emit_iterations && E > 0 && N > 0) {
      int64_t wmax = 0;
      for (int e = 0; e < E; ++e) wmax = std::max(wmax, entry_work[e]);
      // curve slots of an entry: its collectives and (at most two, else
      // not tabulated) distinct p2p curves
      auto slots_of = [&](int e) {
        const int p = int(ent[e] / F);
        std::vector<int32_t> d;
        for (int b = P->p2p_begin[p]; b < P->p2p_begin[p + 1]; ++b)
          if (std::find(d.begin(), d.end(), p2p_tab[b]) == d.end()) d.push_back(p2p_tab[b]);
        return d.size() > 2 ? -1 : P->coll_begin[p + 1] - P->coll_begin[p] + int(d.size());
      };
      std::vector<int32_t> sel;
      for (int e = 0; e < E; ++e)
        if (!entry_missing[e] && (mode == 2 || double(entry_work[e]) >= frac * double(wmax)) &&
            slots_of(e) >= 0)
          sel.push_back(e);
      if (!sel.empty()) {
        // distinct context lengths: a dense rank map over [0, max] (one pass
        // each way) unless the lengths are sparse in a huge range
        std::vector<int32_t> dense;
        if (item_max < (int64_t(1) << 22) || item_max < 8 * N) {
          dense.assign(size_t(item_max) + 1, 0);
          for (int64_t i = 0; i < N; ++i) dense[size_t(T->context_len[i])] = 1;
          for (int64_t c = 0; c <= item_max; ++c)
            if (dense[size_t(c)]) {
              dense[size_t(c)] = int32_t(mt_ctx.size());
              mt_ctx.push_back(c);
            }
        } else {
          mt_ctx.assign(T->context_len, T->context_len + N);
          std::sort(mt_ctx.begin(), mt_ctx.end());
          mt_ctx.erase(std::unique(mt_ctx.begin(), mt_ctx.end()), mt_ctx.end());
        }
        const int64_t R = int64_t(mt_ctx.size());
        auto need = [&](size_t n) { return R * int64_t(mt_w) * 32 * int64_t(n); };
        if (need(sel.size()) > cap_bytes || sel.size() > 65535) {  // the longest chains first
          std::stable_sort(sel.begin(), sel.end(),
                           [&](int32_t a, int32_t b) { return entry_work[a] > entry_work[b]; });
          sel.resize(std::min<size_t>({sel.size(), size_t(cap_bytes / need(1)), 65535}));
        }
        // Worth it when the table costs (measured ~23 ps a row on B200) well
        // under what it saves the longest chain: ~1,500 cycles (0.76 us) per
        // mixed iteration priced on the serial path, about one per request —
        // all of them without speculation, ~30% with it (its misses).
        const double cost = 23e-12 * double(need(sel.size())) / 32.0;
        const double gain = 0.76e-6 * double(wmax) * (speculate == 1 ? 0.3 : 1.0);
        if (mode == 1 && !(cost < 0.5 * gain)) sel.clear();
        if (!sel.empty()) {
          t_crank.resize(N);
          if (!dense.empty()) {
            for (int64_t i = 0; i < N; ++i) t_crank[i] = dense[size_t(T->context_len[i])];
          } else {
            for (int64_t i = 0; i < N; ++i)
              t_crank[i] = int32_t(std::lower_bound(mt_ctx.begin(), mt_ctx.end(), T->context_len[i]) -
                                   mt_ctx.begin());
          }
          int64_t rows = 0;
          for (const int32_t e : sel) {
            moff[e] = rows;
            rows += R * mt_w;
          }
          mt_ent = sel;
          mt_bytes = rows * 32;
          // load test inputs (mixsel_kernel): arrival rate of each entry's
          // longest unit over the trace's arrival span, mean generation length
          double a0 = T->arrival[0], a1 = T->arrival[0], g = 0.0;
          for (int64_t i = 0; i < N; ++i) {
            a0 = std::min(a0, T->arrival[i]);
            a1 = std::max(a1, T->arrival[i]);
            g += double(std::max<int64_t>(T->gen_len[i], 1));
          }
          mt_gen = g / double(N);
          std::vector<int64_t> unit_max(E, 0);
          for (const auto& u : units) unit_max[u.entry] = std::max<int64_t>(unit_max[u.entry], u.n_req);
          for (const int32_t e : sel)
            mt_lam.push_back(a1 > a0 ? double(unit_max[e]) / (a1 - a0) : 0.0);
          for (const int32_t e : sel) mt_nq = std::max(mt_nq, slots_of(e));
          mt_T = mt_ctx.back() + mt_w;
          ct_bytes = (int64_t(sel.size()) * mt_T + 1) * mt_nq * 16;  // + one padding row
          if (host_timing)
            std::fprintf(stderr, "psg mixtab: %zu entries x %lld lengths x %d (%.1f MB, est %.2f ms vs %.2f ms)\n",
                         sel.size(), (long long)R, mt_w, double(mt_bytes) / 1e6, cost * 1e3, gain * 1e3);
        }
      }
    }
  }

  // curves staged per unit in shared memory up to 96 KB; a plan with larger
  // curves stages them in the unit's global region instead
  constexpr int64_t kTabSmemCap = 96 * 1024 / int64_t(sizeof(double));
  int64_t tab_cap = 1;
  for (int e = 0; e < E; ++e) tab_cap = std::max(tab_cap, plan_tab_need[ent[e] / F]);
  const int tab_smem = int(std::min(tab_cap, kTabSmemCap));
  int64_t gtab_total = 0;
  for (auto& u : units) {
    const int64_t need = plan_tab_need[u.plan];
    u.gtab = need > tab_smem ? gtab_total : -1;
    if (need > tab_smem) gtab_total += (need + 1) & ~int64_t(1);
  }

  host_mark(5);
  // ---- pack inputs ----
  Packer pk;
  const size_t o_model_dp = pk.add(P->model_dp, np), o_stages = pk.add(P->num_stages, np),
               o_sdev = pk.add(P->stage_devices, np), o_reps = pk.add(P->stage_repetitions, np),
               o_dtype = pk.add(P->compute_dtype, np), o_enc = pk.add(P->enc_rank, np),
               o_kv = pk.add(P->kv_bytes_per_token, np), o_budget = pk.add(P->kv_budget_per_replica, np),
               o_p2pppt = pk.add(P->p2p_payload_per_token, np), o_hid = pk.add(P->shape_hidden, np),
               o_head = pk.add(P->shape_head_dim, np), o_kve = pk.add(P->shape_kv_elems, np),
               o_cb = pk.add(P->cell_begin, np + 1), o_cop = pk.add(P->cell_op, n_cells),
               o_ct = pk.add(P->cell_tasks, n_cells), o_cw = pk.add(P->cell_width, n_cells),
               o_cs = pk.add(P->cell_token_scale, n_cells), o_kb = pk.add(P->coll_begin, np + 1),
               o_kk = pk.add(P->coll_kind, n_colls), o_kd = pk.add(P->coll_devices, n_colls),
               o_kn = pk.add(P->coll_nodes, n_colls), o_kg = pk.add(P->coll_groups, n_colls),
               o_kp = pk.add(P->coll_ppt, n_colls), o_ksh = pk.add(P->coll_share, n_colls),
               o_pb = pk.add(P->p2p_begin, np + 1), o_pn = pk.add(P->p2p_nodes, n_p2p);
  int64_t n_knots = 0, n_vals = 0, n_kpts = 0;
  for (int t = 0; t < S->n_compute; ++t) {
    n_knots = std::max<int64_t>(n_knots, S->c_knot_begin[t] + S->c_n_ctx[t] + S->c_n_tasks[t] + S->c_n_width[t]);
    n_vals = std::max<int64_t>(n_vals, S->c_value_begin[t] + int64_t(S->c_n_ctx[t]) * S->c_n_tasks[t] * S->c_n_width[t]);
  }
  for (int u = 0; u < S->n_curves; ++u) n_kpts = std::max<int64_t>(n_kpts, S->k_begin[u] + S->k_n[u]);
  const size_t o_snc = pk.add(S->c_n_ctx, S->n_compute), o_snt = pk.add(S->c_n_tasks, S->n_compute),
               o_snw = pk.add(S->c_n_width, S->n_compute), o_skb = pk.add(S->c_knot_begin, S->n_compute),
               o_svb = pk.add(S->c_value_begin, S->n_compute), o_sk = pk.add(S->c_knots, n_knots),
               o_ss = pk.add(S->c_seconds, n_vals), o_sj = pk.add(S->c_joules, n_vals),
               o_kn2 = pk.add(S->k_n, S->n_curves), o_kbeg = pk.add(S->k_begin, S->n_curves),
               o_kpay = pk.add(S->k_payload, n_kpts), o_ksec = pk.add(S->k_seconds, n_kpts),
               o_kjou = pk.add(S->k_joules, n_kpts);
  const size_t o_tctx = pk.add(T->context_len, N), o_tgen = pk.add(T->gen_len, N),
               o_tarr = pk.add(T->arrival, N), o_tslot = pk.add(slot.data(), N),
               o_tseq = pk.add(seq.data(), seq.size()), o_sid = pk.add(slot_id.data(), N),
               o_sgen = pk.add(slot_gen.data(), N);
  const size_t o_freqs = pk.add(freqs.data(), freqs.size()),
               o_celltab = pk.add(cell_tab.data(), cell_tab.size()),
               o_colltab = pk.add(coll_tab.data(), coll_tab.size()),
               o_p2ptab = pk.add(p2p_tab.data(), p2p_tab.size()),
               o_bslot = pk.add(bslot.data(), bslot.size()),
               o_emiss = pk.add(entry_missing.data(), E),
               o_units = pk.add(units.data(), units.size()),
               o_eub = pk.add(entry_unit_begin.data(), E + 1),
               o_eu = pk.add(entry_units.data(), entry_units.size()),
               o_bk0 = pk.add(block_k0.data(), block_k0.size()),
               o_bk1 = pk.add(block_k1.data(), block_k1.size()),
               o_egr = pk.add(entry_groups.data(), entry_groups.size()),
               o_xpr = pk.add(exp_pr.data(), exp_pr.size()),
               o_xpo = pk.add(pr_off0.data(), pr_off0.size()),
               o_xro = pk.add(rj_off0.data(), rj_off0.size()),
               o_epeak = pk.add(entry_peak.data(), E), o_eenc = pk.add(entry_enc.data(), E),
               o_efreq = pk.add(entry_freq.data(), E), o_eglob = pk.add(ent.data(), E);
  const size_t o_pmb = cfg->entry_max_batch_size ? pk.add(cfg->entry_max_batch_size, size_t(E)) : 0;
  const size_t o_sgt = pk.add(sig_table.data(), sig_table.size()),
               o_sgo = pk.add(sig_op.data(), sig_op.size()),
               o_sgs = pk.add(sig_scale.data(), sig_scale.size()),
               o_sgk = pk.add(sig_tasks.data(), sig_tasks.size()),
               o_sgw = pk.add(sig_width.data(), sig_width.size()),
               o_sgh = pk.add(sig_hidden.data(), sig_hidden.size()),
               o_sghd = pk.add(sig_head.data(), sig_head.size()),
               o_sgkv = pk.add(sig_kv.data(), sig_kv.size()),
               o_sgr = pk.add(sig_rows.data(), sig_rows.size()), o_qoff = pk.add(qoff.data(), qoff.size()),
               o_csig = pk.add(cell_sig.data(), cell_sig.size()),
               o_eplan = pk.add(ent_plan.data(), ent_plan.size()),
               o_efs = pk.add(ent_fslot.data(), ent_fslot.size()),
               o_erows = pk.add(ent_rows.data(), ent_rows.size()),
               o_doff = pk.add(doff.data(), doff.size());
  const size_t o_crank = pk.add(t_crank.data(), t_crank.size()),
               o_mctx = pk.add(mt_ctx.data(), mt_ctx.size()),
               o_ment = pk.add(mt_ent.data(), mt_ent.size()),
               o_moff = pk.add(moff.data(), moff.size()),
               o_mlam = pk.add(mt_lam.data(), mt_lam.size());
  const size_t in_bytes = pk.size;

  host_mark(6);
  // ---- device buffers ----
  const size_t slots = size_t(E) * size_t(N);
  PSG_CUDA(ctx->d_in.ensure(in_bytes));
  PSG_CUDA(ctx->h_in.ensure(in_bytes));
  PSG_CUDA(ctx->d_slot_f64.ensure(std::max<size_t>(slots, 1) * 3 * sizeof(double)));
  PSG_CUDA(ctx->d_slot_u8.ensure(std::max<size_t>(slots, 1)));
  PSG_CUDA(ctx->d_scratch_i32.ensure(std::max<int64_t>(scratch_total, 1) * kScratchI32 * sizeof(int32_t)));
  PSG_CUDA(ctx->d_scratch_f64.ensure(std::max<int64_t>(scratch_total, 1) * kScratchF64 * sizeof(double)));
  // chunk minima once a unit's slots migrate: unit k uses [S_k/32 + 2k, +n_req/32 + 2)
  PSG_CUDA(ctx->d_scratch_cm.ensure((scratch_total / 32 + 2 * int64_t(n_units) + 2) * sizeof(int64_t)));
  PSG_CUDA(ctx->d_qtab.ensure(size_t(std::max<int64_t>(qrows, 1)) * 4 * sizeof(double)));
  PSG_CUDA(ctx->d_dtab.ensure(size_t(std::max<int64_t>(drows, 1)) * 4 * sizeof(double)));
  if (mt_bytes > 0) {
    // the tables are an optimization: without the memory, search without them
    if (ctx->d_mtab.ensure(size_t(mt_bytes)) != cudaSuccess ||
        ctx->d_ctab.ensure(size_t(ct_bytes)) != cudaSuccess) {
      cudaGetLastError();
      ctx->d_mtab.release();
      ctx->d_ctab.release();
      std::fill(moff.begin(), moff.end(), int64_t(-1));
      mt_bytes = ct_bytes = 0;
    }
  }
  // work: uout, eout, keys, order, pr_off, rj_off, totals, clamp flags
  Packer wk;  // offsets only
  const size_t w_uout = wk.add<UnitOut>(nullptr, n_units), w_eout = wk.add<EntryOut>(nullptr, E),
               w_keys = wk.add<psg_rank_key>(nullptr, E), w_order = wk.add<int64_t>(nullptr, E),
               w_proff = wk.add<int64_t>(nullptr, E), w_rjoff = wk.add<int64_t>(nullptr, E),
               w_tot = wk.add<int64_t>(nullptr, 2), w_cc = wk.add<uint32_t>(nullptr, S->n_compute),
               w_kc = wk.add<uint32_t>(nullptr, S->n_curves),
               w_ok = wk.add<int32_t>(nullptr, E);
  PSG_CUDA(ctx->d_work.ensure(wk.size + 64));
  PSG_CUDA(ctx->h_out.ensure(wk.size + 64));

  unsigned char* hin = static_cast<unsigned char*>(ctx->h_in.p);
  pk.write(hin);
  unsigned char* din = static_cast<unsigned char*>(ctx->d_in.p);
  unsigned char* dw = static_cast<unsigned char*>(ctx->d_work.p);
  auto D = [&](size_t off) { return static_cast<void*>(din + off); };
  auto W = [&](size_t off) { return static_cast<void*>(dw + off); };

  SimParams sp{};
  sp.P = DPlans{np,
                (const int32_t*)D(o_model_dp), (const int32_t*)D(o_stages), (const int32_t*)D(o_sdev),
                (const int32_t*)D(o_reps), (const int32_t*)D(o_dtype), (const int32_t*)D(o_enc),
                (const double*)D(o_kv), (const double*)D(o_budget), (const double*)D(o_p2pppt),
                (const double*)D(o_hid), (const double*)D(o_head), (const double*)D(o_kve),
                (const int32_t*)D(o_cb), (const int32_t*)D(o_cop), (const double*)D(o_ct),
                (const double*)D(o_cw), (const double*)D(o_cs), (const int32_t*)D(o_kb),
                (const int32_t*)D(o_kk), (const int32_t*)D(o_kd), (const int32_t*)D(o_kn),
                (const int32_t*)D(o_kg), (const double*)D(o_kp), (const double*)D(o_ksh),
                (const int32_t*)D(o_pb), (const int32_t*)D(o_pn)};
  sp.S = DStore{(const int32_t*)D(o_snc), (const int32_t*)D(o_snt), (const int32_t*)D(o_snw),
                (const int64_t*)D(o_skb), (const int64_t*)D(o_svb), (const double*)D(o_sk),
                (const double*)D(o_ss), (const double*)D(o_sj), (const int32_t*)D(o_kn2),
                (const int64_t*)D(o_kbeg), (const double*)D(o_kpay), (const double*)D(o_ksec),
                (const double*)D(o_kjou)};
  sp.T = DTrace{N, (const int64_t*)D(o_tctx), (const int64_t*)D(o_tgen), (const double*)D(o_tarr),
                (const int32_t*)D(o_tslot), sorted ? nullptr : (const int32_t*)D(o_tseq)};
  sp.freqs = (const double*)D(o_freqs);
  sp.cell_tab = (const int32_t*)D(o_celltab);
  sp.coll_tab = (const int32_t*)D(o_colltab);
  sp.p2p_tab = (const int32_t*)D(o_p2ptab);
  sp.p2p_bslot = (const uint8_t*)D(o_bslot);
  PSG_CUDA(ctx->d_gtab.ensure(size_t(std::max<int64_t>(gtab_total, 1)) * sizeof(double)));
  sp.g_tab = static_cast<double*>(ctx->d_gtab.p);
  sp.entry_missing = (const int32_t*)D(o_emiss);
  sp.n_cells_total = n_cells;
  sp.units = (const Unit*)D(o_units);
  sp.entry_max_bs = cfg->entry_max_batch_size ? (const int64_t*)D(o_pmb) : nullptr;
  sp.emit_it = nullptr;
  sp.emit_sec = sp.emit_jou = nullptr;
  sp.emit_off = nullptr;
  sp.emit_S = 0;
  sp.n_units = n_units;
  sp.batch_mode = cfg->batch_mode;
  sp.chunk_size = cfg->chunk_size;
  sp.max_batch_size = cfg->max_batch_size;
  sp.anchor = cfg->ttft_anchor;
  sp.memo_cap = 256;
  sp.tab_smem = tab_smem;
  sp.chain_replicas = chain;
  sp.speculate = speculate;
  sp.spec_sleep_ns = 20;
  if (const char* v = std::getenv("PSG_SPEC_SLEEP_NS")) sp.spec_sleep_ns = std::max(0, std::atoi(v));  // dev knob
  {
    // Active slots live in shared memory while they fit: give each unit as
    // many as keeps every unit resident in one wave (the kernel's time is its
    // longest unit), at least 256, at most the largest unit's request count.
    int64_t max_nr = 0;
    for (const auto& u : units) max_nr = std::max<int64_t>(max_nr, u.n_req);
    const int64_t want = std::max<int64_t>(256, (max_nr + 31) / 32 * 32);
    const int blocks = std::max(sim_blocks, chain == 2 ? ctx->concurrent_groups : ctx->concurrent_blocks);
    const int per_sm = std::max(1, (blocks + ctx->n_sm - 1) / std::max(ctx->n_sm, 1));
    const int64_t budget = std::min<int64_t>(ctx->smem_block_max, ctx->smem_sm / per_sm - 1024) -
                           ctx->sim_static_smem;
    int64_t cap = 256;
    for (int64_t c = want; c > 256; c -= 32) {
      const int64_t l2 = (std::max<int64_t>(c, max_nr) + 1023) / 1024 + 1;
      if (int64_t(sim_smem_bytes(int(c), sp.memo_cap, tab_smem, int(l2))) <= budget) {
        cap = c;
        break;
      }
    }
    sp.smem_cap = int(cap);
    if (const char* v = std::getenv("PSG_SMEM_CAP"))  // dev knob
      sp.smem_cap = int(std::max<int64_t>(256, std::min<int64_t>(std::atoi(v), cap)) / 32 * 32);
  }
  sp.serial_run = 96;  // (C1 -12%, C4 -1%, C2 / C5 within noise vs 128; measured)
  if (const char* v = std::getenv("PSG_SERIAL_RUN")) sp.serial_run = std::max(1, std::atoi(v));  // dev knob
  {
    int64_t max_len = sp.smem_cap;  // active slots never exceed max(smem_cap, n_req)
    for (const auto& u : units) max_len = std::max<int64_t>(max_len, u.n_req);
    sp.cm2_cap = int((max_len + 1023) / 1024 + 1);
  }
  sp.cell_sig = (const int32_t*)D(o_csig);
  sp.qtab = static_cast<const double*>(ctx->d_qtab.p);
  sp.qoff = (const int64_t*)D(o_qoff);
  sp.dectab = static_cast<const double*>(ctx->d_dtab.p);
  sp.doff = (const int64_t*)D(o_doff);
  sp.mixtab = mt_bytes > 0 ? static_cast<const double*>(ctx->d_mtab.p) : nullptr;
  sp.moff = (const int64_t*)D(o_moff);
  sp.t_crank = mt_bytes > 0 ? (const int32_t*)D(o_crank) : nullptr;
  sp.mt_w = mt_w;

  TabParams tp{};
  tp.P = sp.P;
  tp.S = sp.S;
  tp.n_sig = n_sig;
  tp.sig_table = (const int32_t*)D(o_sgt);
  tp.sig_op = (const int32_t*)D(o_sgo);
  tp.sig_scale = (const double*)D(o_sgs);
  tp.sig_tasks = (const double*)D(o_sgk);
  tp.sig_width = (const double*)D(o_sgw);
  tp.sig_hidden = (const double*)D(o_sgh);
  tp.sig_head = (const double*)D(o_sghd);
  tp.sig_kv = (const double*)D(o_sgkv);
  tp.sig_rows = (const int64_t*)D(o_sgr);
  tp.qoff = sp.qoff;
  tp.qtab = static_cast<double*>(ctx->d_qtab.p);
  tp.n_entries = E;
  tp.ent_plan = (const int32_t*)D(o_eplan);
  tp.ent_fslot = (const int32_t*)D(o_efs);
  tp.ent_rows = (const int64_t*)D(o_erows);
  tp.doff = sp.doff;
  tp.cell_sig = sp.cell_sig;
  tp.n_cells_total = n_cells;
  tp.coll_tab = sp.coll_tab;
  tp.p2p_tab = sp.p2p_tab;
  tp.entry_missing = sp.entry_missing;
  tp.dectab = static_cast<double*>(ctx->d_dtab.p);
  tp.n_mt = int32_t(mt_ent.size());
  tp.mt_w = mt_w;
  tp.mt_R = int64_t(mt_ctx.size());
  tp.mt_ent = (const int32_t*)D(o_ment);
  tp.mt_ctx = (const int64_t*)D(o_mctx);
  tp.moff = sp.moff;
  tp.mixtab = static_cast<double*>(ctx->d_mtab.p);
  tp.mt_T = mt_T;
  tp.mt_nq = mt_nq;
  tp.ctab = static_cast<double*>(ctx->d_ctab.p);
  tp.mt_lam = (const double*)D(o_mlam);
  tp.mt_gen = mt_gen;
  tp.moff_rw = (int64_t*)D(o_moff);
  sp.n_slots = N;
  sp.uout = (UnitOut*)W(w_uout);
  double* slot_f = static_cast<double*>(ctx->d_slot_f64.p);
  sp.slot_ttft = slot_f;
  sp.slot_tpot = slot_f + slots;
  sp.slot_e2e = slot_f + 2 * slots;
  sp.slot_status = static_cast<uint8_t*>(ctx->d_slot_u8.p);
  sp.clamp_compute = (uint32_t*)W(w_cc);
  sp.clamp_curve = (uint32_t*)W(w_kc);
  sp.prof = nullptr;
  const char* prof_path = std::getenv("PSG_PHASE_PROFILE");
  if (prof_path && !*prof_path) prof_path = nullptr;
  if (prof_path) {  // dev builds: per-unit phase counters dumped after the run
    PSG_CUDA(ctx->d_prof.ensure(sizeof(unsigned long long) * kProfSlots * std::max(n_units, 1)));
    PSG_CUDA(cudaMemsetAsync(ctx->d_prof.p, 0, sizeof(unsigned long long) * kProfSlots * std::max(n_units, 1), ctx->stream));
    sp.prof = static_cast<unsigned long long*>(ctx->d_prof.p);
  }
  sp.g_i32 = static_cast<int32_t*>(ctx->d_scratch_i32.p);
  sp.g_f64 = static_cast<double*>(ctx->d_scratch_f64.p);
  sp.g_cm = static_cast<int64_t*>(ctx->d_scratch_cm.p);
  if (stream) {  // the result arrays, pinned and mapped, sized before the launch
    PSG_CUDA(ctx->h_pr.ensure(std::max<int64_t>(tot_pr0, 1) * sizeof(psg_request_metrics)));
    PSG_CUDA(ctx->h_rj.ensure(std::max<int64_t>(tot_rj0, 1) * sizeof(int64_t)));
    void *dpr = nullptr, *drj = nullptr;
    if (cudaHostGetDevicePointer(&dpr, ctx->h_pr.p, 0) == cudaSuccess &&
        cudaHostGetDevicePointer(&drj, ctx->h_rj.p, 0) == cudaSuccess) {
      sp.out_pr = static_cast<psg_request_metrics*>(dpr);
      sp.out_rj = static_cast<int64_t*>(drj);
      sp.out_n_pr = (const int64_t*)D(o_xpr);
      sp.out_pr_off = (const int64_t*)D(o_xpo);
      sp.out_rj_off = (const int64_t*)D(o_xro);
      sp.out_ok = (int32_t*)W(w_ok);
      sp.slot_id = (const int64_t*)D(o_sid);
      sp.slot_gen = (const int64_t*)D(o_sgen);
    } else {
      cudaGetLastError();
      stream = false;
    }
  }
  if (chain == 2) {
    PSG_CUDA(ctx->d_rlog.ensure(size_t(std::max<int64_t>(rlog_total, 1)) * sizeof(double2)));
    PSG_CUDA(ctx->d_edone.ensure(size_t(std::max(E, 1)) * sizeof(int32_t)));
    sp.rlog = static_cast<double2*>(ctx->d_rlog.p);
    sp.entry_done = static_cast<int32_t*>(ctx->d_edone.p);
    sp.block_k0 = (const int32_t*)D(o_bk0);
    sp.block_k1 = (const int32_t*)D(o_bk1);
    sp.entry_groups = (const int32_t*)D(o_egr);
  }

  ReduceParams rp{};
  rp.n_slots = N;
  rp.slot_status = sp.slot_status;
  rp.slot_ttft = sp.slot_ttft;
  rp.slot_tpot = sp.slot_tpot;
  rp.slot_e2e = sp.slot_e2e;
  rp.slot_gen = (const int64_t*)D(o_sgen);
  rp.slot_id = (const int64_t*)D(o_sid);
  rp.uout = sp.uout;
  rp.entry_unit_begin = (const int32_t*)D(o_eub);
  rp.entry_units = (const int32_t*)D(o_eu);
  rp.entry_peak = (const double*)D(o_epeak);
  rp.entry_enc_rank = (const int32_t*)D(o_eenc);
  rp.entry_freq = (const double*)D(o_efreq);
  rp.entry_global = (const int64_t*)D(o_eglob);
  rp.mem_bw = cl->peak_mem_bandwidth;
  rp.total_devices = cl->total_devices;
  rp.objective = cfg->objective;
  rp.extras = 1;
  rp.ttft_slo = cfg->ttft_slo > 0.0 ? cfg->ttft_slo : 0.0;
  rp.slo_quantile = cfg->slo_quantile > 0.0 ? cfg->slo_quantile : 0.99;
  rp.chain_replicas = sp.chain_replicas;
  rp.cand_cap = kReduceCandCap;
  if (const char* v = std::getenv("PSG_REDUCE_CANDIDATES")) rp.cand_cap = std::max(0, std::min(kReduceCandCap, std::atoi(v)));  // dev knob
  sp.entry_unit_begin = rp.entry_unit_begin;
  sp.entry_units = rp.entry_units;
  rp.eout = (EntryOut*)W(w_eout);
  rp.keys = (psg_rank_key*)W(w_keys);

  cudaStream_t st = ctx->stream;
  int64_t launches = 0;
  PSG_CUDA(cudaEventRecord(ctx->ev[0], st));
  PSG_CUDA(cudaMemcpyAsync(din, hin, in_bytes, cudaMemcpyHostToDevice, st));
  PSG_CUDA(cudaMemsetAsync(sp.slot_status, 0, std::max<size_t>(slots, 1), st));
  PSG_CUDA(cudaMemsetAsync(W(w_cc), 0, wk.size - w_cc, st));
  PSG_CUDA(cudaEventRecord(ctx->ev[1], st));
  if (ctx->gate && !ctx->gate_passed) {
    ctx->gate_passed = true;
    ctx->gate->arrive(true);
  }
  const size_t smem = sim_smem_bytes(sp.smem_cap, sp.memo_cap, sp.tab_smem, sp.cm2_cap);
  if (prof_path) std::fprintf(stderr, "psg: units=%d smem_cap=%d smem=%zu B\n", n_units, sp.smem_cap, smem);
  if (n_sig > 0) {  // cell-query tables, then decode-only iteration tables
    // grid.y covers the longest table (row loops in the kernels beyond 65535 x 256)
    qtab_kernel<<<dim3(unsigned(n_sig), unsigned(std::min<int64_t>((max_qrows + 255) / 256, 65535))),
                  256, 0, st>>>(tp);
    ++launches;
  }
  if (E > 0) {
    dectab_kernel<<<dim3(unsigned(E), unsigned(std::min<int64_t>((max_drows + 255) / 256, 65535))),
                    256, 0, st>>>(tp);
    ++launches;
  }
  if (mt_bytes > 0) {  // mixed-iteration rows (read the cell-query and curve-value tables)
    const char* ms = std::getenv("PSG_MIXSEL");  // dev knob
    const bool mixsel = !ms || std::atoi(ms) != 0;
    if (mixsel) {
      mixsel_kernel<<<unsigned((tp.n_mt + 127) / 128), 128, 0, st>>>(tp);
      ++launches;
    }
    colltab_kernel<<<dim3(unsigned(tp.n_mt), unsigned(std::min<int64_t>((mt_T + 255) / 256, 65535))),
                     256, 0, st>>>(tp);
    mixtab_kernel<<<dim3(unsigned(std::min<int64_t>(tp.mt_R, 65535)), unsigned(tp.n_mt)),
                    unsigned(std::min(mt_w, 256)), 0, st>>>(tp);
    ++launches;
  }
  if (n_units > 0) {
    if (chain == 2) PSG_CUDA(cudaMemsetAsync(sp.entry_done, 0, size_t(E) * sizeof(int32_t), st));
    launch_sim(sim_blocks, smem, st, sp);
    ++launches;
    PSG_CUDA(cudaGetLastError());
  }
  int64_t n_emit = 0;
  int emit_S = 0;
  if (cfg->emit_iterations && n_units > 0) {
    // Second pass without macro-stepping, one record per iteration; the
    // first pass sized the log exactly (per-unit iteration counts).
    std::vector<UnitOut> uo(n_units);
    PSG_CUDA(cudaMemcpyAsync(uo.data(), sp.uout, n_units * sizeof(UnitOut), cudaMemcpyDeviceToHost, st));
    PSG_CUDA(cudaStreamSynchronize(st));
    bool failed = false;
    for (const UnitOut& u : uo) failed |= u.err != 0;
    if (!failed) {
      std::vector<int64_t> off(n_units, 0);
      for (int k = entry_unit_begin[0]; k < entry_unit_begin[1]; ++k) {  // replica order
        off[entry_units[k]] = n_emit;
        n_emit += uo[entry_units[k]].iterations;
      }
      emit_S = P->num_stages[ent[0] / F];
      const int64_t nr = std::max<int64_t>(n_emit, 1);
      PSG_CUDA(ctx->d_it.ensure(nr * sizeof(psg_iteration)));
      PSG_CUDA(ctx->d_isec.ensure(nr * emit_S * sizeof(double)));
      PSG_CUDA(ctx->d_ijou.ensure(nr * emit_S * sizeof(double)));
      PSG_CUDA(ctx->d_ioff.ensure(n_units * sizeof(int64_t)));
      PSG_CUDA(cudaMemcpyAsync(ctx->d_ioff.p, off.data(), n_units * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      sp.emit_it = static_cast<psg_iteration*>(ctx->d_it.p);
      sp.emit_sec = static_cast<double*>(ctx->d_isec.p);
      sp.emit_jou = static_cast<double*>(ctx->d_ijou.p);
      sp.emit_off = static_cast<const int64_t*>(ctx->d_ioff.p);
      sp.emit_S = emit_S;
      launch_sim(sim_blocks, smem, st, sp);
      ++launches;
      PSG_CUDA(cudaGetLastError());
      // the stepwise pass is a replay: the first pass's outputs are rewritten bit-identically
      PSG_CUDA(cudaStreamSynchronize(st));
      PSG_CUDA(cudaMemcpyAsync(uo.data(), sp.uout, n_units * sizeof(UnitOut), cudaMemcpyDeviceToHost, st));
      PSG_CUDA(cudaStreamSynchronize(st));
      int64_t n2 = 0;
      for (const UnitOut& u : uo) n2 += u.iterations;
      if (n2 != n_emit) return fail(ctx, PSG_ERR_CUDA, "iteration log: replay diverged");
    }
  }
  PSG_CUDA(cudaEventRecord(ctx->ev[2], st));
  entry_reduce_kernel<<<E, kReduceThreads, size_t(rp.cand_cap) * kReduceStats * sizeof(uint64_t), st>>>(rp);
  offsets_kernel<<<1, 32, 0, st>>>(rp.eout, E, (int64_t*)W(w_proff), (int64_t*)W(w_rjoff),
                                   (int64_t*)W(w_tot));
  launches += 2;
  if (cfg->rank) {
    rank_kernel<<<unsigned((E + 255) / 256), 256, 0, st>>>(rp.keys, E, (int64_t*)W(w_order));
    ++launches;
  }
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cudaEventRecord(ctx->ev[3], st));
  // everything from uout onwards is small: one D2H
  PSG_CUDA(cudaMemcpyAsync(ctx->h_out.p, dw, wk.size, cudaMemcpyDeviceToHost, st));
  PSG_CUDA(cudaEventRecord(ctx->ev[4], st));
  PSG_CUDA(cudaStreamSynchronize(st));
  const unsigned char* ho = static_cast<const unsigned char*>(ctx->h_out.p);
  auto H = [&](size_t off) { return ho + off; };
  const auto* eo = reinterpret_cast<const EntryOut*>(H(w_eout));
  const auto* order = reinterpret_cast<const int64_t*>(H(w_order));
  const auto* tot = reinterpret_cast<const int64_t*>(H(w_tot));
  const auto* proff = reinterpret_cast<const int64_t*>(H(w_proff));
  const auto* rjoff = reinterpret_cast<const int64_t*>(H(w_rjoff));

  host_mark(7);
  // ---- errors: the lowest global entry index that failed (jobs=1 order) ----
  {
    int64_t worst = INT64_MAX;
    int we = -1;
    for (int e = 0; e < E; ++e)
      if (eo[e].err && ent[e] < worst) {
        worst = ent[e];
        we = e;
      }
    for (int e = 0; e < E; ++e)
      if (eo[e].err == 9) {  // a replica's tally log overflowed (evictions): rerun chained
        ctx->chain_fallback = true;
        const int rc = search_impl(ctx, P, cl, S, T, cfg, out);
        ctx->chain_fallback = false;
        return rc;
      }
    if (we >= 0) {
      const int code = eo[we].err;
      if (code == 1) return fail(ctx, PSG_ERR_DATA, "chunked prefill requires chunk_size >= 1");
      if (code == 2) return fail(ctx, PSG_ERR_DATA, missing_msg[we]);
      const int p = int(ent[we] / F);
      return fail(ctx, PSG_ERR_DATA, std::string("device has no peak_flops entry for dtype ") +
                                         dtype_name(P->compute_dtype[p]));
    }
  }

  // ---- per-request arrays ----
  const int64_t n_pr = cfg->detail ? tot[0] : 0, n_rj = cfg->detail ? tot[1] : 0;
  bool streamed = stream && n_pr == tot_pr0 && n_rj == tot_rj0;
  if (streamed) {  // every entry wrote its records during the simulation
    const auto* okf = reinterpret_cast<const int32_t*>(H(w_ok));
    for (int e = 0; e < E && streamed; ++e) streamed = okf[e] == 1 && eo[e].completed == exp_pr[e];
  }
  PSG_CUDA(cudaEventRecord(ctx->ev[5], st));
  if (cfg->detail && !streamed) {
    PSG_CUDA(ctx->d_pr.ensure(std::max<int64_t>(n_pr, 1) * sizeof(psg_request_metrics)));
    PSG_CUDA(ctx->d_rj.ensure(std::max<int64_t>(n_rj, 1) * sizeof(int64_t)));
    PSG_CUDA(ctx->h_pr.ensure(std::max<int64_t>(n_pr, 1) * sizeof(psg_request_metrics)));
    PSG_CUDA(ctx->h_rj.ensure(std::max<int64_t>(n_rj, 1) * sizeof(int64_t)));
    compact_kernel<<<E, 256, 0, st>>>(rp, (const int64_t*)W(w_proff), (const int64_t*)W(w_rjoff),
                                      static_cast<psg_request_metrics*>(ctx->d_pr.p),
                                      static_cast<int64_t*>(ctx->d_rj.p));
    ++launches;
    PSG_CUDA(cudaGetLastError());
  }
  PSG_CUDA(cudaEventRecord(ctx->ev[6], st));
  if (cfg->detail && !streamed) {
    if (n_pr)
      PSG_CUDA(cudaMemcpyAsync(ctx->h_pr.p, ctx->d_pr.p, n_pr * sizeof(psg_request_metrics),
                               cudaMemcpyDeviceToHost, st));
    if (n_rj)
      PSG_CUDA(cudaMemcpyAsync(ctx->h_rj.p, ctx->d_rj.p, n_rj * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
  }
  if (n_emit > 0) {
    PSG_CUDA(ctx->h_it.ensure(n_emit * sizeof(psg_iteration)));
    PSG_CUDA(ctx->h_isec.ensure(n_emit * emit_S * sizeof(double)));
    PSG_CUDA(ctx->h_ijou.ensure(n_emit * emit_S * sizeof(double)));
    PSG_CUDA(cudaMemcpyAsync(ctx->h_it.p, ctx->d_it.p, n_emit * sizeof(psg_iteration), cudaMemcpyDeviceToHost, st));
    PSG_CUDA(cudaMemcpyAsync(ctx->h_isec.p, ctx->d_isec.p, n_emit * emit_S * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    PSG_CUDA(cudaMemcpyAsync(ctx->h_ijou.p, ctx->d_ijou.p, n_emit * emit_S * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
  }
  PSG_CUDA(cudaEventRecord(ctx->ev[7], st));
  PSG_CUDA(cudaStreamSynchronize(st));

  if (prof_path) {
    std::vector<unsigned long long> pr(size_t(kProfSlots) * n_units);
    cudaMemcpy(pr.data(), ctx->d_prof.p, pr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(prof_path, "wb")) {
      for (int u = 0; u < n_units; ++u) {  // unit -> (global entry, replica, counters)
        const long long meta[2] = {(long long)ent[units[u].entry], (long long)units[u].replica};
        std::fwrite(meta, sizeof meta, 1, f);
        std::fwrite(pr.data() + size_t(u) * kProfSlots, sizeof(unsigned long long), kProfSlots, f);
      }
      std::fclose(f);
    }
  }
  host_mark(8);
  // ---- assemble result ----
  ctx->entries.resize(E);
  for (int k = 0; k < E; ++k) {
    const int e = cfg->rank ? int(order[k]) : k;
    const EntryOut& o = eo[e];
    psg_entry& r = ctx->entries[k];
    r.entry_index = ent[e];
    r.plan_index = ent[e] / F;
    r.freq_ghz = freqs[ent[e] % F];
    r.e2e_latency = o.e2e;
    r.total_energy = o.energy;
    r.p95_latency = o.p95;
    r.mean_ttft = o.mean_ttft;
    r.mean_tpot = o.mean_tpot;
    r.mfu = o.mfu;
    r.mbu = o.mbu;
    r.num_completed = o.completed;
    r.num_rejected = o.rejected;
    r.num_iterations = o.iterations;
    r.max_batch_observed = o.max_batch;
    r.p50_ttft = o.p50_ttft;
    r.p99_ttft = o.p99_ttft;
    r.p50_tpot = o.p50_tpot;
    r.p99_tpot = o.p99_tpot;
    r.slo_ttft = o.slo_ttft;
    r.slo_met = rp.ttft_slo > 0.0 && o.completed > 0 && o.slo_ttft <= rp.ttft_slo ? 1 : 0;
    r.per_request_offset = cfg->detail ? proff[e] : 0;
    r.rejected_offset = cfg->detail ? rjoff[e] : 0;
  }
  const auto* cc = reinterpret_cast<const uint32_t*>(H(w_cc));
  const auto* kc = reinterpret_cast<const uint32_t*>(H(w_kc));
  ctx->compute_clamp.assign(cc, cc + S->n_compute);
  ctx->curve_clamp.assign(kc, kc + S->n_curves);

  auto* res = new psg_result();
  res->n_entries = E;
  res->entries = ctx->entries.data();
  res->n_per_request = n_pr;
  res->per_request = static_cast<psg_request_metrics*>(ctx->h_pr.p);
  res->n_rejected = n_rj;
  res->rejected_ids = static_cast<int64_t*>(ctx->h_rj.p);
  res->n_compute = S->n_compute;
  res->compute_clamp = ctx->compute_clamp.data();
  res->n_curves = S->n_curves;
  res->curve_clamp = ctx->curve_clamp.data();
  res->gpu_launches = launches;
  int64_t iters = 0, sb = 0, adm = 0, fin = 0;
  for (int e = 0; e < E; ++e) {
    iters += eo[e].iterations;
    sb += eo[e].sum_batch;
    adm += eo[e].admissions;
    fin += eo[e].completed;
  }
  res->total_iterations = iters;
  res->sum_batch = sb;
  res->admissions = adm;
  res->finishes = fin;
  res->n_iterations = n_emit;
  res->iterations = n_emit ? static_cast<psg_iteration*>(ctx->h_it.p) : nullptr;
  res->n_stages = emit_S;
  res->stage_seconds = n_emit ? static_cast<double*>(ctx->h_isec.p) : nullptr;
  res->stage_joules = n_emit ? static_cast<double*>(ctx->h_ijou.p) : nullptr;
  res->h2d_bytes = int64_t(in_bytes);
  res->d2h_bytes = int64_t(wk.size) + n_pr * int64_t(sizeof(psg_request_metrics)) +
                   n_rj * int64_t(sizeof(int64_t)) +
                   n_emit * int64_t(sizeof(psg_iteration) + 2 * sizeof(double) * emit_S);
  float a = 0, b = 0;
  cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
  res->ms_h2d = a;
  cudaEventElapsedTime(&a, ctx->ev[1], ctx->ev[2]);
  res->ms_sim = a;
  cudaEventElapsedTime(&a, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&b, ctx->ev[5], ctx->ev[6]);
  res->ms_reduce = double(a) + double(b);
  cudaEventElapsedTime(&a, ctx->ev[3], ctx->ev[4]);
  cudaEventElapsedTime(&b, ctx->ev[6], ctx->ev[7]);
  res->ms_d2h = double(a) + double(b);
  res->ms_total = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
  if (host_timing) {
    std::fprintf(stderr, "psg host ms: tables %.3f trace %.3f units %.3f stream %.3f sigs %.3f pack %.3f bufs %.3f | errors %.3f assemble %.3f | total %.3f\n",
                 host_t[0], host_t[1], host_t[2], host_t[3], host_t[4], host_t[5], host_t[6], host_t[7], host_t[8], res->ms_total);
  }
  *out = res;
  return PSG_OK;
}

int psg_search_many(psg_context* const* ctxs, int n, const psg_plan_set* const* plans,
                    const psg_cluster* const* clusters, const psg_store* const* stores,
                    const psg_trace* const* traces, const psg_config* const* configs,
                    psg_result** outs, double* kernel_span_ms) {
  if (n <= 0 || !ctxs || !plans || !clusters || !stores || !traces || !configs || !outs)
    return PSG_ERR_USAGE;
  // every search's simulation blocks share the device: size shared memory so
  // they are all resident in one wave
  int total = 0, total_groups = 0;
  const int groups = replica_groups();
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !plans[i] || !configs[i]) return PSG_ERR_USAGE;
    for (int j = 0; j < i; ++j)
      if (ctxs[j] == ctxs[i]) return PSG_ERR_USAGE;  // one context per search
    const psg_config* c = configs[i];
    const psg_plan_set* P = plans[i];
    const int F = std::max(1, c->n_freqs);
    auto count = [&](int64_t g) {  // global entry g = plan * F + frequency
      if (g < 0 || g >= int64_t(P->n_plans) * F) return;
      const int dp = std::max(1, P->model_dp[g / F]);
      ++total;
      total_groups += std::min(dp, groups);
    };
    if (c->n_entry_subset > 0) {
      for (int k = 0; k < c->n_entry_subset; ++k) count(c->entry_subset[k]);
    } else {
      for (int64_t g = 0; g < int64_t(P->n_plans) * F; ++g) count(g);
    }
  }
  std::vector<int> rc(size_t(n), PSG_OK);
  StartGate gate;
  gate.expected = n;
  const bool gated = !std::getenv("PSG_NO_START_GATE");  // dev knob
  auto run = [&](int i) {
    ctxs[i]->concurrent_blocks = total;
    ctxs[i]->concurrent_groups = total_groups;
    ctxs[i]->gate = gated ? &gate : nullptr;
    ctxs[i]->gate_passed = false;
    rc[size_t(i)] = psg_search(ctxs[i], plans[i], clusters[i], stores[i], traces[i], configs[i], &outs[i]);
    if (gated && !ctxs[i]->gate_passed) gate.arrive(false);  // failed before the gate
    ctxs[i]->gate = nullptr;
    ctxs[i]->concurrent_blocks = 0;
    ctxs[i]->concurrent_groups = 0;
  };
  const int spawn = guarded(ctxs[0], [&] {
    std::vector<std::thread> pool;
    for (int i = 1; i < n; ++i) pool.emplace_back(run, i);
    run(0);
    for (auto& t : pool) t.join();
    return PSG_OK;
  });
  if (spawn != PSG_OK) return spawn;
  for (int i = 0; i < n; ++i)
    if (rc[size_t(i)] != PSG_OK) return rc[size_t(i)];
  if (kernel_span_ms) {
    // device span of the searches' kernels: earliest end of input H2D (ev[1])
    // to the latest end of the reduction kernels (ev[3]), across streams
    int first = 0;
    for (int i = 1; i < n; ++i) {
      float d = 0.f;
      if (cudaEventElapsedTime(&d, ctxs[first]->ev[1], ctxs[i]->ev[1]) == cudaSuccess && d < 0.f) first = i;
    }
    double span = 0.0;
    for (int i = 0; i < n; ++i) {
      float d = 0.f;
      cudaEventElapsedTime(&d, ctxs[first]->ev[1], ctxs[i]->ev[3]);
      float extra = 0.f;  // compaction kernel of a detail search (ev[5] -> ev[6])
      cudaEventElapsedTime(&extra, ctxs[i]->ev[5], ctxs[i]->ev[6]);
      span = std::max(span, double(d) + double(extra));
    }
    *kernel_span_ms = span;
  }
  return PSG_OK;
}

}  // extern "C"
