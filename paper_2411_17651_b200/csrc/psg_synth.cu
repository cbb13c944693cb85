// psg_synth.cu — analytical roofline profile tables on the device
// (synth_profiles, /root/reference/proj/src/cost.cpp:454-509; SURVEY.md §8(f)
// row 4).  One thread per grid point (dtype x frequency, op, context, tasks,
// width): seconds = max(flops / (peak * scale), bytes / bandwidth), joules =
// seconds * power, with op_flops / op_bytes in the reference's order.  The
// host inserts the values in the reference's loop order, so the finalized
// store is byte-identical to the CPU synthesis (tests/test_gpu_synth.py).
#include "psg_device.cuh"
#include "psg_reduce.cuh"

namespace psg {

namespace {

// op_bytes (cost.cpp:60-68) at the table's element width
__device__ __forceinline__ double op_bytes_eb(int op, double t, double k, double w, double hidden,
                                              double kv_elems, double e) {
  double b = __dmul_rn(__dmul_rn(__dmul_rn(k, hidden), w), e);
  b = __dadd_rn(b, __dmul_rn(__dmul_rn(__dmul_rn(2.0, t), hidden), e));
  if (op == PSG_OP_ATTENTION)
    b = __dadd_rn(b, __dmul_rn(__dmul_rn(__dmul_rn(t, k), kv_elems), e));
  return b;
}

}  // namespace

__global__ void __launch_bounds__(256) synth_compute_kernel(const psg_synth_grid g, double* sec,
                                                            double* jou) {
  const int64_t nt = g.n_ctx, nk = g.n_tasks, nw = g.n_width;
  const int64_t per_op = nt * nk * nw;
  const int64_t total = int64_t(g.n_variants) * 3 * per_op;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = i;
    const int wi = int(r % nw);
    r /= nw;
    const int ki = int(r % nk);
    r /= nk;
    const int ti = int(r % nt);
    r /= nt;
    const int oi = int(r % 3);
    const int v = int(r / 3);
    const int op = oi == 0 ? PSG_OP_ATTENTION : oi == 1 ? PSG_OP_GEMM : PSG_OP_MOE_GEMM;
    const double t = g.ctx[ti], k = g.tasks[ki], w = g.width[wi];
    const double flops = op_flops(op, t, k, w, g.hidden, g.head_dim);
    const double bytes = op_bytes_eb(op, t, k, w, g.hidden, g.kv_elems, g.elem_bytes[v]);
    const double a = __ddiv_rn(flops, g.peak_scaled[v]);
    const double b = __ddiv_rn(bytes, g.mem_bw);
    const double s = a < b ? b : a;  // std::max(a, b)
    sec[i] = s;
    jou[i] = __dmul_rn(s, g.power[v]);
  }
}

}  // namespace psg

extern "C" int psg_synth_compute(psg_context* ctx, const psg_synth_grid* g, double* seconds,
                                 double* joules) {
  return psg::synth_compute(ctx, g, seconds, joules);
}
