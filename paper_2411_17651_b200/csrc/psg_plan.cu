// psg_plan.cu — plan enumeration and device mapping on the GPU
// (generate_plans, /root/reference/proj/src/planner.cpp:188-389, and
// map_devices, cluster.cpp:118-198).
//
//   plan_map_kernel        one block per candidate group (model_dp, stages):
//                          thread 0 places the stages (smallest aligned subtree
//                          with room, lowest index first; fragmented trees fall
//                          back to the lowest free devices), then the block
//                          computes the worst span (tree level, then node count)
//                          of every group size that divides the stage width
//                          over all its concrete group instances, and the p2p
//                          boundary node counts.
//   plan_candidate_kernel  one thread per candidate (a per-cell choice
//                          combination, last cell fastest): reshard collectives
//                          (planner.cpp:121-152) resolved against the group's
//                          spans, and the memory ledger (finalize_plan,
//                          planner.cpp:307-370) in the reference's order.
//   plan_emit_kernel       the kept candidates compacted into the psg_plan_set
//                          SoA the search consumes (psg_plan_emit).
#include <cub/block/block_scan.cuh>

#include "psg_device.cuh"
#include "psg_reduce.cuh"

namespace psg {

namespace {

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

}  // namespace

// span_nodes[g * n + gsize] = worst node count of size-gsize groups; span_level likewise
__global__ void plan_map_kernel(const psg_plan_space s, int32_t* phys_out, const int64_t* p2p_off,
                                int32_t* p2p_out, int32_t* span_nodes, int32_t* span_level) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int n = s.n_devices;
  int32_t* phys = reinterpret_cast<int32_t*>(sm);
  unsigned char* used = sm + sizeof(int32_t) * size_t(n);
  const int g = blockIdx.x;
  const int dp = s.group_dp[g], stages = s.group_stages[g], sdev = s.group_sdev[g];
  for (int i = threadIdx.x; i < n; i += blockDim.x) used[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int len = 0;
    auto take = [&](int lo, int hi, int want) {
      for (int i = lo; i < hi && want > 0; ++i)
        if (!used[i]) {
          used[i] = 1;
          phys[len++] = i;
          --want;
        }
    };
    for (int block = 0; block < dp * stages; ++block) {
      bool placed = false;
      for (int level = 0; level <= s.n_levels && !placed; ++level) {
        const int cap = s.subtree_cap[level];
        if (cap < sdev) continue;
        for (int base = 0; base + cap <= n && !placed; base += cap) {
          int free_here = 0;
          for (int i = base; i < base + cap; ++i) free_here += used[i] ? 0 : 1;
          if (free_here >= sdev) {
            take(base, base + cap, sdev);
            placed = true;
          }
        }
      }
      if (!placed) take(0, n, sdev);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) phys_out[size_t(g) * n + i] = phys[i];
  // p2p boundary b: first device of stages b and b+1 of replica 0 (planner.cpp:336-342)
  for (int b = threadIdx.x; b + 1 < stages; b += blockDim.x) {
    const int a = phys[b * sdev], c = phys[(b + 1) * sdev];
    p2p_out[p2p_off[g] + b] = a / s.per_node == c / s.per_node ? 1 : 2;
  }
  // worst span of every group size dividing the stage width
  for (int gs = 2; gs <= sdev; ++gs) {
    if (sdev % gs) continue;
    const int groups = sdev / gs;
    const int inst = dp * stages * groups;
    int best_level = -1, best_nodes = -1;
    for (int q = threadIdx.x; q < inst; q += blockDim.x) {
      const int gi = q % groups, rs = q / groups;  // rs = r * stages + st
      const int* ids = phys + (rs * sdev + gi * gs);
      int nodes = 0;
      for (int j = 0; j < gs; ++j) {
        const int nj = ids[j] / s.per_node;
        bool seen = false;
        for (int i = 0; i < j && !seen; ++i) seen = ids[i] / s.per_node == nj;
        nodes += seen ? 0 : 1;
      }
      int level = s.n_levels;
      for (int l = 0; l <= s.n_levels; ++l) {
        const int cap = s.subtree_cap[l];
        bool same = true;
        for (int j = 1; j < gs && same; ++j) same = ids[j] / cap == ids[0] / cap;
        if (same) {
          level = l;
          break;
        }
      }
      if (level > best_level || (level == best_level && nodes > best_nodes)) {
        best_level = level;
        best_nodes = nodes;
      }
    }
    // block max of (level, nodes), lexicographic
    __shared__ int red_key[256];
    red_key[threadIdx.x] = best_level < 0 ? -1 : best_level * (1 << 20) + best_nodes;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red_key[threadIdx.x] = max(red_key[threadIdx.x], red_key[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      span_level[size_t(g) * n + gs] = red_key[0] >> 20;
      span_nodes[size_t(g) * n + gs] = red_key[0] & ((1 << 20) - 1);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) plan_candidate_kernel(const psg_plan_space s,
                                                             const int32_t* span_nodes,
                                                             psg_plan_record* out) {
  const int64_t total = s.group_first[s.n_groups];
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int lo = 0, hi = s.n_groups - 1;  // group of this candidate
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (s.group_first[mid] <= idx) lo = mid; else hi = mid - 1;
  }
  const int g = lo;
  const int nc = s.n_cells, sdev = s.group_sdev[g];
  int mode[PSG_PLAN_MAX_CELLS], cdp[PSG_PLAN_MAX_CELLS], intra[PSG_PLAN_MAX_CELLS];
  double wgt[PSG_PLAN_MAX_CELLS];
  int64_t k = idx - s.group_first[g];
  for (int ci = nc - 1; ci >= 0; --ci) {  // mixed radix, last cell fastest
    const int b = s.choice_begin[g * nc + ci], m = s.choice_begin[g * nc + ci + 1] - b;
    const int c = b + int(k % m);
    k /= m;
    mode[ci] = s.ch_mode[c];
    cdp[ci] = s.ch_cdp[c];
    intra[ci] = s.ch_intra[c];
    wgt[ci] = s.ch_weight[c];
  }
  psg_plan_record r;
  r.n_colls = 0;
  auto resolve = [&](int kind, double share, int gsize) {  // planner.cpp:277-303
    if (gsize < 2) return;                                 // single-device group: elided
    const int q = r.n_colls++;
    r.coll_kind[q] = kind;
    r.coll_share[q] = share;
    r.coll_devices[q] = gsize;
    r.coll_nodes[q] = span_nodes[size_t(g) * s.n_devices + gsize];
    r.coll_groups[q] = sdev / gsize;
  };
  for (int i = 0; i < nc; ++i) {  // reshards between cell i and i+1 (planner.cpp:121-152)
    const int j = (i + 1) % nc;
    const bool l_ep = mode[i] == 1 && intra[i] > 1, r_ep = mode[j] == 1 && intra[j] > 1;
    if (l_ep) resolve(PSG_COLL_ALL_TO_ALL, 1.0 / cdp[i], intra[i]);
    if (r_ep) {
      resolve(PSG_COLL_ALL_TO_ALL, 1.0 / cdp[j], intra[j]);
    } else if (cdp[i] == cdp[j]) {
      if (!l_ep && intra[i] > 1) resolve(PSG_COLL_ALLREDUCE, 1.0 / cdp[i], intra[i]);
    } else {
      resolve(PSG_COLL_ALL_TO_ALL, 1.0, sdev);
      if (intra[j] > 1) resolve(PSG_COLL_ALLGATHER, 1.0 / cdp[j], intra[j]);
    }
  }
  // memory ledger (planner.cpp:344-369)
  double per_device = 0.0;
  for (int i = 0; i < nc; ++i) per_device = __dadd_rn(per_device, wgt[i]);
  per_device = __dmul_rn(per_device, double(s.group_reps[g]));
  const double emb = s.include_embedding ? s.emb_bytes : 0.0;
  double last_stage = per_device;
  if (s.include_embedding) last_stage = __dadd_rn(last_stage, __ddiv_rn(emb, double(sdev)));
  r.static_bytes_per_device = dmax(per_device, last_stage);
  const int replica_devices = s.group_stages[g] * sdev;
  const double replica_static =
      __dadd_rn(__dmul_rn(per_device, double(replica_devices)), s.include_embedding ? emb : 0.0);
  const double replica_capacity = __dmul_rn(s.memory_capacity, double(replica_devices));
  r.kv_budget_per_replica =
      dmax(0.0, __dsub_rn(__dmul_rn(replica_capacity, __dsub_rn(1.0, s.activation_reserve)),
                          replica_static));
  double per_layer = 0.0;
  for (int i = 0; i < nc; ++i) {
    if (!s.cell_is_attention[i]) continue;
    const double kv_instances = dmax(s.cell_kv_heads[i], double(intra[i]));
    per_layer = __dadd_rn(per_layer, __dmul_rn(__dmul_rn(__dmul_rn(2.0, s.cell_head_dim[i]),
                                                         kv_instances), s.kv_elem_bytes));
  }
  r.kv_bytes_per_token = __dmul_rn(per_layer, double(s.num_layers));
  r.feasible = r.static_bytes_per_device <= s.memory_capacity ? 1 : 0;
  out[idx] = r;
}

// plan_emit_kernel: one block compacts the kept candidates (host keep flag
// = first occurrence of the encoding, device feasibility) in candidate order
// straight into the psg_plan_set arrays (PlanSoA's layout, search.cpp), three
// block scans per 1024-candidate tile: plan index, collective offset, p2p
// offset.
__global__ void __launch_bounds__(kEmitThreads) plan_emit_kernel(const psg_plan_space s,
                                                                 const psg_plan_record* rec,
                                                                 const PlanEmitArgs a,
                                                                 PlanEmitOut o) {
  using Scan = cub::BlockScan<int, kEmitThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry[3];
  const int64_t total = s.group_first[s.n_groups];
  const int nc = s.n_cells;
  if (threadIdx.x == 0) carry[0] = carry[1] = carry[2] = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < total; t0 += kEmitThreads) {
    const int64_t idx = t0 + threadIdx.x;
    int g = 0;
    bool kept = false;
    if (idx < total) {
      int lo = 0, hi = s.n_groups - 1;  // group of this candidate
      while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (s.group_first[mid] <= idx) lo = mid; else hi = mid - 1;
      }
      g = lo;
      kept = a.keep[idx] && rec[idx].feasible;
    }
    const int nk = kept ? rec[idx].n_colls : 0, np2 = kept ? s.group_stages[g] - 1 : 0;
    int pi, ko, po, tp, tk, tpp;
    Scan(tmp).ExclusiveSum(int(kept), pi, tp);
    __syncthreads();
    Scan(tmp).ExclusiveSum(nk, ko, tk);
    __syncthreads();
    Scan(tmp).ExclusiveSum(np2, po, tpp);
    pi += carry[0];
    ko += carry[1];
    po += carry[2];
    if (kept) {
      const psg_plan_record& r = rec[idx];
      o.model_dp[pi] = s.group_dp[g];
      o.num_stages[pi] = s.group_stages[g];
      o.stage_devices[pi] = s.group_sdev[g];
      o.stage_reps[pi] = s.group_reps[g];
      o.dtype[pi] = a.compute_dtype;
      o.enc_rank[pi] = a.enc_rank[idx];
      o.kv[pi] = r.kv_bytes_per_token;
      o.budget[pi] = r.kv_budget_per_replica;
      o.p2p_ppt[pi] = a.payload_per_token;
      o.sh_hidden[pi] = a.shape_hidden;
      o.sh_head[pi] = a.shape_head_dim;
      o.sh_kv[pi] = a.shape_kv_elems;
      o.candidate[pi] = idx;
      int64_t k = idx - s.group_first[g];
      for (int ci = nc - 1; ci >= 0; --ci) {  // mixed radix, last cell fastest
        const int b = s.choice_begin[g * nc + ci], m = s.choice_begin[g * nc + ci + 1] - b;
        const int c = b + int(k % m);
        k /= m;
        const int q = pi * nc + ci;
        o.cell_op[q] = a.ch_op[c];
        o.cell_tasks[q] = a.ch_tasks[c];
        o.cell_width[q] = a.ch_width[c];
        o.cell_scale[q] = a.ch_scale[c];
      }
      o.cell_begin[pi] = pi * nc;
      o.coll_begin[pi] = ko;
      for (int q = 0; q < r.n_colls; ++q) {
        o.coll_kind[ko + q] = r.coll_kind[q];
        o.coll_devices[ko + q] = r.coll_devices[q];
        o.coll_nodes[ko + q] = r.coll_nodes[q];
        o.coll_groups[ko + q] = r.coll_groups[q];
        o.coll_ppt[ko + q] = a.payload_per_token;
        o.coll_share[ko + q] = r.coll_share[q];
      }
      o.p2p_begin[pi] = po;
      for (int b = 0; b < np2; ++b) o.p2p_nodes[po + b] = a.p2p[a.p2p_off[g] + b];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += tp;
      carry[1] += tk;
      carry[2] += tpp;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // the closing offsets and the counts
    o.cell_begin[carry[0]] = carry[0] * nc;
    o.coll_begin[carry[0]] = carry[1];
    o.p2p_begin[carry[0]] = carry[2];
    o.counts[0] = carry[0];
    o.counts[1] = carry[1];
    o.counts[2] = carry[2];
  }
}

}  // namespace psg

extern "C" int psg_plan_compute(psg_context* ctx, const psg_plan_space* space,
                                psg_plan_record* records, int32_t* phys, const int64_t* p2p_offset,
                                int32_t* p2p) {
  return psg::plan_compute(ctx, space, records, phys, p2p_offset, p2p);
}

extern "C" int psg_plan_emit(psg_context* ctx, const psg_plan_space* space, const psg_plan_emit_in* in,
                             psg_plan_soa** out) {
  return psg::plan_emit(ctx, space, in, out);
}

extern "C" void psg_plan_soa_free(psg_plan_soa* soa) { psg::plan_soa_free(soa); }
