// psg_reduce.cu — per-entry metric reduction, output compaction and ranking.
//
//  entry_reduce_kernel  simulate_plan's reduction (simulator.cpp:196-238):
//                       e2e = max over replicas, energy summed in replica
//                       order, mean TTFT/TPOT summed in ascending-id order
//                       (one serial FP64 chain, as the reference), p95 by
//                       nearest rank via a fused MSB radix select (also the
//                       additive p50/p99 TTFT/TPOT outputs), MFU/MBU.
//  compact_kernel       per_request sorted by id / rejected_ids sorted
//                       (simulator.cpp:205-207) as dense arrays for one D2H.
//  rank_kernel          search()'s comparator (simulator.cpp:283-294):
//                       (num_rejected, objective, other, encoding, freq),
//                       after the TTFT-SLO flag when an SLO is set.
#include <cub/block/block_scan.cuh>

#include "psg_device.cuh"
#include "psg_reduce.cuh"

namespace psg {

namespace {

__device__ __forceinline__ uint64_t order_key(double v) {
  const uint64_t b = __double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_order_key(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(b);
}

// Nearest-rank index of simulator.cpp:224-225.
__device__ __forceinline__ int64_t nearest_rank(double q, int64_t n) {
  const int64_t rank = int64_t(ceil(__dmul_rn(q, double(n))));
  const int64_t idx = rank == 0 ? 0 : rank - 1;
  return idx < n - 1 ? idx : n - 1;
}

}  // namespace

__global__ void __launch_bounds__(kReduceThreads, 4) entry_reduce_kernel(const ReduceParams r) {
  const int e = blockIdx.x;
  constexpr int kStats = kReduceStats;
  __shared__ unsigned sel_hist[kStats][256];
  __shared__ uint64_t sel_prefix[kStats];
  __shared__ int64_t sel_k[kStats];
  __shared__ double sh_sums[2];
  __shared__ unsigned long long sh_cnt[2];
  __shared__ double sh_q[kStats];
  // after four full 8-bit passes, each statistic's remaining candidates (the
  // keys matching its 24-bit prefix) are gathered here and the four later
  // passes sweep only them; a statistic with more candidates keeps sweeping
  // every slot
  extern __shared__ __align__(16) unsigned char red_smem[];
  uint64_t* cand = reinterpret_cast<uint64_t*>(red_smem);  // [kStats][cand_cap]
  __shared__ unsigned cand_n[kStats];
  const int cand_cap = r.cand_cap;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const size_t base = size_t(e) * size_t(r.n_slots);
  const uint8_t* st = r.slot_status + base;
  const double* ttft = r.slot_ttft + base;
  double* tpot = r.slot_tpot + base;
  const double* e2e = r.slot_e2e + base;
  const int64_t* gen = r.slot_gen;  // per slot (id order), shared by entries

  // The simulation stores tpot's numerator (finish clock - first token);
  // the division (simulator.cpp:150-152) runs here, off its serial path;
  // the same sweep counts the completed requests and those with a TPOT.
  if (threadIdx.x < 2) sh_cnt[threadIdx.x] = 0;
  if (threadIdx.x < kStats) sh_q[threadIdx.x] = 0.0;
  __syncthreads();
  {
    unsigned lc = 0, lp = 0;
    for (int64_t i0 = threadIdx.x; i0 < r.n_slots; i0 += kSweepU * blockDim.x) {
      uint8_t s[kSweepU];
      int64_t g[kSweepU];
      double t[kSweepU];
#pragma unroll
      for (int u = 0; u < kSweepU; ++u) {  // independent loads first
        const int64_t i = i0 + int64_t(u) * blockDim.x;
        const bool in = i < r.n_slots;
        s[u] = in ? st[i] : 0;
        g[u] = in ? gen[i] : 0;
        t[u] = in ? tpot[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kSweepU; ++u)
        if (s[u] == 1) {
          const bool g2 = g[u] >= 2;
          tpot[i0 + int64_t(u) * blockDim.x] = g2 ? __ddiv_rn(t[u], double(g[u] - 1)) : 0.0;
          ++lc;
          lp += g2;
        }
    }
    lc = __reduce_add_sync(0xffffffffu, lc);
    lp = __reduce_add_sync(0xffffffffu, lp);
    if (lane == 0) {
      atomicAdd(&sh_cnt[0], (unsigned long long)lc);
      atomicAdd(&sh_cnt[1], (unsigned long long)lp);
    }
  }
  __syncthreads();
  const int64_t ncomp = int64_t(sh_cnt[0]), ntpot = int64_t(sh_cnt[1]);
  const bool slo = r.ttft_slo > 0.0;
  const bool ext = r.extras != 0, tp = ext && ntpot > 0;
  const bool act[kStats] = {true, ext, ext, tp, tp, slo};
  if (ncomp > 0 && threadIdx.x < kStats) {
    const int j = threadIdx.x;
    const double q = j == 0 ? 0.95 : (j == 1 || j == 3) ? 0.50 : j == 5 ? r.slo_quantile : 0.99;
    sel_k[j] = nearest_rank(q, j == 3 || j == 4 ? (ntpot > 0 ? ntpot : 1) : ncomp);
    sel_prefix[j] = 0;
  }
  __syncthreads();

  if (warp == 0) {
    // ---- ordered means (warp 0, beside the order statistics): one serial
    // chain per mean in ascending id order; the lanes load 128 slots at a
    // time and broadcast them in order.  A slot that does not count adds
    // +0.0, which leaves the non-negative (never -0) sums bit-identical. ----
    constexpr int kU = 4;
    double ts = 0.0, ps = 0.0;
    double nt[kU], np[kU];  // the next 128 slots, loaded while the chain runs
    auto load = [&](int64_t b0) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = b0 + u * 32 + lane;
        const bool in = i < r.n_slots;
        const uint8_t s = in ? st[i] : 0;
        const int64_t g = in ? gen[i] : 0;
        const double a = in ? ttft[i] : 0.0, b = in ? tpot[i] : 0.0;
        nt[u] = s == 1 ? a : 0.0;
        np[u] = s == 1 && g >= 2 ? b : 0.0;
      }
    };
    load(0);
    for (int64_t b0 = 0; b0 < r.n_slots; b0 += kU * 32) {
      double vt[kU], vp[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        vt[u] = nt[u];
        vp[u] = np[u];
      }
      if (b0 + kU * 32 < r.n_slots) load(b0 + kU * 32);
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          ts = __dadd_rn(ts, __shfl_sync(0xffffffffu, vt[u], q));
          ps = __dadd_rn(ps, __shfl_sync(0xffffffffu, vp[u], q));
        }
    }
    if (lane == 0) {
      sh_sums[0] = ts;
      sh_sums[1] = ps;
    }
  } else if (ncomp > 0) {
    // ---- order statistics (warps 1..): p95 latency (simulator.cpp:222-225),
    // the p50/p99 TTFT/TPOT extras and the SLO quantile of TTFT, all by one
    // fused MSB radix select: each 8-bit pass sweeps the slots once and builds
    // the active statistics' histograms, one warp per statistic picks its
    // digit.  Named barrier 1 syncs these warps only. ----
    const int tid = threadIdx.x - 32, nthr = blockDim.x - 32;
    auto sync_sel = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory"); };
    uint64_t mask = 0;
    bool full[kStats];  // the statistic still sweeps every slot
    for (int j = 0; j < kStats; ++j) full[j] = true;
    for (int pass = 7; pass >= 0; --pass) {
      const int shift = pass * 8;
      for (int i = tid; i < kStats * 256; i += nthr) sel_hist[i / 256][i % 256] = 0;
      const bool collect = pass == 4 && cand_cap > 0;  // gather the candidates of the 24-bit prefixes
      if (collect && tid < kStats) cand_n[tid] = 0;
      sync_sel();
      const uint64_t pe = sel_prefix[0], pt50 = sel_prefix[1], pt99 = sel_prefix[2],
                     pp50 = sel_prefix[3], pp99 = sel_prefix[4], pslo = sel_prefix[5];
      const bool sweep = full[0] || full[1] || full[2] || full[3] || full[4] || full[5];
      auto visit = [&](double ve, double vt, double vp, int64_t g) {
        const uint64_t ke = order_key(ve), m8 = (ke >> shift) & 255u;
        if (full[0] && (ke & mask) == pe) {
          atomicAdd(&sel_hist[0][m8], 1u);
          if (collect) {
            const unsigned c = atomicAdd(&cand_n[0], 1u);
            if (c < unsigned(cand_cap)) cand[c] = ke;
          }
        }
        if (ext || slo) {
          const uint64_t kt = order_key(vt), d = (kt >> shift) & 255u;
          if (ext && full[1] && (kt & mask) == pt50) {
            atomicAdd(&sel_hist[1][d], 1u);
            if (collect) {
              const unsigned c = atomicAdd(&cand_n[1], 1u);
              if (c < unsigned(cand_cap)) cand[size_t(cand_cap) + c] = kt;
            }
          }
          if (ext && full[2] && (kt & mask) == pt99) {
            atomicAdd(&sel_hist[2][d], 1u);
            if (collect) {
              const unsigned c = atomicAdd(&cand_n[2], 1u);
              if (c < unsigned(cand_cap)) cand[2 * size_t(cand_cap) + c] = kt;
            }
          }
          if (slo && full[5] && (kt & mask) == pslo) {
            atomicAdd(&sel_hist[5][d], 1u);
            if (collect) {
              const unsigned c = atomicAdd(&cand_n[5], 1u);
              if (c < unsigned(cand_cap)) cand[5 * size_t(cand_cap) + c] = kt;
            }
          }
          if (tp && g >= 2) {
            const uint64_t kp = order_key(vp), dp = (kp >> shift) & 255u;
            if (full[3] && (kp & mask) == pp50) {
              atomicAdd(&sel_hist[3][dp], 1u);
              if (collect) {
                const unsigned c = atomicAdd(&cand_n[3], 1u);
                if (c < unsigned(cand_cap)) cand[3 * size_t(cand_cap) + c] = kp;
              }
            }
            if (full[4] && (kp & mask) == pp99) {
              atomicAdd(&sel_hist[4][dp], 1u);
              if (collect) {
                const unsigned c = atomicAdd(&cand_n[4], 1u);
                if (c < unsigned(cand_cap)) cand[4 * size_t(cand_cap) + c] = kp;
              }
            }
          }
        }
      };
      for (int64_t i0 = tid; sweep && i0 < r.n_slots; i0 += kSweepU * nthr) {
        uint8_t s[kSweepU];
        int64_t g[kSweepU];
        double ve[kSweepU], vt[kSweepU], vp[kSweepU];
#pragma unroll
        for (int u = 0; u < kSweepU; ++u) {  // independent loads first
          const int64_t i = i0 + int64_t(u) * nthr;
          const bool in = i < r.n_slots;
          s[u] = in ? st[i] : 0;
          ve[u] = in ? e2e[i] : 0.0;
          vt[u] = in && (ext || slo) ? ttft[i] : 0.0;
          g[u] = in && tp ? gen[i] : 0;
          vp[u] = in && tp ? tpot[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kSweepU; ++u)
          if (s[u] == 1) visit(ve[u], vt[u], vp[u], g[u]);
      }
      // the statistics swept from their candidates (every key matching the
      // prefix, so the counts are the full sweep's)
      for (int j = 0; j < kStats; ++j) {
        if (full[j] || !act[j]) continue;
        const uint64_t pj = sel_prefix[j];
        const uint64_t* cj = cand + size_t(j) * size_t(cand_cap);
        for (unsigned c = tid; c < cand_n[j]; c += nthr) {
          const uint64_t k = cj[c];
          if ((k & mask) == pj) atomicAdd(&sel_hist[j][(k >> shift) & 255u], 1u);
        }
      }
      sync_sel();
      if (collect)  // from the next pass on, statistics whose candidates fit sweep only them
        for (int j = 0; j < kStats; ++j) full[j] = cand_n[j] > unsigned(cand_cap);
      const int w = warp - 1;  // warps 1..kStats pick the digits
      if (w >= 0 && w < kStats && act[w]) {  // first digit whose inclusive count exceeds k (as the serial scan)
        const int64_t k = sel_k[w];
        unsigned part = 0;
        for (int b = 0; b < 8; ++b) part += sel_hist[w][lane * 8 + b];
        unsigned incl = part;
        for (int off = 1; off < 32; off <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        const int64_t excl = int64_t(incl - part);
        const bool here = excl <= k && k < excl + int64_t(part);
        const unsigned hm = __ballot_sync(0xffffffffu, here);
        if (hm) {
          if (lane == __ffs(hm) - 1) {
            int64_t kk = k - excl;
            int d = lane * 8;
            for (; d < lane * 8 + 7; ++d) {
              if (kk < int64_t(sel_hist[w][d])) break;
              kk -= sel_hist[w][d];
            }
            sel_k[w] = kk;
            sel_prefix[w] |= uint64_t(d) << shift;
          }
        } else if (lane == 31) {  // k beyond every count: digit 255, as the serial scan
          sel_k[w] = k - (excl + int64_t(part) - int64_t(sel_hist[w][255]));
          sel_prefix[w] |= uint64_t(255) << shift;
        }
      }
      mask |= uint64_t(255) << shift;
      sync_sel();
    }
    if (tid == 0) {
      sh_q[0] = from_order_key(sel_prefix[0]);
      if (act[1]) {
        sh_q[1] = from_order_key(sel_prefix[1]);
        sh_q[2] = from_order_key(sel_prefix[2]);
      }
      if (act[3]) {
        sh_q[3] = from_order_key(sel_prefix[3]);
        sh_q[4] = from_order_key(sel_prefix[4]);
      }
      if (act[5]) sh_q[5] = from_order_key(sel_prefix[5]);
    }
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    EntryOut o;
    o.e2e = 0.0;
    o.energy = 0.0;
    o.flops = 0.0;
    o.bytes = 0.0;
    o.iterations = 0;
    o.max_batch = 0;
    o.rejected = 0;
    o.sum_batch = 0;
    o.admissions = 0;
    o.err = 0;
    for (int k = r.entry_unit_begin[e]; k < r.entry_unit_begin[e + 1]; ++k) {
      const UnitOut& u = r.uout[r.entry_units[k]];
      o.e2e = o.e2e < u.clock ? u.clock : o.e2e;
      o.energy = __dadd_rn(o.energy, u.energy);
      if (r.chain_replicas) {  // one WorkTally across replicas (simulator.cpp:195-201)
        o.flops = u.flops;
        o.bytes = u.bytes;
      } else {
        o.flops = __dadd_rn(o.flops, u.flops);
        o.bytes = __dadd_rn(o.bytes, u.bytes);
      }
      o.iterations += u.iterations;
      o.max_batch = o.max_batch > u.max_batch ? o.max_batch : u.max_batch;
      o.rejected += u.rejected;
      o.sum_batch += u.sum_batch;
      o.admissions += u.admissions;
      if (!o.err && u.err) o.err = u.err;
    }
    o.completed = ncomp;
    o.mean_ttft = ncomp > 0 ? __ddiv_rn(sh_sums[0], double(ncomp)) : 0.0;
    o.mean_tpot = ntpot > 0 ? __ddiv_rn(sh_sums[1], double(ntpot)) : 0.0;
    o.mfu = 0.0;
    o.mbu = 0.0;
    if (o.e2e > 0) {
      const double pf = r.entry_peak[e];
      if (!(pf > 0)) {
        if (!o.err) o.err = 3;  // peak_flops_for() throws DataError
      } else {
        o.mfu = __ddiv_rn(o.flops, __dmul_rn(o.e2e, pf));
        o.mbu = __ddiv_rn(o.bytes, __dmul_rn(__dmul_rn(o.e2e, r.mem_bw),
                                             double(r.total_devices)));
      }
    }
    const double tslo = sh_q[5];
    o.p95 = sh_q[0];
    o.p50_ttft = sh_q[1];
    o.p99_ttft = sh_q[2];
    o.p50_tpot = sh_q[3];
    o.p99_tpot = sh_q[4];
    o.slo_ttft = tslo;
    r.eout[e] = o;
    psg_rank_key k;
    const bool lat = r.objective == PSG_OBJ_LATENCY;
    k.num_rejected = o.rejected;
    k.objective_metric = lat ? o.e2e : o.energy;
    k.other_metric = lat ? o.energy : o.e2e;
    k.enc_rank = r.entry_enc_rank[e];
    // an entry with no completed request cannot meet a TTFT SLO
    k.slo_miss = slo && !(ncomp > 0 && tslo <= r.ttft_slo) ? 1 : 0;
    k.freq_ghz = r.entry_freq[e];
    k.entry_index = r.entry_global[e];
    r.keys[e] = k;
  }
}

// Exclusive scan of per-entry completed / rejected counts (one warp, 32
// entries per step: shuffle scan, running totals carried across steps).
__global__ void offsets_kernel(const EntryOut* eout, int n_entries, int64_t* pr_off,
                               int64_t* rj_off, int64_t* totals) {
  const int lane = threadIdx.x;
  if (lane >= 32) return;
  int64_t a = 0, b = 0;  // totals of the entries before this step
  for (int e0 = 0; e0 < n_entries; e0 += 32) {
    const int e = e0 + lane;
    const int64_t ca = e < n_entries ? eout[e].completed : 0;
    const int64_t cb = e < n_entries ? eout[e].rejected : 0;
    int64_t ia = ca, ib = cb;  // inclusive scans
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t ya = __shfl_up_sync(0xffffffffu, ia, off);
      const int64_t yb = __shfl_up_sync(0xffffffffu, ib, off);
      if (lane >= off) {
        ia += ya;
        ib += yb;
      }
    }
    if (e < n_entries) {
      pr_off[e] = a + ia - ca;
      rj_off[e] = b + ib - cb;
    }
    a += __shfl_sync(0xffffffffu, ia, 31);
    b += __shfl_sync(0xffffffffu, ib, 31);
  }
  if (lane == 0) {
    totals[0] = a;
    totals[1] = b;
  }
}

// Dense per_request / rejected_ids in ascending id order per entry.
__global__ void __launch_bounds__(256) compact_kernel(const ReduceParams r,
                                                     const int64_t* pr_off,
                                                     const int64_t* rj_off,
                                                     psg_request_metrics* out_pr,
                                                     int64_t* out_rj) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry[2];
  const int e = blockIdx.x;
  const size_t base = size_t(e) * size_t(r.n_slots);
  if (threadIdx.x == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < r.n_slots; b0 += 256) {
    const int64_t i = b0 + threadIdx.x;
    const uint8_t s = i < r.n_slots ? r.slot_status[base + i] : 0;
    int c = s == 1, j = s == 2;
    int cp, jp, ct, jt;
    Scan(tmp).ExclusiveSum(c, cp, ct);
    __syncthreads();
    Scan(tmp).ExclusiveSum(j, jp, jt);
    if (c) {
      psg_request_metrics m;
      m.id = r.slot_id[i];
      m.ttft = r.slot_ttft[base + i];
      m.tpot = r.slot_tpot[base + i];
      m.e2e = r.slot_e2e[base + i];
      m.gen_len = r.slot_gen[i];
      out_pr[pr_off[e] + carry[0] + cp] = m;
    }
    if (j) out_rj[rj_off[e] + carry[1] + jp] = r.slot_id[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += ct;
      carry[1] += jt;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ bool key_less(const psg_rank_key& a, const psg_rank_key& b) {
  if (a.slo_miss != b.slo_miss) return a.slo_miss < b.slo_miss;  // SLO met first (0 when off)
  if (a.num_rejected != b.num_rejected) return a.num_rejected < b.num_rejected;
  if (a.objective_metric != b.objective_metric) return a.objective_metric < b.objective_metric;
  if (a.other_metric != b.other_metric) return a.other_metric < b.other_metric;
  if (a.enc_rank != b.enc_rank) return a.enc_rank < b.enc_rank;
  if (a.freq_ghz != b.freq_ghz) return a.freq_ghz < b.freq_ghz;
  return a.entry_index < b.entry_index;  // total order (reference: unspecified)
}

// Rank by counting: pos(i) = #{j : key_j < key_i}.  Keys are tiled through
// shared memory; the grid covers the entries in 256-wide blocks.
__global__ void __launch_bounds__(256) rank_kernel(const psg_rank_key* keys, int64_t n,
                                                   int64_t* order) {
  __shared__ psg_rank_key tile[256];
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  psg_rank_key mine;
  if (i < n) mine = keys[i];
  int64_t pos = 0;
  for (int64_t t0 = 0; t0 < n; t0 += 256) {
    if (t0 + threadIdx.x < n) tile[threadIdx.x] = keys[t0 + threadIdx.x];
    __syncthreads();
    const int m = int(n - t0 < 256 ? n - t0 : 256);
    if (i < n)
      for (int j = 0; j < m; ++j) pos += key_less(tile[j], mine);
    __syncthreads();
  }
  if (i < n) order[pos] = i;
}

}  // namespace psg
