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

__global__ void __launch_bounds__(kReduceThreads) entry_reduce_kernel(const ReduceParams r) {
  const int e = blockIdx.x;
  constexpr int kStats = 6;  // p95 e2e, p50/p99 TTFT, p50/p99 TPOT, TTFT at the SLO quantile
  __shared__ unsigned sel_hist[kStats][256];
  __shared__ uint64_t sel_prefix[kStats];
  __shared__ int64_t sel_k[kStats];
  __shared__ double sh_sums[2];
  __shared__ int64_t sh_cnt[2];

  const size_t base = size_t(e) * size_t(r.n_slots);
  const uint8_t* st = r.slot_status + base;
  const double* ttft = r.slot_ttft + base;
  double* tpot = r.slot_tpot + base;
  const double* e2e = r.slot_e2e + base;
  const int64_t* gen = r.slot_gen;  // per slot (id order), shared by entries

  // The simulation stores tpot's numerator (finish clock - first token);
  // the division (simulator.cpp:150-152) runs here, off its serial path.
  for (int64_t i = threadIdx.x; i < r.n_slots; i += blockDim.x)
    if (st[i] == 1) tpot[i] = gen[i] >= 2 ? __ddiv_rn(tpot[i], double(gen[i] - 1)) : 0.0;
  __syncthreads();

  // ---- ordered means: one serial chain in ascending id order ----
  // The block stages tiles of the slot arrays in shared memory (coalesced),
  // thread 0 runs the chain from there.  A slot that does not count adds
  // +0.0, which leaves the non-negative (never -0) sums bit-identical, so the
  // chain needs no branches.
  constexpr int kTile = 1024;
  __shared__ double tile_t[kTile], tile_p[kTile];
  __shared__ unsigned char tile_c[kTile], tile_g[kTile];
  double ts = 0.0, ps = 0.0;
  int64_t pn = 0, cn = 0;
  for (int64_t b0 = 0; b0 < r.n_slots; b0 += kTile) {
    const int len = int(min(int64_t(kTile), r.n_slots - b0));
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const int64_t q = b0 + i;
      const bool c = st[q] == 1, g2 = c && gen[q] >= 2;
      tile_c[i] = c;
      tile_g[i] = g2;
      tile_t[i] = c ? ttft[q] : 0.0;
      tile_p[i] = g2 ? tpot[q] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0;
      for (; i + 8 <= len; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          ts = __dadd_rn(ts, tile_t[i + u]);
          ps = __dadd_rn(ps, tile_p[i + u]);
          cn += tile_c[i + u];
          pn += tile_g[i + u];
        }
      }
      for (; i < len; ++i) {
        ts = __dadd_rn(ts, tile_t[i]);
        ps = __dadd_rn(ps, tile_p[i]);
        cn += tile_c[i];
        pn += tile_g[i];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sh_sums[0] = ts;
    sh_sums[1] = ps;
    sh_cnt[0] = cn;
    sh_cnt[1] = pn;
  }
  __syncthreads();
  const int64_t ncomp = sh_cnt[0], ntpot = sh_cnt[1];

  EntryOut o;
  if (threadIdx.x == 0) {
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
  }

  // ---- order statistics: p95 latency (simulator.cpp:222-225), the
  // p50/p99 TTFT/TPOT extras and the SLO quantile of TTFT, all by one fused
  // MSB radix select: each 8-bit pass sweeps the slots once and builds the
  // active statistics' histograms, one warp per statistic picks its digit ----
  const bool slo = r.ttft_slo > 0.0;
  double p95 = 0.0, t50 = 0.0, t99 = 0.0, q50 = 0.0, q99 = 0.0, tslo = 0.0;
  if (ncomp > 0) {
    const bool ext = r.extras != 0, tp = ext && ntpot > 0;
    const bool act[kStats] = {true, ext, ext, tp, tp, slo};
    if (threadIdx.x < kStats) {
      const int j = threadIdx.x;
      const double q = j == 0 ? 0.95 : (j == 1 || j == 3) ? 0.50 : j == 5 ? r.slo_quantile : 0.99;
      sel_k[j] = nearest_rank(q, j == 3 || j == 4 ? (ntpot > 0 ? ntpot : 1) : ncomp);
      sel_prefix[j] = 0;
    }
    uint64_t mask = 0;
    for (int pass = 7; pass >= 0; --pass) {
      const int shift = pass * 8;
      for (int i = threadIdx.x; i < kStats * 256; i += blockDim.x) sel_hist[i / 256][i % 256] = 0;
      __syncthreads();
      const uint64_t pe = sel_prefix[0], pt50 = sel_prefix[1], pt99 = sel_prefix[2],
                     pp50 = sel_prefix[3], pp99 = sel_prefix[4], pslo = sel_prefix[5];
      for (int64_t i = threadIdx.x; i < r.n_slots; i += blockDim.x) {
        if (st[i] != 1) continue;
        const uint64_t ke = order_key(e2e[i]) , m8 = (ke >> shift) & 255u;
        if ((ke & mask) == pe) atomicAdd(&sel_hist[0][m8], 1u);
        if (ext || slo) {
          const uint64_t kt = order_key(ttft[i]), d = (kt >> shift) & 255u;
          if (ext && (kt & mask) == pt50) atomicAdd(&sel_hist[1][d], 1u);
          if (ext && (kt & mask) == pt99) atomicAdd(&sel_hist[2][d], 1u);
          if (slo && (kt & mask) == pslo) atomicAdd(&sel_hist[5][d], 1u);
          if (tp && gen[i] >= 2) {
            const uint64_t kp = order_key(tpot[i]), dp = (kp >> shift) & 255u;
            if ((kp & mask) == pp50) atomicAdd(&sel_hist[3][dp], 1u);
            if ((kp & mask) == pp99) atomicAdd(&sel_hist[4][dp], 1u);
          }
        }
      }
      __syncthreads();
      const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
      if (w < kStats && act[w]) {  // first digit whose inclusive count exceeds k (as the serial scan)
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
      __syncthreads();
    }
    p95 = from_order_key(sel_prefix[0]);
    if (act[1]) {
      t50 = from_order_key(sel_prefix[1]);
      t99 = from_order_key(sel_prefix[2]);
    }
    if (act[3]) {
      q50 = from_order_key(sel_prefix[3]);
      q99 = from_order_key(sel_prefix[4]);
    }
    if (act[5]) tslo = from_order_key(sel_prefix[5]);
  }
  if (threadIdx.x == 0) {
    o.p95 = p95;
    o.p50_ttft = t50;
    o.p99_ttft = t99;
    o.p50_tpot = q50;
    o.p99_tpot = q99;
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
