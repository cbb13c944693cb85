// restate.cpp — TEST INFRASTRUCTURE: a literal, iteration-by-iteration CPU
// restatement of the reference's evaluate-all-plans path over the same
// structure-of-arrays ABI as the GPU engine (include/psg.h).  It exists so
// tests can run both engines on identical inputs; it is validated against the
// compiled reference itself (oracle/_ref/refdrv) on the reference's own
// known-answer fixtures and the C1-C4 configurations (tests/test_oracle*.py).
//
// It is NOT on the product path: only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load oracle/build/liboracle.so.
//
// Followed line by line (all paths under /root/reference/proj):
//   search             src/simulator.cpp:242-296
//   simulate_plan      src/simulator.cpp:176-240
//   run_replica        src/simulator.cpp:98-172
//   iteration_time     src/simulator.cpp:17-87
//   BatchState         src/batching.cpp:11-125
//   query_time/energy  src/cost.cpp:85-102, :196-291
//   op_flops/op_bytes  src/cost.cpp:51-68
//   TTFT-SLO ranking   an addition (psg.h psg_config.ttft_slo); unpinned by the
//                      reference, which has no SLO; tests derive it from the
//                      reference's own per-request TTFTs instead
// Deliberately naive: std::deque / std::vector state, per-query key lookup,
// O(B) ledger recomputation — no event skipping, so it is an independent
// check of the GPU engine's macro-stepping.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "psg.h"

namespace {

struct DataErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Req {
  int64_t id, ctx, gen;
  double arrival;
};

struct Act {
  Req r;
  bool prefill = true;
  int64_t generated = 0, prefill_done = 0;
};

struct Pos {
  size_t lo = 0, hi = 0;
  double t = 0.0;
};

// cost.cpp:85-102
Pos locate(const double* k, size_t n, double x) {
  Pos p;
  if (x <= k[0]) return p;
  if (x >= k[n - 1]) {
    p.lo = p.hi = n - 1;
    return p;
  }
  const double* it = std::upper_bound(k, k + n, x);
  p.hi = size_t(it - k);
  p.lo = p.hi - 1;
  p.t = (x - k[p.lo]) / (k[p.hi] - k[p.lo]);
  return p;
}

struct Store {
  const psg_store* s;
  std::map<std::tuple<int, int, long long>, int> cmap;
  std::map<std::tuple<int, int, int>, int> kmap;

  explicit Store(const psg_store* st) : s(st) {
    for (int t = 0; t < s->n_compute; ++t)
      cmap[{s->c_op[t], s->c_dtype[t], (long long)s->c_freq_micro[t]}] = t;
    for (int u = 0; u < s->n_curves; ++u)
      kmap[{s->k_kind[u], s->k_devices[u], s->k_nodes[u]}] = u;
  }

  // cost.cpp:196-260 (time and energy share the weights)
  void compute(int op, int dtype, double freq, double ctx, double tasks, double width,
               double& sec, double& joule) const {
    auto it = cmap.find({op, dtype, llround(freq * 1e6)});
    if (it == cmap.end()) throw DataErr("profile: no compute table");
    const int t = it->second;
    const double* kn = s->c_knots + s->c_knot_begin[t];
    const size_t nc = size_t(s->c_n_ctx[t]), nt = size_t(s->c_n_tasks[t]),
                 nw = size_t(s->c_n_width[t]);
    const Pos pi = locate(kn, nc, ctx), pj = locate(kn + nc, nt, tasks),
              pk = locate(kn + nc + nt, nw, width);
    const double* vs = s->c_seconds + s->c_value_begin[t];
    const double* vj = s->c_joules + s->c_value_begin[t];
    double as = 0.0, aj = 0.0;
    for (int ci = 0; ci < 2; ++ci) {
      const double wi = ci ? pi.t : 1.0 - pi.t;
      if (wi == 0.0) continue;
      for (int cj = 0; cj < 2; ++cj) {
        const double wj = cj ? pj.t : 1.0 - pj.t;
        if (wj == 0.0) continue;
        for (int ck = 0; ck < 2; ++ck) {
          const double wk = ck ? pk.t : 1.0 - pk.t;
          if (wk == 0.0) continue;
          const size_t i = ci ? pi.hi : pi.lo, j = cj ? pj.hi : pj.lo,
                       k = ck ? pk.hi : pk.lo;
          as += wi * wj * wk * vs[(i * nt + j) * nw + k];
          aj += wi * wj * wk * vj[(i * nt + j) * nw + k];
        }
      }
    }
    sec = as;
    joule = aj;
  }

  // cost.cpp:262-291
  void collective(int kind, int devices, int nodes, double payload, double& sec,
                  double& joule) const {
    auto it = kmap.find({kind, devices, nodes});
    if (it == kmap.end()) throw DataErr("profile: no collective table");
    const int u = it->second;
    const double* x = s->k_payload + s->k_begin[u];
    const Pos p = locate(x, size_t(s->k_n[u]), payload);
    const double* sv = s->k_seconds + s->k_begin[u];
    const double* jv = s->k_joules + s->k_begin[u];
    sec = (1.0 - p.t) * sv[p.lo] + p.t * sv[p.hi];
    joule = (1.0 - p.t) * jv[p.lo] + p.t * jv[p.hi];
  }
};

double op_flops(int op, double t, double k, double w, double H, double hd) {
  double f = 2.0 * t * k * H * w;
  if (op == PSG_OP_ATTENTION) f += 4.0 * t * t * k * hd;
  return f;
}
double op_bytes(int op, double t, double k, double w, double H, double kve) {
  const double e = 2.0;
  double b = k * H * w * e;
  b += 2.0 * t * H * e;
  if (op == PSG_OP_ATTENTION) b += t * k * kve * e;
  return b;
}

struct Workload {
  std::vector<int64_t> prefill;  // tokens, admission order
  int64_t decode = 0;
  int64_t total() const {
    int64_t t = decode;
    for (int64_t v : prefill) t += v;
    return t;
  }
};

struct Plan {
  const psg_plan_set* P;
  int p;
};

// simulator.cpp:17-87: returns (duration, energy) and adds to the tally.
void iteration_time(const Plan& pl, const Store& st, double freq, const Workload& w,
                    double& dur, double& energy, double& tf, double& tb) {
  const psg_plan_set* P = pl.P;
  const int p = pl.p;
  const double total = double(w.total());
  double bs = 0.0, bj = 0.0, bf = 0.0, bb = 0.0;
  for (int c = P->cell_begin[p]; c < P->cell_begin[p + 1]; ++c) {
    auto q = [&](double tokens) {
      const double x = tokens * P->cell_token_scale[c];
      double s, j;
      st.compute(P->cell_op[c], P->compute_dtype[p], freq, x, P->cell_tasks[c],
                 P->cell_width[c], s, j);
      bs += s;
      bj += j * P->stage_devices[p];
      bf += op_flops(P->cell_op[c], x, P->cell_tasks[c], P->cell_width[c],
                     P->shape_hidden[p], P->shape_head_dim[p]);
      bb += op_bytes(P->cell_op[c], x, P->cell_tasks[c], P->cell_width[c],
                     P->shape_hidden[p], P->shape_kv_elems[p]);
    };
    for (int64_t tok : w.prefill) q(double(tok));
    if (w.decode > 0) q(double(w.decode));
  }
  for (int k = P->coll_begin[p]; k < P->coll_begin[p + 1]; ++k) {
    double s, j;
    st.collective(P->coll_kind[k], P->coll_devices[k], P->coll_nodes[k],
                  P->coll_ppt[k] * total * P->coll_share[k], s, j);
    bs += s;
    bj += j * P->coll_groups[k];
  }
  const int S = P->num_stages[p];
  const double reps = double(P->stage_repetitions[p]);
  std::vector<double> ss(size_t(S), bs * reps), sj(size_t(S), bj * reps);
  for (int b = 0; b < P->p2p_begin[p + 1] - P->p2p_begin[p]; ++b) {
    double s, j;
    st.collective(PSG_COLL_P2P, 2, P->p2p_nodes[P->p2p_begin[p] + b],
                  P->p2p_payload_per_token[p] * total, s, j);
    ss[size_t(b) + 1] += s;
    sj[size_t(b) + 1] += j;
  }
  tf += bf * P->stage_devices[p] * reps * S;
  tb += bb * P->stage_devices[p] * reps * S;
  dur = 0.0;
  energy = 0.0;
  for (int i = 0; i < S; ++i) {
    dur = std::max(dur, ss[size_t(i)]);
    energy += sj[size_t(i)];
  }
}

struct ReplicaOut {
  double clock = 0, energy = 0;
  int64_t iterations = 0, max_batch = 0;
};

struct EntryResult {
  psg_entry e{};
  std::vector<psg_request_metrics> pr;
  std::vector<int64_t> rej;
};

// run_replica over BatchState (simulator.cpp:98-172, batching.cpp:11-125).
ReplicaOut run_replica(const Plan& pl, const Store& st, const psg_config* cfg,
                       double freq, std::vector<Req> reqs, double& tf, double& tb,
                       EntryResult& er) {
  const psg_plan_set* P = pl.P;
  const double kv = P->kv_bytes_per_token[pl.p];
  const double cap = P->kv_budget_per_replica[pl.p];
  std::stable_sort(reqs.begin(), reqs.end(),
                   [](const Req& a, const Req& b) { return a.arrival < b.arrival; });
  std::deque<Req> pending(reqs.begin(), reqs.end());
  std::vector<Act> active;
  std::map<int64_t, Req> by_id;
  for (const Req& r : reqs) by_id[r.id] = r;
  std::map<int64_t, double> first_token_at, admitted_at;
  const bool chunked = cfg->batch_mode == PSG_BATCH_CHUNKED;
  auto mem_used = [&]() {
    double u = 0.0;
    for (const Act& a : active) u += double(a.r.ctx + a.generated) * kv;
    return u;
  };
  ReplicaOut out;
  while (!(pending.empty() && active.empty())) {
    // admit
    double used = mem_used();
    while (!pending.empty() && pending.front().arrival <= out.clock) {
      const Req& h = pending.front();
      const double ckv = double(h.ctx) * kv;
      if (ckv > cap) {
        er.rej.push_back(h.id);
        pending.pop_front();
        continue;
      }
      if (cfg->max_batch_size > 0 && int64_t(active.size()) >= cfg->max_batch_size) break;
      if (used + ckv > cap) break;
      Act a;
      a.r = h;
      active.push_back(a);
      used += ckv;
      admitted_at[h.id] = out.clock;
      pending.pop_front();
    }
    if (active.empty()) {
      if (pending.empty()) break;
      out.clock = std::max(out.clock, pending.front().arrival);
      continue;
    }
    // step
    if (chunked && cfg->chunk_size < 1)
      throw DataErr("chunked prefill requires chunk_size >= 1");
    Workload w;
    for (const Act& a : active) {
      if (a.prefill) {
        int64_t tok = a.r.ctx - a.prefill_done;
        if (chunked) tok = std::min(tok, cfg->chunk_size);
        w.prefill.push_back(tok);
      } else {
        ++w.decode;
      }
    }
    std::vector<int64_t> prefilled, finished;
    for (Act& a : active) {
      if (a.prefill) {
        int64_t tok = a.r.ctx - a.prefill_done;
        if (chunked) tok = std::min(tok, cfg->chunk_size);
        a.prefill_done += tok;
        if (a.prefill_done == a.r.ctx) {
          a.prefill = false;
          a.generated = 1;
          prefilled.push_back(a.r.id);
        }
      } else {
        ++a.generated;
      }
    }
    for (auto it = active.begin(); it != active.end();) {
      if (!it->prefill && it->generated >= it->r.gen) {
        finished.push_back(it->r.id);
        it = active.erase(it);
      } else {
        ++it;
      }
    }
    std::vector<int64_t> evicted, rejected;
    while (active.size() > 1 && mem_used() > cap) {
      evicted.push_back(active.back().r.id);
      pending.push_front(active.back().r);
      active.pop_back();
    }
    if (active.size() == 1 && mem_used() > cap) {
      rejected.push_back(active.front().r.id);
      active.clear();
    }
    double dur, en;
    iteration_time(pl, st, freq, w, dur, en, tf, tb);
    out.clock += dur;
    out.energy += en;
    ++out.iterations;
    out.max_batch = std::max<int64_t>(out.max_batch, int64_t(w.prefill.size()) + w.decode);
    for (int64_t id : prefilled) first_token_at[id] = out.clock;
    for (int64_t id : evicted) {
      first_token_at.erase(id);
      admitted_at.erase(id);
    }
    for (int64_t id : rejected) er.rej.push_back(id);
    for (int64_t id : finished) {
      const Req& r = by_id.at(id);
      psg_request_metrics m{};
      m.id = id;
      m.gen_len = r.gen;
      m.e2e = out.clock - r.arrival;
      const double anchor =
          cfg->ttft_anchor == PSG_ANCHOR_ARRIVAL ? r.arrival : admitted_at.at(id);
      m.ttft = first_token_at.at(id) - anchor;
      if (r.gen >= 2) m.tpot = (out.clock - first_token_at.at(id)) / double(r.gen - 1);
      er.pr.push_back(m);
    }
  }
  return out;
}

double nearest(std::vector<double> v, double q) {
  std::sort(v.begin(), v.end());
  const size_t rank = size_t(std::ceil(q * double(v.size())));
  return v[std::min(v.size() - 1, rank == 0 ? 0 : rank - 1)];
}

// simulate_plan (simulator.cpp:176-240)
EntryResult simulate(const Plan& pl, const psg_cluster* cl, const psg_trace* T,
                     const Store& st, const psg_config* cfg, double freq) {
  const psg_plan_set* P = pl.P;
  EntryResult er;
  const size_t R = size_t(P->model_dp[pl.p]);
  std::vector<std::vector<Req>> split(R);
  for (int64_t i = 0; i < T->n; ++i)
    split[size_t(i) % R].push_back({T->id[i], T->context_len[i], T->gen_len[i], T->arrival[i]});
  double tf = 0.0, tb = 0.0;
  psg_entry& e = er.e;
  for (size_t r = 0; r < R; ++r) {
    const ReplicaOut o = run_replica(pl, st, cfg, freq, split[r], tf, tb, er);
    e.e2e_latency = std::max(e.e2e_latency, o.clock);
    e.total_energy += o.energy;
    e.num_iterations += o.iterations;
    e.max_batch_observed = std::max(e.max_batch_observed, o.max_batch);
  }
  std::sort(er.pr.begin(), er.pr.end(),
            [](const psg_request_metrics& a, const psg_request_metrics& b) { return a.id < b.id; });
  std::sort(er.rej.begin(), er.rej.end());
  e.num_completed = int64_t(er.pr.size());
  e.num_rejected = int64_t(er.rej.size());
  if (!er.pr.empty()) {
    std::vector<double> e2e, ttft, tpot;
    double ts = 0.0, ps = 0.0;
    int64_t pn = 0;
    for (const auto& m : er.pr) {
      e2e.push_back(m.e2e);
      ttft.push_back(m.ttft);
      ts += m.ttft;
      if (m.gen_len >= 2) {
        ps += m.tpot;
        tpot.push_back(m.tpot);
        ++pn;
      }
    }
    e.p95_latency = nearest(e2e, 0.95);
    e.mean_ttft = ts / double(er.pr.size());
    e.mean_tpot = pn > 0 ? ps / double(pn) : 0.0;
    e.p50_ttft = nearest(ttft, 0.50);
    e.p99_ttft = nearest(ttft, 0.99);
    if (!tpot.empty()) {
      e.p50_tpot = nearest(tpot, 0.50);
      e.p99_tpot = nearest(tpot, 0.99);
    }
    // TTFT-SLO-constrained ranking (psg.h psg_config.ttft_slo): nearest-rank
    // quantile of TTFT, the p95 rule of simulator.cpp:223-225
    if (cfg->ttft_slo > 0.0) {
      e.slo_ttft = nearest(ttft, cfg->slo_quantile > 0.0 ? cfg->slo_quantile : 0.99);
      e.slo_met = e.slo_ttft <= cfg->ttft_slo ? 1 : 0;
    }
  }
  if (e.e2e_latency > 0) {
    const int dt = P->compute_dtype[pl.p];
    const double pf = cl->peak_flops[dt];
    if (!(pf > 0)) throw DataErr("device has no peak_flops entry");
    const double peak = pf * cl->total_devices;
    e.mfu = tf / (e.e2e_latency * peak);
    e.mbu = tb / (e.e2e_latency * cl->peak_mem_bandwidth * cl->total_devices);
  }
  return er;
}

std::string g_err;

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

// Same contract as psg_search (entry subset honoured; result memory owned by
// the returned struct, released with oracle_result_free).
int oracle_search(const psg_plan_set* P, const psg_cluster* cl, const psg_store* S,
                  const psg_trace* T, const psg_config* cfg, psg_result** out) {
  *out = nullptr;
  g_err.clear();
  if (P->n_plans <= 0) {
    g_err = "search: no feasible plan";
    return PSG_ERR_INFEASIBLE;
  }
  std::vector<double> freqs(cfg->freqs, cfg->freqs + std::max(0, cfg->n_freqs));
  if (freqs.empty()) freqs.push_back(cl->max_frequency_ghz);
  const int64_t F = int64_t(freqs.size());
  std::vector<int64_t> ent;
  if (cfg->n_entry_subset > 0) {
    ent.assign(cfg->entry_subset, cfg->entry_subset + cfg->n_entry_subset);
  } else {
    ent.resize(size_t(P->n_plans * F));
    std::iota(ent.begin(), ent.end(), 0);
  }
  const Store st(S);
  std::vector<EntryResult> res;
  try {
    for (int64_t g : ent) {
      EntryResult er = simulate(Plan{P, int(g / F)}, cl, T, st, cfg, freqs[size_t(g % F)]);
      er.e.entry_index = g;
      er.e.plan_index = g / F;
      er.e.freq_ghz = freqs[size_t(g % F)];
      res.push_back(std::move(er));
    }
  } catch (const DataErr& e) {
    g_err = e.what();
    return PSG_ERR_DATA;
  }
  std::vector<size_t> order(res.size());
  std::iota(order.begin(), order.end(), 0);
  if (cfg->rank) {
    const bool lat = cfg->objective == PSG_OBJ_LATENCY;
    auto obj = [&](const psg_entry& e, bool l) { return l ? e.e2e_latency : e.total_energy; };
    // simulator.cpp:283-294 (encoding compared through its precomputed rank)
    std::sort(order.begin(), order.end(), [&](size_t ia, size_t ib) {
      const psg_entry& a = res[ia].e;
      const psg_entry& b = res[ib].e;
      if (a.slo_met != b.slo_met) return a.slo_met > b.slo_met;  // SLO met first (0 when off)
      if (a.num_rejected != b.num_rejected) return a.num_rejected < b.num_rejected;
      if (obj(a, lat) != obj(b, lat)) return obj(a, lat) < obj(b, lat);
      if (obj(a, !lat) != obj(b, !lat)) return obj(a, !lat) < obj(b, !lat);
      const int ra = P->enc_rank[a.plan_index], rb = P->enc_rank[b.plan_index];
      if (ra != rb) return ra < rb;
      if (a.freq_ghz != b.freq_ghz) return a.freq_ghz < b.freq_ghz;
      return a.entry_index < b.entry_index;
    });
  }
  auto* r = new psg_result();
  std::memset(r, 0, sizeof(*r));
  r->n_entries = int64_t(res.size());
  r->entries = new psg_entry[res.size() ? res.size() : 1];
  int64_t npr = 0, nrj = 0;
  for (const auto& er : res) {
    npr += int64_t(er.pr.size());
    nrj += int64_t(er.rej.size());
  }
  r->per_request = new psg_request_metrics[npr ? npr : 1];
  r->rejected_ids = new int64_t[nrj ? nrj : 1];
  int64_t a = 0, b = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    EntryResult& er = res[order[k]];
    er.e.per_request_offset = a;
    er.e.rejected_offset = b;
    r->entries[k] = er.e;
    std::copy(er.pr.begin(), er.pr.end(), r->per_request + a);
    std::copy(er.rej.begin(), er.rej.end(), r->rejected_ids + b);
    a += int64_t(er.pr.size());
    b += int64_t(er.rej.size());
    r->total_iterations += er.e.num_iterations;
  }
  r->n_per_request = a;
  r->n_rejected = b;
  *out = r;
  return PSG_OK;
}

void oracle_result_free(psg_result* r) {
  if (!r) return;
  delete[] r->entries;
  delete[] r->per_request;
  delete[] r->rejected_ids;
  delete r;
}

}  // extern "C"
