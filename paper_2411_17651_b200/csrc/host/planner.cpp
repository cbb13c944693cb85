// Plan enumeration, device mapping, collective resolution and the memory
// ledger: the producer of the engine's plan SoA.  Semantics follow
// /root/reference/proj/src/planner.cpp:15-418 (Alg. 1 of the APEX paper),
// verified field-for-field against the reference's plan dump in
// tests/test_host_planner.py.
#include <algorithm>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>

#include "nlohmann/json.hpp"
#include "psb/plansim_b200.hpp"

namespace psb {

const char* op_kind_str(OpKind k) {
  switch (k) {
    case OpKind::Attention: return "attention";
    case OpKind::GEMM: return "gemm";
    case OpKind::MoEGEMM: return "moe_gemm";
  }
  return "?";
}

const char* collective_kind_str(CollectiveKind k) {
  switch (k) {
    case CollectiveKind::AllReduce: return "allreduce";
    case CollectiveKind::AllGather: return "allgather";
    case CollectiveKind::ReduceScatter: return "reduce_scatter";
    case CollectiveKind::AllToAll: return "all_to_all";
    case CollectiveKind::P2P: return "p2p";
  }
  return "?";
}

bool template_valid(const CellSpec& cell, int devices, ParallelMode mode) {
  if (devices < 1) return false;
  if (mode == ParallelMode::EP)
    return cell.kind == CellKind::MoE && devices <= cell.num_experts &&
           cell.num_experts % devices == 0;
  const int granularity = cell.kind == CellKind::MoE ? cell.tp_slices : cell.num_tasks;
  return granularity % devices == 0;
}

namespace {

// Per-device weight bytes of one cell shard (planner.cpp:26-71).
double shard_weight_bytes(const CellSpec& cell, int devices, ParallelMode mode) {
  if (!template_valid(cell, devices, mode))
    throw DataError(std::string("template: cannot split ") + cell_kind_str(cell.kind) +
                    " cell across " + std::to_string(devices) + " devices");
  if (mode == ParallelMode::EP || cell.kind == CellKind::MoE || !cell.is_attention())
    return cell.weight_bytes() / devices;
  // query heads shard evenly; kv heads shard until the split outruns them,
  // after which every shard keeps one replicated kv head
  const int heads_here = cell.num_tasks / devices;
  const double kv_here = cell.kv_heads >= devices ? double(cell.kv_heads) / devices : 1.0;
  return heads_here * cell.qo_weight_bytes_per_task + kv_here * cell.kv_weight_bytes_per_kv_head;
}

CellScheme cell_scheme(const CellSpec& cell, ParallelMode mode, int cell_dp, int intra) {
  CellScheme s;
  s.cell = cell;
  s.mode = intra == 1 ? ParallelMode::TP : mode;  // EP over one device is TP
  s.cell_dp = cell_dp;
  s.intra_degree = intra;
  s.weight_bytes_per_device = shard_weight_bytes(cell, intra, s.mode);
  s.query_width = cell.task_width;
  const double token_split = 1.0 / cell_dp;
  if (cell.kind == CellKind::MoE) {
    s.op = OpKind::MoEGEMM;
    const double routing = double(cell.experts_per_token) / cell.num_experts;
    if (s.mode == ParallelMode::EP) {
      s.query_tasks = double(cell.num_experts) / intra;
      s.token_scale = token_split * routing;
    } else {  // every expert sliced 1/intra; the slice folds into the token axis
      s.query_tasks = double(cell.num_experts);
      s.token_scale = token_split * routing / intra;
    }
  } else {
    s.op = cell.is_attention() ? OpKind::Attention : OpKind::GEMM;
    s.query_tasks = double(cell.num_tasks) / intra;
    s.token_scale = token_split;
  }
  return s;
}

// Reshard collectives between adjacent cells (planner.cpp:121-152).
std::vector<CollectiveOp> reshard(const CellScheme& l, const CellScheme& r, const ModelSpec& m) {
  const double per_token = double(m.hidden_size) * m.activation_dtype.bytes_per_element;
  const bool l_ep = l.mode == ParallelMode::EP && l.intra_degree > 1;
  const bool r_ep = r.mode == ParallelMode::EP && r.intra_degree > 1;
  std::vector<CollectiveOp> ops;
  auto add = [&](CollectiveKind k, double share, GroupScope scope) {
    ops.push_back({k, per_token, share, scope});
  };
  if (l_ep) add(CollectiveKind::AllToAll, 1.0 / l.cell_dp, GroupScope::LeftIntra);
  if (r_ep) {
    add(CollectiveKind::AllToAll, 1.0 / r.cell_dp, GroupScope::RightIntra);
  } else if (l.cell_dp == r.cell_dp) {
    if (!l_ep && l.intra_degree > 1)
      add(CollectiveKind::AllReduce, 1.0 / l.cell_dp, GroupScope::LeftIntra);
  } else {
    add(CollectiveKind::AllToAll, 1.0, GroupScope::Stage);
    if (r.intra_degree > 1) add(CollectiveKind::AllGather, 1.0 / r.cell_dp, GroupScope::RightIntra);
  }
  return ops;
}

ParallelScheme assemble(const ModelSpec& m, const BlockSpec& block, int dp, int stages, int sdev,
                        std::vector<CellScheme> cells) {
  ParallelScheme s;
  s.model_dp = dp;
  s.num_stages = stages;
  s.stage_devices = sdev;
  s.stage_repetitions = block.repeat_count / stages;
  std::ostringstream enc;
  enc << "dp" << dp << ":pp" << stages;
  for (size_t i = 0; i < cells.size(); ++i) {
    const CellScheme& c = cells[i];
    enc << ":" << cell_kind_str(c.cell.kind) << (c.mode == ParallelMode::EP ? "-ep" : "-tp")
        << c.intra_degree << "x" << c.cell_dp;
    s.reshards.push_back(reshard(c, cells[(i + 1) % cells.size()], m));
  }
  s.cells = std::move(cells);
  s.encoding = enc.str();
  return s;
}

struct Span {
  int devices = 0, nodes = 0, level = 0;
};

Span group_span(const ClusterSpec& cl, const std::vector<int>& ids) {
  Span s;
  s.devices = int(ids.size());
  const int per_node = cl.devices_per_node();
  std::set<int> nodes;
  for (int id : ids) nodes.insert(id / per_node);
  s.nodes = int(nodes.size());
  s.level = cl.num_levels();
  for (int level = 0; level <= cl.num_levels(); ++level) {
    const int cap = cl.subtree_capacity(level);
    if (std::all_of(ids.begin(), ids.end(), [&](int id) { return id / cap == ids.front() / cap; })) {
      s.level = level;
      break;
    }
  }
  return s;
}

ExecutionPlan finalize(const ModelSpec& m, const ParallelScheme& scheme, const ClusterSpec& cl,
                       const PlanOptions& opts) {
  ExecutionPlan plan;
  plan.scheme = scheme;
  plan.assignment = map_devices(scheme.model_dp, scheme.num_stages, scheme.stage_devices, cl);
  plan.compute_dtype = m.activation_dtype.name;
  plan.op_shape.model_hidden = m.hidden_size;
  plan.op_shape.head_dim = m.head_dim;
  plan.op_shape.kv_elems_per_task_token =
      2.0 * m.head_dim / (m.num_attention_heads / double(m.num_kv_heads));
  plan.p2p_payload_per_token = double(m.hidden_size) * m.activation_dtype.bytes_per_element;

  const size_t nc = scheme.cells.size();
  for (size_t i = 0; i < nc; ++i) {
    const CellScheme& l = scheme.cells[i];
    const CellScheme& r = scheme.cells[(i + 1) % nc];
    for (const CollectiveOp& op : scheme.reshards[i]) {
      const int gsize = op.scope == GroupScope::LeftIntra    ? l.intra_degree
                        : op.scope == GroupScope::RightIntra ? r.intra_degree
                                                             : scheme.stage_devices;
      if (gsize < 2) continue;  // single-device group: elided
      ResolvedCollective rc;
      rc.kind = op.kind;
      rc.payload_bytes_per_token = op.payload_bytes_per_token;
      rc.token_share = op.token_share;
      rc.groups_per_stage = scheme.stage_devices / gsize;
      // worst span over every concrete group instance (planner.cpp:251-274)
      Span worst;
      bool first = true;
      std::vector<int> ids(static_cast<size_t>(gsize));
      for (int rep = 0; rep < scheme.model_dp; ++rep)
        for (int st = 0; st < scheme.num_stages; ++st)
          for (int g = 0; g < rc.groups_per_stage; ++g) {
            for (int j = 0; j < gsize; ++j)
              ids[size_t(j)] = plan.assignment.device_of(rep, st, g * gsize + j);
            const Span s = group_span(cl, ids);
            if (first || s.level > worst.level || (s.level == worst.level && s.nodes > worst.nodes)) {
              worst = s;
              first = false;
            }
          }
      rc.num_devices = worst.devices;
      rc.num_nodes = worst.nodes;
      if (rc.num_devices >= 2) plan.block_collectives.push_back(rc);
    }
  }

  const int per_node = cl.devices_per_node();
  for (int b = 0; b + 1 < scheme.num_stages; ++b) {
    const int a = plan.assignment.device_of(0, b, 0), c = plan.assignment.device_of(0, b + 1, 0);
    plan.p2p_boundary_nodes.push_back(a / per_node == c / per_node ? 1 : 2);
  }

  double per_device = 0.0;
  for (const auto& cs : scheme.cells) per_device += cs.weight_bytes_per_device;
  per_device *= scheme.stage_repetitions;
  const double emb = opts.include_embedding ? embedding_weight_bytes(m) : 0.0;
  double last_stage = per_device;
  if (opts.include_embedding) last_stage += emb / scheme.stage_devices;
  plan.static_bytes_per_device = std::max(per_device, last_stage);
  const int replica_devices = scheme.num_stages * scheme.stage_devices;
  const double replica_static =
      per_device * replica_devices + (opts.include_embedding ? emb : 0.0);
  const double replica_capacity = cl.device.memory_capacity * replica_devices;
  plan.kv_budget_per_replica =
      std::max(0.0, replica_capacity * (1.0 - opts.activation_reserve) - replica_static);
  double per_layer = 0.0;
  for (const auto& cs : scheme.cells) {
    if (!cs.cell.is_attention()) continue;
    const double kv_instances = std::max(double(cs.cell.kv_heads), double(cs.intra_degree));
    per_layer += 2.0 * cs.cell.head_dim * kv_instances * m.kv_cache_dtype.bytes_per_element;
  }
  plan.kv_bytes_per_token = per_layer * m.num_layers;
  return plan;
}

}  // namespace

std::vector<ParallelScheme> enumerate_schemes(const ModelSpec& m, const BlockSpec& block, int n,
                                              int max_combos) {
  std::vector<ParallelScheme> out;
  std::set<std::string> seen;
  if (n < 1 || block.repeat_count < 1) return out;
  for (const int dp : divisors(n)) {
    const int per_replica = n / dp;
    for (const int stages : divisors(per_replica)) {
      if (stages > block.repeat_count || block.repeat_count % stages) continue;
      const int s = per_replica / stages;
      std::vector<std::vector<CellScheme>> choices(block.cells.size());
      bool viable = true;
      for (size_t ci = 0; ci < block.cells.size() && viable; ++ci) {
        for (const int cdp : divisors(s)) {
          const int intra = s / cdp;
          if (template_valid(block.cells[ci], intra, ParallelMode::TP))
            choices[ci].push_back(cell_scheme(block.cells[ci], ParallelMode::TP, cdp, intra));
          if (intra > 1 && template_valid(block.cells[ci], intra, ParallelMode::EP))
            choices[ci].push_back(cell_scheme(block.cells[ci], ParallelMode::EP, cdp, intra));
        }
        viable = !choices[ci].empty();
      }
      if (!viable) continue;
      long long combos = 1;
      for (const auto& c : choices) combos *= (long long)c.size();
      if (combos > max_combos) {
        std::cerr << "warning: capping cell-scheme combinations at " << max_combos << " (of "
                  << combos << ") for dp=" << dp << " stages=" << stages << "\n";
        combos = max_combos;
      }
      // mixed-radix counter over the per-cell choices, last cell fastest
      std::vector<size_t> digit(block.cells.size(), 0);
      for (long long k = 0; k < combos; ++k) {
        std::vector<CellScheme> cells;
        for (size_t ci = 0; ci < digit.size(); ++ci) cells.push_back(choices[ci][digit[ci]]);
        ParallelScheme sch = assemble(m, block, dp, stages, s, std::move(cells));
        if (seen.insert(sch.encoding).second) out.push_back(std::move(sch));
        for (size_t ci = digit.size(); ci-- > 0;) {
          if (++digit[ci] < choices[ci].size()) break;
          digit[ci] = 0;
        }
      }
    }
  }
  return out;
}

std::vector<ExecutionPlan> generate_plans(const ModelSpec& m, const BlockSpec& block,
                                          const ClusterSpec& cl, const PlanOptions& opts) {
  std::vector<ExecutionPlan> plans;
  for (const auto& sch : enumerate_schemes(m, block, cl.total_devices(), opts.max_cell_combinations)) {
    ExecutionPlan p = finalize(m, sch, cl, opts);
    if (p.static_bytes_per_device <= cl.device.memory_capacity) plans.push_back(std::move(p));
  }
  if (plans.empty()) throw InfeasibleError("no parallel execution plan fits the model on this cluster");
  return plans;
}

namespace {

// The candidate space generate_plans enumerates (groups in enumerate_schemes
// order, per-cell scheme choices, last cell fastest) flattened for the plan
// kernels (psg_plan_space), with the storage its pointers refer to.
struct PlanSpace {
  struct Group {
    int dp, stages, sdev;
    std::vector<std::vector<CellScheme>> choices;
    long long combos;
  };
  std::vector<Group> groups;
  std::vector<int32_t> subtree, att, gdp, gst, gsd, grp, cb, cm, cd, ci_;
  std::vector<double> kvh, hd, cw;
  std::vector<int64_t> gfirst{0}, p2p_off{0};
  psg_plan_space sp{};
};

void build_space(const ModelSpec& m, const BlockSpec& block, const ClusterSpec& cl,
                 const PlanOptions& opts, PlanSpace& S) {
  const int n = cl.total_devices();
  const int nc = int(block.cells.size());
  if (nc < 1 || nc > PSG_PLAN_MAX_CELLS) throw DataError("plan space: unsupported cell count");
  using Group = PlanSpace::Group;
  std::vector<Group>& groups = S.groups;
  if (n >= 1 && block.repeat_count >= 1) {
    for (const int dp : divisors(n)) {
      const int per_replica = n / dp;
      for (const int stages : divisors(per_replica)) {
        if (stages > block.repeat_count || block.repeat_count % stages) continue;
        const int sd = per_replica / stages;
        Group g{dp, stages, sd, std::vector<std::vector<CellScheme>>(static_cast<size_t>(nc)), 1};
        bool viable = true;
        for (int ci = 0; ci < nc && viable; ++ci) {
          for (const int cdp : divisors(sd)) {
            const int intra = sd / cdp;
            if (template_valid(block.cells[size_t(ci)], intra, ParallelMode::TP))
              g.choices[size_t(ci)].push_back(cell_scheme(block.cells[size_t(ci)], ParallelMode::TP, cdp, intra));
            if (intra > 1 && template_valid(block.cells[size_t(ci)], intra, ParallelMode::EP))
              g.choices[size_t(ci)].push_back(cell_scheme(block.cells[size_t(ci)], ParallelMode::EP, cdp, intra));
          }
          viable = !g.choices[size_t(ci)].empty();
        }
        if (!viable) continue;
        for (const auto& c : g.choices) g.combos *= (long long)c.size();
        if (g.combos > opts.max_cell_combinations) {
          std::cerr << "warning: capping cell-scheme combinations at " << opts.max_cell_combinations
                    << " (of " << g.combos << ") for dp=" << dp << " stages=" << stages << "\n";
          g.combos = opts.max_cell_combinations;
        }
        groups.push_back(std::move(g));
      }
    }
  }
  const int G = int(groups.size());
  auto& subtree = S.subtree;
  auto& att = S.att;
  auto& kvh = S.kvh;
  auto& hd = S.hd;
  auto &gdp = S.gdp, &gst = S.gst, &gsd = S.gsd, &grp = S.grp, &cb = S.cb, &cm = S.cm, &cd = S.cd,
       &ci_ = S.ci_;
  auto& cw = S.cw;
  auto &gfirst = S.gfirst, &p2p_off = S.p2p_off;
  subtree.resize(static_cast<size_t>(cl.num_levels()) + 1);
  att.resize(static_cast<size_t>(nc));
  kvh.resize(static_cast<size_t>(nc));
  hd.resize(static_cast<size_t>(nc));
  for (int l = 0; l <= cl.num_levels(); ++l) subtree[size_t(l)] = cl.subtree_capacity(l);
  for (int i = 0; i < nc; ++i) {
    att[size_t(i)] = block.cells[size_t(i)].is_attention() ? 1 : 0;
    kvh[size_t(i)] = double(block.cells[size_t(i)].kv_heads);
    hd[size_t(i)] = block.cells[size_t(i)].head_dim;
  }
  for (const Group& g : groups) {
    gdp.push_back(g.dp);
    gst.push_back(g.stages);
    gsd.push_back(g.sdev);
    grp.push_back(block.repeat_count / g.stages);
    gfirst.push_back(gfirst.back() + g.combos);
    p2p_off.push_back(p2p_off.back() + (g.stages - 1));
    for (const auto& opts_c : g.choices) {
      cb.push_back(int32_t(cm.size()));
      for (const CellScheme& c : opts_c) {
        cm.push_back(c.mode == ParallelMode::EP ? 1 : 0);
        cd.push_back(c.cell_dp);
        ci_.push_back(c.intra_degree);
        cw.push_back(c.weight_bytes_per_device);
      }
    }
  }
  cb.push_back(int32_t(cm.size()));
  psg_plan_space& sp = S.sp;
  sp.n_devices = n;
  sp.per_node = cl.devices_per_node();
  sp.n_levels = cl.num_levels();
  sp.subtree_cap = subtree.data();
  sp.memory_capacity = cl.device.memory_capacity;
  sp.activation_reserve = opts.activation_reserve;
  sp.emb_bytes = embedding_weight_bytes(m);
  sp.kv_elem_bytes = m.kv_cache_dtype.bytes_per_element;
  sp.include_embedding = opts.include_embedding ? 1 : 0;
  sp.num_layers = m.num_layers;
  sp.n_cells = nc;
  sp.cell_is_attention = att.data();
  sp.cell_kv_heads = kvh.data();
  sp.cell_head_dim = hd.data();
  sp.n_groups = G;
  sp.group_dp = gdp.data();
  sp.group_stages = gst.data();
  sp.group_sdev = gsd.data();
  sp.group_reps = grp.data();
  sp.group_first = gfirst.data();
  sp.choice_begin = cb.data();
  sp.ch_mode = cm.data();
  sp.ch_cdp = cd.data();
  sp.ch_intra = ci_.data();
  sp.ch_weight = cw.data();
}

}  // namespace

std::vector<ExecutionPlan> generate_plans_device(const ModelSpec& m, const BlockSpec& block,
                                                 const ClusterSpec& cl, const PlanOptions& opts,
                                                 Engine* engine) {
  // Candidate groups and per-cell choices exactly as enumerate_schemes lists
  // them; the device maps every group and finalizes every candidate.
  PlanSpace S;
  build_space(m, block, cl, opts, S);
  const int n = cl.total_devices();
  const int nc = int(block.cells.size());
  const int G = int(S.groups.size());
  const auto& groups = S.groups;
  const auto& gfirst = S.gfirst;
  const auto& p2p_off = S.p2p_off;
  psg_plan_space& sp = S.sp;
  std::vector<psg_plan_record> rec(static_cast<size_t>(std::max<int64_t>(gfirst.back(), 1)));
  std::vector<int32_t> phys(static_cast<size_t>(std::max(G, 1)) * static_cast<size_t>(n));
  std::vector<int32_t> p2p(static_cast<size_t>(std::max<int64_t>(p2p_off.back(), 1)));
  std::unique_ptr<Engine> own;
  if (!engine) {
    own = std::make_unique<Engine>(0);
    engine = own.get();
  }
  if (G > 0) {
    const int rc = psg_plan_compute(engine->handle(), &sp, rec.data(), phys.data(), p2p_off.data(), p2p.data());
    if (rc != PSG_OK) throw DataError(std::string("plan space on device: ") + psg_last_error(engine->handle()));
  }
  std::vector<ExecutionPlan> plans;
  std::set<std::string> seen;
  const double per_token = double(m.hidden_size) * m.activation_dtype.bytes_per_element;
  for (int gi = 0; gi < G; ++gi) {
    const PlanSpace::Group& g = groups[size_t(gi)];
    std::vector<size_t> digit(static_cast<size_t>(nc), 0);
    for (long long k = 0; k < g.combos; ++k) {
      std::vector<CellScheme> cells;
      for (int c = 0; c < nc; ++c) cells.push_back(g.choices[size_t(c)][digit[size_t(c)]]);
      ParallelScheme sch = assemble(m, block, g.dp, g.stages, g.sdev, std::move(cells));
      const psg_plan_record& r = rec[size_t(gfirst[size_t(gi)] + k)];
      if (seen.insert(sch.encoding).second && r.feasible) {
        ExecutionPlan p;
        p.scheme = std::move(sch);
        p.assignment.model_dp = g.dp;
        p.assignment.num_stages = g.stages;
        p.assignment.stage_devices = g.sdev;
        p.assignment.phys.assign(phys.begin() + size_t(gi) * n, phys.begin() + size_t(gi + 1) * n);
        p.compute_dtype = m.activation_dtype.name;
        p.op_shape.model_hidden = m.hidden_size;
        p.op_shape.head_dim = m.head_dim;
        p.op_shape.kv_elems_per_task_token = 2.0 * m.head_dim / (m.num_attention_heads / double(m.num_kv_heads));
        p.p2p_payload_per_token = per_token;
        for (int q = 0; q < r.n_colls; ++q) {
          ResolvedCollective rc;
          rc.kind = CollectiveKind(r.coll_kind[q]);
          rc.payload_bytes_per_token = per_token;
          rc.token_share = r.coll_share[q];
          rc.num_devices = r.coll_devices[q];
          rc.num_nodes = r.coll_nodes[q];
          rc.groups_per_stage = r.coll_groups[q];
          p.block_collectives.push_back(rc);
        }
        p.p2p_boundary_nodes.assign(p2p.begin() + p2p_off[size_t(gi)], p2p.begin() + p2p_off[size_t(gi) + 1]);
        p.static_bytes_per_device = r.static_bytes_per_device;
        p.kv_budget_per_replica = r.kv_budget_per_replica;
        p.kv_bytes_per_token = r.kv_bytes_per_token;
        plans.push_back(std::move(p));
      }
      for (size_t c = digit.size(); c-- > 0;) {
        if (++digit[c] < g.choices[c].size()) break;
        digit[c] = 0;
      }
    }
  }
  if (plans.empty()) throw InfeasibleError("no parallel execution plan fits the model on this cluster");
  return plans;
}

DevicePlanSet::~DevicePlanSet() {
  if (soa) psg_plan_soa_free(soa);
}

std::unique_ptr<DevicePlanSet> generate_plans_direct(const ModelSpec& m, const BlockSpec& block,
                                                     const ClusterSpec& cl, const PlanOptions& opts,
                                                     Engine* engine) {
  PlanSpace S;
  build_space(m, block, cl, opts, S);
  const int nc = int(block.cells.size());
  const int64_t total = S.gfirst.back();
  // host-side per candidate: its encoding (assemble's format, planner.cpp:111-129
  // here) -> first-occurrence flag and rank; per choice: the CellScheme query
  // constants, in build_space's choice order
  std::vector<std::string> enc(static_cast<size_t>(total));
  std::vector<int32_t> ch_op;
  std::vector<double> ch_t, ch_w, ch_s;
  int64_t k0 = 0;
  for (const auto& g : S.groups) {
    for (const auto& opts_c : g.choices)
      for (const CellScheme& c : opts_c) {
        ch_op.push_back(int32_t(c.op));
        ch_t.push_back(c.query_tasks);
        ch_w.push_back(c.query_width);
        ch_s.push_back(c.token_scale);
      }
    std::vector<size_t> digit(static_cast<size_t>(nc), 0);
    for (long long k = 0; k < g.combos; ++k) {
      std::string e = "dp" + std::to_string(g.dp) + ":pp" + std::to_string(g.stages);
      for (int c = 0; c < nc; ++c) {
        const CellScheme& cs = g.choices[size_t(c)][digit[size_t(c)]];
        e += ":";
        e += cell_kind_str(cs.cell.kind);
        e += cs.mode == ParallelMode::EP ? "-ep" : "-tp";
        e += std::to_string(cs.intra_degree) + "x" + std::to_string(cs.cell_dp);
      }
      enc[size_t(k0 + k)] = std::move(e);
      for (size_t c = digit.size(); c-- > 0;) {
        if (++digit[c] < g.choices[c].size()) break;
        digit[c] = 0;
      }
    }
    k0 += g.combos;
  }
  std::vector<uint8_t> keep(static_cast<size_t>(std::max<int64_t>(total, 1)), 0);
  std::vector<int32_t> rank(static_cast<size_t>(std::max<int64_t>(total, 1)), 0);
  {
    std::vector<std::string> uniq(enc);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    std::set<std::string> seen;
    for (int64_t k = 0; k < total; ++k) {
      keep[size_t(k)] = seen.insert(enc[size_t(k)]).second ? 1 : 0;
      rank[size_t(k)] = int32_t(std::lower_bound(uniq.begin(), uniq.end(), enc[size_t(k)]) - uniq.begin());
    }
  }
  psg_plan_emit_in in{};
  in.keep = keep.data();
  in.enc_rank = rank.data();
  in.ch_op = ch_op.empty() ? nullptr : ch_op.data();
  in.ch_tasks = ch_t.empty() ? nullptr : ch_t.data();
  in.ch_width = ch_w.empty() ? nullptr : ch_w.data();
  in.ch_scale = ch_s.empty() ? nullptr : ch_s.data();
  in.compute_dtype = int32_t(m.activation_dtype.name);
  in.payload_per_token = double(m.hidden_size) * m.activation_dtype.bytes_per_element;
  in.shape_hidden = m.hidden_size;
  in.shape_head_dim = m.head_dim;
  in.shape_kv_elems = 2.0 * m.head_dim / (m.num_attention_heads / double(m.num_kv_heads));
  std::unique_ptr<Engine> own;
  if (!engine) {
    own = std::make_unique<Engine>(0);
    engine = own.get();
  }
  auto out = std::make_unique<DevicePlanSet>();
  const int rc = total > 0 ? psg_plan_emit(engine->handle(), &S.sp, &in, &out->soa) : PSG_ERR_INFEASIBLE;
  if (rc == PSG_ERR_INFEASIBLE)
    throw InfeasibleError("no parallel execution plan fits the model on this cluster");
  if (rc != PSG_OK) throw DataError(std::string("plan space on device: ") + psg_last_error(engine->handle()));
  for (int i = 0; i < out->soa->set.n_plans; ++i) out->encodings.push_back(enc[size_t(out->soa->candidate[i])]);
  // the device wrote ranks among every candidate's encoding; PlanSoA ranks
  // among the plans kept (the same order, other integers): use those, so the
  // two plan sets are identical array for array
  std::vector<std::string> uniq(out->encodings);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  auto* er = const_cast<int32_t*>(out->soa->set.enc_rank);  // library-owned host array
  for (size_t i = 0; i < out->encodings.size(); ++i)
    er[i] = int32_t(std::lower_bound(uniq.begin(), uniq.end(), out->encodings[i]) - uniq.begin());
  return out;
}

ExecutionPlan build_plan(const ModelSpec& m, const BlockSpec& block, const ClusterSpec& cl,
                         int dp, int stages, const std::vector<CellChoice>& choices,
                         const PlanOptions& opts) {
  const int n = cl.total_devices();
  if (dp < 1 || stages < 1 || n % (dp * stages) != 0)
    throw DataError("plan: degrees do not divide the cluster device count");
  const int s = n / (dp * stages);
  if (block.repeat_count % stages != 0)
    throw DataError("plan: stage count does not divide the layer count");
  if (choices.size() != block.cells.size())
    throw DataError("plan: cell scheme count does not match the block");
  std::vector<CellScheme> cells;
  for (size_t i = 0; i < choices.size(); ++i) {
    const CellChoice& ch = choices[i];
    if (ch.cell_dp * ch.intra_degree != s)
      throw DataError("plan: cell_dp * intra_degree must equal stage devices");
    if (!template_valid(block.cells[i], ch.intra_degree, ch.mode))
      throw DataError("plan: invalid template for cell " +
                      std::string(cell_kind_str(block.cells[i].kind)));
    cells.push_back(cell_scheme(block.cells[i], ch.mode, ch.cell_dp, ch.intra_degree));
  }
  return finalize(m, assemble(m, block, dp, stages, s, std::move(cells)), cl, opts);
}

std::string plans_to_json(const std::vector<ExecutionPlan>& plans) {
  using oj = nlohmann::ordered_json;
  oj arr = oj::array();
  for (const auto& p : plans) {
    oj d;
    d["encoding"] = p.scheme.encoding;
    d["model_dp"] = p.scheme.model_dp;
    d["num_stages"] = p.scheme.num_stages;
    d["stage_devices"] = p.scheme.stage_devices;
    d["stage_repetitions"] = p.scheme.stage_repetitions;
    d["compute_dtype"] = int(p.compute_dtype);
    d["kv_bytes_per_token"] = p.kv_bytes_per_token;
    d["kv_budget_per_replica"] = p.kv_budget_per_replica;
    d["static_bytes_per_device"] = p.static_bytes_per_device;
    d["p2p_payload_per_token"] = p.p2p_payload_per_token;
    d["shape"] = {p.op_shape.model_hidden, p.op_shape.head_dim, p.op_shape.kv_elems_per_task_token};
    d["cells"] = oj::array();
    for (const auto& c : p.scheme.cells)
      d["cells"].push_back({{"kind", int(c.cell.kind)},
                            {"mode", int(c.mode)},
                            {"cell_dp", c.cell_dp},
                            {"intra_degree", c.intra_degree},
                            {"op", int(c.op)},
                            {"query_tasks", c.query_tasks},
                            {"query_width", c.query_width},
                            {"token_scale", c.token_scale},
                            {"weight_bytes_per_device", c.weight_bytes_per_device}});
    d["collectives"] = oj::array();
    for (const auto& rc : p.block_collectives)
      d["collectives"].push_back({{"kind", int(rc.kind)},
                                  {"payload_bytes_per_token", rc.payload_bytes_per_token},
                                  {"token_share", rc.token_share},
                                  {"num_devices", rc.num_devices},
                                  {"num_nodes", rc.num_nodes},
                                  {"groups_per_stage", rc.groups_per_stage}});
    d["p2p_boundary_nodes"] = p.p2p_boundary_nodes;
    d["assignment"] = p.assignment.phys;
    arr.push_back(d);
  }
  return arr.dump() + "\n";
}

}  // namespace psb
