// Profile store: JSONL load / serialize, grid finalization into the engine's
// flat tables, and the analytical roofline synthesizer.  Semantics follow
// /root/reference/proj/src/cost.cpp:51-176, :307-509; the serialized text is
// byte-compared with the reference's in tests/test_host_inputs.py.
#include <algorithm>
#include <cmath>
#include <memory>
#include <set>
#include <sstream>

#include "nlohmann/json.hpp"
#include "psb/plansim_b200.hpp"

namespace psb {

namespace {
long long micro(double freq_ghz) { return llround(freq_ghz * 1e6); }

OpKind op_from(const std::string& s) {
  if (s == "attention") return OpKind::Attention;
  if (s == "gemm") return OpKind::GEMM;
  if (s == "moe_gemm") return OpKind::MoEGEMM;
  throw DataError("unknown compute op: " + s);
}
CollectiveKind coll_from(const std::string& s) {
  for (auto k : {CollectiveKind::AllReduce, CollectiveKind::AllGather, CollectiveKind::ReduceScatter,
                 CollectiveKind::AllToAll, CollectiveKind::P2P})
    if (s == collective_kind_str(k)) return k;
  throw DataError("unknown collective op: " + s);
}
}  // namespace

double op_flops(OpKind op, double t, double k, double w, const OpShape& s) {
  double f = 2.0 * t * k * s.model_hidden * w;
  if (op == OpKind::Attention) f += 4.0 * t * t * k * s.head_dim;
  return f;
}

double op_bytes(OpKind op, double t, double k, double w, const OpShape& s, double e) {
  double b = k * s.model_hidden * w * e;
  b += 2.0 * t * s.model_hidden * e;
  if (op == OpKind::Attention) b += t * k * s.kv_elems_per_task_token * e;
  return b;
}

double kv_bytes_per_token(const ModelSpec& m) {
  return 2.0 * m.num_layers * m.num_kv_heads * m.head_dim * m.kv_cache_dtype.bytes_per_element;
}

void ProfileStore::add_compute_entry(OpKind op, Dtype dt, double freq, double ctx, double tasks,
                                     double width, double seconds, double joules) {
  if (seconds < 0 || joules < 0) throw DataError("profile: negative time or energy entry");
  auto& grid = pend_c_[CKey{int(op), int(dt), micro(freq)}];
  if (!grid.emplace(std::array<double, 3>{ctx, tasks, width}, std::make_pair(seconds, joules)).second)
    throw DataError(std::string("profile: duplicate knot in compute table ") + op_kind_str(op));
}

void ProfileStore::add_collective_entry(CollectiveKind kind, int devices, int nodes, double payload,
                                        double seconds, double joules) {
  if (seconds < 0 || joules < 0) throw DataError("profile: negative time or energy entry");
  if (devices < 2) throw DataError("profile: collective with < 2 devices");
  auto& curve = pend_k_[KKey{int(kind), devices, nodes}];
  if (!curve.emplace(payload, std::make_pair(seconds, joules)).second)
    throw DataError(std::string("profile: duplicate knot in collective table ") +
                    collective_kind_str(kind));
}

void ProfileStore::finalize() {
  for (auto* v : {&c_op_, &c_dt_, &c_nc_, &c_nt_, &c_nw_, &k_kind_, &k_dev_, &k_nodes_, &k_n_}) v->clear();
  for (auto* v : {&c_fm_, &c_kb_, &c_vb_, &k_b_}) v->clear();
  for (auto* v : {&c_knots_, &c_sec_, &c_jou_, &k_pay_, &k_sec_, &k_jou_}) v->clear();
  for (const auto& [key, entries] : pend_c_) {
    std::set<double> axes[3];
    for (const auto& kv : entries)
      for (int a = 0; a < 3; ++a) axes[a].insert(kv.first[size_t(a)]);
    const size_t nc = axes[0].size(), nt = axes[1].size(), nw = axes[2].size();
    if (entries.size() != nc * nt * nw)
      throw DataError(std::string("profile: compute table ") +
                      op_kind_str(OpKind(std::get<0>(key))) + " is not a complete grid");
    c_op_.push_back(std::get<0>(key));
    c_dt_.push_back(std::get<1>(key));
    c_fm_.push_back(std::get<2>(key));
    c_nc_.push_back(int32_t(nc));
    c_nt_.push_back(int32_t(nt));
    c_nw_.push_back(int32_t(nw));
    c_kb_.push_back(int64_t(c_knots_.size()));
    c_vb_.push_back(int64_t(c_sec_.size()));
    std::vector<double> ax[3];
    for (int a = 0; a < 3; ++a) {
      ax[a].assign(axes[a].begin(), axes[a].end());
      c_knots_.insert(c_knots_.end(), ax[a].begin(), ax[a].end());
    }
    // std::map iterates the (ctx, tasks, width) keys lexicographically, which
    // is exactly row-major order of the complete grid
    for (const auto& kv : entries) {
      c_sec_.push_back(kv.second.first);
      c_jou_.push_back(kv.second.second);
    }
  }
  for (const auto& [key, curve] : pend_k_) {
    k_kind_.push_back(std::get<0>(key));
    k_dev_.push_back(std::get<1>(key));
    k_nodes_.push_back(std::get<2>(key));
    k_n_.push_back(int32_t(curve.size()));
    k_b_.push_back(int64_t(k_pay_.size()));
    for (const auto& [pay, v] : curve) {
      k_pay_.push_back(pay);
      k_sec_.push_back(v.first);
      k_jou_.push_back(v.second);
    }
  }
}

void ProfileStore::rebind() const {
  auto nz = [](const auto& v) { return v.empty() ? nullptr : v.data(); };
  view_ = psg_store{};
  view_.n_compute = int32_t(c_op_.size());
  view_.c_op = nz(c_op_);
  view_.c_dtype = nz(c_dt_);
  view_.c_freq_micro = nz(c_fm_);
  view_.c_n_ctx = nz(c_nc_);
  view_.c_n_tasks = nz(c_nt_);
  view_.c_n_width = nz(c_nw_);
  view_.c_knot_begin = nz(c_kb_);
  view_.c_value_begin = nz(c_vb_);
  view_.c_knots = nz(c_knots_);
  view_.c_seconds = nz(c_sec_);
  view_.c_joules = nz(c_jou_);
  view_.n_curves = int32_t(k_kind_.size());
  view_.k_kind = nz(k_kind_);
  view_.k_devices = nz(k_dev_);
  view_.k_nodes = nz(k_nodes_);
  view_.k_n = nz(k_n_);
  view_.k_begin = nz(k_b_);
  view_.k_payload = nz(k_pay_);
  view_.k_seconds = nz(k_sec_);
  view_.k_joules = nz(k_jou_);
}

bool ProfileStore::has_compute_table(OpKind op, Dtype dt, double freq) const {
  return pend_c_.count(CKey{int(op), int(dt), micro(freq)}) > 0;
}

void ProfileStore::record_clamps(const uint8_t* cbits, const uint8_t* kbits) const {
  static const char* axis[3] = {"context_tokens", "tasks", "hidden_dim"};
  auto warn = [&](const std::string& key) {
    if (std::find(warn_keys_.begin(), warn_keys_.end(), key) != warn_keys_.end()) return;
    warn_keys_.push_back(key);
    warnings_.push_back("query outside profiled grid, clamped (" + key + ")");
  };
  for (int t = 0; t < int(c_op_.size()); ++t)
    for (int b = 0; b < 6; ++b)
      if (cbits[t] >> b & 1) {
        std::ostringstream ss;
        ss << "compute:" << op_kind_str(OpKind(c_op_[size_t(t)])) << ":"
           << DtypeFormat{Dtype(c_dt_[size_t(t)]), 0}.str() << ":" << c_fm_[size_t(t)] << ":"
           << axis[b / 2] << ":" << (b % 2 ? "above" : "below");
        warn(ss.str());
      }
  for (int u = 0; u < int(k_kind_.size()); ++u)
    for (int b = 0; b < 2; ++b)
      if (kbits[u] >> b & 1) {
        std::ostringstream ss;
        ss << "collective:" << collective_kind_str(CollectiveKind(k_kind_[size_t(u)])) << ":"
           << k_dev_[size_t(u)] << ":" << k_nodes_[size_t(u)] << ":payload:"
           << (b ? "above" : "below");
        warn(ss.str());
      }
}

ProfileStore ProfileStore::load(const std::string& text) {
  ProfileStore store;
  std::istringstream in(text);
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    nlohmann::json rec;
    try {
      rec = nlohmann::json::parse(line);
      const std::string table = rec.at("table").get<std::string>();
      const auto& axes = rec.at("axes");
      const double sec = rec.at("seconds").get<double>(), jou = rec.at("joules").get<double>();
      if (table == "compute") {
        store.add_compute_entry(op_from(rec.at("op").get<std::string>()),
                                DtypeFormat::from_string(rec.at("dtype").get<std::string>()).name,
                                rec.at("freq_ghz").get<double>(),
                                axes.at("context_tokens").get<double>(),
                                axes.at("tasks").get<double>(), axes.at("hidden_dim").get<double>(),
                                sec, jou);
      } else if (table == "collective") {
        store.add_collective_entry(coll_from(rec.at("op").get<std::string>()),
                                   axes.at("num_devices").get<int>(), axes.at("num_nodes").get<int>(),
                                   axes.at("payload_bytes").get<double>(), sec, jou);
      } else {
        throw DataError("unknown table kind: " + table);
      }
    } catch (const nlohmann::json::exception& e) {
      throw DataError("profile line " + std::to_string(lineno) + ": " + e.what());
    }
  }
  store.finalize();
  return store;
}

std::string ProfileStore::serialize() const {
  std::ostringstream out;
  for (const auto& [key, grid] : pend_c_)
    for (const auto& [ax, v] : grid) {
      nlohmann::ordered_json r;
      r["table"] = "compute";
      r["op"] = op_kind_str(OpKind(std::get<0>(key)));
      r["dtype"] = DtypeFormat{Dtype(std::get<1>(key)), 0}.str();
      r["freq_ghz"] = double(std::get<2>(key)) / 1e6;
      r["axes"] = {{"context_tokens", ax[0]}, {"tasks", ax[1]}, {"hidden_dim", ax[2]}};
      r["seconds"] = v.first;
      r["joules"] = v.second;
      out << r.dump() << "\n";
    }
  for (const auto& [key, curve] : pend_k_)
    for (const auto& [pay, v] : curve) {
      nlohmann::ordered_json r;
      r["table"] = "collective";
      r["op"] = collective_kind_str(CollectiveKind(std::get<0>(key)));
      r["axes"] = {{"payload_bytes", pay}, {"num_devices", std::get<1>(key)},
                   {"num_nodes", std::get<2>(key)}};
      r["seconds"] = v.first;
      r["joules"] = v.second;
      out << r.dump() << "\n";
    }
  return out.str();
}

GridSpec GridSpec::for_model(const ModelSpec& model, const ClusterSpec& cluster, double max_context) {
  GridSpec g;
  const BlockSpec block = to_transformer_ir(model);
  g.shape.model_hidden = model.hidden_size;
  g.shape.head_dim = model.head_dim;
  g.shape.kv_elems_per_task_token =
      2.0 * model.head_dim / (model.num_attention_heads / double(model.num_kv_heads));
  // sub-token knots cover cell-DP and routing fractions of the token axis
  for (double c = 1.0 / 4096.0; c < 1.0; c *= 2.0) g.context_knots.push_back(c);
  for (double c = 1.0; c <= max_context; c *= 2.0) g.context_knots.push_back(c);
  if (g.context_knots.back() < max_context) g.context_knots.push_back(g.context_knots.back() * 2.0);
  std::set<double> tasks, widths;
  for (const auto& cell : block.cells) {
    for (int d : divisors(cell.num_tasks)) tasks.insert(double(d));
    widths.insert(cell.task_width);
    if (cell.kind == CellKind::MoE) {
      for (int d : divisors(cell.num_experts)) tasks.insert(double(d));
      tasks.insert(double(cell.num_experts));
    }
  }
  g.task_knots.assign(tasks.begin(), tasks.end());
  g.width_knots.assign(widths.begin(), widths.end());
  g.dtypes.push_back(model.activation_dtype.name);
  const int n = cluster.total_devices(), per_node = cluster.devices_per_node();
  std::set<std::pair<int, int>> groups;
  std::vector<int> sizes = divisors(n);
  sizes.push_back(2);
  for (int d : sizes) {
    if (d < 2) continue;
    const int lo = (d + per_node - 1) / per_node, hi = std::min(d, cluster.num_nodes());
    for (int nodes = lo; nodes <= hi; ++nodes) groups.insert({d, nodes});
    groups.insert({d, std::min(lo, hi)});
  }
  g.collective_groups.assign(groups.begin(), groups.end());
  g.payload_knots = {1.0, 4096.0, double(1 << 20), double(1 << 24), double(1 << 28), 4294967296.0};
  return g;
}

namespace {

// The alpha-beta collective curves of synth_profiles (cost.cpp:489-506).
void add_synth_collectives(ProfileStore& store, const DeviceSpec& hw, const ClusterSpec& net,
                           const GridSpec& grid) {
  for (const auto& [devices, nodes] : grid.collective_groups) {
    int level = 1;  // the link level a group spanning `nodes` nodes must cross
    if (nodes > 1) {
      level = net.num_levels();
      for (int l = 2; l <= net.num_levels(); ++l)
        if (net.subtree_capacity(l) / net.devices_per_node() >= nodes) {
          level = l;
          break;
        }
    }
    const LevelSpec& link = net.levels[size_t(level - 1)];
    const double lat = link.link_latency * (2.0 * std::ceil(std::log2(double(devices))));
    for (const CollectiveKind kind : {CollectiveKind::AllReduce, CollectiveKind::AllGather,
                                      CollectiveKind::ReduceScatter, CollectiveKind::AllToAll,
                                      CollectiveKind::P2P}) {
      if (kind == CollectiveKind::P2P && devices != 2) continue;
      const double d = devices;
      const double factor = kind == CollectiveKind::AllReduce ? 2.0 * (d - 1.0) / d
                            : kind == CollectiveKind::P2P     ? 1.0
                                                              : (d - 1.0) / d;
      for (const double payload : grid.payload_knots) {
        const double sec = lat + payload * factor / link.link_bandwidth;
        store.add_collective_entry(kind, devices, nodes, payload, sec,
                                   sec * devices * 0.25 * hw.tdp_watts);
      }
    }
  }
}

constexpr OpKind kSynthOps[3] = {OpKind::Attention, OpKind::GEMM, OpKind::MoEGEMM};

}  // namespace

ProfileStore synth_profiles(const DeviceSpec& hw, const ClusterSpec& net, const GridSpec& grid) {
  ProfileStore store;
  const double f_max = hw.max_frequency();
  for (const Dtype dt : grid.dtypes) {
    const double peak = hw.peak_flops_for(dt);
    const double eb = dt == Dtype::FP16 ? 2.0 : dt == Dtype::FP8 ? 1.0 : 0.5;
    for (const double f : hw.frequency_options) {
      const double scale = f / f_max;
      const double power = hw.tdp_watts * scale * scale * scale;  // cube-law DVFS power
      for (const OpKind op : kSynthOps)
        for (const double t : grid.context_knots)
          for (const double k : grid.task_knots)
            for (const double w : grid.width_knots) {
              const double sec = std::max(op_flops(op, t, k, w, grid.shape) / (peak * scale),
                                          op_bytes(op, t, k, w, grid.shape, eb) / hw.peak_mem_bandwidth);
              store.add_compute_entry(op, dt, f, t, k, w, sec, sec * power);
            }
    }
  }
  add_synth_collectives(store, hw, net, grid);
  store.finalize();
  return store;
}

ProfileStore synth_profiles_device(const DeviceSpec& hw, const ClusterSpec& net,
                                   const GridSpec& grid, Engine* engine) {
  std::unique_ptr<Engine> own;
  if (!engine) {
    own = std::make_unique<Engine>(0);
    engine = own.get();
  }
  const double f_max = hw.max_frequency();
  std::vector<double> peak_scaled, elem_bytes, power;
  for (const Dtype dt : grid.dtypes) {
    const double peak = hw.peak_flops_for(dt);
    const double eb = dt == Dtype::FP16 ? 2.0 : dt == Dtype::FP8 ? 1.0 : 0.5;
    for (const double f : hw.frequency_options) {
      const double scale = f / f_max;
      peak_scaled.push_back(peak * scale);
      elem_bytes.push_back(eb);
      power.push_back(hw.tdp_watts * scale * scale * scale);
    }
  }
  psg_synth_grid g{};
  g.n_ctx = int32_t(grid.context_knots.size());
  g.n_tasks = int32_t(grid.task_knots.size());
  g.n_width = int32_t(grid.width_knots.size());
  g.n_variants = int32_t(peak_scaled.size());
  g.ctx = grid.context_knots.data();
  g.tasks = grid.task_knots.data();
  g.width = grid.width_knots.data();
  g.peak_scaled = peak_scaled.data();
  g.elem_bytes = elem_bytes.data();
  g.power = power.data();
  g.mem_bw = hw.peak_mem_bandwidth;
  g.hidden = grid.shape.model_hidden;
  g.head_dim = grid.shape.head_dim;
  g.kv_elems = grid.shape.kv_elems_per_task_token;
  const size_t n = size_t(g.n_variants) * 3 * grid.context_knots.size() * grid.task_knots.size() *
                   grid.width_knots.size();
  std::vector<double> sec(n), jou(n);
  ProfileStore store;
  if (n > 0) {
    const int rc = psg_synth_compute(engine->handle(), &g, sec.data(), jou.data());
    if (rc != PSG_OK) throw DataError(std::string("synth on device: ") + psg_last_error(engine->handle()));
  }
  size_t i = 0;  // the values are in the reference's loop order
  for (const Dtype dt : grid.dtypes)
    for (const double f : hw.frequency_options)
      for (const OpKind op : kSynthOps)
        for (const double t : grid.context_knots)
          for (const double k : grid.task_knots)
            for (const double w : grid.width_knots) {
              store.add_compute_entry(op, dt, f, t, k, w, sec[i], jou[i]);
              ++i;
            }
  add_synth_collectives(store, hw, net, grid);
  store.finalize();
  return store;
}

}  // namespace psb
