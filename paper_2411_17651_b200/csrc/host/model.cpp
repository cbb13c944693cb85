// Model IR and cluster description for the host side (mirrors the semantics
// of /root/reference/proj/src/ir.cpp:52-222 and cluster.cpp:14-198).
#include <algorithm>
#include <cctype>
#include <iostream>
#include <set>

#include "nlohmann/json.hpp"
#include "psb/plansim_b200.hpp"

namespace psb {

using json = nlohmann::json;

std::vector<int> divisors(int n) {
  std::vector<int> lo, hi;
  for (int d = 1; d * d <= n; ++d) {
    if (n % d) continue;
    lo.push_back(d);
    if (d != n / d) hi.push_back(n / d);
  }
  lo.insert(lo.end(), hi.rbegin(), hi.rend());
  return lo;
}

namespace {

std::string lower(std::string s) {
  for (auto& ch : s) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

json parse_json(const std::string& text, const char* what) {
  try {
    return json::parse(text);
  } catch (const json::exception& e) {
    throw DataError(std::string(what) + ": " + e.what());
  }
}

// First present key among the aliases.
const json* first_of(const json& doc, std::initializer_list<const char*> keys) {
  for (const char* k : keys)
    if (doc.contains(k)) return &doc.at(k);
  return nullptr;
}

}  // namespace

DtypeFormat DtypeFormat::from_string(const std::string& s) {
  static const std::map<std::string, DtypeFormat> table = {
      {"fp16", {Dtype::FP16, 2.0}},        {"float16", {Dtype::FP16, 2.0}},
      {"half", {Dtype::FP16, 2.0}},        {"bfloat16", {Dtype::FP16, 2.0}},
      {"bf16", {Dtype::FP16, 2.0}},        {"fp8", {Dtype::FP8, 1.0}},
      {"float8", {Dtype::FP8, 1.0}},       {"float8_e4m3fn", {Dtype::FP8, 1.0}},
      {"e4m3", {Dtype::FP8, 1.0}},         {"int4", {Dtype::INT4, 0.5}},
      {"uint4", {Dtype::INT4, 0.5}},       {"w4", {Dtype::INT4, 0.5}}};
  const auto it = table.find(lower(s));
  if (it == table.end()) throw DataError("unknown dtype: " + s);
  return it->second;
}

const char* DtypeFormat::str() const {
  return name == Dtype::FP16 ? "fp16" : name == Dtype::FP8 ? "fp8" : "int4";
}

const char* cell_kind_str(CellKind k) {
  static const char* names[] = {"MHA", "GQA", "MLP", "SwiGLU", "MoE"};
  return names[int(k)];
}

double CellSpec::weight_bytes() const {
  return num_tasks * qo_weight_bytes_per_task + kv_heads * kv_weight_bytes_per_kv_head;
}

ModelSpec parse_model_config(const std::string& text) {
  const json doc = parse_json(text, "model config");
  auto req = [&](std::initializer_list<const char*> keys) {
    const json* v = first_of(doc, keys);
    if (!v) throw DataError(std::string("model config: missing required key \"") + *keys.begin() + "\"");
    return v->get<int>();
  };
  auto opt = [&](std::initializer_list<const char*> keys, int fallback) {
    const json* v = first_of(doc, keys);
    return v ? v->get<int>() : fallback;
  };
  auto opt_str = [&](std::initializer_list<const char*> keys, const std::string& fallback) {
    for (const char* k : keys)
      if (doc.contains(k) && doc.at(k).is_string()) return doc.at(k).get<std::string>();
    return fallback;
  };
  ModelSpec m;
  m.name = opt_str({"name", "model_name", "model_type"}, "model");
  m.num_layers = req({"num_hidden_layers", "num_layers"});
  m.hidden_size = req({"hidden_size"});
  m.num_attention_heads = req({"num_attention_heads"});
  m.intermediate_size = req({"intermediate_size"});
  m.vocab_size = req({"vocab_size"});
  m.num_kv_heads = opt({"num_key_value_heads", "num_kv_heads"}, m.num_attention_heads);
  m.head_dim = opt({"head_dim"}, m.num_attention_heads > 0 ? m.hidden_size / m.num_attention_heads : 0);
  m.num_experts = opt({"num_local_experts", "num_experts"}, 0);
  m.experts_per_token = opt({"num_experts_per_tok", "experts_per_token"}, 0);
  const std::string wd = opt_str({"weight_dtype", "torch_dtype"}, "fp16");
  m.weight_dtype = DtypeFormat::from_string(wd);
  m.activation_dtype = DtypeFormat::from_string(opt_str({"activation_dtype"}, wd));
  m.kv_cache_dtype = DtypeFormat::from_string(opt_str({"kv_cache_dtype"}, m.activation_dtype.str()));
  m.ffn_activation = lower(opt_str({"hidden_act", "hidden_activation"}, "silu"));

  auto positive = [](int v, const char* what) {
    if (v <= 0) throw DataError(std::string("model config: non-positive ") + what);
  };
  if (m.num_layers < 0) throw DataError("model config: negative num_layers");
  positive(m.hidden_size, "hidden_size");
  positive(m.num_attention_heads, "num_attention_heads");
  positive(m.num_kv_heads, "num_key_value_heads");
  positive(m.head_dim, "head_dim");
  positive(m.intermediate_size, "intermediate_size");
  positive(m.vocab_size, "vocab_size");
  if (m.hidden_size != m.num_attention_heads * m.head_dim)
    throw DataError("model config: hidden_size must equal heads * head_dim");
  if (m.num_attention_heads % m.num_kv_heads != 0)
    throw DataError("model config: num_attention_heads not divisible by num_key_value_heads");
  if (m.num_experts < 0 || m.experts_per_token < 0)
    throw DataError("model config: negative expert count");
  if ((m.num_experts == 0) != (m.experts_per_token == 0))
    throw DataError("model config: num_local_experts and num_experts_per_tok must both be zero or both be positive");
  if (m.num_experts > 0 && m.experts_per_token > m.num_experts)
    throw DataError("model config: experts_per_token exceeds num_local_experts");
  return m;
}

BlockSpec to_transformer_ir(const ModelSpec& m) {
  const double wb = m.weight_dtype.bytes_per_element;
  BlockSpec b;
  b.repeat_count = m.num_layers;

  CellSpec att;  // heads are the tasks; K/V projections are shared per kv group
  att.kind = m.is_gqa() ? CellKind::GQA : CellKind::MHA;
  att.num_tasks = m.num_attention_heads;
  att.kv_group_fanin = m.num_attention_heads / m.num_kv_heads;
  att.tp_slices = m.num_attention_heads;
  att.head_dim = m.head_dim;
  att.kv_heads = m.num_kv_heads;
  att.task_width = m.head_dim * (2.0 + 2.0 / att.kv_group_fanin);
  att.qo_weight_bytes_per_task = 2.0 * m.hidden_size * m.head_dim * wb;
  att.kv_weight_bytes_per_kv_head = 2.0 * m.hidden_size * m.head_dim * wb;
  b.cells.push_back(att);

  CellSpec ffn;
  if (m.is_moe()) {
    ffn.kind = CellKind::MoE;
    ffn.num_tasks = m.num_experts;
    ffn.tp_slices = m.num_attention_heads;
    ffn.num_experts = m.num_experts;
    ffn.experts_per_token = m.experts_per_token;
    ffn.task_width = 3.0 * m.intermediate_size;
    ffn.qo_weight_bytes_per_task = m.hidden_size * ffn.task_width * wb;
  } else {
    static const std::set<std::string> gated = {"silu", "swiglu", "silu_and_mul"};
    static const std::set<std::string> plain = {"gelu", "relu", "gelu_new", "gelu_pytorch_tanh"};
    int mats;
    if (gated.count(m.ffn_activation)) {
      ffn.kind = CellKind::SwiGLU;
      mats = 3;
    } else if (plain.count(m.ffn_activation)) {
      ffn.kind = CellKind::MLP;
      mats = 2;
    } else {
      throw DataError("no registered cell for hidden_act \"" + m.ffn_activation + "\"");
    }
    ffn.num_tasks = m.num_attention_heads;
    ffn.tp_slices = m.num_attention_heads;
    ffn.task_width = double(mats) * m.intermediate_size / m.num_attention_heads;
    ffn.qo_weight_bytes_per_task = m.hidden_size * ffn.task_width * wb;
  }
  b.cells.push_back(ffn);
  return b;
}

double embedding_weight_bytes(const ModelSpec& m) {
  return double(m.vocab_size) * m.hidden_size * m.weight_dtype.bytes_per_element;
}

double model_weight_bytes(const ModelSpec& m, bool include_embedding) {
  double per_layer = 0.0;
  if (m.num_layers > 0)
    for (const auto& c : to_transformer_ir(m).cells) per_layer += c.weight_bytes();
  double total = per_layer * m.num_layers;
  if (include_embedding) total += embedding_weight_bytes(m);
  return total;
}

// ---- cluster -------------------------------------------------------------------

double DeviceSpec::peak_flops_for(Dtype dt) const {
  const auto it = peak_flops.find(dt);
  if (it == peak_flops.end())
    throw DataError(std::string("device has no peak_flops entry for dtype ") +
                    DtypeFormat{dt, 0}.str());
  return it->second;
}

int ClusterSpec::total_devices() const {
  int n = 1;
  for (const auto& l : levels) n *= l.fan_out;
  return n;
}

int ClusterSpec::subtree_capacity(int level) const {
  int n = 1;
  for (int i = 0; i < level && i < int(levels.size()); ++i) n *= levels[size_t(i)].fan_out;
  return n;
}

ClusterSpec parse_cluster_spec(const std::string& text) {
  const json doc = parse_json(text, "cluster spec");
  ClusterSpec c;
  if (!doc.contains("levels") || !doc["levels"].is_array() || doc["levels"].empty())
    throw DataError("cluster spec: missing levels array");
  for (const auto& l : doc["levels"]) {
    LevelSpec lv;
    lv.fan_out = l.at("fan_out").get<int>();
    lv.link_bandwidth = l.at("link_bandwidth_bytes_per_s").get<double>();
    lv.link_latency = l.value("link_latency_s", 0.0);
    if (lv.fan_out < 1) throw DataError("cluster spec: fan_out must be >= 1");
    if (lv.link_bandwidth <= 0) throw DataError("cluster spec: bandwidth must be > 0");
    if (lv.link_latency < 0) throw DataError("cluster spec: negative latency");
    c.levels.push_back(lv);
  }
  if (!doc.contains("device")) throw DataError("cluster spec: missing device");
  const json& d = doc["device"];
  c.device.name = d.value("name", "device");
  c.device.memory_capacity = d.at("memory_capacity_bytes").get<double>();
  c.device.peak_mem_bandwidth = d.at("peak_mem_bandwidth_bytes_per_s").get<double>();
  c.device.tdp_watts = d.value("tdp_watts", 700.0);
  if (c.device.memory_capacity <= 0) throw DataError("cluster spec: memory capacity must be > 0");
  if (c.device.peak_mem_bandwidth <= 0) throw DataError("cluster spec: memory bandwidth must be > 0");
  if (!d.contains("peak_flops") || d["peak_flops"].empty())
    throw DataError("cluster spec: missing peak_flops table");
  for (auto it = d["peak_flops"].begin(); it != d["peak_flops"].end(); ++it) {
    const double v = it.value().get<double>();
    if (v <= 0) throw DataError("cluster spec: peak_flops must be > 0");
    c.device.peak_flops[DtypeFormat::from_string(it.key()).name] = v;
  }
  if (d.contains("frequency_options_ghz"))
    for (const auto& f : d["frequency_options_ghz"]) c.device.frequency_options.push_back(f.get<double>());
  if (c.device.frequency_options.empty())
    c.device.frequency_options.push_back(d.value("frequency_ghz", 1.0));
  std::sort(c.device.frequency_options.begin(), c.device.frequency_options.end());
  if (c.device.frequency_options.front() <= 0) throw DataError("cluster spec: frequencies must be > 0");
  for (size_t i = 1; i < c.levels.size(); ++i)
    if (c.levels[i].link_bandwidth > c.levels[i - 1].link_bandwidth)
      std::cerr << "warning: cluster level " << (i + 1) << " has higher bandwidth than level " << i
                << "; expected non-increasing bandwidth up the tree\n";
  return c;
}

int DeviceAssignment::device_of(int r, int s, int slot) const {
  if (r < 0 || r >= model_dp || s < 0 || s >= num_stages || slot < 0 || slot >= stage_devices)
    throw DataError("device assignment: role out of range");
  return phys[size_t((r * num_stages + s) * stage_devices + slot)];
}

DeviceAssignment map_devices(int model_dp, int num_stages, int stage_devices,
                             const ClusterSpec& cluster) {
  const int n = cluster.total_devices();
  if (model_dp * num_stages * stage_devices != n)
    throw DataError("device mapper: scheme uses " +
                    std::to_string(model_dp * num_stages * stage_devices) +
                    " logical devices but the cluster has " + std::to_string(n));
  DeviceAssignment a;
  a.model_dp = model_dp;
  a.num_stages = num_stages;
  a.stage_devices = stage_devices;
  a.phys.reserve(size_t(n));
  std::vector<char> used(size_t(n), 0);
  // Each stage goes into the smallest aligned subtree with room (lowest index
  // first); a fragmented tree falls back to the lowest free devices.
  auto take = [&](int lo, int hi, int want) {
    for (int i = lo; i < hi && want > 0; ++i)
      if (!used[size_t(i)]) {
        used[size_t(i)] = 1;
        a.phys.push_back(i);
        --want;
      }
  };
  for (int block = 0; block < model_dp * num_stages; ++block) {
    bool placed = false;
    for (int level = 0; level <= cluster.num_levels() && !placed; ++level) {
      const int cap = cluster.subtree_capacity(level);
      if (cap < stage_devices) continue;
      for (int base = 0; base + cap <= n && !placed; base += cap) {
        const int free_here = int(std::count(used.begin() + base, used.begin() + base + cap, 0));
        if (free_here >= stage_devices) {
          take(base, base + cap, stage_devices);
          placed = true;
        }
      }
    }
    if (!placed) take(0, n, stage_devices);
  }
  return a;
}

}  // namespace psb
