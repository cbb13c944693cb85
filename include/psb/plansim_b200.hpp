// plansim_b200.hpp — native C++ host API of the B200 plan-search engine.
//
// It mirrors the reference's public C++ surface (/root/reference/proj/include/
// plansim/*.hpp) so callers of plansim::search switch by namespace: the model
// IR, cluster, planner, profile store and trace types keep the reference's
// names and field meanings, and psb::search / psb::simulate_plan run on the
// GPU through the C ABI in include/psg.h.  Everything here is host-side
// preparation (parsing, plan enumeration, table synthesis) — the evaluation
// hot path is the CUDA engine.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "psg.h"

namespace psb {

// ---- errors (common.hpp:13-20) -------------------------------------------
struct DataError : std::runtime_error {
  explicit DataError(const std::string& m) : std::runtime_error(m) {}
};
struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

std::vector<int> divisors(int n);

// ---- model IR (ir.hpp) ----------------------------------------------------
enum class Dtype { FP16 = PSG_DTYPE_FP16, FP8 = PSG_DTYPE_FP8, INT4 = PSG_DTYPE_INT4 };

struct DtypeFormat {
  Dtype name = Dtype::FP16;
  double bytes_per_element = 2.0;
  static DtypeFormat from_string(const std::string& s);
  const char* str() const;
};

struct ModelSpec {
  std::string name;
  int num_layers = 0, hidden_size = 0, num_attention_heads = 0, num_kv_heads = 0;
  int head_dim = 0, intermediate_size = 0, vocab_size = 0;
  int num_experts = 0, experts_per_token = 0;
  DtypeFormat weight_dtype, activation_dtype, kv_cache_dtype;
  std::string ffn_activation;
  bool is_moe() const { return num_experts > 0; }
  bool is_gqa() const { return num_kv_heads < num_attention_heads; }
};

enum class CellKind { MHA, GQA, MLP, SwiGLU, MoE };
const char* cell_kind_str(CellKind k);

struct CellSpec {
  CellKind kind = CellKind::MHA;
  int num_tasks = 0, kv_group_fanin = 1, tp_slices = 0;
  double task_width = 0.0, head_dim = 0.0;
  int kv_heads = 0;
  double qo_weight_bytes_per_task = 0.0, kv_weight_bytes_per_kv_head = 0.0;
  int num_experts = 0, experts_per_token = 0;
  double weight_bytes() const;
  bool is_attention() const { return kind == CellKind::MHA || kind == CellKind::GQA; }
};

struct BlockSpec {
  std::vector<CellSpec> cells;
  int repeat_count = 0;
};

ModelSpec parse_model_config(const std::string& json_text);
BlockSpec to_transformer_ir(const ModelSpec& model);
double embedding_weight_bytes(const ModelSpec& model);
double model_weight_bytes(const ModelSpec& model, bool include_embedding = true);

// ---- cluster (cluster.hpp) --------------------------------------------------
struct LevelSpec {
  int fan_out = 1;
  double link_bandwidth = 0.0, link_latency = 0.0;
};

struct DeviceSpec {
  std::string name;
  double memory_capacity = 0.0;
  std::map<Dtype, double> peak_flops;
  double peak_mem_bandwidth = 0.0;
  std::vector<double> frequency_options;  // ascending
  double tdp_watts = 700.0;
  double max_frequency() const { return frequency_options.back(); }
  double peak_flops_for(Dtype dt) const;
};

struct ClusterSpec {
  std::vector<LevelSpec> levels;  // leaf first
  DeviceSpec device;
  int total_devices() const;
  int devices_per_node() const { return levels.front().fan_out; }
  int num_nodes() const { return total_devices() / devices_per_node(); }
  int subtree_capacity(int level) const;
  int num_levels() const { return int(levels.size()); }
};

ClusterSpec parse_cluster_spec(const std::string& json_text);

struct DeviceAssignment {
  int model_dp = 1, num_stages = 1, stage_devices = 1;
  std::vector<int> phys;  // ((r * stages) + s) * stage_devices + slot
  int device_of(int replica, int stage, int slot) const;
};

DeviceAssignment map_devices(int model_dp, int num_stages, int stage_devices,
                             const ClusterSpec& cluster);

// ---- planner (planner.hpp) ----------------------------------------------------
enum class ParallelMode { TP, EP };
enum class OpKind { Attention = PSG_OP_ATTENTION, GEMM = PSG_OP_GEMM, MoEGEMM = PSG_OP_MOE_GEMM };
enum class CollectiveKind {
  AllReduce = PSG_COLL_ALLREDUCE,
  AllGather = PSG_COLL_ALLGATHER,
  ReduceScatter = PSG_COLL_REDUCE_SCATTER,
  AllToAll = PSG_COLL_ALL_TO_ALL,
  P2P = PSG_COLL_P2P
};
const char* op_kind_str(OpKind k);
const char* collective_kind_str(CollectiveKind k);

struct CellScheme {
  CellSpec cell;
  ParallelMode mode = ParallelMode::TP;
  int cell_dp = 1, intra_degree = 1;
  double weight_bytes_per_device = 0.0;
  OpKind op = OpKind::GEMM;
  double query_tasks = 0.0, query_width = 0.0, token_scale = 1.0;
};

enum class GroupScope { LeftIntra, RightIntra, Stage };

struct CollectiveOp {
  CollectiveKind kind = CollectiveKind::AllReduce;
  double payload_bytes_per_token = 0.0, token_share = 1.0;
  GroupScope scope = GroupScope::LeftIntra;
};

struct ParallelScheme {
  int model_dp = 1, num_stages = 1, stage_devices = 1, stage_repetitions = 1;
  std::vector<CellScheme> cells;
  std::vector<std::vector<CollectiveOp>> reshards;
  std::string encoding;
};

struct ResolvedCollective {
  CollectiveKind kind = CollectiveKind::AllReduce;
  double payload_bytes_per_token = 0.0, token_share = 1.0;
  int num_devices = 0, num_nodes = 1, groups_per_stage = 1;
};

struct OpShape {
  double model_hidden = 0.0, head_dim = 0.0, kv_elems_per_task_token = 0.0;
};

struct ExecutionPlan {
  ParallelScheme scheme;
  DeviceAssignment assignment;
  std::vector<ResolvedCollective> block_collectives;
  std::vector<int> p2p_boundary_nodes;
  double p2p_payload_per_token = 0.0;
  double static_bytes_per_device = 0.0, kv_budget_per_replica = 0.0, kv_bytes_per_token = 0.0;
  Dtype compute_dtype = Dtype::FP16;
  OpShape op_shape;
  const std::string& encoding() const { return scheme.encoding; }
};

struct PlanOptions {
  double activation_reserve = 0.10;
  bool include_embedding = true;
  int max_cell_combinations = 65536;
};

struct CellChoice {
  ParallelMode mode = ParallelMode::TP;
  int cell_dp = 1, intra_degree = 1;
};

bool template_valid(const CellSpec& cell, int devices, ParallelMode mode);
std::vector<ParallelScheme> enumerate_schemes(const ModelSpec& model, const BlockSpec& block,
                                              int n, int max_cell_combinations = 65536);
std::vector<ExecutionPlan> generate_plans(const ModelSpec& model, const BlockSpec& block,
                                          const ClusterSpec& cluster,
                                          const PlanOptions& opts = {});
class Engine;
// generate_plans with the device mapping, collective resolution and memory
// ledger of every candidate computed on the GPU (psg_plan_compute; SURVEY.md
// §8(f) row 3); the same plans, field for field.
std::vector<ExecutionPlan> generate_plans_device(const ModelSpec& model, const BlockSpec& block,
                                                 const ClusterSpec& cluster,
                                                 const PlanOptions& opts = {},
                                                 Engine* engine = nullptr);
// generate_plans straight into the engine's plan SoA: the plan kernels map,
// finalize and compact the candidates on the device (psg_plan_emit) and the
// search consumes that SoA as is — no ExecutionPlan objects on the host.
// The same plans, in the same order, field for field (tests/test_gpu_planner.py).
struct DevicePlanSet {
  psg_plan_soa* soa = nullptr;          // library-owned (psg_plan_soa_free)
  std::vector<std::string> encodings;   // per plan, scheme.encoding
  DevicePlanSet() = default;
  DevicePlanSet(const DevicePlanSet&) = delete;
  DevicePlanSet& operator=(const DevicePlanSet&) = delete;
  ~DevicePlanSet();
  const psg_plan_set& view() const { return soa->set; }
  size_t size() const { return encodings.size(); }
};
std::unique_ptr<DevicePlanSet> generate_plans_direct(const ModelSpec& model, const BlockSpec& block,
                                                     const ClusterSpec& cluster,
                                                     const PlanOptions& opts = {},
                                                     Engine* engine = nullptr);
ExecutionPlan build_plan(const ModelSpec& model, const BlockSpec& block,
                         const ClusterSpec& cluster, int model_dp, int num_stages,
                         const std::vector<CellChoice>& cells, const PlanOptions& opts = {});
// The plan fields in the oracle driver's JSON schema (tests compare them).
std::string plans_to_json(const std::vector<ExecutionPlan>& plans);

// ---- profile store (cost.hpp) ------------------------------------------------
double op_flops(OpKind op, double tokens, double tasks, double width, const OpShape& s);
double op_bytes(OpKind op, double tokens, double tasks, double width, const OpShape& s,
                double elem_bytes);
double kv_bytes_per_token(const ModelSpec& m);

class ProfileStore {
 public:
  static ProfileStore load(const std::string& jsonl_text);
  std::string serialize() const;
  void add_compute_entry(OpKind op, Dtype dt, double freq_ghz, double ctx, double tasks,
                         double width, double seconds, double joules);
  void add_collective_entry(CollectiveKind kind, int num_devices, int num_nodes,
                            double payload, double seconds, double joules);
  void finalize();
  bool has_compute_table(OpKind op, Dtype dt, double freq_ghz) const;
  // Flat structure-of-arrays view for the engine (valid while *this lives
  // and is not modified).
  const psg_store& view() const {
    rebind();
    return view_;
  }
  // Clamp-warning log (cost.cpp:191-194): reproduced from the engine's
  // per-table clamp flags after a search.
  std::vector<std::string> warnings() const { return warnings_; }
  size_t warning_count() const { return warnings_.size(); }
  void record_clamps(const uint8_t* compute_bits, const uint8_t* curve_bits) const;

 private:
  using CKey = std::tuple<int, int, long long>;
  using KKey = std::tuple<int, int, int>;
  std::map<CKey, std::map<std::array<double, 3>, std::pair<double, double>>> pend_c_;
  std::map<KKey, std::map<double, std::pair<double, double>>> pend_k_;
  // flat storage behind view_
  std::vector<int32_t> c_op_, c_dt_, c_nc_, c_nt_, c_nw_, k_kind_, k_dev_, k_nodes_, k_n_;
  std::vector<int64_t> c_fm_, c_kb_, c_vb_, k_b_;
  std::vector<double> c_knots_, c_sec_, c_jou_, k_pay_, k_sec_, k_jou_;
  mutable psg_store view_{};
  void rebind() const;  // points view_ at this object's storage (copy-safe)
  mutable std::vector<std::string> warnings_;
  mutable std::vector<std::string> warn_keys_;
};

struct GridSpec {
  std::vector<double> context_knots, task_knots, width_knots;
  std::vector<Dtype> dtypes;
  OpShape shape;
  std::vector<std::pair<int, int>> collective_groups;
  std::vector<double> payload_knots;
  static GridSpec for_model(const ModelSpec& model, const ClusterSpec& cluster,
                            double max_context = 131072.0);
};

ProfileStore synth_profiles(const DeviceSpec& hw, const ClusterSpec& net, const GridSpec& grid);
class Engine;
// The same store with the compute tables computed on the GPU (psg_synth_compute;
// SURVEY.md §8(f) row 4); byte-identical to synth_profiles.
ProfileStore synth_profiles_device(const DeviceSpec& hw, const ClusterSpec& net,
                                   const GridSpec& grid, Engine* engine = nullptr);

// ---- traces (traces.hpp) -------------------------------------------------------
struct Request {
  int64_t id = 0, context_len = 0, gen_len = 0;
  double arrival = 0.0;
};
struct Trace {
  std::vector<Request> requests;
};
Trace load_trace(const std::string& jsonl_text);
std::string serialize_trace(const Trace& trace);
struct LengthDistribution {
  double mean = 0.0, stddev = 0.0;
};
Trace synth_trace(const LengthDistribution& ctx, const LengthDistribution& gen, double rate,
                  int64_t n, uint64_t seed);

// ---- evaluation (simulator.hpp) --------------------------------------------------
enum class BatchMode { Contiguous, ChunkedPrefill };
struct BatchPolicy {
  BatchMode mode = BatchMode::Contiguous;
  int64_t chunk_size = 0, max_batch_size = 0;
};
enum class TtftAnchor { Arrival, Admission };
struct SimConfig {
  double freq_ghz = 0.0;
  BatchPolicy policy;
  TtftAnchor ttft_anchor = TtftAnchor::Arrival;
  bool emit_iterations = false;  // simulate_plan only (simulator.hpp:77)
  // TTFT-SLO-constrained ranking (psg.h psg_config.ttft_slo; not in the
  // reference): > 0 ranks entries whose slo_quantile TTFT meets it first
  double ttft_slo = 0.0, slo_quantile = 0.0;
};

// plansim::IterationRecord (simulator.hpp:35-42).
struct IterationRecord {
  double clock_start = 0.0, duration = 0.0, energy = 0.0;
  int64_t batch_size = 0;
  std::vector<double> stage_seconds, stage_joules;
};
enum class Objective { Latency, Energy };

struct RequestMetrics {
  int64_t id = 0;
  double ttft = 0.0, tpot = 0.0, e2e = 0.0;
  int64_t gen_len = 0;
};
static_assert(sizeof(RequestMetrics) == sizeof(psg_request_metrics), "layout");

struct SimulationReport {
  std::string plan_encoding;
  double frequency_ghz = 0.0, e2e_latency = 0.0, total_energy = 0.0, p95_latency = 0.0;
  double mean_ttft = 0.0, mean_tpot = 0.0, mfu = 0.0, mbu = 0.0;
  int64_t num_completed = 0, num_rejected = 0, num_iterations = 0, max_batch_observed = 0;
  // additive outputs (not in the reference)
  double p50_ttft = 0.0, p99_ttft = 0.0, p50_tpot = 0.0, p99_tpot = 0.0;
  double slo_ttft = 0.0;  // TTFT at SimConfig::slo_quantile (ttft_slo > 0)
  bool slo_met = false;
  std::vector<RequestMetrics> per_request;
  std::vector<int64_t> rejected_ids;
  std::vector<IterationRecord> iterations;  // emit_iterations
};

// plansim::SweepRow / SweepTable (simulator.hpp:105-115).
struct SweepRow {
  int64_t max_batch_size = 0;
  double mean_tpot = 0.0, mean_ttft = 0.0, e2e_latency = 0.0;
};
struct SweepTable {
  int64_t observed_max_batch = 0;
  std::vector<SweepRow> rows;
};

struct SearchEntry {
  size_t plan_index = 0;
  double freq_ghz = 0.0;
  SimulationReport report;
};
struct RankedPlans {
  std::vector<SearchEntry> entries;
};

// Flat SoA of a plan vector (owned storage + psg_plan_set view).
class PlanSoA {
 public:
  explicit PlanSoA(const std::vector<ExecutionPlan>& plans);
  const psg_plan_set& view() const { return view_; }

 private:
  std::vector<int32_t> dp_, st_, sd_, reps_, dt_, enc_, cb_, cop_, kb_, kk_, kd_, kn_, kg_, pb_, pn_;
  std::vector<double> kv_, bud_, p2p_, hid_, head_, kve_, ct_, cw_, cs_, kp_, ksh_;
  psg_plan_set view_{};
};

psg_cluster cluster_view(const ClusterSpec& cluster);

// The GPU engine handle; one per device.
class Engine {
 public:
  explicit Engine(int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  psg_context* handle() const { return ctx_; }

 private:
  psg_context* ctx_ = nullptr;
};

// plansim::search (simulator.hpp:99-103): `jobs` is accepted for signature
// compatibility; the engine's parallelism is the device.  Throws DataError /
// InfeasibleError exactly where the reference would.
RankedPlans search(const std::vector<ExecutionPlan>& plans, const ModelSpec& model,
                   const ClusterSpec& cluster, const Trace& trace, const ProfileStore& store,
                   Objective objective, const std::vector<double>& frequencies,
                   const SimConfig& cfg, int jobs = 1, Engine* engine = nullptr);

// plansim::simulate_plan (simulator.hpp:80-82), emit_iterations included.
SimulationReport simulate_plan(const ExecutionPlan& plan, const ModelSpec& model,
                               const ClusterSpec& cluster, const Trace& trace,
                               const ProfileStore& store, const SimConfig& cfg,
                               Engine* engine = nullptr);

// plansim::sweep_max_batch (simulator.hpp:117-122): the capped simulations
// run in one launch.
SweepTable sweep_max_batch(const ExecutionPlan& plan, const ModelSpec& model,
                           const ClusterSpec& cluster, const Trace& trace,
                           const ProfileStore& store, const SimConfig& cfg, int segments,
                           int64_t subset_size = 256, Engine* engine = nullptr);

// Report materialization (simulator.cpp:331-397, tools/plansim_main.cpp:
// 128-131, :184-199): byte-identical to the reference's nlohmann output,
// streamed without a JSON document.
std::string report_to_json(const SimulationReport& report);
std::string iterations_to_jsonl(const SimulationReport& report);
std::string report_summary_line(const SimulationReport& report);
void write_ranked_json(const RankedPlans& ranked, const std::string& path);  // CLI ranked.json
std::string sweep_to_json(const SweepTable& table);                          // CLI sweep --out

}  // namespace psb
