// TEST INFRASTRUCTURE: byte-compares the streaming report writers
// (psb::report_to_json / iterations_to_jsonl / report_summary_line /
// write_ranked_json / sweep_to_json, paper_2411_17651_b200/csrc/host/report.cpp)
// with the reference's own (plansim::report_to_json etc., simulator.cpp:331-397,
// and the CLI recipes tools/plansim_main.cpp:128-131, :184-199) on random
// reports with edge-case doubles.  Built against oracle/_ref (tests/test_cpu_report.py).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <sstream>
#include <string>

#include "json.hpp"
#include "plansim/simulator.hpp"
#include "psb/plansim_b200.hpp"

static std::mt19937_64 rng(2026);

static double edge_double() {
  static const double edges[] = {0.0, 1.0, 2.0, 0.1, 1e-5, 1e-4, 9.999e-5, 1e15, 1e16, 1e17,
                                 123456789012345678.0, 0.30000000000000004, 5e-324, 1.7976931348623157e308,
                                 2.2250738585072014e-308, 1e21, 1e22, 3.0e-7, 12345.678, 0.5, 1024.0,
                                 4503599627370496.0, 9007199254740993.0};
  std::uniform_real_distribution<double> U(0.0, 1.0);
  switch (rng() % 4) {
    case 0: return edges[rng() % (sizeof edges / sizeof edges[0])];
    case 1: return std::ldexp(U(rng), int(rng() % 120) - 60);
    case 2: return double(rng() % 100000);
    default: return U(rng) * std::pow(10.0, double(int(rng() % 40) - 20));
  }
}

int main() {
  long bad = 0;
  plansim::RankedPlans ra;
  psb::RankedPlans rb;
  for (int t = 0; t < 300; ++t) {
    plansim::SimulationReport a;
    psb::SimulationReport b;
    a.plan_encoding = b.plan_encoding = "dp" + std::to_string(t) + ":pp2:GQA-tp2x1:SwiGLU-tp1x2" +
                                        (t % 7 == 0 ? std::string("\"q\\\t") : std::string());
    a.frequency_ghz = b.frequency_ghz = edge_double();
    a.e2e_latency = b.e2e_latency = edge_double();
    a.total_energy = b.total_energy = edge_double();
    a.p95_latency = b.p95_latency = edge_double();
    a.mean_ttft = b.mean_ttft = edge_double();
    a.mean_tpot = b.mean_tpot = edge_double();
    a.mfu = b.mfu = edge_double();
    a.mbu = b.mbu = edge_double();
    a.num_completed = b.num_completed = int64_t(rng() % 1000);
    a.num_rejected = b.num_rejected = int64_t(rng() % 5);
    a.num_iterations = b.num_iterations = int64_t(rng() % 100000);
    a.max_batch_observed = b.max_batch_observed = int64_t(rng() % 300);
    const int npr = int(rng() % 6), nrj = int(rng() % 3), nit = t % 3 == 0 ? int(rng() % 4) : 0;
    for (int i = 0; i < npr; ++i) {
      plansim::RequestMetrics m;
      m.id = int64_t(rng() % 100000);
      m.ttft = edge_double();
      m.tpot = edge_double();
      m.e2e = edge_double();
      m.gen_len = int64_t(rng() % 5000);
      a.per_request.push_back(m);
      b.per_request.push_back({m.id, m.ttft, m.tpot, m.e2e, m.gen_len});
    }
    for (int i = 0; i < nrj; ++i) {
      const int64_t id = int64_t(rng() % 100000);
      a.rejected_ids.push_back(id);
      b.rejected_ids.push_back(id);
    }
    for (int i = 0; i < nit; ++i) {
      plansim::IterationRecord x;
      psb::IterationRecord y;
      x.clock_start = y.clock_start = edge_double();
      x.duration = y.duration = edge_double();
      x.energy = y.energy = edge_double();
      x.batch_size = y.batch_size = int64_t(rng() % 64);
      const int S = int(rng() % 4);
      for (int s = 0; s < S; ++s) {
        const double u = edge_double(), v = edge_double();
        x.stage_seconds.push_back(u);
        y.stage_seconds.push_back(u);
        x.stage_joules.push_back(v);
        y.stage_joules.push_back(v);
      }
      a.iterations.push_back(x);
      b.iterations.push_back(y);
    }
    if (plansim::report_to_json(a) != psb::report_to_json(b)) {
      if (!bad++) std::printf("report_to_json differs:\n%s\nvs\n%s\n", plansim::report_to_json(a).c_str(),
                              psb::report_to_json(b).c_str());
    }
    if (plansim::iterations_to_jsonl(a) != psb::iterations_to_jsonl(b)) {
      if (!bad++) std::printf("iterations_to_jsonl differs\n");
    }
    if (plansim::report_summary_line(a) != psb::report_summary_line(b)) {
      if (!bad++) std::printf("summary differs: %s | %s\n", plansim::report_summary_line(a).c_str(),
                              psb::report_summary_line(b).c_str());
    }
    a.iterations.clear();
    b.iterations.clear();
    ra.entries.push_back({size_t(t), a.frequency_ghz, a});
    rb.entries.push_back({size_t(t), b.frequency_ghz, b});
  }
  // ranked.json: the CLI's parse -> array -> dump(2)
  nlohmann::ordered_json doc = nlohmann::ordered_json::array();
  for (const auto& e : ra.entries) doc.push_back(nlohmann::ordered_json::parse(plansim::report_to_json(e.report)));
  const std::string ref_ranked = doc.dump(2) + "\n";
  const char* path = "report_check_ranked.json";
  psb::write_ranked_json(rb, path);
  std::ifstream f(path);
  std::stringstream ss;
  ss << f.rdbuf();
  if (ss.str() != ref_ranked) {
    if (!bad++) std::printf("ranked.json differs (%zu vs %zu bytes)\n", ss.str().size(), ref_ranked.size());
  }
  std::remove(path);
  // sweep table
  for (int t = 0; t < 50; ++t) {
    psb::SweepTable st;
    st.observed_max_batch = int64_t(rng() % 1000);
    nlohmann::ordered_json d;
    d["observed_max_batch"] = st.observed_max_batch;
    d["rows"] = nlohmann::ordered_json::array();
    for (int i = 0; i < int(rng() % 6); ++i) {
      psb::SweepRow r{int64_t(rng() % 500), edge_double(), edge_double(), edge_double()};
      st.rows.push_back(r);
      d["rows"].push_back({{"max_batch_size", r.max_batch_size},
                           {"mean_tpot_s", r.mean_tpot},
                           {"mean_ttft_s", r.mean_ttft},
                           {"e2e_latency_s", r.e2e_latency}});
    }
    if (psb::sweep_to_json(st) != d.dump(2) + "\n") {
      if (!bad++) std::printf("sweep differs:\n%s\nvs\n%s\n", psb::sweep_to_json(st).c_str(), (d.dump(2) + "\n").c_str());
    }
  }
  std::printf("report_check bad=%ld\n", bad);
  return bad ? 1 : 0;
}
