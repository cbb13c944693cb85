// Request traces: JSONL load / serialize and the truncated-normal Poisson
// generator.  Semantics of /root/reference/proj/src/traces.cpp:17-139
// (including its hand-rolled draws over the standardized mt19937_64 stream,
// so output is byte-identical to the reference's; tests/test_host_inputs.py).
#include <algorithm>
#include <cmath>
#include <random>
#include <sstream>

#include "nlohmann/json.hpp"
#include "psb/plansim_b200.hpp"

namespace psb {

Trace load_trace(const std::string& text) {
  Trace t;
  std::istringstream in(text);
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    nlohmann::json rec;
    try {
      rec = nlohmann::json::parse(line);
    } catch (const nlohmann::json::exception& e) {
      throw DataError("trace line " + std::to_string(lineno) + ": " + e.what());
    }
    auto integer = [&](std::initializer_list<const char*> keys, int64_t fallback, bool required) {
      for (const char* k : keys) {
        if (!rec.contains(k)) continue;
        const auto& v = rec.at(k);
        return v.is_string() ? int64_t(std::stoll(v.get<std::string>())) : v.get<int64_t>();
      }
      if (required)
        throw DataError("trace line " + std::to_string(lineno) + ": missing " + *keys.begin());
      return fallback;
    };
    Request r;
    r.id = integer({"id"}, int64_t(t.requests.size()), false);
    r.context_len = integer({"context_len", "context_tokens", "ContextTokens"}, 0, true);
    r.gen_len = integer({"gen_len", "generated_tokens", "GeneratedTokens"}, 0, true);
    r.arrival = 0.0;
    for (const char* k : {"arrival_s", "timestamp", "TIMESTAMP"})
      if (rec.contains(k)) {
        r.arrival = rec.at(k).get<double>();
        break;
      }
    if (r.context_len < 1 || r.gen_len < 1)
      throw DataError("trace line " + std::to_string(lineno) + ": lengths must be >= 1");
    if (r.arrival < 0) throw DataError("trace line " + std::to_string(lineno) + ": negative arrival");
    t.requests.push_back(r);
  }
  std::stable_sort(t.requests.begin(), t.requests.end(),
                   [](const Request& a, const Request& b) { return a.arrival < b.arrival; });
  return t;
}

std::string serialize_trace(const Trace& trace) {
  std::ostringstream out;
  for (const auto& r : trace.requests) {
    nlohmann::ordered_json rec;
    rec["id"] = r.id;
    rec["context_len"] = r.context_len;
    rec["gen_len"] = r.gen_len;
    rec["arrival_s"] = r.arrival;
    out << rec.dump() << "\n";
  }
  return out.str();
}

namespace {
// (0, 1] from the top 53 bits of one mt19937_64 draw
double unit_open0(std::mt19937_64& g) { return (double(g() >> 11) + 1.0) * 0x1p-53; }
}  // namespace

Trace synth_trace(const LengthDistribution& ctx, const LengthDistribution& gen, double rate,
                  int64_t n, uint64_t seed) {
  if (rate <= 0) throw DataError("synth_trace: rate must be > 0");
  if (n < 0) throw DataError("synth_trace: negative request count");
  Trace t;
  t.requests.reserve(size_t(n));
  std::mt19937_64 g(seed);
  // Box-Muller on two uniform draws, rounded and truncated at one token
  auto length = [&](const LengthDistribution& d) {
    const double u1 = unit_open0(g), u2 = unit_open0(g);
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    return std::max<int64_t>(1, llround(d.mean + d.stddev * z));
  };
  double clock = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    Request r;
    r.id = i;
    clock += -std::log(unit_open0(g)) / rate;
    r.arrival = clock;
    r.context_len = length(ctx);
    r.gen_len = length(gen);
    t.requests.push_back(r);
  }
  return t;
}

}  // namespace psb
