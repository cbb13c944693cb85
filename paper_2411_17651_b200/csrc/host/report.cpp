// report.cpp — report materialization without a JSON DOM.
//
// The reference builds an nlohmann::ordered_json per report
// (report_to_json, /root/reference/proj/src/simulator.cpp:331-369), and its
// CLI re-parses every report to assemble ranked.json
// (tools/plansim_main.cpp:128-131: parse -> push_back -> dump(2)).  For a
// 10k-request C2 search that is 151 MB through a DOM twice.  These writers
// stream the same bytes directly: the layout of nlohmann's pretty printer
// (indent 2, "key": value, one array element per line, "[]" / "{}" when
// empty) and its number formatting (nlohmann::detail::to_chars, the same
// header the reference links: nlohmann/json 3.11.3) — so the output is
// byte-identical to the reference's, which tests/test_gpu_report.py checks.
#include <algorithm>
#include <atomic>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "nlohmann/json.hpp"
#include "psb/plansim_b200.hpp"
#include "psg_host.h"

namespace psb {
namespace {

class Out {
 public:
  explicit Out(std::string& s) : s_(s) {}
  void raw(const char* p, size_t n) { s_.append(p, n); }
  void raw(const char* p) { s_.append(p); }
  void ch(char c) { s_.push_back(c); }
  void indent(int n) { s_.append(size_t(n), ' '); }
  void num(double v) {  // serializer::dump_float
    if (!std::isfinite(v)) {
      raw("null", 4);
      return;
    }
    char buf[64];
    char* end = nlohmann::detail::to_chars(buf, buf + sizeof buf, v);
    raw(buf, size_t(end - buf));
  }
  void num(int64_t v) {
    char buf[32];
    const int n = std::snprintf(buf, sizeof buf, "%" PRId64, v);
    raw(buf, size_t(n));
  }
  void str(const std::string& v) {  // serializer::dump_escaped, ensure_ascii = false
    ch('"');
    for (unsigned char c : v) {
      switch (c) {
        case '"': raw("\\\"", 2); break;
        case '\\': raw("\\\\", 2); break;
        case '\b': raw("\\b", 2); break;
        case '\f': raw("\\f", 2); break;
        case '\n': raw("\\n", 2); break;
        case '\r': raw("\\r", 2); break;
        case '\t': raw("\\t", 2); break;
        default:
          if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", unsigned(c));
            raw(buf, 6);
          } else {
            ch(char(c));
          }
      }
    }
    ch('"');
  }
  // pretty object member prefix: indent, "key":
  void key(int ind, const char* k) {
    indent(ind);
    ch('"');
    raw(k);
    raw("\": ", 3);
  }

 private:
  std::string& s_;
};

// Everything report_to_json reads, as flat views (SimulationReport or psg arrays).
struct ReportView {
  const std::string* encoding;
  double freq, e2e, energy, p95, ttft, tpot, mfu, mbu;
  int64_t completed, rejected, iterations, max_batch;
  const psg_request_metrics* per_request;
  int64_t n_per_request;
  const int64_t* rejected_ids;
  int64_t n_rejected;
  const IterationRecord* its;  // emitted iterations (C++ reports only)
  int64_t n_its;
};

// The nlohmann header a build links decides one layout detail: the copy in
// this image (cudnn_frontend's, which the reference oracle also links) prints
// an array whose first element is an integer on one line ("[1,2,3]"); stock
// nlohmann prints one element per line.  Probe the linked header once and
// follow it, so the bytes match whatever the reference is built against.
bool compact_int_arrays() {
  static const bool v = nlohmann::ordered_json::array({1, 2}).dump(2).find('\n') == std::string::npos;
  return v;
}

void int_array(Out& o, int ind, int64_t n, const int64_t* v) {
  if (n == 0) {
    o.raw("[]", 2);
    return;
  }
  if (compact_int_arrays()) {
    o.ch('[');
    for (int64_t i = 0; i < n; ++i) {
      if (i) o.ch(',');
      o.num(v[i]);
    }
    o.ch(']');
    return;
  }
  o.raw("[\n", 2);
  for (int64_t i = 0; i < n; ++i) {
    o.indent(ind + 2);
    o.num(v[i]);
    if (i + 1 < n) o.raw(",\n", 2);
  }
  o.ch('\n');
  o.indent(ind);
  o.ch(']');
}

template <typename Elem>
void pretty_array(Out& o, int ind, int64_t n, Elem&& elem) {
  if (n == 0) {
    o.raw("[]", 2);
    return;
  }
  o.raw("[\n", 2);
  for (int64_t i = 0; i < n; ++i) {
    o.indent(ind + 2);
    elem(i, ind + 2);
    if (i + 1 < n) o.raw(",\n", 2);
  }
  o.ch('\n');
  o.indent(ind);
  o.ch(']');
}

void doubles_pretty(Out& o, int ind, const std::vector<double>& v) {
  pretty_array(o, ind, int64_t(v.size()), [&](int64_t i, int) { o.num(v[size_t(i)]); });
}

// report_to_json's object (simulator.cpp:331-369) at indentation `ind`.
void report_object(Out& o, const ReportView& r, int ind) {
  const int m = ind + 2;
  o.raw("{\n", 2);
  o.key(m, "plan");
  o.str(*r.encoding);
  o.raw(",\n", 2);
  o.key(m, "frequency_ghz");
  o.num(r.freq);
  o.raw(",\n", 2);
  o.key(m, "metrics");
  {
    const int k = m + 2;
    o.raw("{\n", 2);
    o.key(k, "e2e_latency_s"); o.num(r.e2e); o.raw(",\n", 2);
    o.key(k, "total_energy_j"); o.num(r.energy); o.raw(",\n", 2);
    o.key(k, "p95_latency_s"); o.num(r.p95); o.raw(",\n", 2);
    o.key(k, "mean_ttft_s"); o.num(r.ttft); o.raw(",\n", 2);
    o.key(k, "mean_tpot_s"); o.num(r.tpot); o.raw(",\n", 2);
    o.key(k, "mfu"); o.num(r.mfu); o.raw(",\n", 2);
    o.key(k, "mbu"); o.num(r.mbu); o.raw(",\n", 2);
    o.key(k, "num_completed"); o.num(r.completed); o.raw(",\n", 2);
    o.key(k, "num_rejected"); o.num(r.rejected); o.raw(",\n", 2);
    o.key(k, "num_iterations"); o.num(r.iterations); o.raw(",\n", 2);
    o.key(k, "max_batch_observed"); o.num(r.max_batch); o.ch('\n');
    o.indent(m);
    o.ch('}');
  }
  o.raw(",\n", 2);
  o.key(m, "per_request");
  pretty_array(o, m, r.n_per_request, [&](int64_t i, int ei) {
    const psg_request_metrics& q = r.per_request[i];
    const int k = ei + 2;
    o.raw("{\n", 2);
    o.key(k, "id"); o.num(q.id); o.raw(",\n", 2);
    o.key(k, "ttft_s"); o.num(q.ttft); o.raw(",\n", 2);
    o.key(k, "tpot_s"); o.num(q.tpot); o.raw(",\n", 2);
    o.key(k, "e2e_s"); o.num(q.e2e); o.raw(",\n", 2);
    o.key(k, "gen_len"); o.num(q.gen_len); o.ch('\n');
    o.indent(ei);
    o.ch('}');
  });
  o.raw(",\n", 2);
  o.key(m, "rejected");
  int_array(o, m, r.n_rejected, r.rejected_ids);
  if (r.n_its > 0) {
    o.raw(",\n", 2);
    o.key(m, "iterations");
    pretty_array(o, m, r.n_its, [&](int64_t i, int ei) {
      const IterationRecord& it = r.its[i];
      const int k = ei + 2;
      o.raw("{\n", 2);
      o.key(k, "clock_start_s"); o.num(it.clock_start); o.raw(",\n", 2);
      o.key(k, "duration_s"); o.num(it.duration); o.raw(",\n", 2);
      o.key(k, "energy_j"); o.num(it.energy); o.raw(",\n", 2);
      o.key(k, "batch_size"); o.num(it.batch_size); o.raw(",\n", 2);
      o.key(k, "stage_seconds"); doubles_pretty(o, k, it.stage_seconds); o.raw(",\n", 2);
      o.key(k, "stage_joules"); doubles_pretty(o, k, it.stage_joules); o.ch('\n');
      o.indent(ei);
      o.ch('}');
    });
  }
  o.ch('\n');
  o.indent(ind);
  o.ch('}');
}

ReportView view_of(const SimulationReport& r) {
  ReportView v{};
  v.encoding = &r.plan_encoding;
  v.freq = r.frequency_ghz;
  v.e2e = r.e2e_latency;
  v.energy = r.total_energy;
  v.p95 = r.p95_latency;
  v.ttft = r.mean_ttft;
  v.tpot = r.mean_tpot;
  v.mfu = r.mfu;
  v.mbu = r.mbu;
  v.completed = r.num_completed;
  v.rejected = r.num_rejected;
  v.iterations = r.num_iterations;
  v.max_batch = r.max_batch_observed;
  v.per_request = reinterpret_cast<const psg_request_metrics*>(r.per_request.data());
  v.n_per_request = int64_t(r.per_request.size());
  v.rejected_ids = r.rejected_ids.data();
  v.n_rejected = int64_t(r.rejected_ids.size());
  v.its = r.iterations.data();
  v.n_its = int64_t(r.iterations.size());
  return v;
}

// Streams `s` to `path` in chunks as it grows.
class FileSink {
 public:
  explicit FileSink(const std::string& path) : f_(std::fopen(path.c_str(), "wb")) {
    if (!f_) throw DataError("cannot write " + path);
    buf_.reserve(kChunk * 2);
  }
  ~FileSink() {
    if (f_) std::fclose(f_);
  }
  std::string& buf() { return buf_; }
  void maybe_flush() {
    if (buf_.size() >= kChunk) flush();
  }
  void flush() {
    if (!buf_.empty() && std::fwrite(buf_.data(), 1, buf_.size(), f_) != buf_.size())
      throw DataError("write failed");
    buf_.clear();
  }
  void close() {
    flush();
    if (std::fclose(f_) != 0) {
      f_ = nullptr;
      throw DataError("write failed");
    }
    f_ = nullptr;
  }

 private:
  static constexpr size_t kChunk = size_t(8) << 20;
  std::FILE* f_;
  std::string buf_;
};

// ranked.json: entries are formatted in parallel on host threads (each into
// its own buffer), then written in order.
template <typename Each>
void ranked_stream(FileSink& sink, int64_t n, Each&& view_at) {
  Out o(sink.buf());
  if (n == 0) {
    o.raw("[]\n", 3);
    return;
  }
  std::vector<std::string> parts(static_cast<size_t>(n));
  std::atomic<int64_t> next{0};
  std::atomic<bool> failed{false};
  std::string why;
  std::mutex mu;
  auto work = [&]() {
    for (int64_t i; (i = next.fetch_add(1)) < n && !failed.load();) {
      try {
        Out p(parts[size_t(i)]);
        p.indent(2);
        report_object(p, view_at(i), 2);
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> g(mu);
        why = e.what();
        failed = true;
      }
    }
  };
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t T = std::min<int64_t>({hw, n, 64});
  std::vector<std::thread> pool;
  for (int64_t t = 1; t < T; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  if (failed) throw DataError(why);
  o.raw("[\n", 2);
  for (int64_t i = 0; i < n; ++i) {
    sink.buf() += parts[size_t(i)];
    std::string().swap(parts[size_t(i)]);
    if (i + 1 < n) o.raw(",\n", 2);
    sink.maybe_flush();
  }
  o.raw("\n]\n", 3);
}

}  // namespace

std::string report_to_json(const SimulationReport& r) {
  std::string s;
  Out o(s);
  report_object(o, view_of(r), 0);
  s.push_back('\n');
  return s;
}

std::string iterations_to_jsonl(const SimulationReport& r) {  // simulator.cpp:371-385
  std::string s;
  Out o(s);
  for (const IterationRecord& it : r.iterations) {
    o.raw("{\"clock_start_s\":");
    o.num(it.clock_start);
    o.raw(",\"duration_s\":");
    o.num(it.duration);
    o.raw(",\"energy_j\":");
    o.num(it.energy);
    o.raw(",\"batch_size\":");
    o.num(it.batch_size);
    for (int pass = 0; pass < 2; ++pass) {
      o.raw(pass == 0 ? ",\"stage_seconds\":[" : ",\"stage_joules\":[");
      const auto& v = pass == 0 ? it.stage_seconds : it.stage_joules;
      for (size_t k = 0; k < v.size(); ++k) {
        if (k) o.ch(',');
        o.num(v[k]);
      }
      o.ch(']');
    }
    o.raw("}\n", 2);
  }
  return s;
}

std::string report_summary_line(const SimulationReport& r) {  // simulator.cpp:387-397
  std::ostringstream ss;
  ss << r.plan_encoding << " @" << r.frequency_ghz << "GHz"
     << "  e2e=" << r.e2e_latency << "s"
     << "  energy=" << r.total_energy << "J"
     << "  p95=" << r.p95_latency << "s"
     << "  ttft=" << r.mean_ttft << "s"
     << "  tpot=" << r.mean_tpot << "s"
     << "  mfu=" << r.mfu << "  mbu=" << r.mbu
     << "  completed=" << r.num_completed << "  rejected=" << r.num_rejected;
  return ss.str();
}

void write_ranked_json(const RankedPlans& ranked, const std::string& path) {
  FileSink sink(path);
  ranked_stream(sink, int64_t(ranked.entries.size()),
                [&](int64_t i) { return view_of(ranked.entries[size_t(i)].report); });
  sink.close();
}

std::string sweep_to_json(const SweepTable& t) {  // tools/plansim_main.cpp:184-199
  std::string s;
  Out o(s);
  o.raw("{\n");
  o.key(2, "observed_max_batch");
  o.num(t.observed_max_batch);
  o.raw(",\n", 2);
  o.key(2, "rows");
  pretty_array(o, 2, int64_t(t.rows.size()), [&](int64_t i, int ei) {
    const SweepRow& r = t.rows[size_t(i)];
    const int k = ei + 2;
    o.raw("{\n", 2);
    o.key(k, "max_batch_size"); o.num(r.max_batch_size); o.raw(",\n", 2);
    o.key(k, "mean_tpot_s"); o.num(r.mean_tpot); o.raw(",\n", 2);
    o.key(k, "mean_ttft_s"); o.num(r.mean_ttft); o.raw(",\n", 2);
    o.key(k, "e2e_latency_s"); o.num(r.e2e_latency); o.ch('\n');
    o.indent(ei);
    o.ch('}');
  });
  o.raw("\n}\n", 3);
  return s;
}

}  // namespace psb

// ---- C ABI over psg_search results (include/psg_host.h) ----

namespace {

psb::ReportView view_of_entry(const psg_entry& e, const std::string* enc,
                              const psg_request_metrics* per_request, const int64_t* rejected_ids) {
  psb::ReportView v{};
  v.encoding = enc;
  v.freq = e.freq_ghz;
  v.e2e = e.e2e_latency;
  v.energy = e.total_energy;
  v.p95 = e.p95_latency;
  v.ttft = e.mean_ttft;
  v.tpot = e.mean_tpot;
  v.mfu = e.mfu;
  v.mbu = e.mbu;
  v.completed = e.num_completed;
  v.rejected = e.num_rejected;
  v.iterations = e.num_iterations;
  v.max_batch = e.max_batch_observed;
  v.per_request = per_request + e.per_request_offset;
  v.n_per_request = e.num_completed;
  v.rejected_ids = rejected_ids + e.rejected_offset;
  v.n_rejected = e.num_rejected;
  return v;
}

int write_text(const std::string& text, const char* path) {
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return PSG_ERR_DATA;
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  return (std::fclose(f) == 0 && ok) ? PSG_OK : PSG_ERR_DATA;
}

}  // namespace

extern "C" int psgh_write_report_json(const psg_entry* entry, const psg_request_metrics* per_request,
                                      const int64_t* rejected_ids, const char* plan_encoding,
                                      const char* path) {
  try {
    const std::string enc(plan_encoding);
    std::string s;
    psb::Out o(s);
    psb::report_object(o, view_of_entry(*entry, &enc, per_request, rejected_ids), 0);
    s.push_back('\n');
    return write_text(s, path);
  } catch (const std::exception&) {
    return PSG_ERR_DATA;
  }
}

extern "C" int psgh_write_iterations_jsonl(const psg_iteration* its, int64_t n,
                                           const double* stage_seconds, const double* stage_joules,
                                           int32_t n_stages, const char* path) {
  try {
    psb::SimulationReport r;
    r.iterations.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) {
      psb::IterationRecord& it = r.iterations[size_t(i)];
      it.clock_start = its[i].clock_start;
      it.duration = its[i].duration;
      it.energy = its[i].energy;
      it.batch_size = its[i].batch_size;
      it.stage_seconds.assign(stage_seconds + i * n_stages, stage_seconds + (i + 1) * n_stages);
      it.stage_joules.assign(stage_joules + i * n_stages, stage_joules + (i + 1) * n_stages);
    }
    return write_text(psb::iterations_to_jsonl(r), path);
  } catch (const std::exception&) {
    return PSG_ERR_DATA;
  }
}

extern "C" int psgh_write_sweep_json(int64_t observed_max_batch, const int64_t* caps,
                                     const double* mean_tpot, const double* mean_ttft,
                                     const double* e2e, int32_t n_rows, const char* path) {
  try {
    psb::SweepTable t;
    t.observed_max_batch = observed_max_batch;
    for (int32_t i = 0; i < n_rows; ++i) t.rows.push_back({caps[i], mean_tpot[i], mean_ttft[i], e2e[i]});
    return write_text(psb::sweep_to_json(t), path);
  } catch (const std::exception&) {
    return PSG_ERR_DATA;
  }
}

extern "C" int psgh_write_ranked_json(const psg_entry* entries, int64_t n_entries,
                                      const psg_request_metrics* per_request,
                                      const int64_t* rejected_ids,
                                      const char* const* plan_encodings, int32_t n_plans,
                                      const char* path) {
  try {
    std::vector<std::string> enc(plan_encodings, plan_encodings + n_plans);
    psb::FileSink sink(path);
    psb::ranked_stream(sink, n_entries, [&](int64_t i) {
      const psg_entry& e = entries[i];
      if (e.plan_index < 0 || e.plan_index >= n_plans) throw psb::DataError("plan index out of range");
      return view_of_entry(e, &enc[size_t(e.plan_index)], per_request, rejected_ids);
    });
    sink.close();
    return PSG_OK;
  } catch (const std::exception&) {
    return PSG_ERR_DATA;
  }
}
