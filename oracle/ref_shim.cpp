// TEST INFRASTRUCTURE -- C entry points over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp compiled in place by oracle/Makefile into
// oracle/_ref/libmemsched_ref.so). Used only by tests/, by
// tests/golden/make_golden.py (fixture generation) and by bench.py's
// reference / cpu_baseline arm. Never linked into the product.
//
// Everything crosses this boundary as JSON in the reference's own formats:
// graphs as save_graph/load_graph documents (graph.cpp:187-243), plans as
// save_plans documents (plan.cpp:30-65) and reports as PeakReport::to_json
// (peak.cpp:258-272).
#include <algorithm>
#include <chrono>
#include <random>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "memsched/latency.hpp"
#include "memsched/orchestrator.hpp"
#include "memsched/peak.hpp"
#include "memsched/plan.hpp"
#include "memsched/scenario.hpp"
#include "memsched/simulator.hpp"
#include "memsched/swap_planner.hpp"
#include "memsched/workload.hpp"
// test_support.hpp is header-only reference test code (random_job,
// planned_random_job, replay_oracle); compiled where it lies.
#include "test_support.hpp"

using namespace memsched;
using json = nlohmann::json;
using ojson = nlohmann::ordered_json;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

std::string lat_doc(const std::map<OpId, Tick>& lat) {
  ojson d = ojson::object();
  for (const auto& [op, t] : lat) d[op] = t;
  return d.dump();
}

PlannerConfig parse_config(const json& c) {
  PlannerConfig cfg;
  cfg.pcie_bandwidth = c.at("pcie_bandwidth").get<Bytes>();
  cfg.transfer_setup = c.at("transfer_setup").get<Tick>();
  cfg.memory_budget = c.at("memory_budget").get<Bytes>();
  if (c.contains("ewma_alpha")) cfg.ewma_alpha = c["ewma_alpha"].get<double>();
  if (c.contains("replan_threshold"))
    cfg.replan_threshold = c["replan_threshold"].get<double>();
  if (c.contains("stall_epsilon")) cfg.stall_epsilon = c["stall_epsilon"].get<double>();
  if (c.contains("stall_min_iters")) cfg.stall_min_iters = c["stall_min_iters"].get<int>();
  // JSON has no NaN / infinity: oracle/ref.py sends non-finite ratios as the
  // strings "nan" / "inf" / "-inf" (PlannerConfig::validate lets NaN through)
  if (c.contains("max_swap_ratios"))
    for (const auto& [k, v] : c["max_swap_ratios"].items())
      cfg.max_swap_ratios[k] = v.is_string() ? std::stod(v.get<std::string>()) : v.get<double>();
  return cfg;
}

using JobList = std::vector<std::pair<ComputeGraph, std::map<OpId, Tick>>>;

JobList parse_jobs(const json& req) {
  JobList jobs;
  for (const auto& j : req.at("jobs")) {
    ComputeGraph g = load_graph(j.at("graph").dump());
    std::map<OpId, Tick> lat;
    for (const auto& [k, v] : j.at("latencies").items()) lat[k] = v.get<Tick>();
    jobs.emplace_back(std::move(g), std::move(lat));
  }
  return jobs;
}

json report_json(const PeakReport& r) { return json::parse(r.to_json()); }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// generate_workload + true_latency_table (workload.cpp:96-209).
int ref_generate_workload(const char* family, int batch, std::uint64_t seed, int depth,
                          const char* job_id, std::uint64_t lat_seed, double usage,
                          char** graph_json, char** lat_json) {
  return guarded([&] {
    WorkloadSpec spec;
    spec.family = family;
    spec.batch_size = batch;
    spec.seed = seed;
    spec.depth = depth;
    spec.job_id = job_id ? job_id : "";
    ComputeGraph g = generate_workload(spec);
    *graph_json = dup(save_graph(g));
    *lat_json = dup(lat_doc(true_latency_table(g, lat_seed, usage)));
  });
}

// testsup::random_job (test_support.hpp:166-178).
int ref_random_job(std::uint64_t seed, char** graph_json, char** lat_json) {
  return guarded([&] {
    auto [g, lat] = testsup::random_job(seed);
    *graph_json = dup(save_graph(g));
    *lat_json = dup(lat_doc(lat));
  });
}

// Initial per-job peaks (make_job_context, swap_planner.cpp:156-169).
int ref_initial_peaks(const char* request, char** out_json) {
  return guarded([&] {
    json req = json::parse(request);
    JobList jobs = parse_jobs(req);
    ojson out = ojson::object();
    for (auto& [g, lat] : jobs) {
      JobContext ctx = make_job_context(g, lat);
      out[g.job_id()] = ctx.report.memory_peak;
    }
    *out_json = dup(out.dump());
  });
}

// build_plan (orchestrator.cpp:8-70), timed `repeats` times around the call
// (make_job_context included, JSON parsing excluded).
int ref_build_plan(const char* request, int repeats, char** plans_json, char** result_json) {
  return guarded([&] {
    json req = json::parse(request);
    PlannerConfig cfg = parse_config(req.at("config"));
    JobList jobs = parse_jobs(req);
    BuildResult r;
    std::vector<double> times;
    for (int i = 0; i < std::max(1, repeats); ++i) {
      auto t0 = std::chrono::steady_clock::now();
      r = build_plan(jobs, cfg);
      auto t1 = std::chrono::steady_clock::now();
      times.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    std::size_t n_acc = 0;
    for (auto& [g, lat] : jobs)
      n_acc += generate_access_sequence(g, lat).accesses.size();
    ojson out;
    out["merged_peak_history"] = r.merged_peak_history;
    out["final_merged_peak"] = r.final_merged_peak;
    out["within_budget"] = r.within_budget;
    out["diagnostic"] = r.diagnostic;
    ojson reps = ojson::object();
    for (const auto& [job, rep] : r.reports) reps[job] = ojson::parse(rep.to_json());
    out["reports"] = reps;
    out["n_accesses"] = n_acc;
    out["times_ms"] = times;
    *plans_json = dup(save_plans(r.plans));
    *result_json = dup(out.dump());
  });
}

// testsup::planned_random_job + analyzer + replay_oracle
// (test_support.hpp:52-226): golden vectors for the footprint evaluator.
int ref_planned_random_job(std::uint64_t seed, int max_swaps, std::int64_t bw,
                           std::int64_t setup, char** out_json) {
  return guarded([&] {
    PlannerConfig cfg;
    cfg.pcie_bandwidth = bw;
    cfg.transfer_setup = setup;
    JobContext job = testsup::planned_random_job(seed, max_swaps, cfg);
    testsup::OracleResult o = testsup::replay_oracle(job.seq, job.plan, job.catalog);
    auto [g, lat] = testsup::random_job(seed);
    ojson out;
    out["graph"] = ojson::parse(save_graph(g));
    out["latencies"] = ojson::parse(lat_doc(lat));
    out["plan"] = ojson::parse(save_plans({{job.seq.job_id, job.plan}}))[job.seq.job_id];
    out["report"] = ojson::parse(job.report.to_json());
    ojson oo;
    oo["peak"] = o.peak;
    oo["peak_time"] = o.peak_time;
    oo["tensors"] = std::vector<std::string>(o.tensors.begin(), o.tensors.end());
    out["replay_oracle"] = oo;
    *out_json = dup(out.dump());
  });
}

// analyze_job (peak.cpp:246-250) on a caller-supplied plan for one job.
// request: {"graph":…, "latencies":…, "plan": <save_plans entry>}
int ref_analyze_job(const char* request, char** out_json) {
  return guarded([&] {
    json req = json::parse(request);
    ComputeGraph g = load_graph(req.at("graph").dump());
    std::map<OpId, Tick> lat;
    for (const auto& [k, v] : req.at("latencies").items()) lat[k] = v.get<Tick>();
    JobContext ctx = make_job_context(g, lat);
    json wrapped;
    wrapped[g.job_id()] = req.at("plan");
    auto plans = load_plans(wrapped.dump());
    SchedulingPlan plan = plans.at(g.job_id());
    PeakReport rep = analyze_job(ctx.seq, plan, ctx.catalog);
    *out_json = dup(rep.to_json());
  });
}

// The reference CLI's `plan` subcommand (tools/memsched_cli.cpp:136-153):
// load_scenario + plan_scenario, outputs formatted exactly as the CLI writes
// plans.json / peaks.json; *diag = plan_diagnostic.
int ref_plan_scenario(const char* document, const char* base_dir, char** plans_json, char** peaks_json,
                      char** diag) {
  return guarded([&] {
    ScenarioConfig cfg = load_scenario(document, base_dir);
    ScenarioResult result = plan_scenario(cfg);
    *plans_json = dup(save_plans(result.plans));
    std::string o = "{\n";
    bool first = true;
    for (const auto& [job, rep] : result.peak_reports) {
      if (!first) o += ",\n";
      first = false;
      o += "\"" + job + "\": " + rep.to_json();
    }
    o += "}\n";
    *peaks_json = dup(o);
    *diag = dup(result.plan_diagnostic);
  });
}

// generate_training_samples (workload.cpp:211-248) for a graph:
// [[op_kind, [values...], label], ...].
int ref_training_samples(const char* graph_json, std::uint64_t seed, int per_op, double noise, char** out_json) {
  return guarded([&] {
    ComputeGraph g = load_graph(graph_json);
    ojson o = ojson::array();
    for (const auto& [fv, y] : generate_training_samples(g, seed, per_op, noise))
      o.push_back({fv.op_kind, fv.values, y});
    *out_json = dup(o.dump());
  });
}

// The reference unit test's linear_samples (test_latency.cpp:44-62):
// latency = 2 * dim0 + 5 with optional multiplicative noise.
int ref_linear_samples(double noise_fraction, std::uint64_t seed, char** out_json) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> usage(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    ojson o = ojson::array();
    for (int i = 1; i <= 60; ++i) {
      std::vector<double> v = {static_cast<double>(i), usage(rng)};
      double label = 2.0 * v[0] + 5.0;
      if (noise_fraction > 0) label *= 1.0 + noise_fraction * gauss(rng);
      o.push_back({"k", v, label});
    }
    *out_json = dup(o.dump());
  });
}

// LatencyPredictor::from_json -> to_json (the reference's text of a document).
int ref_predictor_roundtrip(const char* doc, char** out) {
  return guarded([&] { *out = dup(LatencyPredictor::from_json(doc).to_json()); });
}

// predict_latencies (orchestrator.cpp:72-87) with a predictor document.
int ref_predict_latencies(const char* graph_json, const char* predictor_doc, double usage, char** out_json) {
  return guarded([&] {
    ComputeGraph g = load_graph(graph_json);
    ojson o = ojson::object();
    for (const auto& [op, t] : predict_latencies(g, LatencyPredictor::from_json(predictor_doc), usage)) o[op] = t;
    *out_json = dup(o.dump());
  });
}

// memsched::simulate (simulator.cpp:573-582) on caller plans.
// request: {"jobs": [{"graph", "latencies" (TRUE latencies), "launch_tick"}],
//           "plans": <save_plans document>, "config": {"mode": "vanilla" |
//           "scheduled" | "passive", "iterations", "memory_budget",
//           "pcie_bandwidth", "transfer_setup", "slowdown": {jobs: mult},
//           "ticks_per_iteration_limit"}}
// out: the trace in tsl_sim_trace_json's layout + "csv" (to_csv).
int ref_simulate(const char* request, char** out_json) {
  return guarded([&] {
    json req = json::parse(request);
    std::vector<SimJob> jobs;
    for (const auto& j : req.at("jobs")) {
      SimJob sj;
      sj.graph = load_graph(j.at("graph").dump());
      for (const auto& [k, v] : j.at("latencies").items()) sj.true_latencies[k] = v.get<Tick>();
      sj.launch_tick = j.value("launch_tick", Tick{0});
      jobs.push_back(std::move(sj));
    }
    std::map<JobId, SchedulingPlan> plans;
    if (req.contains("plans")) plans = load_plans(req["plans"].dump());
    const json& c = req.at("config");
    SimConfig cfg;
    const std::string mode = c.value("mode", std::string("vanilla"));
    cfg.mode = mode == "scheduled" ? SimMode::Scheduled : mode == "passive" ? SimMode::Passive : SimMode::Vanilla;
    cfg.iterations = c.value("iterations", 1);
    cfg.memory_budget = c.value("memory_budget", Bytes{0});
    cfg.pcie_bandwidth = c.value("pcie_bandwidth", Bytes{1});
    cfg.transfer_setup = c.value("transfer_setup", Tick{0});
    if (c.contains("ticks_per_iteration_limit")) cfg.ticks_per_iteration_limit = c["ticks_per_iteration_limit"].get<Tick>();
    if (c.contains("slowdown"))
      for (const auto& [k, v] : c["slowdown"].items()) cfg.gpu_slowdown_curve[std::stoi(k)] = v.get<double>();
    SimulationTrace t = simulate(jobs, plans, cfg);
    ojson o;
    o["peak"] = t.peak;
    o["blocked_ticks"] = t.blocked_ticks;
    o["passive_swap_count"] = t.passive_swap_count;
    ojson js = ojson::array();
    for (const auto& sj : jobs) {
      const JobId id = sj.graph.job_id();
      ojson e;
      e["job_id"] = id;
      e["peak"] = t.per_job_peak.count(id) ? t.per_job_peak.at(id) : 0;
      e["iteration_times"] = t.iteration_times.count(id) ? t.iteration_times.at(id) : std::vector<Tick>{};
      e["plan_versions"] = t.plan_versions.count(id) ? t.plan_versions.at(id) : std::vector<std::int64_t>{};
      ojson curve = ojson::array();
      if (t.per_job_curve.count(id))
        for (const auto& [tick, b] : t.per_job_curve.at(id)) curve.push_back({tick, b});
      e["footprint_curve"] = curve;
      js.push_back(e);
    }
    o["jobs"] = js;
    ojson tr = ojson::array();
    for (const auto& x : t.transfers) tr.push_back({x.start, x.end, x.job_id, x.tensor_id, x.kind});
    o["transfers"] = tr;
    o["safety_violations"] = t.safety_violations;
    ojson pe = ojson::array();
    for (const auto& [j, it, s] : t.passive_events) pe.push_back({j, it, s});
    o["passive_events"] = pe;
    o["csv"] = t.to_csv();
    *out_json = dup(o.dump());
  });
}

// run_scenario (scenario.cpp:223-262): the modes' ModeStats::to_json texts,
// the scheduled plans (save_plans) and replan count, and each mode's trace CSV.
int ref_run_scenario(const char* document, const char* base_dir, const char* modes_csv, char** out_json) {
  return guarded([&] {
    ScenarioConfig cfg = load_scenario(document, base_dir);
    std::set<std::string> modes;
    std::string m = modes_csv, cur;
    for (char ch : m + ",") {
      if (ch == ',') { if (!cur.empty()) modes.insert(cur); cur.clear(); }
      else cur += ch;
    }
    ScenarioResult r = run_scenario(cfg, modes);
    ojson o;
    ojson st = ojson::object();
    for (const auto& [mode, s] : r.stats) st[mode] = s.to_json();
    o["stats"] = st;
    ojson csv = ojson::object();
    for (const auto& [mode, t] : r.traces) csv[mode] = t.to_csv();
    o["csv"] = csv;
    o["plans"] = save_plans(r.plans);
    o["replan_count"] = r.replan_count;
    o["diagnostic"] = r.plan_diagnostic;
    *out_json = dup(o.dump());
  });
}

}  // extern "C"
