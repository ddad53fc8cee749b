// Drop-in replacement for the reference's orchestrator translation unit
// (/root/reference/proj/src/orchestrator.cpp) that plans on the B200 through
// the C-ABI in include/tensile_b200.h.
//
// A maintainer links this file INSTEAD of orchestrator.cpp (that TU defines
// build_plan, predict_latencies and Orchestrator together, so both cannot be
// linked) plus paper_2105_13336_b200/libtensile_b200.so. Everything above the
// planner -- scenario.cpp, the CLI, the reference's own tests -- links
// unchanged against the reference headers:
//
//   memsched::build_plan           orchestrator.hpp:26-28 -> tsl_build_plan
//   memsched::predict_latencies    orchestrator.hpp:32-34 (host arithmetic)
//   memsched::Orchestrator         orchestrator.hpp:39-67 (replan lifecycle)
//
// Errors keep the reference contract: PlannerConfig::validate() runs first
// (config.hpp:25-35), every validation failure reported by the library is
// rethrown as memsched::ValidationError with the same text, anything else
// (no CUDA device, capacity) as std::runtime_error.
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "memsched/orchestrator.hpp"
#include "tensile_b200.h"

namespace memsched {
namespace {

int8_t kind_code(TensorKind k) {
  switch (k) {
    case TensorKind::Input: return TSL_KIND_INPUT;
    case TensorKind::Interim: return TSL_KIND_INTERIM;
    case TensorKind::Parameter: return TSL_KIND_PARAMETER;
    case TensorKind::UpdatedParameter: return TSL_KIND_UPDATED_PARAMETER;
    case TensorKind::Output: return TSL_KIND_OUTPUT;
  }
  return TSL_KIND_INTERIM;
}

tsl_ctx* device_context() {
  static std::once_flag once;
  static tsl_ctx* ctx = nullptr;
  static std::string err;
  std::call_once(once, [] {
    const char* dev = std::getenv("TSL_DEVICE");
    if (tsl_create(dev ? std::atoi(dev) : 0, &ctx) != TSL_OK) err = tsl_last_error();
  });
  if (!ctx) throw std::runtime_error("B200 planner unavailable: " + err);
  return ctx;
}

[[noreturn]] void rethrow(int rc) {
  if (rc == TSL_ERR_VALIDATION) throw ValidationError(tsl_last_error());
  throw std::runtime_error(tsl_last_error());
}

// One job packed into the C-ABI's integer SoA form; owns the buffers.
struct PackedJob {
  std::vector<const char*> tids, oids, okinds;
  std::vector<int64_t> sizes, lat;
  std::vector<int8_t> kinds, phases;
  std::vector<int32_t> in_off{0}, ins, out_off{0}, outs;
  tsl_job_desc desc{};

  PackedJob(const ComputeGraph& g, const std::map<OpId, Tick>& latencies) {
    std::map<TensorId, int32_t> index;
    for (const auto& t : g.tensors()) {
      index.emplace(t.id, static_cast<int32_t>(tids.size()));
      tids.push_back(t.id.c_str());
      sizes.push_back(t.size);
      kinds.push_back(kind_code(t.kind));
    }
    for (const auto& op : g.ops()) {
      oids.push_back(op.id.c_str());
      okinds.push_back(op.kind.c_str());
      phases.push_back(op.phase == OpPhase::Optimize ? TSL_PHASE_OPTIMIZE : TSL_PHASE_FORWARD_BACKWARD);
      for (const auto& t : op.inputs) ins.push_back(index.at(t));
      for (const auto& t : op.outputs) outs.push_back(index.at(t));
      in_off.push_back(static_cast<int32_t>(ins.size()));
      out_off.push_back(static_cast<int32_t>(outs.size()));
      auto it = latencies.find(op.id);
      lat.push_back(it == latencies.end() ? TSL_LATENCY_MISSING : it->second);
    }
    desc.job_id = g.job_id().c_str();
    desc.n_tensors = static_cast<int32_t>(tids.size());
    desc.tensor_ids = tids.data();
    desc.tensor_sizes = sizes.data();
    desc.tensor_kinds = kinds.data();
    desc.n_ops = static_cast<int32_t>(oids.size());
    desc.op_ids = oids.data();
    desc.op_kinds = okinds.data();
    desc.op_phases = phases.data();
    desc.op_in_offsets = in_off.data();
    desc.op_inputs = ins.data();
    desc.op_out_offsets = out_off.data();
    desc.op_outputs = outs.data();
    desc.op_latencies = lat.data();
  }
};

SchedulingPlan unpack_plan(const tsl_job_view& v, const ComputeGraph& g) {
  const auto& ts = g.tensors();
  SchedulingPlan plan;
  plan.job_id = v.job_id;
  plan.version = v.version;
  for (int32_t i = 0; i < v.n_swap; ++i) {
    SwapEvent e;
    e.event_id = v.ev_id[i];
    e.job_id = plan.job_id;
    e.tensor_id = ts[static_cast<size_t>(v.ev_tensor[i])].id;
    e.direction = v.ev_dir[i] == 0 ? SwapDirection::Out : SwapDirection::In;
    e.trigger_access = v.ev_trigger[i];
    e.delta_time = v.ev_delta[i];
    e.start_time = v.ev_start[i];
    e.end_time = v.ev_end[i];
    e.earliest_time = v.ev_earliest[i];
    e.latest_time = v.ev_latest[i];
    e.wraps_iteration = v.ev_wraps[i] != 0;
    e.pair_id = v.ev_pair[i];
    e.serves_access = v.ev_serves[i];
    plan.swap_events.push_back(std::move(e));
  }
  for (int32_t i = 0; i < v.n_recompute; ++i) {
    RecomputeEvent e;
    e.event_id = v.rc_id[i];
    e.job_id = plan.job_id;
    e.tensor_id = ts[static_cast<size_t>(v.rc_tensor[i])].id;
    e.target_access = v.rc_target[i];
    e.regen_op = g.ops()[static_cast<size_t>(v.rc_regen_op[i])].id;
    e.recompute_latency = v.rc_latency[i];
    e.memory_saving = v.rc_saving[i];
    plan.recompute_events.push_back(std::move(e));
  }
  for (int32_t i = 0; i < v.n_release; ++i) plan.release_flags.insert(v.release_flags[i]);
  return plan;
}

PeakReport unpack_report(const tsl_job_view& v, const ComputeGraph& g) {
  PeakReport r;
  r.memory_peak = v.memory_peak;
  r.peak_time = v.peak_time;
  if (v.has_last_input_access) r.last_input_access = v.last_input_access;
  for (int32_t i = 0; i < v.n_peak_tensors; ++i)
    r.peak_tensors.insert(g.tensors()[static_cast<size_t>(v.peak_tensors[i])].id);
  for (int32_t i = 0; i < v.n_curve; ++i) r.footprint_curve.emplace_back(v.curve_time[i], v.curve_bytes[i]);
  return r;
}

}  // namespace

BuildResult build_plan(const std::vector<std::pair<ComputeGraph, std::map<OpId, Tick>>>& jobs,
                       const PlannerConfig& config) {
  config.validate();
  BuildResult result;
  if (jobs.empty()) return result;
  std::vector<PackedJob> packed;
  packed.reserve(jobs.size());
  for (const auto& [g, lat] : jobs) packed.emplace_back(g, lat);
  std::vector<tsl_job_desc> descs;
  for (const auto& p : packed) descs.push_back(p.desc);
  tsl_config cfg;
  tsl_config_default(&cfg);
  cfg.pcie_bandwidth = config.pcie_bandwidth;
  cfg.transfer_setup = config.transfer_setup;
  cfg.memory_budget = config.memory_budget;
  cfg.ewma_alpha = config.ewma_alpha;
  cfg.replan_threshold = config.replan_threshold;
  cfg.stall_epsilon = config.stall_epsilon;
  cfg.stall_min_iters = config.stall_min_iters;
  cfg.cold_start_gpu_usage = config.cold_start_gpu_usage;
  std::vector<const char*> ratio_jobs;  // PlannerConfig::max_swap_ratios, every entry
  std::vector<double> ratio_values;
  for (const auto& [job, r] : config.max_swap_ratios) {
    ratio_jobs.push_back(job.c_str());
    ratio_values.push_back(r);
  }
  cfg.n_max_swap_ratios = static_cast<int32_t>(ratio_jobs.size());
  cfg.max_swap_ratio_jobs = ratio_jobs.data();
  cfg.max_swap_ratio_values = ratio_values.data();
  tsl_result* r = nullptr;
  const int rc = tsl_build_plan(device_context(), descs.data(), static_cast<int32_t>(descs.size()), &cfg, &r);
  if (rc != TSL_OK) rethrow(rc);
  std::map<std::string, const ComputeGraph*> graph_of;
  for (const auto& [g, lat] : jobs) graph_of[g.job_id()] = &g;
  for (int32_t i = 0; i < tsl_result_n_jobs(r); ++i) {
    tsl_job_view v;
    tsl_result_job(r, i, &v);
    const ComputeGraph& g = *graph_of.at(v.job_id);
    result.plans[v.job_id] = unpack_plan(v, g);
    result.reports[v.job_id] = unpack_report(v, g);
  }
  const int64_t* hist = nullptr;
  const int32_t nh = tsl_result_history(r, &hist);
  result.merged_peak_history.assign(hist, hist + nh);
  result.final_merged_peak = tsl_result_final_merged_peak(r);
  result.within_budget = tsl_result_within_budget(r) != 0;
  result.diagnostic = tsl_result_diagnostic(r);
  tsl_result_destroy(r);
  return result;
}

// Latency table from the cold-start predictor at a fixed usage level
// (orchestrator.hpp:32-34): one input-dimension slot per input (its bytes).
std::map<OpId, Tick> predict_latencies(const ComputeGraph& graph, const LatencyPredictor& predictor,
                                       double gpu_usage) {
  const auto layouts = derive_layouts(graph);
  std::map<OpId, Tick> out;
  for (const auto& op : graph.ops()) {
    std::map<TensorId, std::vector<double>> dims;
    for (const auto& t : op.inputs) dims[t] = {static_cast<double>(graph.tensor(t).size)};
    const FeatureVector f = extract_features(op, dims, gpu_usage, layouts.at(op.kind));
    out[op.id] = static_cast<Tick>(std::llround(predictor.predict(f)));
  }
  return out;
}

// ---- replan lifecycle (orchestrator.hpp:39-67) -----------------------------
Orchestrator::Orchestrator(PlannerConfig config, std::vector<ComputeGraph> graphs)
    : config_(std::move(config)), graphs_(std::move(graphs)) {
  config_.validate();
  for (const auto& g : graphs_) versions_[g.job_id()] = 0;
}

BuildResult Orchestrator::rebuild() {
  std::vector<std::pair<ComputeGraph, std::map<OpId, Tick>>> jobs;
  Tick total = 0;
  for (const auto& g : graphs_) {
    const auto& lat = latencies_.at(g.job_id());
    for (const auto& kv : lat) total += kv.second;
    jobs.emplace_back(g, lat);
  }
  BuildResult result = build_plan(jobs, config_);
  last_plan_sum_ = total;
  for (auto& kv : result.plans) kv.second.version = ++versions_[kv.first];  // strictly monotone
  return result;
}

BuildResult Orchestrator::plan_with_latencies(const std::map<JobId, std::map<OpId, Tick>>& latencies) {
  latencies_ = latencies;
  return rebuild();
}

BuildResult Orchestrator::plan_cold_start(const LatencyPredictor& predictor) {
  latencies_.clear();
  for (const auto& g : graphs_)
    latencies_[g.job_id()] = predict_latencies(g, predictor, config_.cold_start_gpu_usage);
  return rebuild();
}

std::optional<std::map<JobId, SchedulingPlan>> Orchestrator::replan_if_needed(
    const std::map<JobId, std::map<OpId, Tick>>& observed) {
  // Drift is judged on the summed execution time: observed ops plus the
  // current estimate of every op the round did not report.
  Tick current = 0;
  for (const auto& [job, ops] : latencies_) {
    auto seen = observed.find(job);
    for (const auto& [op, est] : ops) {
      if (seen != observed.end()) {
        auto o = seen->second.find(op);
        if (o != seen->second.end()) continue;
      }
      current += est;
    }
  }
  for (const auto& [job, ops] : observed)
    for (const auto& kv : ops) current += kv.second;
  ReplanState state;
  state.last_sum = last_plan_sum_;
  state.current_sum = current;
  state.threshold = config_.replan_threshold;
  // The EWMA correction applies whether or not the trigger fires.
  for (const auto& [job, ops] : observed) {
    auto est = latencies_.find(job);
    if (est == latencies_.end()) continue;
    for (const auto& [op, t] : ops) {
      auto e = est->second.find(op);
      if (e != est->second.end()) e->second = ewma_update(e->second, t, config_.ewma_alpha);
    }
  }
  if (!should_replan(state)) return std::nullopt;
  ++replan_count_;
  return rebuild().plans;
}

}  // namespace memsched
