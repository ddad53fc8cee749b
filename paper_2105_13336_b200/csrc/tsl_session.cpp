// Planning session: the reference's Orchestrator (orchestrator.cpp:89-159)
// over the C-ABI -- the replan lifecycle around the device planner. A session
// holds the active job set (jobs arrive and depart), each job's latency
// estimates and plan version; every rebuild is one tsl_build_plan over the
// active set (one device launch), versions bump per job, and
// replan_if_needed applies the EWMA correction to observed op latencies and
// rebuilds only when the summed latency drifted past replan_threshold
// (latency.cpp:151-174). Every rebuild's latency is recorded.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tensile_b200.h"
#include "tsl_graph.h"

using namespace tsl::hostg;

namespace {

// A caller's job descriptor copied into owned storage (the C-ABI contract:
// inputs are caller-owned and copied at call time).
struct OwnedJob {
  std::string job_id;
  std::vector<std::string> tid, oid, okind;
  std::vector<const char*> tid_p, oid_p, okind_p;
  std::vector<int64_t> size;
  std::vector<int8_t> kind, phase;
  std::vector<int32_t> in_off, in, out_off, out;
  std::vector<int64_t> lat;  // current estimates (Orchestrator::latencies_), TSL_LATENCY_MISSING if none
  bool has_lat = false;
  tsl_job_desc desc{};

  explicit OwnedJob(const tsl_job_desc& d) {
    job_id = d.job_id ? d.job_id : "";
    const int32_t T = d.n_tensors, O = d.n_ops;
    if (T < 0 || O < 0) fail(TSL_ERR_ARGUMENT, "negative tensor/op count in job " + job_id);
    for (int32_t t = 0; t < T; ++t) tid.emplace_back(d.tensor_ids && d.tensor_ids[t] ? d.tensor_ids[t] : "");
    for (int32_t o = 0; o < O; ++o) {
      oid.emplace_back(d.op_ids && d.op_ids[o] ? d.op_ids[o] : "");
      okind.emplace_back(d.op_kinds && d.op_kinds[o] ? d.op_kinds[o] : "");
    }
    if (T > 0) {
      size.assign(d.tensor_sizes, d.tensor_sizes + T);
      kind.assign(d.tensor_kinds, d.tensor_kinds + T);
    }
    if (O > 0) {
      phase.assign(d.op_phases, d.op_phases + O);
      in_off.assign(d.op_in_offsets, d.op_in_offsets + O + 1);
      out_off.assign(d.op_out_offsets, d.op_out_offsets + O + 1);
      in.assign(d.op_inputs, d.op_inputs + in_off[O]);
      out.assign(d.op_outputs, d.op_outputs + out_off[O]);
    } else {
      in_off.assign(1, 0);
      out_off.assign(1, 0);
    }
    lat.assign(O, TSL_LATENCY_MISSING);
    if (d.op_latencies) {
      lat.assign(d.op_latencies, d.op_latencies + O);
      has_lat = true;
    }
    for (auto& s : tid) tid_p.push_back(s.c_str());
    for (auto& s : oid) oid_p.push_back(s.c_str());
    for (auto& s : okind) okind_p.push_back(s.c_str());
    desc.job_id = job_id.c_str();
    desc.n_tensors = T;
    desc.tensor_ids = tid_p.data();
    desc.tensor_sizes = size.data();
    desc.tensor_kinds = kind.data();
    desc.n_ops = O;
    desc.op_ids = oid_p.data();
    desc.op_kinds = okind_p.data();
    desc.op_phases = phase.data();
    desc.op_in_offsets = in_off.data();
    desc.op_inputs = in.data();
    desc.op_out_offsets = out_off.data();
    desc.op_outputs = out.data();
    desc.op_latencies = lat.data();
  }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return TSL_OK;
  } catch (const Fail& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TSL_ERR_INTERNAL;
  }
}

// ewma_update (latency.cpp:137-149), the Tick overload.
int64_t ewma(int64_t estimate, int64_t observation, double alpha) {
  if (alpha < 0.0 || alpha > 1.0) fail(TSL_ERR_VALIDATION, "ewma alpha out of [0,1]");
  if (estimate < 0 || observation < 0) fail(TSL_ERR_VALIDATION, "ewma inputs must be nonnegative");
  return int64_t(std::llround(alpha * double(observation) + (1.0 - alpha) * double(estimate)));
}

// should_replan (latency.cpp:162-174).
bool should_replan(int64_t last_sum, int64_t current_sum, double threshold) {
  if (threshold <= 0.0) fail(TSL_ERR_VALIDATION, "replan threshold must be positive");
  if (last_sum < 0 || current_sum < 0) fail(TSL_ERR_VALIDATION, "replan sums must be nonnegative");
  if (last_sum == 0) return current_sum > 0;
  return std::abs(double(current_sum - last_sum)) / double(last_sum) > threshold;
}

}  // namespace

struct tsl_session {
  tsl_ctx* ctx = nullptr;
  tsl_config cfg{};
  std::vector<std::string> ratio_jobs;
  std::vector<const char*> ratio_ptrs;
  std::vector<double> ratio_vals;
  std::vector<std::unique_ptr<OwnedJob>> jobs;  // Orchestrator::graphs_ order (arrival order)
  std::map<std::string, int64_t> versions;      // survive a job's departure, like the reference's map
  int64_t last_plan_sum = 0;
  int32_t replan_count = 0;
  std::vector<double> rebuild_ms;               // wall time of every rebuild (validation..results)

  OwnedJob* find(const std::string& id) {
    for (auto& j : jobs)
      if (j->job_id == id) return j.get();
    return nullptr;
  }

  // Orchestrator::rebuild (orchestrator.cpp:96-110).
  tsl_result* rebuild() {
    int64_t sum = 0;
    std::vector<tsl_job_desc> descs;
    for (auto& j : jobs) {
      if (!j->has_lat) fail(TSL_ERR_VALIDATION, "map::at");  // latencies_.at(job)
      for (int64_t t : j->lat) sum += t;
      descs.push_back(j->desc);
    }
    const auto t0 = std::chrono::steady_clock::now();
    tsl_result* res = nullptr;
    const int rc = tsl_build_plan(ctx, descs.data(), int32_t(descs.size()), &cfg, &res);
    if (rc) fail(rc, tsl_last_error());
    rebuild_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    last_plan_sum = sum;
    for (auto& j : jobs) tsl_result_set_version(res, j->job_id.c_str(), ++versions[j->job_id]);
    return res;
  }
};

extern "C" {

int tsl_session_create(tsl_ctx* ctx, const tsl_config* cfg, tsl_session** out) {
  if (!ctx || !cfg || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto s = std::make_unique<tsl_session>();
    s->ctx = ctx;
    s->cfg = *cfg;
    for (int32_t i = 0; i < cfg->n_max_swap_ratios; ++i) {
      s->ratio_jobs.emplace_back(cfg->max_swap_ratio_jobs[i] ? cfg->max_swap_ratio_jobs[i] : "");
      s->ratio_vals.push_back(cfg->max_swap_ratio_values[i]);
    }
    for (auto& r : s->ratio_jobs) s->ratio_ptrs.push_back(r.c_str());
    s->cfg.max_swap_ratio_jobs = s->ratio_ptrs.data();
    s->cfg.max_swap_ratio_values = s->ratio_vals.data();
    // the reference's constructor validates the config (orchestrator.cpp:89-94)
    const int rc = tsl_validate_config(&s->cfg);
    if (rc) fail(rc, tsl_last_error());
    *out = s.release();
  });
}

void tsl_session_destroy(tsl_session* s) { delete s; }

int tsl_session_add_job(tsl_session* s, const tsl_job_desc* job) {
  if (!s || !job) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto j = std::make_unique<OwnedJob>(*job);
    if (s->find(j->job_id)) fail(TSL_ERR_ARGUMENT, "duplicate job id " + j->job_id + " in session");
    s->versions.emplace(j->job_id, 0);
    s->jobs.push_back(std::move(j));
  });
}

int tsl_session_remove_job(tsl_session* s, const char* job_id) {
  if (!s || !job_id) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto it = std::find_if(s->jobs.begin(), s->jobs.end(), [&](const auto& j) { return j->job_id == job_id; });
    if (it == s->jobs.end()) fail(TSL_ERR_ARGUMENT, std::string("no job ") + job_id + " in session");
    s->jobs.erase(it);
  });
}

int tsl_session_set_latencies(tsl_session* s, const char* job_id, const int64_t* latencies) {
  if (!s || !job_id || !latencies) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    OwnedJob* j = s->find(job_id);
    if (!j) fail(TSL_ERR_ARGUMENT, std::string("no job ") + job_id + " in session");
    j->lat.assign(latencies, latencies + j->desc.n_ops);
    j->desc.op_latencies = j->lat.data();
    j->has_lat = true;
  });
}

int tsl_session_rebuild(tsl_session* s, tsl_result** out) {
  if (!s || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] { *out = s->rebuild(); });
}

// Orchestrator::replan_if_needed (orchestrator.cpp:126-159): observed[k] are
// job_ids[k]'s op ticks (op order, < 0 = not observed).
int tsl_session_replan_if_needed(tsl_session* s, int32_t n, const char* const* job_ids,
                                 const int64_t* const* observed, tsl_result** out) {
  if (!s || !out || (n > 0 && (!job_ids || !observed))) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    *out = nullptr;
    // the observation per (job, op); a job reported twice keeps the last report
    std::map<std::string, const int64_t*> obs;
    for (int32_t k = 0; k < n; ++k) obs[job_ids[k] ? job_ids[k] : ""] = observed[k];
    int64_t observed_sum = 0;
    for (const auto& [id, ticks] : obs) {
      OwnedJob* j = s->find(id);
      const int32_t O = j ? j->desc.n_ops : 0;
      if (!j) continue;  // (ops of unknown jobs carry no op ids we could match)
      for (int32_t o = 0; o < O; ++o)
        if (ticks[o] >= 0) observed_sum += ticks[o];
    }
    // ops not covered by this round keep their current estimate in the sum
    for (auto& j : s->jobs) {
      auto it = obs.find(j->job_id);
      for (int32_t o = 0; o < j->desc.n_ops; ++o)
        if (it == obs.end() || it->second[o] < 0) observed_sum += j->lat[o];
    }
    // the EWMA correction happens regardless of the trigger (before it is tested)
    for (const auto& [id, ticks] : obs) {
      OwnedJob* j = s->find(id);
      if (!j) continue;
      for (int32_t o = 0; o < j->desc.n_ops; ++o)
        if (ticks[o] >= 0) j->lat[o] = ewma(j->lat[o], ticks[o], s->cfg.ewma_alpha);
    }
    if (!should_replan(s->last_plan_sum, observed_sum, s->cfg.replan_threshold)) return;
    ++s->replan_count;
    *out = s->rebuild();
  });
}

int32_t tsl_session_replan_count(const tsl_session* s) { return s ? s->replan_count : 0; }

int32_t tsl_session_rebuild_times(const tsl_session* s, const double** ms) {
  if (!s) return 0;
  if (ms) *ms = s->rebuild_ms.data();
  return int32_t(s->rebuild_ms.size());
}

int32_t tsl_session_n_jobs(const tsl_session* s) { return s ? int32_t(s->jobs.size()) : 0; }

int tsl_session_latencies(const tsl_session* s, const char* job_id, int64_t* out) {
  if (!s || !job_id || !out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    const OwnedJob* j = const_cast<tsl_session*>(s)->find(job_id);
    if (!j) fail(TSL_ERR_ARGUMENT, std::string("no job ") + job_id + " in session");
    std::copy(j->lat.begin(), j->lat.end(), out);
  });
}

}  // extern "C"
