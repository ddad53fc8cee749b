// Host side of the C-ABI (include/tensile_b200.h): graph validation and
// topological order (graph.cpp:49-119, 245-282), integer/rank packing, one
// H2D copy, one kernel launch for all groups, one D2H copy, and the
// reference's output formats (save_plans, PeakReport::to_json).
//
// Everything on the planning path runs in tsl_plan_kernel (tsl_kernel.cu);
// this file never computes a plan. Without a CUDA device every entry point
// fails with TSL_ERR_CUDA -- there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <queue>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "tensile_b200.h"
#include "tsl_exec.h"
#include "tsl_kernel.h"
#include "tsl_graph.h"

using namespace tsl;
using namespace tsl::hostg;

namespace {

thread_local std::string g_err;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TSL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// PlannerConfig::max_swap_ratios as the std::map<JobId,double> it restates
// (a repeated id keeps its last value, like repeated map assignment).
std::map<std::string, double> ratio_map(const tsl_config& c) {
  std::map<std::string, double> m;
  if (c.n_max_swap_ratios < 0) fail(TSL_ERR_ARGUMENT, "negative n_max_swap_ratios");
  if (c.n_max_swap_ratios > 0 && (!c.max_swap_ratio_jobs || !c.max_swap_ratio_values))
    fail(TSL_ERR_ARGUMENT, "null max_swap_ratios arrays");
  for (int32_t i = 0; i < c.n_max_swap_ratios; ++i)
    m[c.max_swap_ratio_jobs[i] ? c.max_swap_ratio_jobs[i] : ""] = c.max_swap_ratio_values[i];
  return m;
}

// PlannerConfig::max_swap_ratio, config.hpp:20-23.
double ratio_of(const std::map<std::string, double>& m, const std::string& job) {
  auto it = m.find(job);
  return it == m.end() ? 1.0 : it->second;
}

// PlannerConfig::validate, config.hpp:25-35 (every map entry, in key order;
// the same predicate, so a NaN ratio passes as it does there).
void validate_config(const tsl_config& c) {
  if (c.pcie_bandwidth <= 0) fail(TSL_ERR_VALIDATION, "pcie_bandwidth must be positive");
  if (c.transfer_setup < 0) fail(TSL_ERR_VALIDATION, "transfer_setup must be nonnegative");
  if (c.memory_budget < 0) fail(TSL_ERR_VALIDATION, "memory_budget must be nonnegative");
  if (c.ewma_alpha < 0 || c.ewma_alpha > 1) fail(TSL_ERR_VALIDATION, "ewma_alpha out of [0,1]");
  if (c.replan_threshold <= 0) fail(TSL_ERR_VALIDATION, "replan_threshold must be positive");
  if (c.stall_epsilon <= 0 || c.stall_epsilon >= 1) fail(TSL_ERR_VALIDATION, "stall_epsilon out of (0,1)");
  for (auto& [job, r] : ratio_map(c))
    if (r <= 0 || r > 1) fail(TSL_ERR_VALIDATION, "max swap ratio for " + job + " out of (0,1]");
}

// ---------------------------------------------------------------------------
// Device buffer layout
// ---------------------------------------------------------------------------
struct Layout {
  size_t off = 0;
  template <class T>
  size_t take(size_t n) {
    off = (off + 15) & ~size_t(15);
    size_t o = off;
    off += n * sizeof(T);
    return o;
  }
};

struct JobPlace {  // byte offsets into the device buffer
  size_t topo, o_lat, o_in_off, o_in, o_out_off, o_out, t_size, t_kind, t_rank, t_store, t_upd, t_prod, inflag;
  size_t a_tensor, a_store, a_type, a_start, a_end, a_base, a_flag, a_owned, s_off, s_acc, t_wfirst, t_utga;
  size_t ev[12], bz_s, bz_e, pd_s, pd_e, pd_ts, pd_te, bzi_s, bzi_e, ai_e, st_evcnt, swapped, rc[6], in_peak, ev_drop, res_init, curve_t, curve_b;
  size_t bk_a_start, bk_a_end, bk_flag, bk_in_peak, bk_ev, bk_rc, bk_bz, bk_evcnt, bk_curve, pk_list;
  int32_t Scap, Rcap, Ecap, ti_nb;
};

struct GroupPlace {
  size_t hist, c_info, c_hull, dev_list, c_comp, pr_pool, w_pool, wbuf, cb_idx, cb_ent, bs_key = 0, bs_val = 0;
  int64_t c_cap = 0;
  size_t coop = 0, tile_hist = 0, coop_gsh = 0, cta_part = 0, c_wscratch = 0;
  int64_t c_wscap = 0;
  int64_t pr_cap, w_cap, wcap, cb_cap;
  int32_t cb_nb = 1024;
  size_t k_key, k_val, x_time, x_fp, x_store, x_aid, x_type, x_job, x_state, x_seq2, x_key2, x_order;
  int32_t hist_cap;
  // incremental timeline order (one-job big builds)
  bool ec = false;
  int64_t ec_dcap = 0;
  size_t ec_act, ec_ract, ec_rpos, ec_gbt, ec_gbst, ec_gty, ec_gst, ec_bt, ec_bl, ec_bs, ec_gt, ec_gl, ec_gb, ec_ginv, ec_posb, ec_sc, ec_dord, ec_dins, ec_dgrp, ec_gins, ec_nw, ec_posd, ec_dl;
};

}  // namespace

// ---------------------------------------------------------------------------
// Results
// ---------------------------------------------------------------------------
struct JobOut {
  const Graph* g = nullptr;
  int32_t version = 0;
  JobState st{};
  std::vector<int64_t> ev_id, ev_trig, ev_delta, ev_start, ev_end, ev_earl, ev_late, ev_pair, ev_serves;
  std::vector<int32_t> ev_tensor;
  std::vector<int8_t> ev_dir, ev_wraps;
  std::vector<int64_t> rc_id, rc_target, rc_lat, rc_saving;
  std::vector<int32_t> rc_tensor, rc_regen;
  std::vector<int64_t> flags;
  std::vector<int32_t> peak_tensors;
  std::vector<int64_t> curve_t, curve_b;
};

using GraphP = std::shared_ptr<const Graph>;

struct tsl_result {
  std::vector<GraphP> graphs;  // shared with the plan (and across groups)
  std::vector<JobOut> jobs;  // job-id order
  std::vector<int64_t> history;
  int64_t final_merged = 0;
  bool within = true;
  std::string diagnostic;
  tsl_stats stats{};
};

// Device buffer + pinned staging buffer. One-shot calls reuse the context's;
// a prepared plan owns its own so its resident inputs survive other calls.
struct Buffers {
  void* dbuf = nullptr;
  size_t dcap = 0;
  uint8_t* hbuf = nullptr;
  size_t hcap = 0;
  void release() {
    if (dbuf) cudaFree(dbuf);
    if (hbuf) cudaFreeHost(hbuf);
    dbuf = nullptr;
    hbuf = nullptr;
    dcap = hcap = 0;
  }
};

struct tsl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  Buffers buf;
};

struct tsl_plan {
  tsl_ctx* ctx = nullptr;
  Buffers* buf = nullptr;  // ctx->buf, or own_buf for a prepared plan
  Buffers own_buf;
  ~tsl_plan() {
    if (done) cudaEventDestroy(done);
    own_buf.release();
  }
  int mode = 0;  // 0 build_plan, 1 analyze_job
  int32_t n_groups = 0;
  std::vector<std::vector<GraphP>> graphs;  // per group, caller order (a descriptor seen twice is loaded once)
  std::vector<std::vector<JobPlace>> jp;
  std::vector<GroupPlace> gp;
  std::vector<tsl_config> cfgs;
  size_t h2d_bytes = 0;          // [0, h2d_bytes) uploaded
  size_t d2h_off = 0, d2h_bytes = 0;
  size_t stage_end = 0;     // end of the group / state / job headers
  size_t d2h_done = 0;      // bytes the last download moved
  size_t groups_off = 0, jobs_off = 0, states_off = 0;
  std::vector<int32_t> group_job_base;  // first JobDev index of each group
  double last_kernel_ms = 0;
  double prep_ms = 0;
  int32_t max_jobs = 1;
  int32_t ipt = 1;        // block-sort tile of this launch
  int64_t sort_cap = 0;   // NT * ipt
  int64_t ecap = 0;       // timeline scratch capacity (== sort_cap unless big)
  bool big = false;       // a job exceeds one sort tile
  bool coop = false;      // big and one group: cooperative launch, one CTA per SM
  size_t res_bytes = 0;   // shared memory for resident job arrays (build mode)
  tsl::CoopCtl coop_init{};  // initial cooperative control block (uploaded before each launch)
  cudaEvent_t done = nullptr;  // recorded after the last asynchronous launch (tsl_plan_launch_async)
  int64_t n_accesses = 0;
};

namespace {

// The device buffer holds inputs, outputs and the workspace; the pinned host
// staging buffer only the inputs and outputs (host_need <= need).
void grow(Buffers* c, size_t need, size_t host_need) {
  if (need > c->dcap) {
    if (c->dbuf) cudaFree(c->dbuf);
    c->dbuf = nullptr;
    size_t cap = std::max(need, c->dcap * 2);
    cuda_check(cudaMalloc(&c->dbuf, cap), "cudaMalloc");
    c->dcap = cap;
  }
  if (host_need > c->hcap) {
    if (c->hbuf) cudaFreeHost(c->hbuf);
    c->hbuf = nullptr;
    size_t cap = std::max(host_need, c->hcap * 2);
    cuda_check(cudaMallocHost(reinterpret_cast<void**>(&c->hbuf), cap), "cudaMallocHost");
    c->hcap = cap;
  }
}

template <class T>
T* hp(Buffers* c, size_t off) { return reinterpret_cast<T*>(c->hbuf + off); }
template <class T>
T* dp(Buffers* c, size_t off) { return reinterpret_cast<T*>(static_cast<uint8_t*>(c->dbuf) + off); }

template <class T>
void put(Buffers* c, size_t off, const std::vector<T>& v) {
  if (!v.empty()) std::memcpy(c->hbuf + off, v.data(), v.size() * sizeof(T));
}

// A caller plan for analyze mode (tsl_plan_desc), kept with its job.
struct CallerPlan {
  const tsl_plan_desc* p = nullptr;
};

tsl_plan* prepare(tsl_ctx* cx, const tsl_job_desc* jobs, const int32_t* offs, int32_t n_groups,
                  const tsl_config* cfgs, int32_t n_cfgs, int mode, const tsl_plan_desc* caller, bool own) {
  if (n_cfgs != 1 && n_cfgs != n_groups) fail(TSL_ERR_ARGUMENT, "n_cfgs must be 1 or n_groups");
  auto t0 = std::chrono::steady_clock::now();
  auto* P = new tsl_plan();
  P->ctx = cx;
  P->buf = own ? &P->own_buf : &cx->buf;
  Buffers* ctx = P->buf;
  P->mode = mode;
  P->n_groups = n_groups;
  P->cfgs.assign(cfgs, cfgs + n_cfgs);
  for (auto& c : P->cfgs) {  // the ratio map is read during prepare only
    c.n_max_swap_ratios = 0;
    c.max_swap_ratio_jobs = nullptr;
    c.max_swap_ratio_values = nullptr;
  }
  P->graphs.resize(n_groups);
  // 1. validate graphs (caller order), then the config, then latencies
  {
    // identical descriptors (same arrays) within one call are one graph: the
    // C5 replans of a shard repeat each resident workload in every request
    std::map<std::vector<uintptr_t>, GraphP> seen;
    for (int gi = 0; gi < n_groups; ++gi) {
      for (int32_t k = offs[gi]; k < offs[gi + 1]; ++k) {
        const tsl_job_desc& d = jobs[k];
        std::vector<uintptr_t> key = {
            uintptr_t(d.job_id), uintptr_t(d.n_tensors), uintptr_t(d.tensor_ids), uintptr_t(d.tensor_sizes),
            uintptr_t(d.tensor_kinds), uintptr_t(d.n_ops), uintptr_t(d.op_ids), uintptr_t(d.op_kinds),
            uintptr_t(d.op_phases), uintptr_t(d.op_in_offsets), uintptr_t(d.op_inputs), uintptr_t(d.op_out_offsets),
            uintptr_t(d.op_outputs), uintptr_t(d.op_latencies)};
        auto it = seen.find(key);
        if (it == seen.end()) it = seen.emplace(std::move(key), std::make_shared<const Graph>(load_graph(d))).first;
        P->graphs[gi].push_back(it->second);
      }
    }
  }
  const auto t_load = std::chrono::steady_clock::now();
  for (int gi = 0; gi < n_groups; ++gi) {
    if (mode == 0) validate_config(cfgs[n_cfgs == 1 ? 0 : gi]);
    std::set<std::string> ids;
    for (auto& gp : P->graphs[gi]) {
      const Graph& g = *gp;
      if (!ids.insert(g.job_id).second)
        fail(TSL_ERR_ARGUMENT, "duplicate job id " + g.job_id + " in one build (unsupported)");
      check_latencies(g);
      if (g.T >= (1 << 24)) fail(TSL_ERR_CAPACITY, "job " + g.job_id + " has too many tensors");
    }
    if (P->graphs[gi].size() > 128) fail(TSL_ERR_CAPACITY, "more than 128 jobs in one group");
  }
  // Sort tile: the largest block sort of any group -- CSR of a job's
  // accesses, one job's whole timeline (<= 2A + S + R with S <= 2A + 2 and
  // R <= T + 1), a pass's candidates (<= sum T). Busy rebuilds and
  // evaluation batches are split to fit it.
  {
    int64_t need = 1;
    for (auto& gs : P->graphs) {
      int64_t sumT = 0;
      for (auto& gp : gs) {
        const Graph& g = *gp;
        need = std::max<int64_t>(need, 4 * int64_t(g.A) + g.T + 4);
        need = std::max<int64_t>(need, g.O + 1);
        sumT += g.T;
      }
      need = std::max<int64_t>(need, sumT);
    }
    P->ipt = sort_ipt_for(need);
    P->sort_cap = int64_t(NT) * P->ipt;
    P->ecap = P->sort_cap;
    if (need > P->sort_cap) {
      // above one sort tile: block-wide radix sorts through global ping-pong
      // buffers (DevX::sort_big), timeline scratch sized for the largest job
      if (need > (int64_t(1) << 30))
        fail(TSL_ERR_CAPACITY, "build exceeds the planner capacity (2^30 timeline events per job)");
      P->big = true;
      P->ecap = (need + 15) & ~int64_t(15);
      const char* ce = std::getenv("TSL_COOP");
      P->coop = n_groups == 1 && !(ce && ce[0] == '0');
      // a grid-wide evaluation scans one release count per global thread
      // (<= 256 SMs x NT) inside the timeline scratch
      if (P->coop) P->ecap = std::max<int64_t>(P->ecap, int64_t(256) * NT);
    }
  }
  const auto t_val = std::chrono::steady_clock::now();
  // 2. layout: [static inputs][groups|states|jobs][outputs][workspace]
  Layout L;
  P->jp.resize(n_groups);
  P->gp.resize(n_groups);
  for (int gi = 0; gi < n_groups; ++gi) {
    for (auto& gp : P->graphs[gi]) {
      const Graph& g = *gp;
      JobPlace p{};
      p.topo = L.take<int32_t>(g.O);
      p.o_lat = L.take<int64_t>(g.O);
      p.o_in_off = L.take<int32_t>(g.O + 1);
      p.o_in = L.take<int32_t>(g.in.size());
      p.o_out_off = L.take<int32_t>(g.O + 1);
      p.o_out = L.take<int32_t>(g.out.size());
      p.t_size = L.take<int64_t>(g.T);
      p.t_kind = L.take<int8_t>(g.T);
      p.t_rank = L.take<int32_t>(g.T);
      p.t_store = L.take<int32_t>(g.T);
      p.t_upd = L.take<int32_t>(g.T);
      p.t_prod = L.take<int32_t>(g.T);
      p.inflag = mode == 1 ? L.take<uint8_t>(g.A) : 0;
      p.Scap = 2 * g.A + 2;
      p.Rcap = g.T + 1;
      p.Ecap = 2 * g.A + p.Scap + p.Rcap;
      // time-index buckets (per job; a finer index for the big jobs measured
      // only 7 % faster re-score queries on C4 -- the bisection steps after
      // the coarse index mostly hit L1 -- and made index rebuilds costlier)
      p.ti_nb = tsl::TI_NB_HOST;
      if (P->big)
        if (const char* e = std::getenv("TSL_TI_NB")) p.ti_nb = std::max(16, std::min(1 << 20, std::atoi(e)));
      P->n_accesses += g.A;
      P->jp[gi].push_back(p);
    }
  }
  P->groups_off = L.take<GroupDev>(n_groups);
  int32_t nj = 0;
  for (auto& v : P->graphs) {
    P->group_job_base.push_back(nj);
    nj += static_cast<int32_t>(v.size());
    P->max_jobs = std::max<int32_t>(P->max_jobs, static_cast<int32_t>(v.size()));
  }
  // shared-memory residency of the job arrays: the largest group's arrays
  // when they fit (RES_FULL_MAX keeps most of the SM's L1)
  if (mode == 0 && P->max_jobs <= RES_MAX_JOBS && !P->big) {
    size_t need = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
      size_t sum = 0;
      for (size_t k = 0; k < P->graphs[gi].size(); ++k)
        sum += resident_bytes_for(P->graphs[gi][k]->A, P->graphs[gi][k]->T, P->jp[gi][k].Scap);
      need = std::max(need, sum);
    }
    const size_t with = kernel_smem_bytes(P->max_jobs, P->ipt, 16) - 16;
    const size_t limit = size_t(227) * 1024;
    // all or nothing: a partly resident group gains little and loses L1
    size_t res = (with < limit && need <= limit - with && need <= RES_FULL_MAX) ? need : 0;
    if (const char* e = std::getenv("TSL_RES_BYTES")) res = std::min<size_t>(res, std::strtoull(e, nullptr, 10));
    P->res_bytes = res & ~size_t(15);
  }
  P->states_off = L.take<JobState>(nj);
  P->jobs_off = L.take<JobDev>(nj);
  const size_t stage_end = L.off;
  // outputs (read back)
  for (int gi = 0; gi < n_groups; ++gi) {
    int64_t sumT = 0;
    for (auto& g : P->graphs[gi]) sumT += g->T;
    P->gp[gi].hist_cap = static_cast<int32_t>(2 * sumT + 16);
    P->gp[gi].hist = L.take<int64_t>(P->gp[gi].hist_cap);
    for (size_t k = 0; k < P->graphs[gi].size(); ++k) {
      const Graph& g = *P->graphs[gi][k];
      JobPlace& p = P->jp[gi][k];
      for (int f = 0; f < 12; ++f) {
        size_t w = (f == 1) ? 4 : (f == 2 || f == 3) ? 1 : 8;  // tensor int32, dir/wraps int8
        p.ev[f] = L.take<uint8_t>(w * p.Scap);
      }
      for (int f = 0; f < 6; ++f) {
        size_t w = (f == 1 || f == 3) ? 4 : 8;
        p.rc[f] = L.take<uint8_t>(w * p.Rcap);
      }
      p.a_flag = L.take<uint8_t>(g.A);
      p.in_peak = L.take<uint8_t>(g.T);
      p.curve_t = L.take<int64_t>(p.Ecap + 1);
      p.curve_b = L.take<int64_t>(p.Ecap + 1);
    }
  }
  const size_t out_end = L.off;
  // workspace
  for (int gi = 0; gi < n_groups; ++gi) {
    for (size_t k = 0; k < P->graphs[gi].size(); ++k) {
      const Graph& g = *P->graphs[gi][k];
      JobPlace& p = P->jp[gi][k];
      p.a_tensor = L.take<int32_t>(g.A);
      p.a_store = L.take<int32_t>(g.A);
      p.a_type = L.take<int8_t>(g.A);
      p.a_start = L.take<int64_t>(g.A);
      p.a_end = L.take<int64_t>(g.A);
      p.a_base = L.take<uint8_t>(g.A);
      p.a_owned = L.take<uint8_t>(g.A);
      p.s_off = L.take<int32_t>(g.T + 1);
      p.s_acc = L.take<int32_t>(g.A);
      p.t_wfirst = L.take<int32_t>(g.T);
      p.t_utga = L.take<int32_t>(g.T);
      p.bz_s = L.take<int64_t>(p.Scap);
      p.bz_e = L.take<int64_t>(p.Scap);
      p.pd_s = L.take<int64_t>(p.Scap);
      p.pd_e = L.take<int64_t>(p.Scap);
      p.pd_ts = L.take<int64_t>(p.Scap);
      p.pd_te = L.take<int64_t>(p.Scap);
      p.bzi_s = L.take<int32_t>(size_t(p.ti_nb) + 1);
      p.bzi_e = L.take<int32_t>(size_t(p.ti_nb) + 1);
      p.ai_e = L.take<int32_t>(size_t(p.ti_nb) + 1);
      p.st_evcnt = L.take<int32_t>(g.T);
      p.swapped = L.take<uint8_t>(g.T);
      p.ev_drop = L.take<uint8_t>(p.Scap);
      p.res_init = L.take<uint8_t>(g.T);
      p.bk_a_start = L.take<int64_t>(g.A);
      p.bk_a_end = L.take<int64_t>(g.A);
      p.bk_flag = L.take<uint8_t>(g.A);
      p.bk_in_peak = L.take<uint8_t>(g.T);
      p.pk_list = L.take<int32_t>(g.T);
      p.bk_ev = L.take<int64_t>(size_t(12) * p.Scap);
      p.bk_rc = L.take<int64_t>(size_t(6) * p.Rcap);
      p.bk_bz = L.take<int64_t>(size_t(2) * p.Scap);
      p.bk_evcnt = L.take<int32_t>(g.T);
      p.bk_curve = L.take<int64_t>(size_t(2) * (p.Ecap + 1));
    }
    GroupPlace& q = P->gp[gi];
    const size_t E = size_t(P->ecap);
    int64_t sumA = 0, sumT = 0;
    for (auto& g : P->graphs[gi]) { sumA += g->A; sumT += g->T; }
    const size_t CC = size_t(std::min<int64_t>(P->ecap, sumT + 16));  // candidates of a pass <= sum T
    if (P->big) {
      q.bs_key = L.take<uint64_t>(E);
      q.bs_val = L.take<int32_t>(E);
    }
    if (P->coop) {
      q.coop = L.take<uint8_t>(sizeof(tsl::CoopCtl));
      q.tile_hist = L.take<int32_t>(size_t((P->ecap + NT * SORT_IPT - 1) / (NT * SORT_IPT)) * 256);
      q.coop_gsh = L.take<int64_t>(1024);  // SH_WORDS (tsl_plan.cuh)
      q.cta_part = L.take<int64_t>(1024);
      // component runs on every warp of the grid: a private interval list of
      // up to 4096 entries per warp (6 words each: list, merge target, scratch)
      int sms = 0;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->ctx->device) != cudaSuccess || sms <= 0)
        sms = 148;
      q.c_wscap = 4096;
      q.c_wscratch = L.take<int64_t>(size_t(sms) * (NT / 32) * 6 * size_t(q.c_wscap));
    }
    q.k_key = L.take<uint64_t>(E);
    q.k_val = L.take<int32_t>(E);
    q.x_time = L.take<int64_t>(2 * E);  // second half: evaluator scan scratch
    q.x_fp = L.take<int64_t>(E);
    q.x_store = L.take<int32_t>(E);
    q.x_aid = L.take<int32_t>(E);
    q.x_type = L.take<int8_t>(E);
    q.x_job = L.take<int8_t>(E);
    q.x_state = L.take<uint8_t>(E);
    q.x_seq2 = L.take<int32_t>(E);
    q.x_key2 = L.take<uint64_t>(E);
    q.x_order = L.take<int32_t>(E);
    q.pr_cap = sumA + sumT + 16;
    q.w_cap = 2 * q.pr_cap + 2 * sumT + 16;
    q.c_info = L.take<int32_t>(CC * 16);
    q.c_hull = L.take<int64_t>(CC * 4);
    q.dev_list = L.take<int64_t>(CC);
    q.c_cap = int64_t(CC);
    q.c_comp = L.take<int32_t>(2 * CC);
    q.pr_pool = L.take<uint8_t>(size_t(q.pr_cap) * tsl::PAIRREC_BYTES);
    q.w_pool = L.take<int64_t>(size_t(2 * q.w_cap));
    int64_t maxS = 0;
    for (auto& p : P->jp[gi]) maxS = std::max<int64_t>(maxS, p.Scap);
    q.wcap = 3 * maxS + 64;
    q.wbuf = L.take<int64_t>(size_t(NT / 32) * 4 * q.wcap);
    q.cb_nb = P->big ? (1 << 16) : 1024;        // buckets of the pair-interval and window indexes
    q.cb_idx = L.take<int32_t>(4 * size_t(q.cb_nb + 2));
    q.cb_cap = std::max<int64_t>(8 * P->sort_cap, 4 * q.pr_cap);
    q.cb_ent = L.take<int32_t>(2 * size_t(q.cb_cap));
    // incremental evaluation (tsl_plan.cuh inc_order): one big job per build
    const char* ie = std::getenv("TSL_EVAL_INC");
    q.ec = mode == 0 && P->big && P->graphs[gi].size() == 1 && !(ie && ie[0] == '0');
    if (q.ec) {
      const size_t NB = 2 * size_t(sumA);
      q.ec_dcap = P->jp[gi][0].Scap + P->jp[gi][0].Rcap;
      const size_t D = size_t(q.ec_dcap);
      q.ec_bt = L.take<int64_t>(NB);
      q.ec_bl = L.take<uint32_t>(NB);
      q.ec_bs = L.take<int32_t>(NB);
      q.ec_gt = L.take<int64_t>(NB);
      q.ec_gl = L.take<uint32_t>(NB);
      q.ec_gb = L.take<int32_t>(NB);
      q.ec_ginv = L.take<int32_t>(NB);
      q.ec_posb = L.take<int32_t>(NB);
      q.ec_sc = L.take<int64_t>(2 * (NB + 1));
      q.ec_dord = L.take<int32_t>(2 * D);
      q.ec_dins = L.take<int32_t>(2 * D);
      q.ec_dgrp = L.take<int32_t>(2 * D);
      q.ec_gins = L.take<int32_t>(2 * D);
      q.ec_nw = L.take<int32_t>(4 * D);
      q.ec_posd = L.take<int32_t>(D);
      q.ec_dl = L.take<uint32_t>(D);
      q.ec_gbt = L.take<int8_t>(NB);
      q.ec_gbst = L.take<int32_t>(NB);
      q.ec_act = L.take<uint8_t>(2 * NB);
      q.ec_ract = L.take<uint8_t>(NB / 2);
      q.ec_rpos = L.take<int32_t>(NB);
      q.ec_gty = L.take<int8_t>(E);
      q.ec_gst = L.take<int32_t>(E);
    }
  }
  const size_t total = L.off;
  const auto t_lay = std::chrono::steady_clock::now();
  grow(ctx, total, out_end);
  const auto t_grow = std::chrono::steady_clock::now();
  // 3. fill the staging buffer
  int32_t jglob = 0;
  for (int gi = 0; gi < n_groups; ++gi) {
    const auto& gs = P->graphs[gi];
    std::vector<std::string> jids;
    for (auto& g : gs) jids.push_back(g->job_id);
    std::vector<int32_t> jrank = lex_rank(jids);
    const tsl_config* cfg = &cfgs[n_cfgs == 1 ? 0 : gi];
    const std::map<std::string, double> ratios = mode == 0 ? ratio_map(*cfg) : std::map<std::string, double>{};
    // jobs interact through SwapBudget::allows (swap_planner.cpp:268-276)
    // unless every ratio is >= 1; a NaN ratio (it passes validate) couples too
    bool coupled = false;
    for (auto& g : gs) coupled = coupled || !(ratio_of(ratios, g->job_id) >= 1.0);
    GroupDev* G = hp<GroupDev>(ctx, P->groups_off) + gi;
    std::memset(G, 0, sizeof *G);
    G->n_jobs = static_cast<int32_t>(gs.size());
    G->coupled = coupled ? 1 : 0;
    G->spec_window = 0;
    if (const char* e = std::getenv("TSL_SPEC_WINDOW")) G->spec_window = std::atoi(e);
    // component speculation (swap_pass phase A2): 1 = on for passes of >= 512
    // candidates (C4's passes re-score ~40 % of their candidates without it)
    G->spec_comp = 1;
    if (const char* e = std::getenv("TSL_SPEC_COMP")) G->spec_comp = std::atoi(e);
    G->grid_conf = 1;
    if (const char* e = std::getenv("TSL_GRID_CONF")) G->grid_conf = std::atoi(e);
    G->hist_cap = P->gp[gi].hist_cap;
    G->cfg.bw = cfg->pcie_bandwidth;
    G->cfg.setup = cfg->transfer_setup;
    G->cfg.budget = cfg->memory_budget;
    G->cfg.stall_eps = cfg->stall_epsilon;
    G->cfg.stall_min_iters = cfg->stall_min_iters;
    G->jobs = dp<JobDev>(ctx, P->jobs_off) + jglob;
    G->st = dp<JobState>(ctx, P->states_off) + jglob;
    const GroupPlace& q = P->gp[gi];
    G->hist = dp<int64_t>(ctx, q.hist);
    G->ecap = int32_t(P->ecap);
    G->coop = P->coop ? reinterpret_cast<tsl::CoopCtl*>(static_cast<uint8_t*>(ctx->dbuf) + q.coop) : nullptr;
    if (P->coop) {  // the device control block starts zeroed; its tile table is set here
      tsl::CoopCtl cc{};
      cc.tile_hist = dp<int32_t>(ctx, q.tile_hist);
      cc.gsh = dp<int64_t>(ctx, q.coop_gsh);
      cc.cta_part = dp<int64_t>(ctx, q.cta_part);
      P->coop_init = cc;
    }
    G->bs_key = P->big ? dp<uint64_t>(ctx, q.bs_key) : nullptr;
    G->bs_val = P->big ? dp<int32_t>(ctx, q.bs_val) : nullptr;
    G->k_key = dp<uint64_t>(ctx, q.k_key);
    G->k_val = dp<int32_t>(ctx, q.k_val);
    G->x_time = dp<int64_t>(ctx, q.x_time);
    G->x_fp = dp<int64_t>(ctx, q.x_fp);
    G->x_store = dp<int32_t>(ctx, q.x_store);
    G->x_aid = dp<int32_t>(ctx, q.x_aid);
    G->x_type = dp<int8_t>(ctx, q.x_type);
    G->x_job = dp<int8_t>(ctx, q.x_job);
    G->x_state = dp<uint8_t>(ctx, q.x_state);
    G->x_seq2 = dp<int32_t>(ctx, q.x_seq2);
    G->x_key2 = dp<uint64_t>(ctx, q.x_key2);
    G->x_order = dp<int32_t>(ctx, q.x_order);
    G->c_info = dp<int32_t>(ctx, q.c_info);
    G->c_hull = dp<int64_t>(ctx, q.c_hull);
    G->dev_list = dp<int64_t>(ctx, q.dev_list);
    G->c_comp = dp<int32_t>(ctx, q.c_comp);
    G->c_cap = q.c_cap;
    G->c_wscratch = P->coop ? dp<int64_t>(ctx, q.c_wscratch) : nullptr;
    G->c_wscap = q.c_wscap;
    G->pr_pool = reinterpret_cast<tsl::PairRec*>(static_cast<uint8_t*>(ctx->dbuf) + q.pr_pool);
    G->w_pool = dp<int64_t>(ctx, q.w_pool);
    G->pr_cap = q.pr_cap;
    G->wbuf = dp<int64_t>(ctx, q.wbuf);
    G->wcap = q.wcap;
    G->cb_idx = dp<int32_t>(ctx, q.cb_idx);
    G->cb_nb = q.cb_nb;
    G->cb_ent = dp<int32_t>(ctx, q.cb_ent);
    G->cb_cap = q.cb_cap;
    G->w_cap = q.w_cap;
    G->ec_S0 = -1;
    if (q.ec) {
      G->ec_dcap = q.ec_dcap;
      G->ec_bt = dp<int64_t>(ctx, q.ec_bt);
      G->ec_bl = dp<uint32_t>(ctx, q.ec_bl);
      G->ec_bs = dp<int32_t>(ctx, q.ec_bs);
      G->ec_gt = dp<int64_t>(ctx, q.ec_gt);
      G->ec_gl = dp<uint32_t>(ctx, q.ec_gl);
      G->ec_gb = dp<int32_t>(ctx, q.ec_gb);
      G->ec_ginv = dp<int32_t>(ctx, q.ec_ginv);
      G->ec_posb = dp<int32_t>(ctx, q.ec_posb);
      G->ec_sc = dp<int64_t>(ctx, q.ec_sc);
      G->ec_dord = dp<int32_t>(ctx, q.ec_dord);
      G->ec_dins = dp<int32_t>(ctx, q.ec_dins);
      G->ec_dgrp = dp<int32_t>(ctx, q.ec_dgrp);
      G->ec_gins = dp<int32_t>(ctx, q.ec_gins);
      G->ec_nw = dp<int32_t>(ctx, q.ec_nw);
      G->ec_posd = dp<int32_t>(ctx, q.ec_posd);
      G->ec_dl = dp<uint32_t>(ctx, q.ec_dl);
      G->ec_gbt = dp<int8_t>(ctx, q.ec_gbt);
      G->ec_gbst = dp<int32_t>(ctx, q.ec_gbst);
      G->ec_act = dp<uint8_t>(ctx, q.ec_act);
      G->ec_ract = dp<uint8_t>(ctx, q.ec_ract);
      G->ec_rpos = dp<int32_t>(ctx, q.ec_rpos);
      G->ec_gty = dp<int8_t>(ctx, q.ec_gty);
      G->ec_gst = dp<int32_t>(ctx, q.ec_gst);
    }
    for (size_t k = 0; k < gs.size(); ++k, ++jglob) {
      const Graph& g = *gs[k];
      const JobPlace& p = P->jp[gi][k];

      std::vector<int32_t> topo = g.topo;
      put(ctx, p.topo, topo);
      put(ctx, p.o_lat, g.lat);
      put(ctx, p.o_in_off, g.in_off);
      put(ctx, p.o_in, g.in);
      put(ctx, p.o_out_off, g.out_off);
      put(ctx, p.o_out, g.out);
      put(ctx, p.t_size, g.size);
      put(ctx, p.t_kind, g.kind);
      put(ctx, p.t_rank, g.trank);
      put(ctx, p.t_store, g.store);
      put(ctx, p.t_upd, g.upd);
      put(ctx, p.t_prod, g.prod);
      JobDev* J = hp<JobDev>(ctx, P->jobs_off) + jglob;
      std::memset(J, 0, sizeof *J);
      J->A = g.A; J->T = g.T; J->O = g.O; J->rank = jrank[k]; J->ratio = ratio_of(ratios, g.job_id);
      J->Scap = p.Scap; J->Rcap = p.Rcap; J->Ecap = p.Ecap; J->ti_nb = p.ti_nb;
      J->topo = dp<int32_t>(ctx, p.topo);
      J->o_lat = dp<int64_t>(ctx, p.o_lat);
      J->o_in_off = dp<int32_t>(ctx, p.o_in_off);
      J->o_in = dp<int32_t>(ctx, p.o_in);
      J->o_out_off = dp<int32_t>(ctx, p.o_out_off);
      J->o_out = dp<int32_t>(ctx, p.o_out);
      J->t_size = dp<int64_t>(ctx, p.t_size);
      J->t_kind = dp<int8_t>(ctx, p.t_kind);
      J->t_rank = dp<int32_t>(ctx, p.t_rank);
      J->t_store = dp<int32_t>(ctx, p.t_store);
      J->t_upd = dp<int32_t>(ctx, p.t_upd);
      J->t_prod = dp<int32_t>(ctx, p.t_prod);
      J->a_inflag = mode == 1 ? dp<uint8_t>(ctx, p.inflag) : nullptr;
      J->a_tensor = dp<int32_t>(ctx, p.a_tensor);
      J->a_store = dp<int32_t>(ctx, p.a_store);
      J->a_type = dp<int8_t>(ctx, p.a_type);
      J->a_start = dp<int64_t>(ctx, p.a_start);
      J->a_end = dp<int64_t>(ctx, p.a_end);
      J->a_base = dp<uint8_t>(ctx, p.a_base);
      J->a_flag = dp<uint8_t>(ctx, p.a_flag);
      J->a_owned = dp<uint8_t>(ctx, p.a_owned);
      J->s_off = dp<int32_t>(ctx, p.s_off);
      J->s_acc = dp<int32_t>(ctx, p.s_acc);
      J->t_wfirst = dp<int32_t>(ctx, p.t_wfirst);
      J->t_utga = dp<int32_t>(ctx, p.t_utga);
      J->ev_id = dp<int64_t>(ctx, p.ev[0]);
      J->ev_tensor = dp<int32_t>(ctx, p.ev[1]);
      J->ev_dir = dp<int8_t>(ctx, p.ev[2]);
      J->ev_wraps = dp<int8_t>(ctx, p.ev[3]);
      J->ev_trig = dp<int64_t>(ctx, p.ev[4]);
      J->ev_delta = dp<int64_t>(ctx, p.ev[5]);
      J->ev_start = dp<int64_t>(ctx, p.ev[6]);
      J->ev_end = dp<int64_t>(ctx, p.ev[7]);
      J->ev_earl = dp<int64_t>(ctx, p.ev[8]);
      J->ev_late = dp<int64_t>(ctx, p.ev[9]);
      J->ev_pair = dp<int64_t>(ctx, p.ev[10]);
      J->ev_serves = dp<int64_t>(ctx, p.ev[11]);
      J->bz_s = dp<int64_t>(ctx, p.bz_s);
      J->bz_e = dp<int64_t>(ctx, p.bz_e);
      J->pd_s = dp<int64_t>(ctx, p.pd_s);
      J->pd_e = dp<int64_t>(ctx, p.pd_e);
      J->pd_ts = dp<int64_t>(ctx, p.pd_ts);
      J->pd_te = dp<int64_t>(ctx, p.pd_te);
      J->bzi_s = dp<int32_t>(ctx, p.bzi_s);
      J->bzi_e = dp<int32_t>(ctx, p.bzi_e);
      J->ai_e = dp<int32_t>(ctx, p.ai_e);
      J->st_evcnt = dp<int32_t>(ctx, p.st_evcnt);
      J->swapped = dp<uint8_t>(ctx, p.swapped);
      J->rc_id = dp<int64_t>(ctx, p.rc[0]);
      J->rc_tensor = dp<int32_t>(ctx, p.rc[1]);
      J->rc_target = dp<int64_t>(ctx, p.rc[2]);
      J->rc_regen = dp<int32_t>(ctx, p.rc[3]);
      J->rc_lat = dp<int64_t>(ctx, p.rc[4]);
      J->rc_saving = dp<int64_t>(ctx, p.rc[5]);
      J->in_peak = dp<uint8_t>(ctx, p.in_peak);
      J->ev_drop = dp<uint8_t>(ctx, p.ev_drop);
      J->res_init = dp<uint8_t>(ctx, p.res_init);
      J->curve_t = dp<int64_t>(ctx, p.curve_t);
      J->curve_b = dp<int64_t>(ctx, p.curve_b);
      J->bk_a_start = dp<int64_t>(ctx, p.bk_a_start);
      J->bk_a_end = dp<int64_t>(ctx, p.bk_a_end);
      J->bk_flag = dp<uint8_t>(ctx, p.bk_flag);
      J->bk_in_peak = dp<uint8_t>(ctx, p.bk_in_peak);
      J->pk_list = dp<int32_t>(ctx, p.pk_list);
      J->bk_ev = dp<int64_t>(ctx, p.bk_ev);
      J->bk_rc = dp<int64_t>(ctx, p.bk_rc);
      J->bk_bz = dp<int64_t>(ctx, p.bk_bz);
      J->bk_evcnt = dp<int32_t>(ctx, p.bk_evcnt);
      J->bk_curve = dp<int64_t>(ctx, p.bk_curve);
      JobState* S = hp<JobState>(ctx, P->states_off) + jglob;
      std::memset(S, 0, sizeof *S);
      if (mode == 1) {
        // caller plan -> ev/rc arrays in the output region + flags
        const tsl_plan_desc& pd = caller[jglob];
        if (pd.n_swap > p.Scap || pd.n_recompute > p.Rcap) fail(TSL_ERR_CAPACITY, "caller plan too large");
        int64_t mx = -1;
        for (int32_t i = 0; i < pd.n_swap; ++i) {
          if (pd.ev_tensor[i] < 0 || pd.ev_tensor[i] >= g.T)
            fail(TSL_ERR_VALIDATION, "unknown tensor #" + std::to_string(pd.ev_tensor[i]) + " in catalog of " + g.job_id);
          hp<int64_t>(ctx, p.ev[0])[i] = pd.ev_id[i];
          hp<int32_t>(ctx, p.ev[1])[i] = pd.ev_tensor[i];
          hp<int8_t>(ctx, p.ev[2])[i] = pd.ev_dir[i];
          hp<int8_t>(ctx, p.ev[3])[i] = pd.ev_wraps[i];
          hp<int64_t>(ctx, p.ev[4])[i] = pd.ev_trigger[i];
          hp<int64_t>(ctx, p.ev[5])[i] = pd.ev_delta[i];
          hp<int64_t>(ctx, p.ev[6])[i] = pd.ev_start[i];
          hp<int64_t>(ctx, p.ev[7])[i] = pd.ev_end[i];
          hp<int64_t>(ctx, p.ev[8])[i] = 0;
          hp<int64_t>(ctx, p.ev[9])[i] = 0;
          hp<int64_t>(ctx, p.ev[10])[i] = pd.ev_pair[i];
          hp<int64_t>(ctx, p.ev[11])[i] = pd.ev_serves[i];
          mx = std::max(mx, pd.ev_id[i]);
        }
        for (int32_t r = 0; r < pd.n_recompute; ++r) {
          if (pd.rc_tensor[r] < 0 || pd.rc_tensor[r] >= g.T)
            fail(TSL_ERR_VALIDATION, "unknown tensor #" + std::to_string(pd.rc_tensor[r]) + " in catalog of " + g.job_id);
          hp<int64_t>(ctx, p.rc[0])[r] = pd.rc_id[r];
          hp<int32_t>(ctx, p.rc[1])[r] = pd.rc_tensor[r];
          hp<int64_t>(ctx, p.rc[2])[r] = pd.rc_target[r];
          hp<int32_t>(ctx, p.rc[3])[r] = pd.rc_regen_op[r];
          hp<int64_t>(ctx, p.rc[4])[r] = pd.rc_latency[r];
          hp<int64_t>(ctx, p.rc[5])[r] = pd.rc_saving[r];
          mx = std::max(mx, pd.rc_id[r]);
        }
        uint8_t* fl = hp<uint8_t>(ctx, p.inflag);
        std::memset(fl, 0, g.A);
        for (int32_t i = 0; i < pd.n_release; ++i)
          if (pd.release_flags[i] >= 0 && pd.release_flags[i] < g.A) fl[pd.release_flags[i]] = 1;
        S->S = pd.n_swap;
        S->R = pd.n_recompute;
        S->next_id = mx + 1;
      }
    }
  }
  P->h2d_bytes = mode == 1 ? out_end : stage_end;
  P->d2h_off = P->groups_off;
  P->d2h_bytes = out_end - P->groups_off;
  P->stage_end = stage_end;
  auto t1 = std::chrono::steady_clock::now();
  P->prep_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  if (std::getenv("TSL_PREP_PROFILE")) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "prep: load %.3f validate %.3f layout %.3f grow %.3f fill %.3f ms\n", ms(t0, t_load),
                 ms(t_load, t_val), ms(t_val, t_lay), ms(t_lay, t_grow), ms(t_grow, t1));
  }
  return P;
}

void upload(tsl_plan* P) {
  Buffers* b = P->buf;
  cuda_check(cudaMemcpyAsync(b->dbuf, b->hbuf, P->h2d_bytes, cudaMemcpyHostToDevice, P->ctx->stream), "H2D");
  if (P->coop)  // (the kernel leaves it reset, so one upload serves every launch)
    cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(b->dbuf) + P->gp[0].coop, &P->coop_init, sizeof P->coop_init,
                               cudaMemcpyHostToDevice, P->ctx->stream), "H2D coop");
}

void launch(tsl_plan* P, int repeats, bool timed) {
  tsl_ctx* c = P->ctx;
  GroupDev* dg = dp<GroupDev>(P->buf, P->groups_off);
  if (timed) cuda_check(cudaEventRecord(c->ev0, c->stream), "event");
  for (int r = 0; r < repeats; ++r) {  // the kernel resets its own group header
    if (P->coop && r == 0)  // (and the control block, unless a launch aborted)
      cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(P->buf->dbuf) + P->gp[0].coop, &P->coop_init,
                                 sizeof P->coop_init, cudaMemcpyHostToDevice, c->stream), "H2D coop");
    cuda_check(launch_plan_kernel(dg, P->n_groups, P->mode, P->max_jobs, P->ipt, P->res_bytes, P->big, P->coop, c->stream), "launch");
  }
  if (timed) cuda_check(cudaEventRecord(c->ev1, c->stream), "event");
}

// Results to the host. Builds of small jobs: the whole output region in one
// copy (a C5 launch's 120 builds would otherwise need thousands of small
// copies). Builds with jobs above one sort tile (C4: ~250 MB of
// capacity-sized arrays): the headers first, then only the used prefix of
// every output array (events, recomputes, history, curve) -- one extra round
// trip for ~4x fewer bytes.
void download(tsl_plan* P, cudaStream_t s) {
  Buffers* b = P->buf;
  size_t moved = 0;
  auto d2h = [&](size_t off, size_t n) {
    if (!n) return;
    cuda_check(cudaMemcpyAsync(b->hbuf + off, static_cast<uint8_t*>(b->dbuf) + off, n, cudaMemcpyDeviceToHost, s),
               "D2H");
    moved += n;
  };
  if (!P->big || P->d2h_bytes <= (size_t(8) << 20) || P->mode != 0) {
    d2h(P->d2h_off, P->d2h_bytes);
    cuda_check(cudaStreamSynchronize(s), "sync");
    P->d2h_done = moved;
    return;
  }
  d2h(P->groups_off, P->stage_end - P->groups_off);
  cuda_check(cudaStreamSynchronize(s), "sync");
  for (int gi = 0; gi < P->n_groups; ++gi) {
    const GroupDev& G = hp<GroupDev>(b, P->groups_off)[gi];
    const GroupPlace& q = P->gp[gi];
    d2h(q.hist, sizeof(int64_t) * size_t(std::max(0, std::min(G.n_hist, G.hist_cap))));
    const int32_t jb = P->group_job_base[gi];
    for (size_t k = 0; k < P->graphs[gi].size(); ++k) {
      const Graph& g = *P->graphs[gi][k];
      const JobPlace& p = P->jp[gi][k];
      const JobState& st = hp<JobState>(b, P->states_off)[jb + k];
      for (int f = 0; f < 12; ++f) d2h(p.ev[f], size_t((f == 1) ? 4 : (f == 2 || f == 3) ? 1 : 8) * size_t(st.S));
      for (int f = 0; f < 6; ++f) d2h(p.rc[f], size_t((f == 1 || f == 3) ? 4 : 8) * size_t(st.R));
      d2h(p.a_flag, size_t(g.A));
      d2h(p.in_peak, size_t(g.T));
      d2h(p.curve_t, sizeof(int64_t) * size_t(st.n_curve));
      d2h(p.curve_b, sizeof(int64_t) * size_t(st.n_curve));
    }
  }
  cuda_check(cudaStreamSynchronize(s), "sync");
  P->d2h_done = moved;
}

std::string err_text(const GroupDev& G, const std::vector<GraphP>& gs) {
  const ErrInfo& e = G.err;
  const Graph* g = (e.job >= 0 && e.job < static_cast<int>(gs.size())) ? gs[e.job].get() : nullptr;
  auto tname = [&](int64_t t) { return (g && t >= 0 && t < g->T) ? g->tid[t] : "#" + std::to_string(t); };
  switch (e.code) {
    case E_DOUBLE_RELEASE: return "double release of tensor " + tname(e.tensor);
    case E_SWAPIN_RESIDENT: return "swap-in of resident tensor " + tname(e.tensor);
    case E_NEG_FOOTPRINT: return "negative footprint at tick " + std::to_string(e.tick);
    case E_NO_TGA: return "tensor " + tname(e.tensor) + " has no TGA in sequence";
    case E_UNKNOWN_ACCESS:
      return "unknown access id " + std::to_string(e.tensor) + " in job " + (g ? g->job_id : std::string("?"));
    case E_CAPACITY: return "device planner capacity exceeded (" + std::to_string(e.tensor) + ")";
    default:
      if (e.code == E_INTERNAL && e.tick >= 1000)
        return "device spin timeout at site " + std::to_string(e.tick - 1000) + ": cooperative launch aborted";
      return "internal planner error";
  }
}

void cp64_now(Buffers* c, std::vector<int64_t>& v, size_t off, int32_t n) {
  v.assign(hp<int64_t>(c, off), hp<int64_t>(c, off) + n);
}

// Runs independent tasks in order, or on up to 8 host threads when `par`.
void run_tasks(std::vector<std::function<void()>>& tasks, bool par) {
  if (!par) {
    for (auto& t : tasks) t();
    return;
  }
  const size_t nt = std::min<size_t>({8, tasks.size(), std::max(1u, std::thread::hardware_concurrency())});
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t i; (i = next.fetch_add(1)) < tasks.size();) tasks[i]();
  };
  std::vector<std::thread> th;
  for (size_t k = 1; k < nt; ++k) th.emplace_back(worker);
  worker();
  for (auto& t : th) t.join();
}

tsl_result* collect_group(tsl_plan* P, int gi) {
  Buffers* c = P->buf;
  const GroupDev& G = hp<GroupDev>(c, P->groups_off)[gi];
  if (G.err.code) {
    int code = G.err.code == E_CAPACITY ? TSL_ERR_CAPACITY
             : G.err.code == E_INTERNAL ? TSL_ERR_INTERNAL : TSL_ERR_VALIDATION;
    fail(code, err_text(G, P->graphs[gi]));
  }
  auto* R = new tsl_result();
  R->graphs = P->graphs[gi];
  const int32_t jb = P->group_job_base[gi];
  std::map<std::string, int> order;
  for (size_t k = 0; k < R->graphs.size(); ++k) order[R->graphs[k]->job_id] = static_cast<int>(k);
  for (auto& kv : order) {
    const int k = kv.second;
    const Graph& g = *R->graphs[k];
    const JobPlace& p = P->jp[gi][k];
    const JobState& st = hp<JobState>(c, P->states_off)[jb + k];
    JobOut o;
    o.g = R->graphs[k].get();
    o.st = st;
    // the copies out of the pinned buffer are independent: a big job's
    // (C4: ~60 MB of events and curve) run on a few host threads
    std::vector<std::function<void()>> tasks;
    auto cp64 = [&](std::vector<int64_t>& v, size_t off, int32_t n) {
      tasks.push_back([&v, c, off, n] { v.assign(hp<int64_t>(c, off), hp<int64_t>(c, off) + n); });
    };
    cp64(o.ev_id, p.ev[0], st.S);
    tasks.push_back([&] {
      o.ev_tensor.assign(hp<int32_t>(c, p.ev[1]), hp<int32_t>(c, p.ev[1]) + st.S);
      o.ev_dir.assign(hp<int8_t>(c, p.ev[2]), hp<int8_t>(c, p.ev[2]) + st.S);
      o.ev_wraps.assign(hp<int8_t>(c, p.ev[3]), hp<int8_t>(c, p.ev[3]) + st.S);
    });
    cp64(o.ev_trig, p.ev[4], st.S);
    cp64(o.ev_delta, p.ev[5], st.S);
    cp64(o.ev_start, p.ev[6], st.S);
    cp64(o.ev_end, p.ev[7], st.S);
    cp64(o.ev_earl, p.ev[8], st.S);
    cp64(o.ev_late, p.ev[9], st.S);
    cp64(o.ev_pair, p.ev[10], st.S);
    cp64(o.ev_serves, p.ev[11], st.S);
    tasks.push_back([&] {
      cp64_now(c, o.rc_id, p.rc[0], st.R);
      o.rc_tensor.assign(hp<int32_t>(c, p.rc[1]), hp<int32_t>(c, p.rc[1]) + st.R);
      cp64_now(c, o.rc_target, p.rc[2], st.R);
      o.rc_regen.assign(hp<int32_t>(c, p.rc[3]), hp<int32_t>(c, p.rc[3]) + st.R);
      cp64_now(c, o.rc_lat, p.rc[4], st.R);
      cp64_now(c, o.rc_saving, p.rc[5], st.R);
    });
    tasks.push_back([&] {
      const uint8_t* fl = hp<uint8_t>(c, p.a_flag);
      for (int32_t a = 0; a < g.A; ++a)
        if (fl[a]) o.flags.push_back(a);
      if (P->mode == 1) o.flags.clear();  // caller flags outside [0, A) are kept verbatim
    });
    tasks.push_back([&] {
      const uint8_t* pk = hp<uint8_t>(c, p.in_peak);
      std::vector<int32_t> byr(g.T);
      for (int32_t t = 0; t < g.T; ++t) byr[g.trank[t]] = t;
      for (int32_t r = 0; r < g.T; ++r)
        if (pk[byr[r]]) o.peak_tensors.push_back(byr[r]);
    });
    cp64(o.curve_t, p.curve_t, st.n_curve);
    cp64(o.curve_b, p.curve_b, st.n_curve);
    run_tasks(tasks, size_t(st.S) + size_t(st.n_curve) + size_t(g.A) > (size_t(1) << 20));
    R->jobs.push_back(std::move(o));
  }
  R->history.assign(hp<int64_t>(c, P->gp[gi].hist), hp<int64_t>(c, P->gp[gi].hist) + std::min(G.n_hist, G.hist_cap));
  R->final_merged = G.final_merged;
  R->within = G.within_budget != 0;
  if (P->mode == 0 && !R->within)
    R->diagnostic = "merged memory peak " + std::to_string(G.final_merged) + " still exceeds budget " +
                    std::to_string(G.cfg.budget) + " after exhausting swap and recomputation";
  tsl_stats& s = R->stats;
  s.kernel_ms = P->last_kernel_ms;
  for (auto& g : R->graphs) s.n_accesses += g->A;
  s.loop_iterations = G.stats.loop_iterations;
  s.evaluations = G.stats.evaluations;
  s.timeline_events = G.stats.timeline_events;
  s.candidates = G.stats.candidates;
  s.candidate_accesses = G.stats.candidate_accesses;
  s.busy_intervals = G.stats.busy_intervals;
  s.algorithmic_bytes = 24 * s.timeline_events + 24 * s.candidate_accesses + 16 * s.busy_intervals + 16 * s.candidates;
  s.kernel_launches = 1;
  s.h2d_bytes = static_cast<int64_t>(P->h2d_bytes);
  s.d2h_bytes = static_cast<int64_t>(P->d2h_done);
  s.prep_ms = P->prep_ms;
  s.rescored = G.stats.rescored;
  s.cyc_sequence = G.stats.cyc[0];
  s.cyc_evaluate = G.stats.cyc[1];
  s.cyc_swap = G.stats.cyc[2];
  s.cyc_recompute = G.stats.cyc[3];
  s.cyc_total = G.stats.cyc[4];
  s.cyc_spec = G.stats.cyc[5];
  s.cyc_conflict = G.stats.cyc[6];
  s.cyc_sweep = G.stats.cyc[7];
  s.cyc_merge = G.stats.cyc[8] + G.stats.cyc[9];
  s.cyc_rescore = G.stats.cyc[10];
  s.cyc_apply = G.stats.cyc[8];
  for (int k = 0; k < 4; ++k) s.debug[k] = G.stats.cyc[12 + k];
  s.cyc_pendsort = G.stats.cyc[11];
  for (int k = 0; k < 4; ++k) s.fitprof[k] = G.stats.cyc[16 + k];
  for (int k = 0; k < 5; ++k) s.fitprof[4 + k] = G.stats.cyc[27 + k];
  for (int k = 0; k < 7; ++k) s.evalprof[k] = G.stats.cyc[20 + k];
  for (int k = 0; k < 16; ++k) s.queryprof[k] = G.stats.prof[k];
  s.comp_rescored = G.stats.comp_rescored;
  for (int k = 0; k < 24; ++k) s.stageprof[k] = G.stats.sprof[k];
  return R;
}

// ---------------------------------------------------------------------------
// JSON (nlohmann ordered_json dump(2) layout, as the reference prints it)
// ---------------------------------------------------------------------------
void jstr(std::string& o, const std::string& s) {
  o += '"';
  for (unsigned char ch : s) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (ch < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", ch);
          o += buf;
        } else {
          o += static_cast<char>(ch);
        }
    }
  }
  o += '"';
}

std::string sp(int n) { return std::string(static_cast<size_t>(n), ' '); }
std::string num(int64_t v) { return std::to_string(v); }

// save_plans, plan.cpp:30-65.
std::string save_plans(const tsl_result& r) {
  if (r.jobs.empty()) return "null\n";
  std::string o = "{\n";
  for (size_t ji = 0; ji < r.jobs.size(); ++ji) {
    const JobOut& j = r.jobs[ji];
    o += sp(2);
    jstr(o, j.g->job_id);
    o += ": {\n" + sp(4) + "\"version\": " + num(j.version) + ",\n" + sp(4) + "\"swap_events\": ";
    const size_t S = j.ev_id.size();
    if (!S) o += "[],\n";
    else {
      o += "[\n";
      for (size_t i = 0; i < S; ++i) {
        o += sp(6) + "{\n";
        o += sp(8) + "\"event_id\": " + num(j.ev_id[i]) + ",\n";
        o += sp(8) + "\"tensor\": ";
        jstr(o, j.g->tid[j.ev_tensor[i]]);
        o += ",\n" + sp(8) + "\"direction\": " + (j.ev_dir[i] == 0 ? "\"out\"" : "\"in\"") + ",\n";
        o += sp(8) + "\"trigger_access\": " + num(j.ev_trig[i]) + ",\n";
        o += sp(8) + "\"delta_time\": " + num(j.ev_delta[i]) + ",\n";
        o += sp(8) + "\"wraps_iteration\": " + (j.ev_wraps[i] ? "true" : "false") + ",\n";
        o += sp(8) + "\"start_time\": " + num(j.ev_start[i]) + ",\n";
        o += sp(8) + "\"end_time\": " + num(j.ev_end[i]) + ",\n";
        o += sp(8) + "\"pair_id\": " + num(j.ev_pair[i]) + ",\n";
        o += sp(8) + "\"serves_access\": " + num(j.ev_serves[i]) + "\n";
        o += sp(6) + (i + 1 < S ? "},\n" : "}\n");
      }
      o += sp(4) + "],\n";
    }
    o += sp(4) + "\"recompute_events\": ";
    const size_t R = j.rc_id.size();
    if (!R) o += "[],\n";
    else {
      o += "[\n";
      for (size_t i = 0; i < R; ++i) {
        o += sp(6) + "{\n";
        o += sp(8) + "\"event_id\": " + num(j.rc_id[i]) + ",\n";
        o += sp(8) + "\"tensor\": ";
        jstr(o, j.g->tid[j.rc_tensor[i]]);
        o += ",\n" + sp(8) + "\"target_access\": " + num(j.rc_target[i]) + ",\n";
        o += sp(8) + "\"regen_op\": ";
        jstr(o, j.g->oid[j.rc_regen[i]]);
        o += ",\n" + sp(8) + "\"recompute_latency\": " + num(j.rc_lat[i]) + ",\n";
        o += sp(8) + "\"memory_saving\": " + num(j.rc_saving[i]) + "\n";
        o += sp(6) + (i + 1 < R ? "},\n" : "}\n");
      }
      o += sp(4) + "],\n";
    }
    // nlohmann 3.11.3 prints an array whose elements are all numbers inline.
    o += sp(4) + "\"release_flags\": [";
    for (size_t k = 0; k < j.flags.size(); ++k) o += (k ? "," : "") + num(j.flags[k]);
    o += "]\n" + sp(2) + (ji + 1 < r.jobs.size() ? "},\n" : "}\n");
  }
  return o + "}\n";
}

// PeakReport::to_json, peak.cpp:258-272.
std::string report_json(const JobOut& j) {
  std::string o = "{\n" + sp(2) + "\"memory_peak\": " + num(j.st.peak) + ",\n" + sp(2) + "\"peak_tensors\": ";
  if (j.peak_tensors.empty()) o += "[],\n";
  else {
    o += "[\n";
    for (size_t i = 0; i < j.peak_tensors.size(); ++i) {
      o += sp(4);
      jstr(o, j.g->tid[j.peak_tensors[i]]);
      o += i + 1 < j.peak_tensors.size() ? ",\n" : "\n";
    }
    o += sp(2) + "],\n";
  }
  o += sp(2) + "\"last_input_access\": " + (j.st.has_lua ? num(j.st.lua) : std::string("null")) + ",\n";
  o += sp(2) + "\"peak_time\": " + num(j.st.peak_time) + ",\n" + sp(2) + "\"footprint_curve\": ";
  if (j.curve_t.empty()) o += "[]\n";
  else {
    o += "[\n";
    for (size_t i = 0; i < j.curve_t.size(); ++i)
      o += sp(4) + "[" + num(j.curve_t[i]) + "," + num(j.curve_b[i]) + (i + 1 < j.curve_t.size() ? "],\n" : "]\n");
    o += sp(2) + "]\n";
  }
  return o + "}\n";
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return TSL_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TSL_ERR_INTERNAL;
  }
}

}  // namespace

namespace tsl {
namespace hostg {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace hostg
}  // namespace tsl

extern "C" {

const char* tsl_last_error(void) { return g_err.c_str(); }

int tsl_validate_config(const tsl_config* cfg) {
  if (!cfg) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] { validate_config(*cfg); });
}

int tsl_result_set_version(tsl_result* r, const char* job_id, int64_t version) {
  if (!r || !job_id) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    for (auto& j : r->jobs)
      if (j.g && j.g->job_id == job_id) { j.version = static_cast<int32_t>(version); return; }
    fail(TSL_ERR_ARGUMENT, std::string("no job ") + job_id + " in result");
  });
}

void tsl_config_default(tsl_config* c) {
  c->pcie_bandwidth = 1;
  c->transfer_setup = 0;
  c->memory_budget = 0;
  c->ewma_alpha = 0.3;
  c->replan_threshold = 0.2;
  c->stall_epsilon = 0.0005;
  c->stall_min_iters = 100;
  c->cold_start_gpu_usage = 0.5;
  c->n_max_swap_ratios = 0;
  c->max_swap_ratio_jobs = nullptr;
  c->max_swap_ratio_values = nullptr;
}

int tsl_create(int device, tsl_ctx** out) {
  if (!out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) fail(TSL_ERR_CUDA, "no CUDA device " + std::to_string(device));
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new tsl_ctx();
    c->device = device;
    cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreate(&c->ev0), "event");
    cuda_check(cudaEventCreate(&c->ev1), "event");
    *out = c;
  });
}

int tsl_destroy(tsl_ctx* c) {
  if (!c) return TSL_OK;
  cudaSetDevice(c->device);
  c->buf.release();
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return TSL_OK;
}

int tsl_plan_prepare(tsl_ctx* ctx, const tsl_job_desc* jobs, const int32_t* group_offsets, int32_t n_groups,
                     const tsl_config* cfgs, int32_t n_cfgs, tsl_plan** out) {
  if (!ctx || !cfgs || !out || !group_offsets || n_groups < 0) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tsl_plan* P = prepare(ctx, jobs, group_offsets, n_groups, cfgs, n_cfgs, 0, nullptr, true);
    try {
      upload(P);
      cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    } catch (...) {
      delete P;
      throw;
    }
    *out = P;
  });
}

int tsl_plan_run(tsl_plan* P, int32_t repeats, double* kernel_ms) {
  if (!P) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    tsl_ctx* c = P->ctx;
    cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
    launch(P, std::max(1, repeats), true);
    cuda_check(cudaEventSynchronize(c->ev1), "sync");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "elapsed");
    P->last_kernel_ms = ms / std::max(1, repeats);
    if (kernel_ms) *kernel_ms = P->last_kernel_ms;
  });
}

int tsl_plan_launch_async(tsl_plan* P, void* stream) {
  if (!P) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    tsl_ctx* c = P->ctx;
    cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
    const cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    cuda_check(launch_plan_kernel(dp<GroupDev>(P->buf, P->groups_off), P->n_groups, P->mode, P->max_jobs, P->ipt,
                                  P->res_bytes, P->big, P->coop, s), "launch");
    if (!P->done) cuda_check(cudaEventCreateWithFlags(&P->done, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(P->done, s), "event record");
  });
}

int tsl_plan_collect(tsl_plan* P, tsl_result** out) {
  if (!P || !out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    cuda_check(cudaSetDevice(P->ctx->device), "cudaSetDevice");
    // the last asynchronous launch may sit on a caller stream: wait for it
    // alone (not the whole device), then read back on the context's stream
    if (P->done) cuda_check(cudaEventSynchronize(P->done), "sync");
    download(P, P->ctx->stream);
    std::vector<tsl_result*> rs;
    try {
      for (int gi = 0; gi < P->n_groups; ++gi) rs.push_back(collect_group(P, gi));
    } catch (...) {
      for (auto* r : rs) delete r;
      throw;
    }
    for (int gi = 0; gi < P->n_groups; ++gi) out[gi] = rs[gi];
  });
}

void tsl_plan_destroy(tsl_plan* P) { delete P; }

int tsl_build_plan_groups(tsl_ctx* ctx, const tsl_job_desc* jobs, const int32_t* group_offsets, int32_t n_groups,
                          const tsl_config* cfgs, int32_t n_cfgs, tsl_result** out) {
  if (!ctx || !cfgs || !out || !group_offsets || n_groups < 0) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tsl_plan* P = prepare(ctx, jobs, group_offsets, n_groups, cfgs, n_cfgs, 0, nullptr, false);
    std::vector<tsl_result*> rs;
    try {
      const auto tp = std::chrono::steady_clock::now();
      upload(P);
      launch(P, 1, true);
      download(P, ctx->stream);
      const auto td = std::chrono::steady_clock::now();
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "elapsed");
      P->last_kernel_ms = ms;
      for (int gi = 0; gi < n_groups; ++gi) rs.push_back(collect_group(P, gi));
      if (std::getenv("TSL_E2E_PROFILE")) {
        auto d = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "e2e: prep %.3f upload+kernel+download %.3f (kernel %.3f, d2h %zu B) collect %.3f ms\n",
                     d(t0, tp), d(tp, td), double(ms), P->d2h_bytes, d(td, std::chrono::steady_clock::now()));
      }
    } catch (...) {
      for (auto* r : rs) delete r;
      delete P;
      throw;
    }
    auto t1 = std::chrono::steady_clock::now();
    const double tot = std::chrono::duration<double, std::milli>(t1 - t0).count();
    for (int gi = 0; gi < n_groups; ++gi) {
      rs[gi]->stats.total_ms = tot;
      out[gi] = rs[gi];
    }
    delete P;
  });
}

int tsl_build_plan(tsl_ctx* ctx, const tsl_job_desc* jobs, int32_t n_jobs, const tsl_config* cfg,
                   tsl_result** out) {
  if (n_jobs < 0) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  const int32_t offs[2] = {0, n_jobs};
  if (n_jobs == 0) {  // build_plan returns an empty result (orchestrator.cpp:12)
    if (!ctx || !cfg || !out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
    return guard([&] {
      validate_config(*cfg);
      *out = new tsl_result();
    });
  }
  return tsl_build_plan_groups(ctx, jobs, offs, 1, cfg, 1, out);
}

int tsl_analyze_job(tsl_ctx* ctx, const tsl_job_desc* job, const tsl_plan_desc* plan, tsl_result** out) {
  if (!ctx || !job || !plan || !out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tsl_config cfg;
    tsl_config_default(&cfg);
    const int32_t offs[2] = {0, 1};
    tsl_plan* P = prepare(ctx, job, offs, 1, &cfg, 1, 1, plan, false);
    tsl_result* r = nullptr;
    try {
      upload(P);
      launch(P, 1, true);
      download(P, ctx->stream);
      r = collect_group(P, 0);
    } catch (...) {
      delete P;
      throw;
    }
    // the caller's plan is echoed verbatim (release flags included)
    JobOut& o = r->jobs[0];
    o.version = static_cast<int32_t>(plan->version);
    o.flags.assign(plan->release_flags, plan->release_flags + plan->n_release);
    std::sort(o.flags.begin(), o.flags.end());
    o.flags.erase(std::unique(o.flags.begin(), o.flags.end()), o.flags.end());
    delete P;
    *out = r;
  });
}

int32_t tsl_result_n_jobs(const tsl_result* r) { return r ? static_cast<int32_t>(r->jobs.size()) : 0; }

int tsl_result_job(const tsl_result* r, int32_t i, tsl_job_view* v) {
  if (!r || !v || i < 0 || i >= static_cast<int32_t>(r->jobs.size())) { g_err = "bad job index"; return TSL_ERR_ARGUMENT; }
  const JobOut& o = r->jobs[static_cast<size_t>(i)];
  std::memset(v, 0, sizeof *v);
  v->job_id = o.g->job_id.c_str();
  v->version = o.version;
  v->n_swap = static_cast<int32_t>(o.ev_id.size());
  v->ev_id = o.ev_id.data();
  v->ev_tensor = o.ev_tensor.data();
  v->ev_dir = o.ev_dir.data();
  v->ev_trigger = o.ev_trig.data();
  v->ev_delta = o.ev_delta.data();
  v->ev_start = o.ev_start.data();
  v->ev_end = o.ev_end.data();
  v->ev_earliest = o.ev_earl.data();
  v->ev_latest = o.ev_late.data();
  v->ev_wraps = o.ev_wraps.data();
  v->ev_pair = o.ev_pair.data();
  v->ev_serves = o.ev_serves.data();
  v->n_recompute = static_cast<int32_t>(o.rc_id.size());
  v->rc_id = o.rc_id.data();
  v->rc_tensor = o.rc_tensor.data();
  v->rc_target = o.rc_target.data();
  v->rc_regen_op = o.rc_regen.data();
  v->rc_latency = o.rc_lat.data();
  v->rc_saving = o.rc_saving.data();
  v->n_release = static_cast<int32_t>(o.flags.size());
  v->release_flags = o.flags.data();
  v->memory_peak = o.st.peak;
  v->peak_time = o.st.peak_time;
  v->has_last_input_access = o.st.has_lua ? 1 : 0;
  v->last_input_access = o.st.has_lua ? o.st.lua : -1;
  v->n_peak_tensors = static_cast<int32_t>(o.peak_tensors.size());
  v->peak_tensors = o.peak_tensors.data();
  v->n_curve = static_cast<int32_t>(o.curve_t.size());
  v->curve_time = o.curve_t.data();
  v->curve_bytes = o.curve_b.data();
  v->iteration_period = o.st.period;
  v->n_accesses = o.g->A;
  return TSL_OK;
}

int32_t tsl_result_history(const tsl_result* r, const int64_t** h) {
  if (!r || !h) return 0;
  *h = r->history.data();
  return static_cast<int32_t>(r->history.size());
}
int64_t tsl_result_final_merged_peak(const tsl_result* r) { return r ? r->final_merged : 0; }
int32_t tsl_result_within_budget(const tsl_result* r) { return r && r->within ? 1 : 0; }
const char* tsl_result_diagnostic(const tsl_result* r) { return r ? r->diagnostic.c_str() : ""; }
int tsl_result_stats(const tsl_result* r, tsl_stats* out) {
  if (!r || !out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  *out = r->stats;
  return TSL_OK;
}
char* tsl_result_save_plans(const tsl_result* r) { return r ? dup(save_plans(*r)) : nullptr; }
char* tsl_result_report_json(const tsl_result* r, int32_t i) {
  if (!r || i < 0 || i >= static_cast<int32_t>(r->jobs.size())) return nullptr;
  return dup(report_json(r->jobs[static_cast<size_t>(i)]));
}
void tsl_result_destroy(tsl_result* r) { delete r; }
void tsl_free(void* p) { std::free(p); }

}  // extern "C"

// ---------------------------------------------------------------------------
// Plan executor host driver (tsl_exec.cu holds the kernels)
// ---------------------------------------------------------------------------
namespace {

struct ExecStepH {
  int32_t op;
  bool regen;
  int64_t ticks;
  int64_t start, end;  // planned ticks within the iteration
  std::vector<int32_t> ins, outs, rel;
  std::vector<int64_t> out_size, rel_size;
  std::vector<int32_t> access_ids;
};

struct ExecXferH {
  int32_t ev;      // plan index
  int32_t storage;
  int dir;         // 0 out, 1 in
  int32_t anchor;  // step index or -1 (iteration start)
  int64_t delta, arrival, dur, size;
  int32_t serve_step;  // swap-in: step that waits for it
};

// One job's replay program: steps (ops + recompute regenerations) and the
// iteration's transfers in channel order (simulator.cpp:168-224).
struct JobProgram {
  const JobOut* o = nullptr;
  const Graph* g = nullptr;
  std::vector<ExecStepH> steps;
  std::vector<ExecXferH> xs;
  std::vector<int32_t> outs_per_iter;
  int64_t period = 0;
  std::vector<int64_t> slot_off, host_off;
  int64_t pool_bytes = 0, host_bytes = 0;
  std::vector<int32_t> i32;
  std::vector<int64_t> i64;
  struct OpOff { size_t ins, outs, rel, osz, rsz; };
  std::vector<OpOff> offs;
  std::vector<int32_t> init_st;
  std::vector<int64_t> init_sz;
  std::set<int32_t> wrapped_in;
};

JobProgram make_program(const JobOut& o, const tsl_config& cfg, const tsl_exec_config& ex) {
  JobProgram P;
  P.o = &o;
  const Graph& g = *o.g;
  P.g = &g;
  // access sequence with the true latencies (simulator.cpp:168-213)
  std::vector<int32_t> acc_op, acc_tensor;
  std::vector<std::vector<int32_t>> op_acc(g.O);
  for (int32_t op : g.topo) {
    for (int32_t i = g.in_off[op]; i < g.in_off[op + 1]; ++i) {
      op_acc[op].push_back(static_cast<int32_t>(acc_op.size()));
      acc_op.push_back(op);
      acc_tensor.push_back(g.in[i]);
    }
    for (int32_t i = g.out_off[op]; i < g.out_off[op + 1]; ++i) {
      op_acc[op].push_back(static_cast<int32_t>(acc_op.size()));
      acc_op.push_back(op);
      acc_tensor.push_back(g.out[i]);
    }
  }
  std::set<int64_t> flags(o.flags.begin(), o.flags.end());
  const bool vanilla = ex.vanilla != 0;
  if (vanilla) {  // activity analysis only (access.cpp:61-78): the last access of every Interim tensor id
    flags.clear();
    std::vector<int32_t> last(g.T, -1);
    for (size_t a = 0; a < acc_tensor.size(); ++a) last[acc_tensor[a]] = static_cast<int32_t>(a);
    for (int32_t t = 0; t < g.T; ++t)
      if (last[t] >= 0 && g.kind[t] == TSL_KIND_INTERIM) flags.insert(last[t]);
  }
  // steps: recompute regenerations right before their target op, then the op
  std::vector<int32_t> op_step(g.O, -1);
  int64_t clock = 0;
  for (int32_t op : g.topo) {
    for (size_t k = 0; k < (vanilla ? 0 : o.rc_id.size()); ++k) {
      if (acc_op[static_cast<size_t>(o.rc_target[k])] != op) continue;
      ExecStepH st{};
      st.op = o.rc_regen[k];
      st.regen = true;
      st.ticks = g.lat[st.op];
      for (int32_t i = g.in_off[st.op]; i < g.in_off[st.op + 1]; ++i) st.ins.push_back(g.store[g.in[i]]);
      const int32_t s = g.store[o.rc_tensor[k]];
      st.outs.push_back(s);
      st.out_size.push_back(g.size[s]);
      st.start = clock;
      clock += st.ticks;
      st.end = clock;
      P.steps.push_back(std::move(st));
    }
    ExecStepH st{};
    st.op = op;
    st.regen = false;
    st.ticks = g.lat[op];
    for (int32_t i = g.in_off[op]; i < g.in_off[op + 1]; ++i) st.ins.push_back(g.store[g.in[i]]);
    for (int32_t i = g.out_off[op]; i < g.out_off[op + 1]; ++i) {
      const int32_t t = g.out[i];
      st.outs.push_back(g.store[t]);
      st.out_size.push_back(g.store[t] != t ? 0 : g.size[t]);  // in-place update: no allocation
    }
    for (int32_t a : op_acc[op])
      if (flags.count(a)) {
        st.rel.push_back(g.store[acc_tensor[a]]);
        st.rel_size.push_back(g.size[g.store[acc_tensor[a]]]);
      }
    st.access_ids = op_acc[op];
    st.start = clock;
    clock += st.ticks;
    st.end = clock;
    op_step[op] = static_cast<int32_t>(P.steps.size());
    P.steps.push_back(std::move(st));
  }
  P.period = clock;
  // transfers of one iteration, in channel (arrival) order
  P.outs_per_iter.assign(g.T, 0);
  for (size_t e = 0; e < (vanilla ? 0 : o.ev_id.size()); ++e) {
    ExecXferH t{};
    t.ev = static_cast<int32_t>(e);
    t.storage = g.store[o.ev_tensor[e]];
    t.dir = o.ev_dir[e];
    t.anchor = o.ev_trig[e] < 0 ? -1 : op_step[acc_op[static_cast<size_t>(o.ev_trig[e])]];
    t.delta = o.ev_delta[e];
    t.arrival = (t.anchor < 0 ? 0 : P.steps[static_cast<size_t>(t.anchor)].end) + t.delta;
    t.size = g.size[t.storage];
    t.dur = (t.size + cfg.pcie_bandwidth - 1) / cfg.pcie_bandwidth + cfg.transfer_setup;
    t.serve_step = (t.dir == 1 && o.ev_serves[e] >= 0) ? op_step[acc_op[static_cast<size_t>(o.ev_serves[e])]] : -1;
    if (t.dir == 0) P.outs_per_iter[t.storage]++;
    P.xs.push_back(t);
  }
  std::stable_sort(P.xs.begin(), P.xs.end(), [](const ExecXferH& a, const ExecXferH& b) { return a.arrival < b.arrival; });
  // device / host slots
  P.slot_off.assign(g.T, 0);
  for (int32_t t = 0; t < g.T; ++t) {
    if (g.store[t] != t) continue;
    P.slot_off[t] = P.pool_bytes;
    P.pool_bytes += ((g.size[t] * ex.bytes_per_unit + 255) / 256) * 256;
  }
  P.host_off.assign(g.T, -1);
  for (auto& t : P.xs)
    if (P.host_off[t.storage] < 0) {
      P.host_off[t.storage] = P.host_bytes;
      P.host_bytes += ((g.size[t.storage] * ex.bytes_per_unit + 255) / 256) * 256;
    }
  for (auto& st : P.steps) {
    JobProgram::OpOff f{};
    f.ins = P.i32.size(); P.i32.insert(P.i32.end(), st.ins.begin(), st.ins.end());
    f.outs = P.i32.size(); P.i32.insert(P.i32.end(), st.outs.begin(), st.outs.end());
    f.rel = P.i32.size(); P.i32.insert(P.i32.end(), st.rel.begin(), st.rel.end());
    f.osz = P.i64.size(); P.i64.insert(P.i64.end(), st.out_size.begin(), st.out_size.end());
    f.rsz = P.i64.size(); P.i64.insert(P.i64.end(), st.rel_size.begin(), st.rel_size.end());
    P.offs.push_back(f);
  }
  for (size_t e = 0; e < (vanilla ? 0 : o.ev_id.size()); ++e)
    if (o.ev_dir[e] == 1 && o.ev_wraps[e]) P.wrapped_in.insert(g.store[o.ev_tensor[e]]);
  for (int32_t t = 0; t < g.T; ++t) {  // initial residency (simulator.cpp:247-269)
    if (g.store[t] != t) continue;
    const int8_t k = g.kind[t];
    if (k != TSL_KIND_PARAMETER && k != TSL_KIND_INPUT && k != TSL_KIND_OUTPUT) continue;
    if (P.wrapped_in.count(t)) continue;
    P.init_st.push_back(t);
    P.init_sz.push_back(g.size[t]);
  }
  return P;
}

// Replays the plans of jobs `jis` of one build result together (the
// reference's scheduled mode, simulator.cpp:112-569): every job's steps on
// its own compute stream, every job's transfers on ONE copy stream (the FIFO
// channel) in planned-arrival order, one allocator counter over all jobs
// (plus per-job counters). A single job is the same program with one stream.
void execute_jobs(tsl_ctx* ctx, const tsl_result* r, const std::vector<int32_t>& jis, const tsl_config& cfg,
                  const tsl_exec_config& ex, std::vector<tsl_exec_report>& per, tsl_exec_report& merged) {
  auto t0 = std::chrono::steady_clock::now();
  if (ex.iterations < 1 || ex.iterations > 8) fail(TSL_ERR_ARGUMENT, "iterations must be in 1..8");
  if (ex.tick_ns <= 0 || ex.bytes_per_unit <= 0) fail(TSL_ERR_ARGUMENT, "tick_ns and bytes_per_unit must be positive");
  if (jis.empty()) fail(TSL_ERR_ARGUMENT, "no job to replay");
  // the host issues the pool's frees at the plan's instants; with several
  // jobs contending for the channel the device's release ownership can drift
  // from them, so the pool-backed replay is a single-job replay
  if (ex.mempool && jis.size() != 1) fail(TSL_ERR_ARGUMENT, "mempool mode replays one job (tsl_execute_plan)");
  std::vector<JobProgram> progs;
  for (int32_t ji : jis) {
    if (ji < 0 || ji >= static_cast<int32_t>(r->jobs.size())) fail(TSL_ERR_ARGUMENT, "bad job index");
    progs.push_back(make_program(r->jobs[static_cast<size_t>(ji)], cfg, ex));
  }
  const int nj = static_cast<int>(progs.size());
  const int iters = ex.iterations;
  // device layout: the shared counters, then every job's block
  struct DevOff {
    size_t dev, ops, i32, i64, slot, res, ver, pend, opi, init, initsz, end, iter, pool, addr;
    size_t host;
  };
  const bool mp = ex.mempool != 0;
  Layout L;
  const size_t o_acct = L.take<ExecAcct>(1);
  std::vector<DevOff> dof(nj);
  int64_t host_total = 0;
  for (int j = 0; j < nj; ++j) {
    const JobProgram& P = progs[j];
    const int32_t T = P.g->T;
    DevOff& f = dof[j];
    f.dev = L.take<ExecDevice>(1);
    f.ops = L.take<ExecOp>(P.steps.size());
    f.i32 = L.take<int32_t>(P.i32.size() + 1);
    f.i64 = L.take<int64_t>(P.i64.size() + 1);
    f.slot = L.take<int64_t>(T);
    f.res = L.take<int32_t>(T);
    f.ver = L.take<int32_t>(T);
    f.pend = L.take<int32_t>(T);
    f.opi = L.take<int32_t>(T);
    f.init = L.take<int32_t>(P.init_st.size() + 1);
    f.initsz = L.take<int64_t>(P.init_sz.size() + 1);
    f.end = L.take<uint64_t>(size_t(iters) * P.steps.size() + 1);
    f.iter = L.take<uint64_t>(iters + 1);
    f.addr = L.take<uint8_t*>(T + 1);  // mempool mode: each storage's current allocation
    f.host = static_cast<size_t>(host_total);
    host_total += P.host_bytes;
  }
  const size_t meta_end = L.off;  // staged by the host
  // fixed slots (mempool mode: the pool holds the data, the slots are unused)
  for (int j = 0; j < nj; ++j) dof[j].pool = L.take<uint8_t>(mp ? 256 : progs[j].pool_bytes + 256);
  const size_t total = L.off;
  uint8_t* dbuf = nullptr;
  uint8_t* hpin = nullptr;
  std::vector<uint8_t> stage(meta_end, 0);
  std::vector<cudaEvent_t> events;
  std::vector<cudaStream_t> cs(nj, nullptr);
  cudaStream_t xs_stream = nullptr;
  // mempool mode: a private pool, every storage's live allocation on the host
  // side, and pinned cells holding the pointer values the device table is fed
  // from in stream order (one cell per allocation event)
  cudaMemPool_t mpool = nullptr;
  std::vector<std::vector<void*>> live(nj);
  int64_t* hptr = nullptr;
  size_t nptr = 0, ptr_cap = 0;
  int64_t n_alloc = 0;
  auto cleanup = [&]() {
    if (mpool) {
      for (auto c : cs) if (c) cudaStreamSynchronize(c);
      if (xs_stream) cudaStreamSynchronize(xs_stream);
      for (auto& v : live)
        for (void* p : v) if (p) cudaFree(p);
      cudaMemPoolDestroy(mpool);
      mpool = nullptr;
    }
    for (auto e : events) cudaEventDestroy(e);
    for (auto c : cs) if (c) cudaStreamDestroy(c);
    if (xs_stream) cudaStreamDestroy(xs_stream);
    if (dbuf) cudaFree(dbuf);
    if (hpin) cudaFreeHost(hpin);
    if (hptr) cudaFreeHost(hptr);
  };
  per.assign(nj, tsl_exec_report{});
  merged = tsl_exec_report{};
  try {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&dbuf), total), "cudaMalloc");
    cuda_check(cudaMallocHost(reinterpret_cast<void**>(&hpin), std::max<int64_t>(host_total, 256)), "cudaMallocHost");
    for (auto& c : cs) cuda_check(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&xs_stream, cudaStreamNonBlocking), "stream");
    auto D = [&](size_t off) { return dbuf + off; };
    if (mp) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = ctx->device;
      cuda_check(cudaMemPoolCreate(&mpool, &props), "cudaMemPoolCreate");
      uint64_t keep = ~uint64_t(0), zero = 0;
      cuda_check(cudaMemPoolSetAttribute(mpool, cudaMemPoolAttrReleaseThreshold, &keep), "pool attr");
      cuda_check(cudaMemPoolSetAttribute(mpool, cudaMemPoolAttrUsedMemHigh, &zero), "pool attr");
      cuda_check(cudaMemPoolSetAttribute(mpool, cudaMemPoolAttrReservedMemHigh, &zero), "pool attr");
      for (int j = 0; j < nj; ++j) {
        live[j].assign(progs[j].g->T, nullptr);
        ptr_cap += progs[j].init_st.size() + size_t(iters) * (progs[j].steps.size() * 4 + progs[j].xs.size() + 1);
        for (const auto& st : progs[j].steps) ptr_cap += size_t(iters) * st.outs.size();
      }
      cuda_check(cudaMallocHost(reinterpret_cast<void**>(&hptr), (ptr_cap + 1) * sizeof(int64_t)), "cudaMallocHost");
    }
    std::vector<ExecDevice*> dptr(nj);
    for (int j = 0; j < nj; ++j) {
      const JobProgram& P = progs[j];
      const DevOff& f = dof[j];
      ExecDevice dev{};
      dev.acct = reinterpret_cast<ExecAcct*>(D(o_acct));
      dev.tick_ns = static_cast<uint64_t>(ex.tick_ns);
      dev.pool = D(f.pool);
      dev.slot_off = reinterpret_cast<const int64_t*>(D(f.slot));
      dev.resident = reinterpret_cast<int32_t*>(D(f.res));
      dev.version = reinterpret_cast<int32_t*>(D(f.ver));
      dev.out_pending = reinterpret_cast<int32_t*>(D(f.pend));
      dev.op_end_ns = reinterpret_cast<uint64_t*>(D(f.end));
      dev.iter_start_ns = reinterpret_cast<uint64_t*>(D(f.iter));
      dev.addr = mp ? reinterpret_cast<uint8_t**>(D(f.addr)) : nullptr;
      std::memcpy(stage.data() + f.dev, &dev, sizeof dev);
      for (size_t k = 0; k < P.steps.size(); ++k) {
        ExecOp op{};
        op.index = static_cast<int32_t>(k);
        op.ticks = P.steps[k].ticks;
        op.start = P.steps[k].start;
        op.n_in = static_cast<int32_t>(P.steps[k].ins.size());
        op.n_out = static_cast<int32_t>(P.steps[k].outs.size());
        op.n_rel = static_cast<int32_t>(P.steps[k].rel.size());
        op.ins = reinterpret_cast<const int32_t*>(D(f.i32)) + P.offs[k].ins;
        op.outs = reinterpret_cast<const int32_t*>(D(f.i32)) + P.offs[k].outs;
        op.rel = reinterpret_cast<const int32_t*>(D(f.i32)) + P.offs[k].rel;
        op.out_size = reinterpret_cast<const int64_t*>(D(f.i64)) + P.offs[k].osz;
        op.rel_size = reinterpret_cast<const int64_t*>(D(f.i64)) + P.offs[k].rsz;
        std::memcpy(stage.data() + f.ops + k * sizeof(ExecOp), &op, sizeof op);
      }
      if (!P.i32.empty()) std::memcpy(stage.data() + f.i32, P.i32.data(), P.i32.size() * 4);
      if (!P.i64.empty()) std::memcpy(stage.data() + f.i64, P.i64.data(), P.i64.size() * 8);
      std::memcpy(stage.data() + f.slot, P.slot_off.data(), P.slot_off.size() * 8);
      std::memcpy(stage.data() + f.opi, P.outs_per_iter.data(), P.outs_per_iter.size() * 4);
      if (!P.init_st.empty()) std::memcpy(stage.data() + f.init, P.init_st.data(), P.init_st.size() * 4);
      if (!P.init_sz.empty()) std::memcpy(stage.data() + f.initsz, P.init_sz.data(), P.init_sz.size() * 8);
      dptr[j] = reinterpret_cast<ExecDevice*>(D(f.dev));
    }
    // mempool mode: the initially resident storages' allocations (stream
    // ordered before each job's init kernel), their pointers staged into the
    // device address tables
    auto mp_alloc = [&](int j, int32_t s, int64_t units, cudaStream_t st) -> void* {
      void* p = nullptr;
      cuda_check(cudaMallocFromPoolAsync(&p, size_t(units * ex.bytes_per_unit), mpool, st), "cudaMallocFromPoolAsync");
      live[j][s] = p;
      ++n_alloc;
      return p;
    };
    if (mp)
      for (int j = 0; j < nj; ++j)
        for (size_t k = 0; k < progs[j].init_st.size(); ++k) {
          void* p = mp_alloc(j, progs[j].init_st[k], progs[j].init_sz[k], cs[j]);
          std::memcpy(stage.data() + dof[j].addr + sizeof(void*) * size_t(progs[j].init_st[k]), &p, sizeof p);
        }
    cuda_check(cudaMemcpy(dbuf, stage.data(), meta_end, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemset(D(dof[0].pool), 0, total - dof[0].pool), "memset");
    auto ev = [&]() {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      events.push_back(e);
      return e;
    };
    int kernels = 0;
    // per job: initial residency and host tags, then the replay's events
    struct JobRun {
      std::vector<cudaEvent_t> op_end, in_done;
      cudaEvent_t it_start, xfer_tail;
    };
    std::vector<JobRun> run(nj);
    std::vector<cudaEvent_t> readies;
    for (int j = 0; j < nj; ++j) {
      const JobProgram& P = progs[j];
      cuda_check(exec_launch_init(dptr[j], reinterpret_cast<const int32_t*>(D(dof[j].init)),
                                  reinterpret_cast<const int64_t*>(D(dof[j].initsz)),
                                  static_cast<int>(P.init_st.size()), cs[j]), "init");
      ++kernels;
      for (int32_t s : P.wrapped_in) {
        cuda_check(exec_launch_host_tag(dptr[j], s, hpin + dof[j].host + P.host_off[s], cs[j]), "host tag");
        ++kernels;
      }
      cudaEvent_t ready = ev();
      cuda_check(cudaEventRecord(ready, cs[j]), "event");
      cuda_check(cudaStreamWaitEvent(xs_stream, ready, 0), "wait");
      readies.push_back(ready);
      run[j].op_end.resize(P.steps.size());
      for (auto& e : run[j].op_end) e = ev();
      run[j].in_done.resize(P.xs.size());
      for (auto& e : run[j].in_done) e = ev();
      run[j].it_start = ev();
      run[j].xfer_tail = ev();
    }
    // every job starts once every job's initial state is on the device
    for (int j = 0; j < nj; ++j)
      for (auto e : readies) cuda_check(cudaStreamWaitEvent(cs[j], e, 0), "wait");
    // each job's action list in its single-job order, with planned global times
    enum { A_BEGIN, A_XFER, A_OP, A_END };
    struct Act { int kind; int it; int idx; int64_t time; };
    std::vector<std::vector<Act>> acts(nj);
    for (int j = 0; j < nj; ++j) {
      const JobProgram& P = progs[j];
      const int32_t nsteps = static_cast<int32_t>(P.steps.size());
      for (int it = 0; it < iters; ++it) {
        const int64_t base = int64_t(it) * P.period;
        acts[j].push_back({A_BEGIN, it, -1, base});
        size_t xi = 0;
        for (int32_t k = 0; k < nsteps; ++k) {
          while (xi < P.xs.size() && P.xs[xi].arrival <= P.steps[static_cast<size_t>(k)].start && P.xs[xi].anchor < k) {
            acts[j].push_back({A_XFER, it, static_cast<int>(xi), base + P.xs[xi].arrival});
            ++xi;
          }
          acts[j].push_back({A_OP, it, k, base + P.steps[static_cast<size_t>(k)].start});
        }
        for (; xi < P.xs.size(); ++xi) acts[j].push_back({A_XFER, it, static_cast<int>(xi), base + P.xs[xi].arrival});
        acts[j].push_back({A_END, it, -1, base + P.period});
      }
    }
    // mempool mode: every transfer's planned completion on the shared FIFO
    // channel (enqueue order = the merged action order below), so the host
    // frees a released storage exactly when the device's release does -- not
    // while a swap-out of it is still pending (simulator.cpp:461-470)
    std::vector<std::vector<std::vector<int64_t>>> done_at(nj);
    if (mp) {
      std::vector<std::tuple<int64_t, int, int, int>> q;  // (time, job, iteration, transfer)
      for (int j = 0; j < nj; ++j) {
        done_at[j].assign(iters, std::vector<int64_t>(progs[j].xs.size(), 0));
        for (const Act& a : acts[j])
          if (a.kind == A_XFER) q.emplace_back(a.time, j, a.it, a.idx);
      }
      std::stable_sort(q.begin(), q.end(), [](const auto& a, const auto& b) {
        return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b) : std::get<1>(a) < std::get<1>(b);
      });
      int64_t chan = 0;
      for (const auto& [t, j, it, xi] : q) {
        chan = std::max(chan, t) + progs[j].xs[size_t(xi)].dur;
        done_at[j][it][size_t(xi)] = chan;
      }
      // The pool accounts allocations and frees in the order the host issues
      // them, so they are issued in the replay's planned time order: a
      // transfer's action moves to its planned channel start (where a swap-in
      // allocates), frees wait in a queue until the timeline reaches their
      // instant (op end / swap-out completion), frees before allocations at
      // equal ticks (simulator.cpp:47-52).
      for (int j = 0; j < nj; ++j) {
        for (Act& a : acts[j])
          if (a.kind == A_XFER) a.time = done_at[j][a.it][size_t(a.idx)] - progs[j].xs[size_t(a.idx)].dur;
        std::stable_sort(acts[j].begin(), acts[j].end(), [](const Act& x, const Act& y) {
          const int px = x.kind == A_END ? 1 : 0, py = y.kind == A_END ? 1 : 0;
          return x.time != y.time ? x.time < y.time : px < py;
        });
      }
    }
    struct PendingFree { int64_t time; uint64_t seq; int j; int32_t s; cudaStream_t st; };
    auto later = [](const PendingFree& a, const PendingFree& b) {
      return a.time != b.time ? a.time > b.time : a.seq > b.seq;
    };
    std::priority_queue<PendingFree, std::vector<PendingFree>, decltype(later)> frees(later);
    uint64_t free_seq = 0;
    auto flush_frees = [&](int64_t upto) {
      while (!frees.empty() && frees.top().time <= upto) {
        const PendingFree f = frees.top();
        frees.pop();
        if (!live[f.j][f.s]) continue;
        cuda_check(cudaFreeAsync(live[f.j][f.s], f.st), "cudaFreeAsync");
        live[f.j][f.s] = nullptr;
      }
    };
    auto set_addr = [&](int j, int32_t s, void* p, cudaStream_t st) {
      if (nptr >= ptr_cap) fail(TSL_ERR_INTERNAL, "mempool pointer cells exhausted");
      hptr[nptr] = reinterpret_cast<int64_t>(p);
      cuda_check(cudaMemcpyAsync(D(dof[j].addr) + sizeof(void*) * size_t(s), &hptr[nptr], sizeof(void*),
                                 cudaMemcpyHostToDevice, st), "H2D addr");
      ++nptr;
    };
    // merge the jobs' lists by planned time (ties: job order); enqueue
    std::vector<size_t> head(nj, 0);
    std::vector<std::vector<char>> enq(nj);
    for (int j = 0; j < nj; ++j) enq[j].assign(progs[j].xs.size(), 0);
    for (;;) {
      int bj = -1;
      for (int j = 0; j < nj; ++j)
        if (head[j] < acts[j].size() && (bj < 0 || acts[j][head[j]].time < acts[bj][head[bj]].time)) bj = j;
      if (bj < 0) break;
      const Act a = acts[bj][head[bj]++];
      if (mp) flush_frees(a.time);
      const JobProgram& P = progs[bj];
      JobRun& R = run[bj];
      ExecDevice* d = dptr[bj];
      const int nsteps = static_cast<int>(P.steps.size());
      const int base = a.it * nsteps;
      if (a.kind == A_BEGIN) {
        std::fill(enq[bj].begin(), enq[bj].end(), 0);
        cuda_check(exec_launch_iter_begin(d, reinterpret_cast<const int32_t*>(D(dof[bj].opi)), P.g->T, a.it, cs[bj]),
                   "iter");
        ++kernels;
        cuda_check(cudaEventRecord(R.it_start, cs[bj]), "event");
      } else if (a.kind == A_XFER) {
        const ExecXferH& t = P.xs[static_cast<size_t>(a.idx)];
        cuda_check(cudaStreamWaitEvent(xs_stream, t.anchor < 0 ? R.it_start : R.op_end[static_cast<size_t>(t.anchor)], 0),
                   "wait");
        cuda_check(exec_launch_delay(d, t.anchor < 0 ? -1 : base + t.anchor, a.it, t.delta, xs_stream), "delay");
        const size_t nbytes = static_cast<size_t>(t.size * ex.bytes_per_unit);
        uint8_t* dev_slot = D(dof[bj].pool) + P.slot_off[t.storage];
        uint8_t* host_slot = hpin + dof[bj].host + P.host_off[t.storage];
        if (mp && t.dir == 1 && !live[bj][t.storage]) {  // a swap-in allocates before its copy
          void* p = mp_alloc(bj, t.storage, t.size, xs_stream);
          set_addr(bj, t.storage, p, xs_stream);
        }
        if (mp) dev_slot = static_cast<uint8_t*>(live[bj][t.storage]);
        if (t.dir == 0) {
          if (dev_slot) cuda_check(cudaMemcpyAsync(host_slot, dev_slot, nbytes, cudaMemcpyDeviceToHost, xs_stream), "D2H");
          per[bj].bytes_d2h += static_cast<int64_t>(nbytes);
        } else {
          cuda_check(cudaMemcpyAsync(dev_slot, host_slot, nbytes, cudaMemcpyHostToDevice, xs_stream), "H2D");
          per[bj].bytes_h2d += static_cast<int64_t>(nbytes);
        }
        cuda_check(exec_launch_done(d, t.storage, t.size, t.dur, t.dir, xs_stream), "done");
        kernels += 2;
        if (mp && t.dir == 0)  // a completed swap-out frees (queued to its completion instant)
          frees.push({done_at[bj][a.it][size_t(a.idx)], free_seq++, bj, t.storage, xs_stream});
        if (t.dir == 1) cuda_check(cudaEventRecord(R.in_done[static_cast<size_t>(a.idx)], xs_stream), "event");
        enq[bj][static_cast<size_t>(a.idx)] = 1;
      } else if (a.kind == A_OP) {
        for (size_t q = 0; q < P.xs.size(); ++q)  // swap-ins serving this step, already on the channel
          if (P.xs[q].serve_step == a.idx && enq[bj][q]) cuda_check(cudaStreamWaitEvent(cs[bj], R.in_done[q], 0), "wait");
        const ExecStepH& stp = P.steps[static_cast<size_t>(a.idx)];
        if (mp)  // outputs allocate at the op's start
          for (size_t k = 0; k < stp.outs.size(); ++k)
            if (stp.out_size[k] > 0 && !live[bj][stp.outs[k]]) {
              void* p = mp_alloc(bj, stp.outs[k], stp.out_size[k], cs[bj]);
              set_addr(bj, stp.outs[k], p, cs[bj]);
            }
        cuda_check(exec_launch_op(d, reinterpret_cast<const ExecOp*>(D(dof[bj].ops)) + a.idx, base, a.it, cs[bj]), "op");
        ++kernels;
        cuda_check(cudaEventRecord(R.op_end[static_cast<size_t>(a.idx)], cs[bj]), "event");
        if (mp) {  // releases at its end, unless a swap-out of the storage is still pending
          const int64_t end_t = int64_t(a.it) * P.period + stp.end;
          for (int32_t s : stp.rel) {
            bool owned = false;
            for (size_t q = 0; q < P.xs.size() && !owned; ++q)
              owned = P.xs[q].dir == 0 && P.xs[q].storage == s && done_at[bj][a.it][q] > end_t;
            if (!owned) frees.push({end_t, free_seq++, bj, s, cs[bj]});
          }
        }
      } else {
        // the iteration ends when its transfers are done (simulator.cpp:478-484)
        cuda_check(cudaEventRecord(R.xfer_tail, xs_stream), "event");
        cuda_check(cudaStreamWaitEvent(cs[bj], R.xfer_tail, 0), "wait");
        if (nj == 1)  // a lone job's channel also waits for its iteration (the channel is its own)
          cuda_check(cudaStreamWaitEvent(xs_stream, R.op_end[static_cast<size_t>(nsteps - 1)], 0), "wait");
      }
    }
    if (mp) flush_frees(std::numeric_limits<int64_t>::max());
    for (int j = 0; j < nj; ++j) {
      cuda_check(exec_launch_iter_begin(dptr[j], reinterpret_cast<const int32_t*>(D(dof[j].opi)), 0, iters, cs[j]),
                 "iter");
      ++kernels;
    }
    for (auto c : cs) cuda_check(cudaStreamSynchronize(c), "sync");
    cuda_check(cudaStreamSynchronize(xs_stream), "sync");
    int64_t pool_used = 0, pool_reserved = 0;
    if (mp) {
      uint64_t v = 0;
      cuda_check(cudaMemPoolGetAttribute(mpool, cudaMemPoolAttrUsedMemHigh, &v), "pool attr");
      pool_used = int64_t(v);
      cuda_check(cudaMemPoolGetAttribute(mpool, cudaMemPoolAttrReservedMemHigh, &v), "pool attr");
      pool_reserved = int64_t(v);
    }
    ExecAcct acct{};
    cuda_check(cudaMemcpy(&acct, D(o_acct), sizeof acct, cudaMemcpyDeviceToHost), "D2H");
    for (int j = 0; j < nj; ++j) {
      const JobProgram& P = progs[j];
      ExecDevice out{};
      cuda_check(cudaMemcpy(&out, dptr[j], sizeof out, cudaMemcpyDeviceToHost), "D2H");
      std::vector<uint64_t> starts(iters + 1);
      cuda_check(cudaMemcpy(starts.data(), D(dof[j].iter), starts.size() * 8, cudaMemcpyDeviceToHost), "D2H");
      tsl_exec_report& rep = per[j];
      rep.predicted_peak = ex.vanilla ? -1 : P.o->st.peak;  // vanilla: no per-job prediction in the result
      rep.hwm = out.hwm;
      rep.final_footprint = out.footprint;
      rep.iterations = iters;
      for (int it = 0; it < iters; ++it) rep.iteration_ms[it] = double(starts[it + 1] - starts[it]) / 1e6;
      rep.planned_iteration_ms = double(P.period) * double(ex.tick_ns) / 1e6;
      rep.swap_outs = out.n_out;
      rep.swap_ins = out.n_in;
      rep.verify_errors = out.verify_errors;
      rep.violations = out.violations;
      if (!ex.vanilla) merged.predicted_peak += rep.predicted_peak;
      merged.swap_outs += rep.swap_outs;
      merged.swap_ins += rep.swap_ins;
      merged.bytes_d2h += rep.bytes_d2h;
      merged.bytes_h2d += rep.bytes_h2d;
      merged.verify_errors += rep.verify_errors;
      merged.violations += rep.violations;
      merged.planned_iteration_ms = std::max(merged.planned_iteration_ms, rep.planned_iteration_ms);
      for (int it = 0; it < iters; ++it) merged.iteration_ms[it] = std::max(merged.iteration_ms[it], rep.iteration_ms[it]);
    }
    if (ex.vanilla)  // the release-at-last-use plan's merged peak: the history's first entry
      merged.predicted_peak = r->history.empty() ? -1 : r->history[0];
    merged.hwm = acct.hwm;
    merged.final_footprint = acct.footprint;
    merged.iterations = iters;
    merged.kernels = kernels;
    merged.pool_used_hwm = pool_used;
    merged.pool_reserved_hwm = pool_reserved;
    merged.pool_allocs = n_alloc;
    for (auto& rep : per) {
      rep.kernels = kernels;
      rep.pool_used_hwm = pool_used;
      rep.pool_reserved_hwm = pool_reserved;
      rep.pool_allocs = n_alloc;
    }
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  merged.total_ms = ms;
  for (auto& rep : per) rep.total_ms = ms;
}

tsl_exec_report execute(tsl_ctx* ctx, const tsl_result* r, int32_t ji, const tsl_config& cfg,
                        const tsl_exec_config& ex) {
  std::vector<tsl_exec_report> per;
  tsl_exec_report merged{};
  execute_jobs(ctx, r, {ji}, cfg, ex, per, merged);
  return per[0];
}

}  // namespace

extern "C" {

void tsl_exec_config_default(tsl_exec_config* c) {
  c->tick_ns = 1000;
  c->iterations = 3;
  c->bytes_per_unit = 16;
  c->vanilla = 0;
  c->mempool = 0;
}

int tsl_execute_plan(tsl_ctx* ctx, const tsl_result* r, int32_t job, const tsl_config* cfg,
                     const tsl_exec_config* ex, tsl_exec_report* out) {
  if (!ctx || !r || !cfg || !ex || !out) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] { *out = execute(ctx, r, job, *cfg, *ex); });
}

int tsl_execute_plans(tsl_ctx* ctx, const tsl_result* r, const tsl_config* cfg, const tsl_exec_config* ex,
                      tsl_exec_report* per_job, tsl_exec_report* merged) {
  if (!ctx || !r || !cfg || !ex || !per_job || !merged) { g_err = "null argument"; return TSL_ERR_ARGUMENT; }
  return guard([&] {
    std::vector<int32_t> jis(r->jobs.size());
    for (size_t k = 0; k < jis.size(); ++k) jis[k] = static_cast<int32_t>(k);
    std::vector<tsl_exec_report> per;
    execute_jobs(ctx, r, jis, *cfg, *ex, per, *merged);
    for (size_t k = 0; k < per.size(); ++k) per_job[k] = per[k];
  });
}

}  // extern "C"
