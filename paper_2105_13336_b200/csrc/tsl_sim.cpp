// Tick-level model of the plan executor: the reference's discrete-event
// simulator (simulator.cpp:26-569, simulate :573-582, compute_metrics
// :598-632) in its three modes -- vanilla (release at last use), scheduled
// (the plan's swap / recompute events drive one FIFO transfer channel, with
// passive fetches as fallback) and passive (LRU eviction under the memory
// budget, every miss fetched on demand) -- plus the SimController hook that
// installs re-planned SchedulingPlans at iteration boundaries
// (simulator.hpp:73-79; Orchestrator::replan_if_needed drives it).
//
// It is the planner's host runtime around the device: the trace it produces
// (footprint curves, blocked ticks, transfers, passive fetches, safety
// violations, plan versions) is the reference's SimulationTrace, compared
// value for value with the reference in tests/test_sim.py; the device replay
// (tsl_exec.cu) executes such a schedule with real copies and allocations.
//
// Everything runs over dense indices: job / tensor / op ids become the
// lexicographic ranks the reference's std::string comparisons induce.
#include <array>
#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "tensile_b200.h"
#include "tsl_graph.h"

using namespace tsl::hostg;

namespace {

enum : int { M_VANILLA = 0, M_SCHEDULED = 1, M_PASSIVE = 2 };
// Event kinds in dispatch order at one tick (simulator.cpp:48-56): op
// completions first, so their releases land before same-tick allocations.
enum : int { E_OP = 0, E_XFER_DONE = 1, E_XFER_ARRIVE = 2, E_LAUNCH = 3 };
enum : int { X_OUT = 0, X_IN = 1, X_PASSIVE = 2 };
const char* const kXferName[] = {"swap_out", "swap_in", "passive_swap_in"};

struct SwapEv {
  int32_t storage;  // the event's tensor, resolved to its storage root
  int8_t dir;       // 0 out, 1 in
  int8_t wraps;
  int64_t trigger;  // access id or -1 (iteration start)
  int64_t delta;
};

struct Plan {  // SchedulingPlan (plan.hpp:46-53) as the executor reads it
  std::vector<SwapEv> swaps;
  std::vector<std::array<int64_t, 3>> rcs;  // (tensor, target access, regen op)
  std::vector<char> release;                // by access id
  int64_t version = 0;
};

struct Step {
  int32_t op;
  bool recompute;
  std::vector<int64_t> accesses;               // the op's access ids (empty for recomputes)
  std::vector<int32_t> inputs;                 // input storages, op.inputs order
  std::vector<std::pair<int32_t, int64_t>> allocs;  // (storage, size)
};

struct Xfer {
  int32_t job, storage;
  int64_t size, duration, arrival;
  uint64_t seq;
  int kind;
};

struct Event {
  int64_t tick;
  int kind;
  int32_t job_rank;  // the reference breaks ties on the job id string
  uint64_t seq;
  int32_t job;
  int64_t payload;
  bool operator>(const Event& o) const {
    if (tick != o.tick) return tick > o.tick;
    if (kind != o.kind) return kind > o.kind;
    if (job_rank != o.job_rank) return job_rank > o.job_rank;
    return seq > o.seq;
  }
};

enum class S { NotLaunched, Ready, WaitingInputs, Running, IterEndWait, Finished };

struct Job {
  int32_t index = 0, rank = 0;
  std::shared_ptr<const Graph> g;
  int64_t launch_tick = 0;
  // access sequence under the true latencies (access.cpp:28-59)
  std::vector<int32_t> a_tensor, a_op;
  std::vector<std::vector<int64_t>> op_acc;
  Plan plan;
  bool has_pending = false;
  Plan pending;
  std::vector<Step> steps;
  std::map<int64_t, std::vector<SwapEv>> triggered;
  std::vector<SwapEv> iter_start;
  std::vector<int32_t> outs_per_iter, outs_remaining;  // by storage
  S state = S::NotLaunched;
  size_t step_idx = 0;
  int iteration = 0;
  int64_t iter_start_tick = 0, wait_start = 0;
  int outstanding = 0;
  std::vector<int32_t> pending_in;         // by storage
  std::vector<int64_t> observed;           // by op, -1: not run this iteration
  std::vector<char> resident, host, pinned;
  std::vector<int64_t> last_use;           // by storage, -1: never (reads as 0)
  int64_t footprint = 0;
};

struct Row {
  int64_t tick;
  int32_t job;
  const char* kind;
  int32_t tensor;  // -1: none
  int64_t footprint;      // global, after the event
  int64_t job_footprint;  // the job's, after the event
};

}  // namespace

struct tsl_sim {
  // inputs
  std::vector<Job> jobs;
  int mode = M_VANILLA;
  int iterations = 1;
  int64_t tick_limit = 10000000;
  int64_t budget = 0, bw = 1, setup = 0;
  std::vector<std::pair<int32_t, double>> slowdown;  // ascending job counts
  tsl_sim_controller_fn ctrl = nullptr;
  void* user = nullptr;
  std::vector<int32_t> name_rank;  // global tensor-name rank of (job, tensor): LRU ties
  std::vector<int32_t> name_base;  // per job offset into name_rank
  // engine
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> events;
  std::vector<Xfer> xfers;
  std::set<std::tuple<int64_t, int32_t, uint64_t, int64_t>> channel;  // (arrival, job rank, seq, xfer)
  bool busy = false;
  int64_t current = 0;
  uint64_t next_seq = 0;
  int64_t now = 0, global_fp = 0, peak = 0;
  int active = 0;
  // trace (SimulationTrace, simulator.hpp:51-68)
  std::vector<Row> rows;
  std::vector<std::vector<int64_t>> iteration_times, plan_versions;
  std::vector<int64_t> per_job_peak;
  int64_t passive_count = 0, blocked = 0;
  struct XferRow { int64_t start, end; int32_t job, storage; int kind; };
  std::vector<XferRow> transfers;
  std::vector<std::string> violations;
  std::vector<std::tuple<int32_t, int32_t, int32_t>> passive_events;  // (job, iteration, storage)
  bool in_controller = false;
};

namespace {

int64_t transfer_duration(int64_t size, int64_t bw, int64_t setup) {  // plan.cpp:22-28
  if (bw <= 0) fail(TSL_ERR_VALIDATION, "bandwidth must be positive");
  if (setup < 0) fail(TSL_ERR_VALIDATION, "setup cost must be nonnegative");
  return (size + bw - 1) / bw + setup;
}

double slowdown_of(const tsl_sim& m, int n) {  // SimConfig::slowdown
  double mult = 1.0;
  for (const auto& [count, v] : m.slowdown)
    if (count <= n) mult = v;
  return mult;
}

const std::string& tname(const Job& js, int32_t t) { return js.g->tid[t]; }

void record(tsl_sim& m, Job& js, const char* kind, int32_t tensor) {
  m.rows.push_back({m.now, js.index, kind, tensor, m.global_fp, js.footprint});
  if (m.global_fp > m.peak) m.peak = m.global_fp;
  m.per_job_peak[js.index] = std::max(m.per_job_peak[js.index], js.footprint);
}

void free_storage(tsl_sim& m, Job& js, int32_t s, const char* kind) {
  if (!js.resident[s]) {
    if (js.host[s]) { js.host[s] = 0; return; }
    m.violations.push_back("double release of " + tname(js, s) + " in job " + js.g->job_id);
    return;
  }
  const int64_t size = js.g->size[s];
  js.resident[s] = 0;
  js.footprint -= size;
  m.global_fp -= size;
  record(m, js, kind, s);
}

// LRU eviction across every job until `incoming` fits under the budget
// (simulator.cpp:270-291): the least recently used unpinned resident storage,
// ties to the smaller storage id (then the earlier job).
void evict_for(tsl_sim& m, int64_t incoming) {
  while (m.global_fp + incoming > m.budget) {
    int32_t vj = -1, vs = -1;
    int64_t oldest = std::numeric_limits<int64_t>::max();
    int32_t vname = 0;
    for (auto& js : m.jobs) {
      const int32_t T = js.g->T;
      for (int32_t s = 0; s < T; ++s) {
        if (!js.resident[s] || js.pinned[s]) continue;
        const int64_t used = js.last_use[s] < 0 ? 0 : js.last_use[s];
        const int32_t nm = m.name_rank[m.name_base[js.index] + s];
        if (used < oldest || (used == oldest && vj >= 0 && nm < vname)) {
          oldest = used;
          vj = js.index;
          vs = s;
          vname = nm;
        }
      }
    }
    if (vj < 0) break;  // nothing evictable: run over budget
    Job& v = m.jobs[vj];
    v.host[vs] = 1;
    free_storage(m, v, vs, "evict");
  }
}

void alloc(tsl_sim& m, Job& js, int32_t s, int64_t size, const char* kind) {
  if (js.resident[s]) return;
  if (m.mode == M_PASSIVE) evict_for(m, size);
  js.resident[s] = 1;
  js.footprint += size;
  m.global_fp += size;
  js.last_use[s] = m.now;
  record(m, js, kind, s);
}

void push(tsl_sim& m, int64_t tick, int kind, const Job& js, uint64_t seq, int64_t payload) {
  m.events.push(Event{tick, kind, js.rank, seq, js.index, payload});
}

// Step list, trigger map and per-iteration swap-out counts for the job's
// current plan (simulator.cpp:157-225).
void prepare(tsl_sim& m, Job& js) {
  const Graph& g = *js.g;
  js.steps.clear();
  js.triggered.clear();
  js.iter_start.clear();
  std::fill(js.outs_per_iter.begin(), js.outs_per_iter.end(), 0);
  std::vector<std::vector<int32_t>> rc_before(g.O);  // recompute events (plan order) before their target op
  for (size_t r = 0; r < js.plan.rcs.size(); ++r) {
    const int64_t tgt = js.plan.rcs[r][1];
    if (tgt < 0 || tgt >= int64_t(js.a_op.size())) fail(TSL_ERR_VALIDATION, "map::at");
    rc_before[js.a_op[tgt]].push_back(int32_t(r));
  }
  for (int32_t o : g.topo) {
    for (int32_t r : rc_before[o]) {
      const auto& ev = js.plan.rcs[r];
      const int32_t regen = int32_t(ev[2]);
      Step s{regen, true, {}, {}, {}};
      const int32_t st = g.store[ev[0]];
      for (int32_t i = g.in_off[regen]; i < g.in_off[regen + 1]; ++i) s.inputs.push_back(g.store[g.in[i]]);
      s.allocs.emplace_back(st, g.size[st]);
      js.steps.push_back(std::move(s));
    }
    Step s{o, false, js.op_acc[o], {}, {}};
    for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) s.inputs.push_back(g.store[g.in[i]]);
    for (int32_t i = g.out_off[o]; i < g.out_off[o + 1]; ++i) {
      const int32_t t = g.out[i];
      if (g.store[t] != t) continue;  // in-place update
      s.allocs.emplace_back(t, g.size[t]);
    }
    js.steps.push_back(std::move(s));
  }
  if (m.mode == M_SCHEDULED)
    for (const SwapEv& ev : js.plan.swaps) {
      if (ev.trigger == -1) js.iter_start.push_back(ev);
      else js.triggered[ev.trigger].push_back(ev);
      if (ev.dir == 0) js.outs_per_iter[ev.storage]++;
    }
}

void schedule_transfer(tsl_sim& m, Job& js, const SwapEv& ev) {
  Xfer t;
  t.job = js.index;
  t.storage = ev.storage;
  t.size = js.g->size[ev.storage];
  t.duration = transfer_duration(t.size, m.bw, m.setup);
  t.kind = ev.dir == 0 ? X_OUT : X_IN;
  t.arrival = m.now + ev.delta;
  t.seq = m.next_seq++;
  m.xfers.push_back(t);
  js.outstanding++;
  if (t.kind == X_IN) js.pending_in[t.storage]++;
  push(m, t.arrival, E_XFER_ARRIVE, js, t.seq, int64_t(m.xfers.size()) - 1);
}

void issue_passive(tsl_sim& m, Job& js, int32_t s) {
  Xfer t;
  t.job = js.index;
  t.storage = s;
  t.size = js.g->size[s];
  t.duration = transfer_duration(t.size, m.bw, m.setup);
  t.kind = X_PASSIVE;
  t.arrival = m.now;
  t.seq = m.next_seq++;
  m.xfers.push_back(t);
  js.outstanding++;
  js.pending_in[s]++;
  m.passive_count++;
  m.passive_events.emplace_back(js.index, js.iteration, s);
  // through the arrival event: this tick's channel dispatch may have run
  push(m, m.now, E_XFER_ARRIVE, js, t.seq, int64_t(m.xfers.size()) - 1);
  record(m, js, "passive_swap_in_issued", s);
}

void start_iteration(tsl_sim& m, Job& js) {
  js.iter_start_tick = m.now;
  js.step_idx = 0;
  js.outs_remaining = js.outs_per_iter;
  js.state = S::Ready;
  for (const SwapEv& ev : js.iter_start) schedule_transfer(m, js, ev);
}

void launch(tsl_sim& m, Job& js) {
  js.state = S::Ready;
  js.iteration = 0;
  m.active++;
  // parameters, inputs and outputs are resident from launch, except storages
  // with an across-iteration prefetch (they arrive through the channel);
  // the reference walks its catalog in tensor-id order
  const Graph& g = *js.g;
  std::vector<char> wrapped_in(g.T, 0);
  for (const SwapEv& ev : js.plan.swaps)
    if (ev.dir == 1 && ev.wraps) wrapped_in[ev.storage] = 1;
  std::vector<int32_t> by_name(g.T);
  for (int32_t t = 0; t < g.T; ++t) by_name[g.trank[t]] = t;
  for (int32_t t : by_name) {
    if (g.store[t] != t) continue;
    const int8_t k = g.kind[t];
    if (k != TSL_KIND_PARAMETER && k != TSL_KIND_INPUT && k != TSL_KIND_OUTPUT) continue;
    if (wrapped_in[t]) continue;
    alloc(m, js, t, g.size[t], "launch");
  }
  start_iteration(m, js);
}

void complete_iteration(tsl_sim& m, Job& js);

void try_start_step(tsl_sim& m, Job& js) {
  const Graph& g = *js.g;
  const Step& step = js.steps[js.step_idx];
  bool all = true;
  for (int32_t s : step.inputs) {
    if (js.resident[s]) continue;
    if (js.pending_in[s] > 0) { all = false; continue; }  // a prefetch or passive fetch is on the way
    if (js.host[s]) { issue_passive(m, js, s); all = false; continue; }
    // a lost tensor: logged, then materialized so the run reports every violation
    m.violations.push_back("read of non-resident tensor " + g.tid[s] + " without host copy, job " + g.job_id +
                           " op " + g.oid[step.op]);
    alloc(m, js, s, g.size[s], "error_materialize");
  }
  if (!all) {
    if (js.state != S::WaitingInputs) {
      js.state = S::WaitingInputs;
      js.wait_start = m.now;
    }
    return;
  }
  if (js.state == S::WaitingInputs) m.blocked += m.now - js.wait_start;
  js.state = S::Running;
  std::fill(js.pinned.begin(), js.pinned.end(), 0);
  for (int32_t s : step.inputs) js.pinned[s] = 1;
  for (const auto& a : step.allocs) js.pinned[a.first] = 1;
  // outputs occupy memory for the whole op execution, as in the analyzer
  for (const auto& a : step.allocs) alloc(m, js, a.first, a.second, step.recompute ? "recompute" : "tga");
  const int64_t base = g.lat[step.op];
  const int64_t dur = int64_t(std::llround(double(base) * slowdown_of(m, m.active)));
  js.observed[step.op] = dur;
  push(m, m.now + dur, E_OP, js, m.next_seq++, 0);
}

void finish_step(tsl_sim& m, Job& js) {
  const Step& step = js.steps[js.step_idx];
  for (int32_t s : step.inputs) js.last_use[s] = m.now;
  for (const auto& a : step.allocs) js.last_use[a.first] = m.now;
  std::fill(js.pinned.begin(), js.pinned.end(), 0);
  for (int64_t aid : step.accesses) {
    auto it = js.triggered.find(aid);
    if (it != js.triggered.end())
      for (const SwapEv& ev : it->second) schedule_transfer(m, js, ev);
  }
  for (int64_t aid : step.accesses) {
    if (!js.plan.release[aid]) continue;
    const int32_t s = js.g->store[js.a_tensor[aid]];
    if (js.outs_remaining[s] > 0) continue;  // the pending swap-out owns this eviction
    if (js.resident[s]) {
      js.host[s] = 0;  // a plain release drops the data
      free_storage(m, js, s, "release");
    }
  }
  js.step_idx++;
  if (js.step_idx < js.steps.size()) {
    js.state = S::Ready;
    try_start_step(m, js);
    return;
  }
  if (js.outstanding > 0) {
    js.state = S::IterEndWait;
    js.wait_start = m.now;
  } else {
    complete_iteration(m, js);
  }
}

void complete_iteration(tsl_sim& m, Job& js) {
  const int64_t elapsed = m.now - js.iter_start_tick;
  if (elapsed > m.tick_limit) fail(TSL_ERR_VALIDATION, "iteration tick limit exceeded for job " + js.g->job_id);
  m.iteration_times[js.index].push_back(elapsed);
  m.plan_versions[js.index].push_back(js.plan.version);
  if (m.ctrl) {
    m.in_controller = true;
    const int rc = m.ctrl(m.user, &m, js.index, js.iteration, js.observed.data());
    m.in_controller = false;
    if (rc) fail(rc, "sim controller failed: " + std::string(tsl_last_error()));
  }
  std::fill(js.observed.begin(), js.observed.end(), -1);
  js.iteration++;
  if (js.iteration >= m.iterations) {
    js.state = S::Finished;
    m.active--;
    record(m, js, "job_finished", -1);
    return;
  }
  if (js.has_pending) {
    js.plan = std::move(js.pending);
    js.has_pending = false;
    prepare(m, js);
  }
  start_iteration(m, js);
}

void finish_transfer(tsl_sim& m) {
  const Xfer t = m.xfers[m.current];
  m.busy = false;
  Job& js = m.jobs[t.job];
  js.outstanding--;
  if (t.kind == X_OUT) {
    js.host[t.storage] = 1;
    js.outs_remaining[t.storage]--;
    if (js.resident[t.storage]) free_storage(m, js, t.storage, "swap_out");
  } else {
    js.pending_in[t.storage]--;
    alloc(m, js, t.storage, t.size, t.kind == X_IN ? "swap_in" : "passive_swap_in");
  }
  if (js.state == S::IterEndWait && js.outstanding == 0) {
    m.blocked += m.now - js.wait_start;
    complete_iteration(m, js);
  }
}

void pump(tsl_sim& m) {
  // the channel: strict FIFO by arrival tick, ties by job then sequence
  if (!m.busy && !m.channel.empty()) {
    const int64_t best = std::get<3>(*m.channel.begin());
    m.channel.erase(m.channel.begin());
    m.busy = true;
    m.current = best;
    const Xfer& t = m.xfers[best];
    m.transfers.push_back({m.now, m.now + t.duration, t.job, t.storage, t.kind});
    push(m, m.now + t.duration, E_XFER_DONE, m.jobs[t.job], t.seq, best);
  }
  for (auto& js : m.jobs)
    if (js.state == S::Ready || js.state == S::WaitingInputs) try_start_step(m, js);
}

void run(tsl_sim& m) {
  for (auto& js : m.jobs) push(m, js.launch_tick, E_LAUNCH, js, m.next_seq++, 0);
  while (!m.events.empty()) {
    m.now = m.events.top().tick;
    // every event of this tick before new work: frees precede allocations
    while (!m.events.empty() && m.events.top().tick == m.now) {
      const Event e = m.events.top();
      m.events.pop();
      Job& js = m.jobs[e.job];
      switch (e.kind) {
        case E_LAUNCH: launch(m, js); break;
        case E_OP: finish_step(m, js); break;
        case E_XFER_ARRIVE: {
          const Xfer& t = m.xfers[e.payload];
          m.channel.insert({t.arrival, m.jobs[t.job].rank, t.seq, e.payload});
          break;
        }
        case E_XFER_DONE: finish_transfer(m); break;
      }
    }
    pump(m);
  }
  for (const auto& js : m.jobs) {
    if (js.state == S::Finished) continue;
    std::string msg = "deadlock: job " + js.g->job_id + " stuck";
    if (js.state == S::WaitingInputs) msg += " waiting for inputs of step " + std::to_string(js.step_idx);
    else if (js.state == S::IterEndWait) msg += " waiting for " + std::to_string(js.outstanding) + " transfers";
    fail(TSL_ERR_VALIDATION, msg);
  }
}

Plan load_plan(const Job& js, const tsl_plan_desc* p) {
  Plan out;
  out.release.assign(js.a_tensor.size(), 0);
  if (!p) return out;
  const Graph& g = *js.g;
  for (int32_t i = 0; i < p->n_swap; ++i) {
    const int32_t t = p->ev_tensor[i];
    if (t < 0 || t >= g.T) fail(TSL_ERR_ARGUMENT, "swap event tensor out of range in job " + g.job_id);
    out.swaps.push_back(SwapEv{g.store[t], p->ev_dir[i], p->ev_wraps[i], p->ev_trigger[i], p->ev_delta[i]});
  }
  for (int32_t i = 0; i < p->n_recompute; ++i) {
    const int32_t t = p->rc_tensor[i], op = p->rc_regen_op[i];
    if (t < 0 || t >= g.T || op < 0 || op >= g.O)
      fail(TSL_ERR_ARGUMENT, "recompute event out of range in job " + g.job_id);
    out.rcs.push_back({t, p->rc_target[i], op});
  }
  for (int32_t i = 0; i < p->n_release; ++i) {
    const int64_t a = p->release_flags[i];
    if (a >= 0 && a < int64_t(out.release.size())) out.release[a] = 1;
  }
  out.version = p->version;
  return out;
}

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

std::string jstr(const std::string& s) {  // a JSON string literal
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else o += c;
  }
  return o + "\"";
}

}  // namespace

extern "C" {

int tsl_simulate(const tsl_job_desc* jobs, const int64_t* launch_ticks, int32_t n_jobs, const tsl_plan_desc* plans,
                 const tsl_sim_config* cfg, tsl_sim_controller_fn controller, void* user, tsl_sim** out) {
  if (!cfg || !out || (n_jobs > 0 && !jobs) || n_jobs < 0) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    auto m = std::make_unique<tsl_sim>();
    if (cfg->iterations < 1) fail(TSL_ERR_VALIDATION, "iterations must be at least 1");
    for (int32_t i = 0; i < cfg->n_slowdown; ++i)
      if (cfg->slowdown_mult[i] < 1.0) fail(TSL_ERR_VALIDATION, "slowdown multipliers must be >= 1");
    if (cfg->mode < M_VANILLA || cfg->mode > M_PASSIVE) fail(TSL_ERR_ARGUMENT, "unknown simulation mode");
    m->mode = cfg->mode;
    m->iterations = cfg->iterations;
    m->tick_limit = cfg->ticks_per_iteration_limit;
    m->budget = cfg->memory_budget;
    m->bw = cfg->pcie_bandwidth;
    m->setup = cfg->transfer_setup;
    {
      std::map<int32_t, double> curve;  // a repeated count keeps its last multiplier
      for (int32_t i = 0; i < cfg->n_slowdown; ++i) curve[cfg->slowdown_jobs[i]] = cfg->slowdown_mult[i];
      m->slowdown.assign(curve.begin(), curve.end());
    }
    m->ctrl = controller;
    m->user = user;
    std::vector<std::string> jids;
    for (int32_t k = 0; k < n_jobs; ++k) {
      Job js;
      js.index = k;
      js.g = std::make_shared<const Graph>(load_graph(jobs[k]));
      check_latencies(*js.g);
      js.launch_tick = launch_ticks ? launch_ticks[k] : 0;
      const Graph& g = *js.g;
      js.op_acc.assign(g.O, {});
      for (int32_t o : g.topo) {  // generate_access_sequence (access.cpp:42-54)
        for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) {
          js.op_acc[o].push_back(int64_t(js.a_tensor.size()));
          js.a_tensor.push_back(g.in[i]);
          js.a_op.push_back(o);
        }
        for (int32_t i = g.out_off[o]; i < g.out_off[o + 1]; ++i) {
          js.op_acc[o].push_back(int64_t(js.a_tensor.size()));
          js.a_tensor.push_back(g.out[i]);
          js.a_op.push_back(o);
        }
      }
      js.plan = load_plan(js, plans ? &plans[k] : nullptr);
      js.outs_per_iter.assign(g.T, 0);
      js.outs_remaining.assign(g.T, 0);
      js.pending_in.assign(g.T, 0);
      js.observed.assign(g.O, -1);
      js.resident.assign(g.T, 0);
      js.host.assign(g.T, 0);
      js.pinned.assign(g.T, 0);
      js.last_use.assign(g.T, -1);
      jids.push_back(g.job_id);
      m->jobs.push_back(std::move(js));
    }
    const std::vector<int32_t> jrank = lex_rank(jids);
    // one name order over every job's tensors (LRU ties compare storage ids
    // across jobs; equal ids keep the earlier job)
    std::vector<std::pair<const std::string*, int64_t>> names;
    for (auto& js : m->jobs) {
      js.rank = jrank[js.index];
      m->name_base.push_back(int32_t(names.size()));
      for (int32_t t = 0; t < js.g->T; ++t) names.emplace_back(&js.g->tid[t], int64_t(names.size()));
    }
    std::sort(names.begin(), names.end(), [](const auto& a, const auto& b) {
      const int c = a.first->compare(*b.first);
      return c != 0 ? c < 0 : a.second < b.second;
    });
    m->name_rank.assign(names.size(), 0);
    for (size_t r = 0; r < names.size(); ++r) m->name_rank[names[r].second] = int32_t(r);
    m->iteration_times.assign(n_jobs, {});
    m->plan_versions.assign(n_jobs, {});
    m->per_job_peak.assign(n_jobs, 0);
    for (auto& js : m->jobs) prepare(*m, js);
    run(*m);
    *out = m.release();
  });
}

int tsl_sim_set_plan(tsl_sim* m, int32_t job, const tsl_plan_desc* plan) {
  if (!m || !plan || job < 0 || job >= int32_t(m->jobs.size())) {
    set_last_error("null argument or job out of range");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    Job& js = m->jobs[job];
    js.pending = load_plan(js, plan);
    js.has_pending = true;
  });
}

int64_t tsl_sim_peak(const tsl_sim* m) { return m ? m->peak : 0; }

// SimulationTrace (simulator.hpp:51-68) as one JSON document: jobs in input
// order, names as the reference prints them.
char* tsl_sim_trace_json(const tsl_sim* m) {
  if (!m) return nullptr;
  std::string o = "{\"peak\": " + std::to_string(m->peak) + ", \"blocked_ticks\": " + std::to_string(m->blocked) +
                  ", \"passive_swap_count\": " + std::to_string(m->passive_count) + ", \"jobs\": [";
  for (size_t k = 0; k < m->jobs.size(); ++k) {
    const Job& js = m->jobs[k];
    if (k) o += ", ";
    o += "{\"job_id\": " + jstr(js.g->job_id) + ", \"peak\": " + std::to_string(m->per_job_peak[k]) +
         ", \"iteration_times\": [";
    for (size_t i = 0; i < m->iteration_times[k].size(); ++i)
      o += (i ? ", " : "") + std::to_string(m->iteration_times[k][i]);
    o += "], \"plan_versions\": [";
    for (size_t i = 0; i < m->plan_versions[k].size(); ++i)
      o += (i ? ", " : "") + std::to_string(m->plan_versions[k][i]);
    o += "], \"footprint_curve\": [";  // per_job_curve
    bool first = true;
    for (const Row& r : m->rows) {
      if (r.job != int32_t(k)) continue;
      o += (first ? "[" : ", [") + std::to_string(r.tick) + ", " + std::to_string(r.job_footprint) + "]";
      first = false;
    }
    o += "]}";
  }
  o += "], \"transfers\": [";
  for (size_t i = 0; i < m->transfers.size(); ++i) {
    const auto& t = m->transfers[i];
    o += (i ? ", [" : "[") + std::to_string(t.start) + ", " + std::to_string(t.end) + ", " +
         jstr(m->jobs[t.job].g->job_id) + ", " + jstr(m->jobs[t.job].g->tid[t.storage]) + ", " +
         jstr(kXferName[t.kind]) + "]";
  }
  o += "], \"safety_violations\": [";
  for (size_t i = 0; i < m->violations.size(); ++i) o += (i ? ", " : "") + jstr(m->violations[i]);
  o += "], \"passive_events\": [";
  for (size_t i = 0; i < m->passive_events.size(); ++i) {
    const auto& [j, it, s] = m->passive_events[i];
    o += (i ? ", [" : "[") + jstr(m->jobs[j].g->job_id) + ", " + std::to_string(it) + ", " +
         jstr(m->jobs[j].g->tid[s]) + "]";
  }
  o += "]}";
  char* p = static_cast<char*>(std::malloc(o.size() + 1));
  std::memcpy(p, o.c_str(), o.size() + 1);
  return p;
}

// SimulationTrace::to_csv (simulator.cpp:584-592): every row with the global
// footprint after it (the footprint curves are these rows' (tick, footprint)).
char* tsl_sim_trace_csv(const tsl_sim* m) {
  if (!m) return nullptr;
  std::string o = "tick,job_id,event_kind,tensor_id,footprint_bytes\n";
  o.reserve(o.size() + m->rows.size() * 40);
  for (const Row& r : m->rows) {
    const Job& js = m->jobs[r.job];
    o += std::to_string(r.tick);
    o += ',';
    o += js.g->job_id;
    o += ',';
    o += r.kind;
    o += ',';
    if (r.tensor >= 0) o += js.g->tid[r.tensor];
    o += ',';
    o += std::to_string(r.footprint);
    o += '\n';
  }
  char* p = static_cast<char*>(std::malloc(o.size() + 1));
  std::memcpy(p, o.c_str(), o.size() + 1);
  return p;
}

void tsl_sim_destroy(tsl_sim* m) { delete m; }

int tsl_base_release_flags(const tsl_job_desc* job, int64_t* out, int32_t cap, int32_t* n_out) {
  if (!job || !n_out) {
    set_last_error("null argument");
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] {
    const Graph g = load_graph(*job);
    // emission order (access.cpp:42-54), last access of each Interim tensor id
    std::vector<int64_t> last(g.T, -1);
    int64_t a = 0;
    for (int32_t o : g.topo) {
      for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) last[g.in[i]] = a++;
      for (int32_t i = g.out_off[o]; i < g.out_off[o + 1]; ++i) last[g.out[i]] = a++;
    }
    std::vector<int64_t> flags;
    for (int32_t t = 0; t < g.T; ++t)
      if (g.kind[t] == TSL_KIND_INTERIM && last[t] >= 0) flags.push_back(last[t]);
    std::sort(flags.begin(), flags.end());
    *n_out = int32_t(flags.size());
    if (out && cap >= int32_t(flags.size())) std::copy(flags.begin(), flags.end(), out);
    else if (out) fail(TSL_ERR_ARGUMENT, "flag buffer too small");
  });
}

}  // extern "C"
