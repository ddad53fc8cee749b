// TEST INFRASTRUCTURE -- restated CPU oracle for the TENSILE plan generator.
//
// A plain, single-threaded restatement of the reference hot path
// (memsched::build_plan and everything under it) over integer tensor/op ids
// with precomputed lexicographic ranks, so every std::string ordering in the
// reference becomes an integer compare. It is the checker for the CUDA
// product (tests/, smoke(), bench.py's cpu_baseline arm); the product never
// links or calls it.
//
// PINNING: this oracle is checked byte-for-byte (save_plans text, PeakReport
// JSON, merged history) against the UNMODIFIED reference compiled from
// /root/reference (oracle/_ref/libmemsched_ref.so) on every golden config and
// on randomized jobs -- tests/test_oracle_vs_reference.py. It is used as the
// parity source only where the reference cannot finish (C4, ~1M accesses).
//
// Each function cites the reference file:line it restates
// (paths relative to /root/reference/proj/).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "tensile_b200.h"

namespace {

thread_local std::string g_err;

struct Invalid : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum { TGA = 0, TUA = 1 };  // AccessType, access.hpp:11
enum { EV_TGA = 0, EV_TUA = 1, EV_SWAPIN = 2, EV_SWAPOUT = 3, EV_RELEASE = 4 };  // peak.hpp:33-39

// ---------------------------------------------------------------- graph ----
struct Graph {
  std::string job_id;
  int T = 0, O = 0;
  std::vector<std::string> tid, oid, okind;
  std::vector<int64_t> size, lat;
  std::vector<int8_t> kind, phase;
  std::vector<std::vector<int>> in, out;
  std::vector<int> producer, alias, updated_by, trank, orank;
  std::vector<std::vector<int>> consumers;
  std::vector<char> has_lat;
  double ratio = 1.0;
};

std::vector<int> lex_rank(const std::vector<std::string>& ids) {
  std::vector<int> idx(ids.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return ids[a] < ids[b]; });
  std::vector<int> rank(ids.size());
  for (size_t r = 0; r < idx.size(); ++r) rank[idx[r]] = static_cast<int>(r);
  return rank;
}

// ComputeGraph::validate, graph.cpp:49-119 (+ topological cycle check).
std::vector<int> topological_order(const Graph& g);

Graph load_graph(const tsl_job_desc& d) {
  Graph g;
  g.job_id = d.job_id ? d.job_id : "";
  g.T = d.n_tensors;
  g.O = d.n_ops;
  std::set<std::string> seen;
  for (int i = 0; i < g.T; ++i) {
    g.tid.emplace_back(d.tensor_ids[i]);
    g.size.push_back(d.tensor_sizes[i]);
    g.kind.push_back(d.tensor_kinds[i]);
    if (g.size[i] <= 0) throw Invalid("nonpositive size for tensor " + g.tid[i]);
    if (!seen.insert(g.tid[i]).second) throw Invalid("duplicate tensor id " + g.tid[i]);
  }
  g.producer.assign(g.T, -1);
  g.consumers.assign(g.T, {});
  std::set<std::string> oseen;
  for (int o = 0; o < g.O; ++o) {
    g.oid.emplace_back(d.op_ids[o]);
    g.okind.emplace_back(d.op_kinds[o]);
    g.phase.push_back(d.op_phases[o]);
    if (!oseen.insert(g.oid[o]).second) throw Invalid("duplicate op id " + g.oid[o]);
    std::vector<int> ins(d.op_inputs + d.op_in_offsets[o], d.op_inputs + d.op_in_offsets[o + 1]);
    std::vector<int> outs(d.op_outputs + d.op_out_offsets[o], d.op_outputs + d.op_out_offsets[o + 1]);
    for (int t : ins) {
      if (t < 0 || t >= g.T)
        throw Invalid("dangling tensor reference #" + std::to_string(t) + " in op " + g.oid[o]);
      g.consumers[t].push_back(o);
    }
    for (int t : outs) {
      if (t < 0 || t >= g.T)
        throw Invalid("dangling tensor reference #" + std::to_string(t) + " in op " + g.oid[o]);
      if (g.producer[t] >= 0) throw Invalid("tensor " + g.tid[t] + " has more than one producer");
      g.producer[t] = o;
    }
    g.in.push_back(ins);
    g.out.push_back(outs);
    int64_t l = d.op_latencies ? d.op_latencies[o] : TSL_LATENCY_MISSING;
    g.has_lat.push_back(l != TSL_LATENCY_MISSING);
    g.lat.push_back(l == TSL_LATENCY_MISSING ? 0 : l);
  }
  for (int t = 0; t < g.T; ++t) {
    if (g.kind[t] == TSL_KIND_INPUT || g.kind[t] == TSL_KIND_PARAMETER) {
      if (g.producer[t] >= 0) throw Invalid("source tensor " + g.tid[t] + " must not have a producing op");
      continue;
    }
    if (g.producer[t] < 0) throw Invalid("tensor " + g.tid[t] + " has no producing op");
  }
  g.alias.assign(g.T, -1);
  g.updated_by.assign(g.T, -1);
  for (int o = 0; o < g.O; ++o) {
    if (g.phase[o] == TSL_PHASE_OPTIMIZE && g.okind[o] == "update") {
      std::vector<int> upd, par;
      for (int t : g.out[o]) if (g.kind[t] == TSL_KIND_UPDATED_PARAMETER) upd.push_back(t);
      if (upd.size() != 1)
        throw Invalid("update op " + g.oid[o] + " must output exactly one updated_parameter");
      for (int t : g.in[o]) if (g.kind[t] == TSL_KIND_PARAMETER) par.push_back(t);
      if (par.size() != 1) throw Invalid("update op " + g.oid[o] + " must read exactly one parameter");
      if (g.size[upd[0]] != g.size[par[0]])
        throw Invalid("updated parameter " + g.tid[upd[0]] + " must match the size of " + g.tid[par[0]]);
      g.alias[upd[0]] = par[0];
      g.updated_by[par[0]] = upd[0];
    }
  }
  for (int t = 0; t < g.T; ++t)
    if (g.kind[t] == TSL_KIND_UPDATED_PARAMETER && g.alias[t] < 0)
      throw Invalid("updated parameter " + g.tid[t] + " is not produced by an update op");
  g.trank = lex_rank(g.tid);
  g.orank = lex_rank(g.oid);
  topological_order(g);
  return g;
}

int storage_of(const Graph& g, int t) { return g.alias[t] >= 0 ? g.alias[t] : t; }  // graph.cpp:159-163

// topological_order, graph.cpp:245-282: Kahn with a min-heap on op id plus
// user -> update edges for every consumer of an updated parameter's param.
std::vector<int> topological_order(const Graph& g) {
  std::vector<int> indeg(g.O, 0);
  std::vector<std::set<int>> succ(g.O);
  for (int o = 0; o < g.O; ++o) {
    for (int t : g.in[o]) {
      int p = g.producer[t];
      if (p >= 0 && p != o && succ[p].insert(o).second) indeg[o]++;
    }
    for (int t : g.out[o]) {
      if (g.kind[t] != TSL_KIND_UPDATED_PARAMETER) continue;
      int param = g.alias[t];
      if (param < 0) continue;
      for (int user : g.consumers[param])
        if (user != o && succ[user].insert(o).second) indeg[o]++;
    }
  }
  auto cmp = [&](int a, int b) { return g.orank[a] > g.orank[b]; };
  std::priority_queue<int, std::vector<int>, decltype(cmp)> ready(cmp);
  for (int o = 0; o < g.O; ++o) if (indeg[o] == 0) ready.push(o);
  std::vector<int> order;
  while (!ready.empty()) {
    int o = ready.top();
    ready.pop();
    order.push_back(o);
    for (int n : succ[o]) if (--indeg[n] == 0) ready.push(n);
  }
  if (static_cast<int>(order.size()) != g.O) throw Invalid("cycle detected in graph of job " + g.job_id);
  return order;
}

// ----------------------------------------------------------------- plan ----
struct Acc {
  int tensor, op;
  int8_t type;
  int64_t start, end;
};
struct Ev {  // SwapEvent, plan.hpp:18-32
  int64_t id = -1;
  int tensor = -1;
  int8_t dir = 0;  // 0 out, 1 in
  int64_t trigger = -1, delta = 0, start = 0, end = 0, earliest = 0, latest = 0;
  bool wraps = false;
  int64_t pair = -1, serves = -1;
};
struct Rc {  // RecomputeEvent, plan.hpp:34-42
  int64_t id = -1;
  int tensor = -1;
  int64_t target = -1;
  int regen = -1;
  int64_t lat = 0, saving = 0;
};
struct Plan {
  std::vector<Ev> sw;
  std::vector<Rc> rc;
  std::set<int64_t> flags;
  int64_t version = 0;
  // plan.cpp:15-20: max event id + 1 over swap and recompute events. Kept up
  // to date by every mutation (note_id) and recounted after removals, instead
  // of the reference's scan per new event.
  int64_t next_id = 0;
  // every swap interval [start, end) by start (busy_intervals' scan over all
  // swap events, swap_planner.cpp:39-50, restricted by an index) + the longest
  std::multiset<std::pair<int64_t, int64_t>> by_start;
  int64_t max_len = 0;
  int64_t next_event_id() const { return next_id; }
  void note_id(int64_t id) { next_id = std::max(next_id, id + 1); }
  void add_sw(const Ev& e) {
    sw.push_back(e);
    note_id(e.id);
    by_start.emplace(e.start, e.end);
    max_len = std::max(max_len, e.end - e.start);
  }
  void reindex() {  // after sw changed wholesale (revalidation, caller plans)
    next_id = 0;
    by_start.clear();
    max_len = 0;
    for (auto& e : sw) {
      note_id(e.id);
      by_start.emplace(e.start, e.end);
      max_len = std::max(max_len, e.end - e.start);
    }
    for (auto& e : rc) note_id(e.id);
  }
};
struct Report {  // PeakReport, peak.hpp:47-56
  int64_t peak = 0, peak_time = 0;
  bool has_lua = false;
  int64_t lua = -1;
  std::vector<int> tensors;  // storage ids, lexicographic order
  std::vector<std::pair<int64_t, int64_t>> curve;
};

int64_t transfer_duration(int64_t size, int64_t bw, int64_t setup) {  // plan.cpp:22-28
  if (bw <= 0) throw Invalid("pcie_bandwidth must be positive");
  if (setup < 0) throw Invalid("transfer_setup must be nonnegative");
  return (size + bw - 1) / bw + setup;
}

struct Job {
  const Graph* g = nullptr;
  int rank = 0;  // job id rank (std::string order)
  std::vector<Acc> acc;
  int64_t period = 0;
  std::vector<std::vector<int>> sacc;  // storage -> access ids sorted (start, id)
  std::set<int64_t> base_flags;
  std::vector<int> last_tga;  // tensor -> its last TGA access (access ids never change)
  Plan plan;
  Report rep;

  const Acc& access(int64_t id) const {  // access.cpp:7-12
    if (id < 0 || id >= static_cast<int64_t>(acc.size()))
      throw Invalid("unknown access id " + std::to_string(id) + " in job " + g->job_id);
    return acc[static_cast<size_t>(id)];
  }
  int storage(int t) const { return storage_of(*g, t); }
  void resort_sacc() {  // storage_accesses ordering, swap_planner.cpp:12-24
    for (auto& v : sacc)
      std::sort(v.begin(), v.end(), [&](int a, int b) {
        if (acc[a].start != acc[b].start) return acc[a].start < acc[b].start;
        return a < b;
      });
  }
};

// generate_access_sequence (access.cpp:28-59) + activity_analysis (access.cpp:61-78).
void make_sequence(Job& j) {
  const Graph& g = *j.g;
  int64_t clock = 0;
  for (int o : topological_order(g)) {
    if (!g.has_lat[o]) throw Invalid("missing latency entry for op " + g.oid[o]);
    if (g.lat[o] < 0) throw Invalid("negative latency for op " + g.oid[o]);
    int64_t s = clock, e = clock + g.lat[o];
    for (int t : g.in[o]) j.acc.push_back({t, o, TUA, s, e});
    for (int t : g.out[o]) j.acc.push_back({t, o, TGA, s, e});
    clock = e;
  }
  j.period = clock;
  std::vector<int> last(g.T, -1);
  for (size_t i = 0; i < j.acc.size(); ++i) last[j.acc[i].tensor] = static_cast<int>(i);
  for (int t = 0; t < g.T; ++t)
    if (last[t] >= 0 && g.kind[t] == TSL_KIND_INTERIM) j.base_flags.insert(last[t]);
  j.last_tga.assign(g.T, -1);
  for (size_t i = 0; i < j.acc.size(); ++i)
    if (j.acc[i].type == TGA) j.last_tga[j.acc[i].tensor] = static_cast<int>(i);
  j.sacc.assign(g.T, {});
  for (size_t i = 0; i < j.acc.size(); ++i) j.sacc[j.storage(j.acc[i].tensor)].push_back(static_cast<int>(i));
  j.resort_sacc();
}

// ------------------------------------------------------------ evaluator ----
struct TEv {
  int64_t time;
  int type;
  int storage;
  int64_t size, delta, aid;
  bool flagged;
};

// build_timeline, peak.cpp:66-174 (sort: peak.cpp:44-62).
std::vector<TEv> build_timeline(const Job& j, const Plan& plan) {
  const Graph& g = *j.g;
  std::vector<TEv> ev;
  // swap-out starts per storage, sorted: the ownership test below asks whether
  // any swap-out of the storage starts in [a.end, next) (peak.cpp:107-130)
  std::map<int, std::vector<int64_t>> out_starts;
  for (const Ev& e : plan.sw)
    if (e.dir == 0) out_starts[j.storage(e.tensor)].push_back(e.start);
  for (auto& kv : out_starts) std::sort(kv.second.begin(), kv.second.end());
  for (size_t i = 0; i < j.acc.size(); ++i) {
    const Acc& a = j.acc[i];
    int s = j.storage(a.tensor);
    int64_t size = g.size[s];
    bool flagged = plan.flags.count(static_cast<int64_t>(i)) > 0;
    if (a.type == TGA)
      ev.push_back({a.start, EV_TGA, s, size, s != a.tensor ? 0 : size, static_cast<int64_t>(i), false});
    else
      ev.push_back({a.end, EV_TUA, s, size, 0, static_cast<int64_t>(i), flagged});
    if (flagged) {
      int64_t next = INT64_MAX;
      for (int b : j.sacc[s]) if (j.acc[b].start >= a.end) next = std::min(next, j.acc[b].start);
      bool owned = false;
      auto os = out_starts.find(s);
      if (os != out_starts.end()) {
        auto it = std::lower_bound(os->second.begin(), os->second.end(), a.end);
        owned = it != os->second.end() && *it < next;
      }
      if (!owned) ev.push_back({a.end, EV_RELEASE, s, size, -size, static_cast<int64_t>(i), false});
    }
  }
  for (const Ev& e : plan.sw) {
    int s = j.storage(e.tensor);
    int64_t size = g.size[s];
    if (e.dir == 0) {
      int64_t when = e.end;
      if (e.trigger != -1) when = std::max(when, j.access(e.trigger).end);
      ev.push_back({when, EV_SWAPOUT, s, size, -size, -1, false});
    } else {
      int64_t when = e.end;
      if (e.wraps && j.period > 0) when = ((when % j.period) + j.period) % j.period;
      ev.push_back({when, EV_SWAPIN, s, size, size, -1, false});
    }
  }
  for (const Rc& r : plan.rc) {
    const Acc& target = j.access(r.target);
    int s = j.storage(r.tensor);
    ev.push_back({target.start - r.lat, EV_TGA, s, g.size[s], g.size[s], -1, false});
  }
  auto is_free = [](const TEv& e) { return e.type == EV_RELEASE || e.type == EV_SWAPOUT; };
  std::stable_sort(ev.begin(), ev.end(), [&](const TEv& a, const TEv& b) {
    if (a.time != b.time) return a.time < b.time;
    if (is_free(a) != is_free(b)) return is_free(a);
    if (a.storage != b.storage) return g.trank[a.storage] < g.trank[b.storage];
    if (a.type != b.type) return a.type < b.type;
    return a.aid < b.aid;
  });
  return ev;
}

// initial_resident_set (peak.cpp:176-190) + analyze_peak (peak.cpp:192-244).
Report analyze(const Job& j, const Plan& plan) {
  const Graph& g = *j.g;
  std::vector<TEv> tl = build_timeline(j, plan);
  std::vector<char> res(g.T, 0);
  for (int t = 0; t < g.T; ++t)
    if (storage_of(g, t) == t &&
        (g.kind[t] == TSL_KIND_PARAMETER || g.kind[t] == TSL_KIND_INPUT || g.kind[t] == TSL_KIND_OUTPUT))
      res[t] = 1;
  for (const Ev& e : plan.sw)
    if (e.dir == 1 && e.wraps) res[j.storage(e.tensor)] = 0;
  Report r;
  int64_t fp = 0;
  for (int t = 0; t < g.T; ++t) if (res[t]) fp += g.size[t];
  r.peak = fp;
  r.peak_time = 0;
  r.curve.emplace_back(0, fp);
  auto snapshot = [&]() {
    r.tensors.clear();
    for (int t = 0; t < g.T; ++t) if (res[t]) r.tensors.push_back(t);
    std::sort(r.tensors.begin(), r.tensors.end(), [&](int a, int b) { return g.trank[a] < g.trank[b]; });
  };
  snapshot();
  // the resident set at the last new maximum is rebuilt by a replay once the
  // walk is done (the reference copies it at every new maximum)
  const std::vector<char> res0 = res;
  int64_t peak_at = -1;  // index in tl of the last new maximum
  bool has_lua = false;
  int64_t lua = -1;
  for (size_t ei = 0; ei < tl.size(); ++ei) {
    const TEv& e = tl[ei];
    switch (e.type) {
      case EV_TGA:
        if (!res[e.storage]) { fp += e.delta; res[e.storage] = 1; }
        break;
      case EV_TUA:
        if (!e.flagged) { has_lua = true; lua = e.aid; }
        break;
      case EV_RELEASE:
      case EV_SWAPOUT:
        if (!res[e.storage]) throw Invalid("double release of tensor " + g.tid[e.storage]);
        fp -= e.size;
        res[e.storage] = 0;
        break;
      case EV_SWAPIN:
        if (res[e.storage]) throw Invalid("swap-in of resident tensor " + g.tid[e.storage]);
        fp += e.size;
        res[e.storage] = 1;
        break;
    }
    if (fp < 0) throw Invalid("negative footprint at tick " + std::to_string(e.time));
    r.curve.emplace_back(e.time, fp);
    if (fp > r.peak) {
      r.peak = fp;
      peak_at = static_cast<int64_t>(ei);
      r.peak_time = e.time;
      r.has_lua = has_lua;
      r.lua = lua;
    }
  }
  if (peak_at >= 0) {
    res = res0;
    for (int64_t ei = 0; ei <= peak_at; ++ei) {
      const TEv& e = tl[static_cast<size_t>(ei)];
      if (e.type == EV_TGA || e.type == EV_SWAPIN) res[e.storage] = 1;
      else if (e.type == EV_RELEASE || e.type == EV_SWAPOUT) res[e.storage] = 0;
    }
    snapshot();
  }
  return r;
}

void refresh(Job& j) { j.rep = analyze(j, j.plan); }  // swap_planner.hpp:28

// ---------------------------------------------------------- swap planner ----
using Iv = std::pair<int64_t, int64_t>;

void lift_into(std::vector<Iv>& busy, int64_t s, int64_t e, int64_t period, int64_t lo, int64_t hi) {
  if (e <= s) return;  // swap_planner.cpp:28-37
  for (int k = -1; k <= 1; ++k) {
    int64_t sh = k * period;
    if (e + sh > lo && s + sh < hi) busy.emplace_back(s + sh, e + sh);
  }
}

std::vector<Iv> busy_intervals(const Job& j, int storage, int64_t lo, int64_t hi, const std::vector<Iv>& extra) {
  std::vector<Iv> busy;  // swap_planner.cpp:39-50
  int64_t period = std::max<int64_t>(1, j.period);
  // the swap events whose lifted copies can reach [lo, hi): for shift k*P,
  // start < hi - kP and end > lo - kP, so start > lo - kP - max_len
  for (int k = -1; k <= 1; ++k) {
    const int64_t sh = k * period;
    auto it = j.plan.by_start.lower_bound({lo - sh - j.plan.max_len, INT64_MIN});
    for (; it != j.plan.by_start.end() && it->first < hi - sh; ++it) {
      const int64_t s = it->first, e = it->second;
      if (e <= s || !(e + sh > lo && s + sh < hi)) continue;
      busy.emplace_back(s + sh, e + sh);
    }
  }
  for (int a : j.sacc[storage]) lift_into(busy, j.acc[a].start, j.acc[a].end, period, lo, hi);
  for (auto& x : extra) lift_into(busy, x.first, x.second, period, lo, hi);
  return busy;
}

std::vector<Iv> feasible_regions(int64_t b, int64_t e, const std::vector<Iv>& busy, int64_t d) {
  if (d <= 0) throw Invalid("duration must be positive");  // swap_planner.cpp:315-337
  std::vector<Iv> regions;
  if (e <= b) return regions;
  std::vector<Iv> sorted;
  for (auto& x : busy) {
    int64_t cs = std::max(x.first, b), ce = std::min(x.second, e);
    if (ce > cs) sorted.emplace_back(cs, ce);
  }
  std::sort(sorted.begin(), sorted.end());
  int64_t cursor = b;
  for (auto& x : sorted) {
    if (x.first > cursor && x.first - cursor >= d) regions.emplace_back(cursor, x.first);
    cursor = std::max(cursor, x.second);
  }
  if (e > cursor && e - cursor >= d) regions.emplace_back(cursor, e);
  return regions;
}

struct Place {
  bool ok = false;
  int64_t s = 0, e = 0;
};
Place place_earliest(const std::vector<Iv>& r, int64_t d) {  // swap_planner.cpp:58-64
  for (auto& x : r) if (x.second - x.first >= d) return {true, x.first, x.first + d};
  return {};
}
Place place_latest(const std::vector<Iv>& r, int64_t d) {  // swap_planner.cpp:66-72
  for (auto it = r.rbegin(); it != r.rend(); ++it)
    if (it->second - it->first >= d) return {true, it->second - d, it->second};
  return {};
}

// anchor, swap_planner.cpp:76-93: the access with the greatest end <= t (ties
// to the larger id). Access ends never decrease with access id (ops are
// stamped back to back and recomputation shifts a suffix), so that access is
// the last one whose end is <= t.
std::pair<int64_t, int64_t> anchor(const Job& j, int64_t t, bool wrapped) {
  if (wrapped && j.period > 0) t = ((t % j.period) + j.period) % j.period;
  size_t lo = 0, hi = j.acc.size();
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (j.acc[mid].end <= t) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return {-1, t};
  return {static_cast<int64_t>(lo - 1), t - j.acc[lo - 1].end};
}

Ev make_event(Job& j, int storage, int dir, int64_t s, int64_t e, int64_t earliest, int64_t latest, bool wrapped,
              int64_t serves) {  // swap_planner.cpp:95-113
  Ev ev;
  ev.id = j.plan.next_event_id();
  ev.tensor = storage;
  ev.dir = static_cast<int8_t>(dir);
  ev.start = s;
  ev.end = e;
  ev.earliest = earliest;
  ev.latest = latest;
  ev.wraps = wrapped;
  ev.serves = serves;
  auto a = anchor(j, s, wrapped);
  ev.trigger = a.first;
  ev.delta = a.second;
  return ev;
}

void flag_release_before(Job& j, int storage, int64_t t) {  // swap_planner.cpp:115-122
  int preceding = -1;
  for (int a : j.sacc[storage]) if (j.acc[a].end <= t) preceding = a;
  if (preceding >= 0) j.plan.flags.insert(preceding);
}

void push_pair(Job& j, Ev out, Ev in) {
  in.pair = out.id;
  out.pair = in.id;
  j.plan.add_sw(out);
  j.plan.add_sw(in);
}

bool try_gap_pair(Job& j, int storage, int64_t lo, int64_t hi, int64_t serves, const tsl_config& c) {
  int64_t d = transfer_duration(j.g->size[storage], c.pcie_bandwidth, c.transfer_setup);  // :126-152
  if (hi - lo < 2 * d) return false;
  auto busy = busy_intervals(j, storage, lo, hi, {});
  Place out = place_earliest(feasible_regions(lo, hi, busy, d), d);
  if (!out.ok) return false;
  busy.emplace_back(out.s, out.e);
  Place in = place_latest(feasible_regions(out.e, hi, busy, d), d);
  if (!in.ok) return false;
  Ev oe = make_event(j, storage, 0, out.s, out.e, lo, hi, false, -1);
  j.plan.note_id(oe.id);  // next_event_id must see the out event first
  Ev ie = make_event(j, storage, 1, in.s, in.e, out.e, hi, false, serves);
  push_pair(j, oe, ie);
  flag_release_before(j, storage, out.s);
  return true;
}

struct Sched {
  bool ok = false, out_ok = false, first = false;
};

Sched schedule_swap(Job& j, int storage, int64_t earliest, int64_t& latest, const tsl_config& c) {
  Sched r;  // swap_planner.cpp:339-399
  int64_t d = transfer_duration(j.g->size[storage], c.pcie_bandwidth, c.transfer_setup);
  Place out = place_earliest(feasible_regions(earliest, latest, busy_intervals(j, storage, earliest, latest, {}), d), d);
  if (!out.ok) return r;
  r.out_ok = true;
  int first = -1;
  for (int a : j.sacc[storage])
    if (j.acc[a].type == TUA && j.acc[a].start >= out.e) { first = a; break; }
  if (first < 0) return r;
  r.first = true;
  int64_t fs = j.acc[first].start;
  Place in = place_latest(feasible_regions(out.e, fs, busy_intervals(j, storage, out.e, fs, {{out.s, out.e}}), d), d);
  if (!in.ok) {
    latest = j.acc[first].end;
    return r;
  }
  Ev oe = make_event(j, storage, 0, out.s, out.e, earliest, latest, false, -1);
  j.plan.note_id(oe.id);
  Ev ie = make_event(j, storage, 1, in.s, in.e, out.e, fs, false, first);
  push_pair(j, oe, ie);
  flag_release_before(j, storage, out.s);
  const std::vector<int> accs = j.sacc[storage];
  for (size_t i = 0; i + 1 < accs.size(); ++i) {
    if (accs[i] < first) continue;
    if (j.acc[accs[i + 1]].type != TUA) continue;
    try_gap_pair(j, storage, j.acc[accs[i]].end, j.acc[accs[i + 1]].start, accs[i + 1], c);
  }
  r.ok = true;
  return r;
}

Sched schedule_wrapped_swap(Job& j, int param, const tsl_config& c) {
  Sched r;  // swap_planner.cpp:401-459
  int updated = j.g->updated_by[param];
  if (updated < 0) return r;
  int64_t d = transfer_duration(j.g->size[param], c.pcie_bandwidth, c.transfer_setup);
  int64_t period = j.period;
  const int lt = j.last_tga[updated];  // the last TGA of the updated version (swap_planner.cpp:412-415)
  const int64_t tga_end = lt >= 0 ? j.acc[lt].end : -1;
  if (tga_end < 0) return r;
  Place out = place_earliest(feasible_regions(tga_end, period, busy_intervals(j, param, tga_end, period, {}), d), d);
  if (!out.ok) return r;
  r.out_ok = true;
  int first = -1;
  for (int a : j.sacc[param])
    if (j.acc[a].tensor == param && j.acc[a].type == TUA) { first = a; break; }
  if (first < 0) return r;
  r.first = true;
  int64_t lo = period, hi = period + j.acc[first].start;
  Place in = place_latest(feasible_regions(lo, hi, busy_intervals(j, param, lo, hi, {{out.s, out.e}}), d), d);
  if (!in.ok) return r;
  Ev oe = make_event(j, param, 0, out.s, out.e, tga_end, period, true, -1);
  j.plan.note_id(oe.id);
  Ev ie = make_event(j, param, 1, in.s, in.e, lo, hi, true, first);
  ie.trigger = -1;
  ie.delta = in.s - period;
  push_pair(j, oe, ie);
  flag_release_before(j, param, out.s);
  r.ok = true;
  return r;
}

struct Budget {  // SwapBudget, swap_planner.cpp:268-288 (keyed by job id rank)
  std::map<int, double> ratio;
  std::map<int, int> son;
  int total = 0;
  std::set<std::pair<int, int>> swapped;
  bool allows(int job) const {
    if (total == 0) return true;
    auto it = ratio.find(job);
    double r = it == ratio.end() ? 1.0 : it->second;
    auto s = son.find(job);
    int n = s == son.end() ? 0 : s->second;
    return static_cast<double>(n + 1) / static_cast<double>(total + 1) <= r;
  }
  void record(int job, int storage) {
    son[job]++;
    total++;
    swapped.insert({job, storage});
  }
};

std::pair<int64_t, int64_t> swap_window(const Job& j, int storage) {  // swap_planner.cpp:290-313
  int64_t latest = j.rep.peak_time, earliest = -1;
  bool has_tga = false;
  for (int a : j.sacc[storage]) {
    if (j.acc[a].type == TGA) {
      has_tga = true;
      earliest = std::max(earliest, j.acc[a].end);
    }
    if (j.acc[a].start < latest) earliest = std::max(earliest, j.acc[a].end);
  }
  if (!has_tga && j.g->kind[storage] == TSL_KIND_INTERIM)
    throw Invalid("tensor " + j.g->tid[storage] + " has no TGA in sequence");
  if (earliest < 0) earliest = 0;
  return {earliest, latest};
}

bool swap_pass(std::vector<Job>& jobs, Budget& budget, const tsl_config& c) {  // :461-520
  struct Cand {
    int64_t size;
    int job, storage;
  };
  std::vector<Cand> cands;
  for (size_t j = 0; j < jobs.size(); ++j)
    for (int t : jobs[j].rep.tensors) cands.push_back({jobs[j].g->size[t], static_cast<int>(j), t});
  std::sort(cands.begin(), cands.end(), [&](const Cand& a, const Cand& b) {
    if (a.size != b.size) return a.size > b.size;
    if (jobs[a.job].rank != jobs[b.job].rank) return jobs[a.job].rank < jobs[b.job].rank;
    return jobs[a.job].g->trank[a.storage] < jobs[b.job].g->trank[b.storage];
  });
  bool changed = false;
  for (const Cand& cd : cands) {
    Job& j = jobs[cd.job];
    int jr = j.rank, s = cd.storage;
    if (budget.swapped.count({jr, s})) continue;
    if (!budget.allows(jr)) continue;
    if (j.g->kind[s] == TSL_KIND_PARAMETER && j.g->updated_by[s] >= 0) {
      if (schedule_wrapped_swap(j, s, c).ok) {
        budget.record(jr, s);
        changed = true;
      }
      continue;
    }
    if (j.sacc[s].size() <= 1) continue;
    auto w = swap_window(j, s);
    int64_t earliest = w.first, latest = w.second;
    Sched r;
    r.out_ok = r.first = true;
    int tries = 0;
    while (!r.ok && latest > earliest && r.out_ok && r.first && tries < 16) {
      r = schedule_swap(j, s, earliest, latest, c);
      ++tries;
    }
    if (r.ok) {
      budget.record(jr, s);
      changed = true;
    }
  }
  return changed;
}

void rebuild_release_flags(Job& j) {  // swap_planner.cpp:171-188
  j.plan.flags = j.base_flags;
  auto flag_preceding = [&](int storage, int64_t before, int64_t skip) {
    int preceding = -1;
    for (int a : j.sacc[storage]) if (j.acc[a].end <= before && a != skip) preceding = a;
    if (preceding >= 0) j.plan.flags.insert(preceding);
  };
  for (const Ev& e : j.plan.sw) if (e.dir == 0) flag_preceding(j.storage(e.tensor), e.start, -2);
  for (const Rc& r : j.plan.rc) flag_preceding(j.storage(r.tensor), j.access(r.target).start, r.target);
}

void revalidate(Job& j, const tsl_config& c) {  // swap_planner.cpp:190-266
  int64_t period = std::max<int64_t>(1, j.period);
  std::map<int64_t, size_t> by_id;
  for (size_t i = 0; i < j.plan.sw.size(); ++i) {
    Ev& e = j.plan.sw[i];
    int64_t base = e.trigger == -1 ? 0 : j.access(e.trigger).end;
    int64_t d = transfer_duration(j.g->size[j.storage(e.tensor)], c.pcie_bandwidth, c.transfer_setup);
    int64_t s = base + e.delta;
    if (e.wraps && e.dir == 1) s += period;
    e.start = s;
    e.end = s + d;
    by_id[e.id] = i;
  }
  auto ov = [&](int64_t s1, int64_t e1, int64_t s2, int64_t e2) {
    for (int k = -1; k <= 1; ++k) {
      int64_t sh = k * period;
      if (s1 + sh < e2 && s2 < e1 + sh) return true;
    }
    return false;
  };
  std::set<int64_t> dropped;
  std::vector<Iv> kept;
  for (size_t i = 0; i < j.plan.sw.size(); ++i) {
    const Ev& e = j.plan.sw[i];
    if (e.dir != 0) continue;
    const Ev* in = (e.pair >= 0 && by_id.count(e.pair)) ? &j.plan.sw[by_id[e.pair]] : nullptr;
    bool ok = in != nullptr && e.end <= in->start;
    if (ok && in->serves >= 0) {
      int64_t deadline = j.access(in->serves).start;
      if (in->wraps) deadline += period;
      ok = in->end <= deadline;
    }
    if (ok) {
      for (int a : j.sacc[j.storage(e.tensor)])
        if (ov(e.start, e.end, j.acc[a].start, j.acc[a].end) || ov(in->start, in->end, j.acc[a].start, j.acc[a].end)) {
          ok = false;
          break;
        }
    }
    if (ok) {
      for (auto& k : kept)
        if (ov(e.start, e.end, k.first, k.second) || ov(in->start, in->end, k.first, k.second)) {
          ok = false;
          break;
        }
    }
    if (!ok) {
      dropped.insert(e.id);
      if (in) dropped.insert(in->id);
    } else {
      kept.emplace_back(e.start, e.end);
      kept.emplace_back(in->start, in->end);
    }
  }
  std::vector<Ev> keep;
  for (const Ev& e : j.plan.sw) if (!dropped.count(e.id)) keep.push_back(e);
  j.plan.sw.swap(keep);
  j.plan.reindex();
  rebuild_release_flags(j);
}

bool recompute_pass(std::vector<Job>& jobs, int64_t budget, const tsl_config& c) {  // recompute_planner.cpp:50-153
  int64_t merged = 0;
  for (auto& j : jobs) merged += j.rep.peak;
  if (merged < budget) return false;
  struct Cand {
    double value;
    int job, tensor;
    int64_t target, preceding;
    int regen;
    int64_t lat, saving;
  };
  std::vector<Cand> cands;
  for (size_t ji = 0; ji < jobs.size(); ++ji) {
    const Job& j = jobs[ji];
    const Graph& g = *j.g;
    auto has_swap = [&](int storage) {
      for (const Ev& e : j.plan.sw) if (j.storage(e.tensor) == storage) return true;
      return false;
    };
    auto has_release = [&](int storage) {
      for (int a : j.sacc[storage]) if (j.plan.flags.count(a)) return true;
      return false;
    };
    for (int tid : j.rep.tensors) {
      if (g.kind[tid] != TSL_KIND_INTERIM) continue;
      bool rec = false;
      for (const Rc& r : j.plan.rc) if (r.tensor == tid) rec = true;
      if (has_swap(tid) || rec) continue;
      int p = g.producer[tid];
      if (p < 0) continue;
      bool resident = true;
      for (int in : g.in[p]) {
        int st = j.storage(in);
        if (has_release(st) || has_swap(st)) { resident = false; break; }
      }
      if (!resident) continue;
      if (!g.has_lat[p] || g.lat[p] <= 0) continue;
      int target = -1, preceding = -1;
      for (int a : j.sacc[tid]) {
        if (j.acc[a].type == TUA && j.acc[a].start > j.rep.peak_time) { target = a; break; }
        preceding = a;
      }
      if (target < 0 || preceding < 0) continue;
      if (j.acc[preceding].end > j.rep.peak_time) continue;
      cands.push_back({static_cast<double>(g.size[tid]) / static_cast<double>(g.lat[p]), static_cast<int>(ji), tid,
                       target, preceding, p, g.lat[p], g.size[tid]});
    }
  }
  if (cands.empty()) return false;
  std::sort(cands.begin(), cands.end(), [&](const Cand& a, const Cand& b) {
    if (a.value != b.value) return a.value > b.value;
    if (jobs[a.job].rank != jobs[b.job].rank) return jobs[a.job].rank < jobs[b.job].rank;
    return jobs[a.job].g->trank[a.tensor] < jobs[b.job].g->trank[b.tensor];
  });
  const Cand best = cands.front();
  Job& j = jobs[best.job];
  Job backup = j;
  Rc ev;
  ev.id = j.plan.next_event_id();
  ev.tensor = best.tensor;
  ev.target = best.target;
  ev.regen = best.regen;
  ev.lat = best.lat;
  ev.saving = best.saving;
  j.plan.rc.push_back(ev);
  j.plan.note_id(ev.id);
  int64_t pivot = j.access(best.target).start;
  for (Acc& a : j.acc)
    if (a.start >= pivot) {
      a.start += best.lat;
      a.end += best.lat;
    }
  j.period += best.lat;
  j.resort_sacc();
  revalidate(j, c);
  refresh(j);
  if (j.rep.peak > backup.rep.peak) {
    j = std::move(backup);
    return false;
  }
  return true;
}

// --------------------------------------------------------------- result ----
struct JobOut {
  std::string job_id;
  const Graph* g;
  Plan plan;
  Report rep;
  int64_t period;
  int n_acc;
  // flattened views
  std::vector<int64_t> ev_id, ev_trigger, ev_delta, ev_start, ev_end, ev_earliest, ev_latest, ev_pair, ev_serves;
  std::vector<int32_t> ev_tensor;
  std::vector<int8_t> ev_dir, ev_wraps;
  std::vector<int64_t> rc_id, rc_target, rc_latency, rc_saving, flags, curve_t, curve_b;
  std::vector<int32_t> rc_tensor, rc_regen, peak_tensors;
};

}  // namespace

struct tslo_result {
  std::vector<Graph> graphs;
  std::vector<JobOut> jobs;  // job-id order (std::map)
  std::vector<int64_t> history;
  int64_t final_merged = 0;
  bool within = true;
  std::string diagnostic;
};

namespace {

void flatten(JobOut& o) {
  for (const Ev& e : o.plan.sw) {
    o.ev_id.push_back(e.id);
    o.ev_tensor.push_back(e.tensor);
    o.ev_dir.push_back(e.dir);
    o.ev_trigger.push_back(e.trigger);
    o.ev_delta.push_back(e.delta);
    o.ev_start.push_back(e.start);
    o.ev_end.push_back(e.end);
    o.ev_earliest.push_back(e.earliest);
    o.ev_latest.push_back(e.latest);
    o.ev_wraps.push_back(e.wraps ? 1 : 0);
    o.ev_pair.push_back(e.pair);
    o.ev_serves.push_back(e.serves);
  }
  for (const Rc& r : o.plan.rc) {
    o.rc_id.push_back(r.id);
    o.rc_tensor.push_back(r.tensor);
    o.rc_target.push_back(r.target);
    o.rc_regen.push_back(r.regen);
    o.rc_latency.push_back(r.lat);
    o.rc_saving.push_back(r.saving);
  }
  o.flags.assign(o.plan.flags.begin(), o.plan.flags.end());
  for (auto& p : o.rep.curve) {
    o.curve_t.push_back(p.first);
    o.curve_b.push_back(p.second);
  }
  o.peak_tensors.assign(o.rep.tensors.begin(), o.rep.tensors.end());
}

std::map<std::string, double> ratios(const tsl_config& c) {  // PlannerConfig::max_swap_ratios
  std::map<std::string, double> m;
  for (int32_t i = 0; i < c.n_max_swap_ratios; ++i) m[c.max_swap_ratio_jobs[i]] = c.max_swap_ratio_values[i];
  return m;
}

void validate_config(const tsl_config& c) {  // config.hpp:25-35
  if (c.pcie_bandwidth <= 0) throw Invalid("pcie_bandwidth must be positive");
  if (c.transfer_setup < 0) throw Invalid("transfer_setup must be nonnegative");
  if (c.memory_budget < 0) throw Invalid("memory_budget must be nonnegative");
  if (c.ewma_alpha < 0 || c.ewma_alpha > 1) throw Invalid("ewma_alpha out of [0,1]");
  if (c.replan_threshold <= 0) throw Invalid("replan_threshold must be positive");
  if (c.stall_epsilon <= 0 || c.stall_epsilon >= 1) throw Invalid("stall_epsilon out of (0,1)");
  for (auto& [job, r] : ratios(c))
    if (r <= 0 || r > 1) throw Invalid("max swap ratio for " + job + " out of (0,1]");
}

// build_plan, orchestrator.cpp:8-70.
tslo_result* build(const tsl_job_desc* descs, int n, const tsl_config& c) {
  auto* res = new tslo_result();
  res->graphs.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) res->graphs.push_back(load_graph(descs[i]));
  validate_config(c);
  const std::map<std::string, double> rmap = ratios(c);
  for (auto& g : res->graphs) {  // PlannerConfig::max_swap_ratio, config.hpp:20-23
    auto it = rmap.find(g.job_id);
    g.ratio = it == rmap.end() ? 1.0 : it->second;
  }
  if (n == 0) return res;
  std::vector<std::string> jids;
  for (auto& g : res->graphs) jids.push_back(g.job_id);
  std::vector<int> jrank = lex_rank(jids);
  // duplicate job ids share one rank (they share the reference's map keys)
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      if (jids[a] == jids[b]) jrank[a] = std::min(jrank[a], jrank[b]);
  std::vector<Job> jobs(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    jobs[i].g = &res->graphs[i];
    jobs[i].rank = jrank[i];
    make_sequence(jobs[i]);
    jobs[i].plan.flags = jobs[i].base_flags;
    refresh(jobs[i]);
  }
  Budget budget;
  for (int i = 0; i < n; ++i) budget.ratio[jrank[i]] = res->graphs[i].ratio;
  std::vector<double> mean_hist;
  bool swap_ok = true, rc_ok = true;
  int iter = 0;
  while (swap_ok || rc_ok) {
    int64_t merged = 0;
    for (auto& j : jobs) {
      refresh(j);
      merged += j.rep.peak;
    }
    res->history.push_back(merged);
    mean_hist.push_back(static_cast<double>(merged) / static_cast<double>(n));
    if (iter > c.stall_min_iters && mean_hist.size() > 3) {
      double before = mean_hist[mean_hist.size() - 4], now = mean_hist.back();
      if (before > 0 && (before - now) / before < c.stall_epsilon) break;
    }
    if (swap_ok)
      swap_ok = swap_pass(jobs, budget, c);
    else if (merged >= c.memory_budget)
      rc_ok = recompute_pass(jobs, c.memory_budget, c);
    else
      rc_ok = false;
    ++iter;
  }
  int64_t merged = 0;
  std::map<std::string, size_t> order;
  for (size_t i = 0; i < jobs.size(); ++i) {
    refresh(jobs[i]);
    merged += jobs[i].rep.peak;
    order[jobs[i].g->job_id] = i;  // later duplicates overwrite, as in result.plans[id] = ...
  }
  for (auto& kv : order) {
    Job& j = jobs[kv.second];
    JobOut o;
    o.job_id = kv.first;
    o.g = j.g;
    o.plan = j.plan;
    o.rep = j.rep;
    o.period = j.period;
    o.n_acc = static_cast<int>(j.acc.size());
    flatten(o);
    res->jobs.push_back(std::move(o));
  }
  res->final_merged = merged;
  res->within = merged <= c.memory_budget;
  if (!res->within)
    res->diagnostic = "merged memory peak " + std::to_string(merged) + " still exceeds budget " +
                      std::to_string(c.memory_budget) + " after exhausting swap and recomputation";
  return res;
}

// ----------------------------------------------------------------- json ----
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
          snprintf(buf, sizeof buf, "\\u%04x", ch);
          o += buf;
        } else {
          o += static_cast<char>(ch);
        }
    }
  }
  o += '"';
}

std::string ind(int n) { return std::string(static_cast<size_t>(n), ' '); }

// save_plans, plan.cpp:30-65 (nlohmann ordered_json dump(2) layout).
std::string save_plans(const tslo_result& r) {
  if (r.jobs.empty()) return "null\n";
  std::string o = "{\n";
  for (size_t ji = 0; ji < r.jobs.size(); ++ji) {
    const JobOut& j = r.jobs[ji];
    o += ind(2);
    jstr(o, j.job_id);
    o += ": {\n" + ind(4) + "\"version\": " + std::to_string(j.plan.version) + ",\n";
    o += ind(4) + "\"swap_events\": ";
    if (j.plan.sw.empty()) o += "[],\n";
    else {
      o += "[\n";
      for (size_t i = 0; i < j.plan.sw.size(); ++i) {
        const Ev& e = j.plan.sw[i];
        o += ind(6) + "{\n";
        o += ind(8) + "\"event_id\": " + std::to_string(e.id) + ",\n";
        o += ind(8) + "\"tensor\": ";
        jstr(o, j.g->tid[e.tensor]);
        o += ",\n";
        o += ind(8) + "\"direction\": " + (e.dir == 0 ? "\"out\"" : "\"in\"") + ",\n";
        o += ind(8) + "\"trigger_access\": " + std::to_string(e.trigger) + ",\n";
        o += ind(8) + "\"delta_time\": " + std::to_string(e.delta) + ",\n";
        o += ind(8) + "\"wraps_iteration\": " + (e.wraps ? "true" : "false") + ",\n";
        o += ind(8) + "\"start_time\": " + std::to_string(e.start) + ",\n";
        o += ind(8) + "\"end_time\": " + std::to_string(e.end) + ",\n";
        o += ind(8) + "\"pair_id\": " + std::to_string(e.pair) + ",\n";
        o += ind(8) + "\"serves_access\": " + std::to_string(e.serves) + "\n";
        o += ind(6) + (i + 1 < j.plan.sw.size() ? "},\n" : "}\n");
      }
      o += ind(4) + "],\n";
    }
    o += ind(4) + "\"recompute_events\": ";
    if (j.plan.rc.empty()) o += "[],\n";
    else {
      o += "[\n";
      for (size_t i = 0; i < j.plan.rc.size(); ++i) {
        const Rc& e = j.plan.rc[i];
        o += ind(6) + "{\n";
        o += ind(8) + "\"event_id\": " + std::to_string(e.id) + ",\n";
        o += ind(8) + "\"tensor\": ";
        jstr(o, j.g->tid[e.tensor]);
        o += ",\n";
        o += ind(8) + "\"target_access\": " + std::to_string(e.target) + ",\n";
        o += ind(8) + "\"regen_op\": ";
        jstr(o, j.g->oid[e.regen]);
        o += ",\n";
        o += ind(8) + "\"recompute_latency\": " + std::to_string(e.lat) + ",\n";
        o += ind(8) + "\"memory_saving\": " + std::to_string(e.saving) + "\n";
        o += ind(6) + (i + 1 < j.plan.rc.size() ? "},\n" : "}\n");
      }
      o += ind(4) + "],\n";
    }
    // The nlohmann/json 3.11.3 in this image (cudnn_frontend's vendored copy,
    // the only one available to build the reference) prints arrays whose
    // first element is an integer on one line: "[0,3,6]".
    o += ind(4) + "\"release_flags\": [";
    {
      size_t k = 0;
      for (int64_t f : j.plan.flags) o += (k++ ? "," : "") + std::to_string(f);
    }
    o += "]\n";
    o += ind(2) + (ji + 1 < r.jobs.size() ? "},\n" : "}\n");
  }
  o += "}\n";
  return o;
}

// PeakReport::to_json, peak.cpp:258-272.
std::string report_json(const JobOut& j) {
  const Report& r = j.rep;
  std::string o = "{\n" + ind(2) + "\"memory_peak\": " + std::to_string(r.peak) + ",\n";
  o += ind(2) + "\"peak_tensors\": ";
  if (r.tensors.empty()) o += "[],\n";
  else {
    o += "[\n";
    for (size_t i = 0; i < r.tensors.size(); ++i) {
      o += ind(4);
      jstr(o, j.g->tid[r.tensors[i]]);
      o += i + 1 < r.tensors.size() ? ",\n" : "\n";
    }
    o += ind(2) + "],\n";
  }
  o += ind(2) + "\"last_input_access\": " + (r.has_lua ? std::to_string(r.lua) : std::string("null")) + ",\n";
  o += ind(2) + "\"peak_time\": " + std::to_string(r.peak_time) + ",\n";
  o += ind(2) + "\"footprint_curve\": ";
  if (r.curve.empty()) o += "[]\n";
  else {
    o += "[\n";
    for (size_t i = 0; i < r.curve.size(); ++i) {
      o += ind(4) + "[" + std::to_string(r.curve[i].first) + "," + std::to_string(r.curve[i].second) +
           (i + 1 < r.curve.size() ? "],\n" : "]\n");
    }
    o += ind(2) + "]\n";
  }
  o += "}\n";
  return o;
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
  } catch (const Invalid& e) {
    g_err = e.what();
    return TSL_ERR_VALIDATION;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TSL_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" {

const char* tslo_last_error(void) { return g_err.c_str(); }

int tslo_build_plan(const tsl_job_desc* jobs, int32_t n, const tsl_config* cfg, tslo_result** out) {
  if (!out || !cfg || (n > 0 && !jobs)) {
    g_err = "null argument";
    return TSL_ERR_ARGUMENT;
  }
  return guard([&] { *out = build(jobs, n, *cfg); });
}

// analyze_job on a caller-supplied plan (peak.cpp:246-250).
// Initial peak of every job (make_job_context's report, swap_planner.cpp:156-169):
// release-at-last-use flags, empty plan. The budget basis of the configs.
int tslo_initial_peaks(const tsl_job_desc* jobs, int32_t n, int64_t* peaks) {
  return guard([&] {
    for (int32_t i = 0; i < n; ++i) {
      Graph g = load_graph(jobs[i]);
      Job j;
      j.g = &g;
      j.rank = 0;
      make_sequence(j);
      j.plan.flags = j.base_flags;
      refresh(j);
      peaks[i] = j.rep.peak;
    }
  });
}

int tslo_analyze_job(const tsl_job_desc* jd, const tsl_plan_desc* pd, tslo_result** out) {
  return guard([&] {
    auto* res = new tslo_result();
    res->graphs.push_back(load_graph(*jd));
    Job j;
    j.g = &res->graphs[0];
    make_sequence(j);
    for (int i = 0; i < pd->n_swap; ++i) {
      Ev e;
      e.id = pd->ev_id[i];
      e.tensor = pd->ev_tensor[i];
      e.dir = pd->ev_dir[i];
      e.trigger = pd->ev_trigger[i];
      e.delta = pd->ev_delta[i];
      e.start = pd->ev_start[i];
      e.end = pd->ev_end[i];
      e.wraps = pd->ev_wraps[i] != 0;
      e.pair = pd->ev_pair[i];
      e.serves = pd->ev_serves[i];
      j.plan.sw.push_back(e);
    }
    for (int i = 0; i < pd->n_recompute; ++i) {
      Rc r;
      r.id = pd->rc_id[i];
      r.tensor = pd->rc_tensor[i];
      r.target = pd->rc_target[i];
      r.regen = pd->rc_regen_op[i];
      r.lat = pd->rc_latency[i];
      r.saving = pd->rc_saving[i];
      j.plan.rc.push_back(r);
    }
    for (int i = 0; i < pd->n_release; ++i) j.plan.flags.insert(pd->release_flags[i]);
    j.plan.version = pd->version;
    j.plan.reindex();
    refresh(j);
    JobOut o;
    o.job_id = j.g->job_id;
    o.g = j.g;
    o.plan = j.plan;
    o.rep = j.rep;
    o.period = j.period;
    o.n_acc = static_cast<int>(j.acc.size());
    flatten(o);
    res->jobs.push_back(std::move(o));
    *out = res;
  });
}

int32_t tslo_result_n_jobs(const tslo_result* r) { return static_cast<int32_t>(r->jobs.size()); }

int tslo_result_job(const tslo_result* r, int32_t i, tsl_job_view* v) {
  if (!r || i < 0 || i >= static_cast<int32_t>(r->jobs.size())) return TSL_ERR_ARGUMENT;
  const JobOut& o = r->jobs[static_cast<size_t>(i)];
  std::memset(v, 0, sizeof *v);
  v->job_id = o.job_id.c_str();
  v->version = o.plan.version;
  v->n_swap = static_cast<int32_t>(o.ev_id.size());
  v->ev_id = o.ev_id.data();
  v->ev_tensor = o.ev_tensor.data();
  v->ev_dir = o.ev_dir.data();
  v->ev_trigger = o.ev_trigger.data();
  v->ev_delta = o.ev_delta.data();
  v->ev_start = o.ev_start.data();
  v->ev_end = o.ev_end.data();
  v->ev_earliest = o.ev_earliest.data();
  v->ev_latest = o.ev_latest.data();
  v->ev_wraps = o.ev_wraps.data();
  v->ev_pair = o.ev_pair.data();
  v->ev_serves = o.ev_serves.data();
  v->n_recompute = static_cast<int32_t>(o.rc_id.size());
  v->rc_id = o.rc_id.data();
  v->rc_tensor = o.rc_tensor.data();
  v->rc_target = o.rc_target.data();
  v->rc_regen_op = o.rc_regen.data();
  v->rc_latency = o.rc_latency.data();
  v->rc_saving = o.rc_saving.data();
  v->n_release = static_cast<int32_t>(o.flags.size());
  v->release_flags = o.flags.data();
  v->memory_peak = o.rep.peak;
  v->peak_time = o.rep.peak_time;
  v->has_last_input_access = o.rep.has_lua ? 1 : 0;
  v->last_input_access = o.rep.lua;
  v->n_peak_tensors = static_cast<int32_t>(o.peak_tensors.size());
  v->peak_tensors = o.peak_tensors.data();
  v->n_curve = static_cast<int32_t>(o.curve_t.size());
  v->curve_time = o.curve_t.data();
  v->curve_bytes = o.curve_b.data();
  v->iteration_period = o.period;
  v->n_accesses = o.n_acc;
  return TSL_OK;
}

int32_t tslo_result_history(const tslo_result* r, const int64_t** h) {
  *h = r->history.data();
  return static_cast<int32_t>(r->history.size());
}
int64_t tslo_result_final_merged_peak(const tslo_result* r) { return r->final_merged; }
int32_t tslo_result_within_budget(const tslo_result* r) { return r->within ? 1 : 0; }
const char* tslo_result_diagnostic(const tslo_result* r) { return r->diagnostic.c_str(); }
char* tslo_result_save_plans(const tslo_result* r) { return dup(save_plans(*r)); }
char* tslo_result_report_json(const tslo_result* r, int32_t i) {
  return dup(report_json(r->jobs[static_cast<size_t>(i)]));
}
void tslo_result_destroy(tslo_result* r) { delete r; }
void tslo_free(void* p) { std::free(p); }

}  // extern "C"
