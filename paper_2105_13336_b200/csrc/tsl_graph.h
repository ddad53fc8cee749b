// Host-side graph model shared by the planner's host code (tsl_host.cpp) and
// the tick-level executor model (tsl_sim.cpp): ComputeGraph
// (graph.hpp:14-62) over dense indices, loaded and validated from a
// tsl_job_desc with the reference's checks and error texts
// (graph.cpp:49-119, 245-282; access.cpp:33-38).
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "tensile_b200.h"

namespace tsl {
namespace hostg {

// Host error: a tsl status code and the reference's message.
struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Fail{code, m}; }


// tsl_last_error()'s thread-local text (tsl_host.cpp).
void set_last_error(const std::string& msg);

// std::sort over up to 8 host threads: chunks sorted in parallel, then merged
// pairwise in parallel rounds (large graphs: C4's 4e5 tensor ids).
template <class T, class Cmp>
inline void par_sort(std::vector<T>& v, Cmp cmp) {
  const size_t n = v.size();
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  size_t parts = 1;
  while (parts * 2 <= std::min<size_t>(8, hw) && n / (parts * 2) >= 32768) parts *= 2;
  if (parts == 1) { std::sort(v.begin(), v.end(), cmp); return; }
  std::vector<size_t> cut(parts + 1);
  for (size_t p = 0; p <= parts; ++p) cut[p] = n * p / parts;
  {
    std::vector<std::thread> th;
    for (size_t p = 0; p < parts; ++p)
      th.emplace_back([&, p] { std::sort(v.begin() + cut[p], v.begin() + cut[p + 1], cmp); });
    for (auto& t : th) t.join();
  }
  std::vector<T> buf(n);
  std::vector<T>* src = &v;
  std::vector<T>* dst = &buf;
  for (size_t w = 1; w < parts; w *= 2) {
    std::vector<std::thread> th;
    for (size_t p = 0; p < parts; p += 2 * w)
      th.emplace_back([&, p] {
        const size_t a = cut[p], m = cut[std::min(parts, p + w)], b = cut[std::min(parts, p + 2 * w)];
        std::merge(src->begin() + a, src->begin() + m, src->begin() + m, src->begin() + b, dst->begin() + a, cmp);
      });
    for (auto& t : th) t.join();
    std::swap(src, dst);
  }
  if (src != &v) v.swap(*src);
}

// fn(i) for i in [0, n), on up to 8 host threads for large n (contiguous ranges).
template <class F>
inline void par_for(size_t n, F fn) {
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t parts = n >= 65536 ? std::min<size_t>(8, hw) : 1;
  if (parts <= 1) { for (size_t i = 0; i < n; ++i) fn(i); return; }
  std::vector<std::thread> th;
  for (size_t p = 1; p < parts; ++p)
    th.emplace_back([&, p] { for (size_t i = n * p / parts; i < n * (p + 1) / parts; ++i) fn(i); });
  for (size_t i = 0; i < n / parts; ++i) fn(i);
  for (auto& t : th) t.join();
}

// Rank of every id in std::string order, ties by index (a stable sort). The
// sort compares a 16-byte big-endian prefix held inline (ids of one job share
// long prefixes, but rarely 16 bytes) and only then the strings.
inline std::vector<int32_t> lex_rank(const std::vector<std::string>& ids) {
  struct K {
    uint64_t k0, k1;
    int32_t i;
  };
  auto be = [](const std::string& s, size_t off) {
    uint64_t v = 0;
    for (size_t b = 0; b < 8; ++b) v = (v << 8) | (off + b < s.size() ? uint8_t(s[off + b]) : 0u);
    return v;
  };
  std::vector<K> keys(ids.size());
  par_for(ids.size(), [&](size_t i) { keys[i] = K{be(ids[i], 0), be(ids[i], 8), int32_t(i)}; });
  par_sort(keys, [&](const K& a, const K& b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    const std::string& x = ids[a.i];
    const std::string& y = ids[b.i];
    // equal 16-byte prefixes (zero-padded): compare the rest, then the index
    const int c = (x.size() > 16 || y.size() > 16) ? x.compare(y) : (x.size() == y.size() ? 0 : x.size() < y.size() ? -1 : 1);
    return c != 0 ? c < 0 : a.i < b.i;
  });
  std::vector<int32_t> rank(ids.size());
  par_for(keys.size(), [&](size_t r) { rank[keys[r].i] = static_cast<int32_t>(r); });
  return rank;
}

// ---------------------------------------------------------------------------
// Graph: ComputeGraph (graph.hpp:14-62) over dense indices.
// ---------------------------------------------------------------------------
struct Graph {
  std::string job_id;
  int32_t T = 0, O = 0, A = 0;
  std::vector<std::string> tid, oid;
  std::vector<int64_t> size, lat;
  std::vector<int8_t> kind;
  std::vector<int32_t> in_off, in, out_off, out;
  std::vector<int32_t> trank, store, upd, prod, topo;
};

inline const char* kind_name(int k) {
  static const char* n[] = {"input", "interim", "parameter", "updated_parameter", "output"};
  return (k >= 0 && k < 5) ? n[k] : "?";
}

// ComputeGraph::validate, graph.cpp:49-119, same checks in the same order and
// the same first error; duplicate ids are found from the lexicographic sort
// the ranks need anyway, successor sets are one sorted edge list.
inline Graph load_graph(const tsl_job_desc& d) {
  Graph g;
  static const bool lp = std::getenv("TSL_PREP_PROFILE") != nullptr;
  auto lt0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!lp) return;
    auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  load %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - lt0).count());
    lt0 = t;
  };
  g.job_id = d.job_id ? d.job_id : "";
  g.T = d.n_tensors;
  g.O = d.n_ops;
  if (g.T < 0 || g.O < 0) fail(TSL_ERR_ARGUMENT, "negative tensor/op count in job " + g.job_id);
  if (g.T > 0 && (!d.tensor_ids || !d.tensor_sizes || !d.tensor_kinds))
    fail(TSL_ERR_ARGUMENT, "null tensor table in job " + g.job_id);
  if (g.O > 0 && (!d.op_ids || !d.op_kinds || !d.op_phases || !d.op_in_offsets || !d.op_out_offsets))
    fail(TSL_ERR_ARGUMENT, "null op table in job " + g.job_id);
  lap("strings");
  // The op side (op id strings, their ranks and duplicates, phases, update
  // kinds) runs on a second thread for big graphs while the tensor side is
  // built; its first error is raised where the sequential order puts it.
  std::vector<int32_t> orank;
  std::vector<char> odup(g.O, 0), is_update(g.O, 0);
  std::vector<int8_t> phase(g.O, 0);
  std::string phase_err;
  auto op_side = [&] {
    g.oid.resize(g.O);
    par_for(size_t(g.O), [&](size_t o) { g.oid[o] = d.op_ids[o] ? d.op_ids[o] : ""; });
    orank = lex_rank(g.oid);
    std::vector<int32_t> by(g.O);
    for (int i = 0; i < g.O; ++i) by[orank[i]] = i;
    for (int r = 1; r < g.O; ++r)
      if (g.oid[by[r]] == g.oid[by[r - 1]]) odup[by[r]] = 1;
    for (int o = 0; o < g.O; ++o) {
      const int8_t ph = d.op_phases[o];
      if (ph != 0 && ph != 1 && phase_err.empty()) phase_err = "unknown op phase: #" + std::to_string(ph);
      phase[o] = ph;
      is_update[o] = d.op_kinds[o] && std::strcmp(d.op_kinds[o], "update") == 0;
    }
  };
  std::thread op_thread;
  struct Join {
    std::thread& t;
    ~Join() { if (t.joinable()) t.join(); }
  } join_on_exit{op_thread};
  if (g.O > 4096) op_thread = std::thread(op_side);
  else op_side();
  g.size.assign(d.tensor_sizes, d.tensor_sizes + g.T);
  g.kind.assign(d.tensor_kinds, d.tensor_kinds + g.T);
  for (int i = 0; i < g.T; ++i)
    if (g.kind[i] < 0 || g.kind[i] > 4) fail(TSL_ERR_VALIDATION, "unknown tensor kind: #" + std::to_string(g.kind[i]));
  g.tid.resize(g.T);
  par_for(size_t(g.T), [&](size_t i) { g.tid[i] = d.tensor_ids[i] ? d.tensor_ids[i] : ""; });
  lap("tid");
  g.trank = lex_rank(g.tid);
  lap("lexrank");
  {
    // first tensor (in order) that is nonpositive or a repeated id
    std::vector<int32_t> by(g.T);
    for (int i = 0; i < g.T; ++i) by[g.trank[i]] = i;
    std::vector<char> dup(g.T, 0);
    for (int r = 1; r < g.T; ++r) {
      if (g.tid[by[r]] != g.tid[by[r - 1]]) continue;
      // equal ids are adjacent in rank order with ascending index (stable sort)
      dup[by[r]] = 1;
    }
    for (int i = 0; i < g.T; ++i) {
      if (g.size[i] <= 0) fail(TSL_ERR_VALIDATION, "nonpositive size for tensor " + g.tid[i]);
      if (dup[i]) fail(TSL_ERR_VALIDATION, "duplicate tensor id " + g.tid[i]);
    }
  }
  lap("ranks+dups");
  std::vector<int32_t> producer(g.T, -1);
  if (op_thread.joinable()) op_thread.join();
  if (!phase_err.empty()) fail(TSL_ERR_VALIDATION, phase_err);
  lap("opkinds+odup");
  g.in_off.assign(1, 0);
  g.out_off.assign(1, 0);
  for (int o = 0; o < g.O; ++o) {
    if (odup[o]) fail(TSL_ERR_VALIDATION, "duplicate op id " + g.oid[o]);
    for (int32_t i = d.op_in_offsets[o]; i < d.op_in_offsets[o + 1]; ++i) {
      int32_t t = d.op_inputs[i];
      if (t < 0 || t >= g.T)
        fail(TSL_ERR_VALIDATION, "dangling tensor reference #" + std::to_string(t) + " in op " + g.oid[o]);
      g.in.push_back(t);
    }
    for (int32_t i = d.op_out_offsets[o]; i < d.op_out_offsets[o + 1]; ++i) {
      int32_t t = d.op_outputs[i];
      if (t < 0 || t >= g.T)
        fail(TSL_ERR_VALIDATION, "dangling tensor reference #" + std::to_string(t) + " in op " + g.oid[o]);
      if (producer[t] >= 0) fail(TSL_ERR_VALIDATION, "tensor " + g.tid[t] + " has more than one producer");
      producer[t] = o;
      g.out.push_back(t);
    }
    g.in_off.push_back(static_cast<int32_t>(g.in.size()));
    g.out_off.push_back(static_cast<int32_t>(g.out.size()));
  }
  lap("csr");
  for (int t = 0; t < g.T; ++t) {
    if (g.kind[t] == TSL_KIND_INPUT || g.kind[t] == TSL_KIND_PARAMETER) {
      if (producer[t] >= 0) fail(TSL_ERR_VALIDATION, "source tensor " + g.tid[t] + " must not have a producing op");
      continue;
    }
    if (producer[t] < 0) fail(TSL_ERR_VALIDATION, "tensor " + g.tid[t] + " has no producing op");
  }
  std::vector<int32_t> alias(g.T, -1);
  g.upd.assign(g.T, -1);
  for (int o = 0; o < g.O; ++o) {
    if (phase[o] != TSL_PHASE_OPTIMIZE || !is_update[o]) continue;
    int32_t u = -1, p = -1, nu = 0, np = 0;
    for (int32_t i = g.out_off[o]; i < g.out_off[o + 1]; ++i)
      if (g.kind[g.out[i]] == TSL_KIND_UPDATED_PARAMETER) { if (nu++ == 0) u = g.out[i]; }
    if (nu != 1) fail(TSL_ERR_VALIDATION, "update op " + g.oid[o] + " must output exactly one updated_parameter");
    for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i)
      if (g.kind[g.in[i]] == TSL_KIND_PARAMETER) { if (np++ == 0) p = g.in[i]; }
    if (np != 1) fail(TSL_ERR_VALIDATION, "update op " + g.oid[o] + " must read exactly one parameter");
    if (g.size[u] != g.size[p])
      fail(TSL_ERR_VALIDATION, "updated parameter " + g.tid[u] + " must match the size of " + g.tid[p]);
    alias[u] = p;
    g.upd[p] = u;
  }
  for (int t = 0; t < g.T; ++t)
    if (g.kind[t] == TSL_KIND_UPDATED_PARAMETER && alias[t] < 0)
      fail(TSL_ERR_VALIDATION, "updated parameter " + g.tid[t] + " is not produced by an update op");
  g.store.resize(g.T);
  for (int t = 0; t < g.T; ++t) g.store[t] = alias[t] >= 0 ? alias[t] : t;
  g.prod = producer;
  // topological_order (graph.cpp:245-282): Kahn with a min-heap on the op id,
  // plus user -> update edges for every consumer of an updated param's param.
  std::vector<std::pair<int32_t, int32_t>> edges;
  edges.reserve(g.in.size() + 16);
  for (int o = 0; o < g.O; ++o)
    for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) {
      int32_t p = producer[g.in[i]];
      if (p >= 0 && p != o) edges.emplace_back(p, o);
    }
  {
    // consumers of a parameter, for the update-after-every-use edges
    std::vector<int32_t> coff(g.T + 1, 0), cons;
    for (int o = 0; o < g.O; ++o)
      for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) coff[g.in[i] + 1]++;
    for (int t = 0; t < g.T; ++t) coff[t + 1] += coff[t];
    cons.resize(coff[g.T]);
    std::vector<int32_t> cur(coff.begin(), coff.end() - 1);
    for (int o = 0; o < g.O; ++o)
      for (int32_t i = g.in_off[o]; i < g.in_off[o + 1]; ++i) cons[cur[g.in[i]]++] = o;
    for (int o = 0; o < g.O; ++o)
      for (int32_t i = g.out_off[o]; i < g.out_off[o + 1]; ++i) {
        const int32_t t = g.out[i];
        if (g.kind[t] != TSL_KIND_UPDATED_PARAMETER || alias[t] < 0) continue;
        for (int32_t k = coff[alias[t]]; k < coff[alias[t] + 1]; ++k)
          if (cons[k] != o) edges.emplace_back(cons[k], o);
      }
  }
  lap("edges");
  // group the edges by source (counting sort), then sort + dedupe each
  // source's short target list: the same (source, target) order as one
  // global sort + unique, in linear time
  std::vector<int32_t> indeg(g.O, 0), soff(g.O + 1, 0);
  {
    std::vector<int32_t> cnt(g.O + 1, 0), tgt(edges.size());
    for (auto& e : edges) cnt[e.first + 1]++;
    for (int o = 0; o < g.O; ++o) cnt[o + 1] += cnt[o];
    std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
    for (auto& e : edges) tgt[cur[e.first]++] = e.second;
    size_t w = 0;
    for (int o = 0; o < g.O; ++o) {
      auto b = tgt.begin() + cnt[o], e = tgt.begin() + cnt[o + 1];
      std::sort(b, e);
      auto u = std::unique(b, e);
      soff[o] = int32_t(w);
      for (auto it = b; it != u; ++it) edges[w++] = {o, *it};
    }
    soff[g.O] = int32_t(w);
    edges.resize(w);
  }
  for (auto& e : edges) indeg[e.second]++;
  lap("sort-edges");
  // the min-heap on the op id is a three-level bitset over the (unique) id
  // ranks: insert and extract-min in a few word operations
  std::vector<int32_t> by_rank(g.O);
  for (int o = 0; o < g.O; ++o) by_rank[orank[o]] = o;
  std::vector<uint64_t> b0((size_t(g.O) + 63) / 64, 0), b1((b0.size() + 63) / 64, 0), b2((b1.size() + 63) / 64, 0);
  int64_t n_ready = 0;
  auto push = [&](int32_t o) {
    const uint32_t r = uint32_t(orank[o]);
    b0[r >> 6] |= uint64_t(1) << (r & 63);
    b1[r >> 12] |= uint64_t(1) << ((r >> 6) & 63);
    b2[r >> 18] |= uint64_t(1) << ((r >> 12) & 63);
    ++n_ready;
  };
  auto pop_min = [&]() -> int32_t {
    size_t w2 = 0;
    while (!b2[w2]) ++w2;
    const size_t w1 = w2 * 64 + size_t(__builtin_ctzll(b2[w2]));
    const size_t w0 = w1 * 64 + size_t(__builtin_ctzll(b1[w1]));
    const uint32_t r = uint32_t(w0 * 64 + size_t(__builtin_ctzll(b0[w0])));
    b0[w0] &= b0[w0] - 1;
    if (!b0[w0]) {
      b1[w1] &= ~(uint64_t(1) << (w0 & 63));
      if (!b1[w1]) b2[w2] &= ~(uint64_t(1) << (w1 & 63));
    }
    --n_ready;
    return by_rank[r];
  };
  for (int o = 0; o < g.O; ++o)
    if (indeg[o] == 0) push(o);
  g.topo.reserve(g.O);
  while (n_ready > 0) {
    const int32_t o = pop_min();
    g.topo.push_back(o);
    for (int32_t k = soff[o]; k < soff[o + 1]; ++k)
      if (--indeg[edges[k].second] == 0) push(edges[k].second);
  }
  if (static_cast<int32_t>(g.topo.size()) != g.O) fail(TSL_ERR_VALIDATION, "cycle detected in graph of job " + g.job_id);
  lap("topo");
  // latency table (generate_access_sequence, access.cpp:33-38), checked in
  // topological order like the reference.
  g.lat.assign(g.O, 0);
  for (int o = 0; o < g.O; ++o) g.lat[o] = d.op_latencies ? d.op_latencies[o] : TSL_LATENCY_MISSING;
  int64_t A = 0;
  for (int o = 0; o < g.O; ++o) A += (g.in_off[o + 1] - g.in_off[o]) + (g.out_off[o + 1] - g.out_off[o]);
  if (A > (1 << 30)) fail(TSL_ERR_CAPACITY, "job " + g.job_id + " has too many accesses");
  g.A = static_cast<int32_t>(A);
  return g;
}

inline void check_latencies(const Graph& g) {
  for (int32_t o : g.topo) {
    if (g.lat[o] == TSL_LATENCY_MISSING) fail(TSL_ERR_VALIDATION, "missing latency entry for op " + g.oid[o]);
    if (g.lat[o] < 0) fail(TSL_ERR_VALIDATION, "negative latency for op " + g.oid[o]);
  }
}

}  // namespace hostg
}  // namespace tsl
