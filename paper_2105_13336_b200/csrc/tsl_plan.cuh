// TENSILE scheduling-plan generator: the whole memsched::build_plan
// (/root/reference/proj/src/orchestrator.cpp:8-70) for one planning group,
// written against an execution context X so that ONE CTA runs it end to end.
//
//   X::tid/nthr          CTA thread index / count
//   X::lane/warp/nwarp   warp geometry (W == 32 on the device)
//   X::sync()            CTA barrier         X::wsync()  warp barrier
//   X::sort(k,v,n,bits)  CTA-collective stable radix sort of (u64 key, i32 value)
//   X::scan(a,n)         CTA-collective inclusive int64 scan in place
//   X::amin/amax/aadd    atomics on shared/global scalars
//   X::sh                CTA-shared scalar scratch (SH_WORDS int64)
//
// The device context lives in tsl_kernel.cu. tests/emu/ compiles this same
// file with a one-thread host context purely to debug the algorithm against
// the oracle on CPU; the product library never contains that build.
//
// Design:
//  * stage 1, timeline builder (access.cpp:28-78): latency scan over the topo
//    order, access emission, activity analysis, CSR-by-storage via a sort.
//  * stage 2, footprint evaluator (peak.cpp:66-244): all events of a batch of
//    jobs get a packed 64-bit key (job, time, frees-first, storage rank, type
//    rank, tie) and one block radix sort; a second stable sort groups the
//    sorted positions by storage so each storage's residency automaton runs
//    independently (one thread per storage); then a block scan gives the
//    footprint curve, a max-reduce + first-index-min gives the first strict
//    maximum, and the per-storage state at that position gives peak_tensors.
//  * stage 3/4, scorer + selector (swap_planner.cpp:461-520): each job's
//    candidate list is walked in the reference's order by one warp; the
//    feasible-region queries are k-way merge sweeps over the job's swap
//    intervals kept sorted by start (they are pairwise disjoint), with early
//    exit; all lanes run the scalar logic redundantly and cooperate on bulk
//    moves. Jobs are independent unless a max_swap_ratio < 1 couples them
//    through SwapBudget, in which case one warp walks the global order.
//  * recomputation (recompute_planner.cpp:50-153): candidates scored by all
//    threads, argmax, commit, shift, revalidate, re-evaluate, rollback.
#pragma once
#include <stdint.h>

#include "tsl_types.h"

#ifdef __CUDACC__
#define TSL_HD __device__ inline
// the query/search helpers are forced inline: in a 255-register kernel a call
// spills and restores live registers through local memory, which costs more
// than the larger body (measured: C2 0.637 -> 0.600 ms)
#define TSL_HD_FORCE __device__ __forceinline__
#else
#define TSL_HD inline
#define TSL_HD_FORCE inline
#endif

#if TSL_EMU_STATS
#include <cstdio>
#include <cstdlib>
#include <vector>
#endif
namespace tsl {

#if TSL_EMU_STATS
// development statistics of the re-scores (emulation build only)
namespace emu_stats {
inline int64_t n_rescore, spec_not_ok, wrapped, spec_pairs, new_pairs, kept_pairs, main_same, main_in_only, now_fail,
    now_ok, with_gaps, passes, comp_max, comp_sum_max, comp_big, conf_over, conf_edges, cands, why_hit, why_over,
    why_nconf, why_diff, why_conf, verify_bad, verified;
struct Printer {
  ~Printer() {
    std::fprintf(stderr,
                 "rescore %lld spec_not_ok %lld wrapped %lld spec_pairs %lld new_pairs %lld kept_pairs %lld "
                 "main_same %lld main_in_only %lld now_fail %lld now_ok %lld with_gaps %lld\n",
                 (long long)n_rescore, (long long)spec_not_ok, (long long)wrapped, (long long)spec_pairs,
                 (long long)new_pairs, (long long)kept_pairs, (long long)main_same, (long long)main_in_only,
                 (long long)now_fail, (long long)now_ok, (long long)with_gaps);
    std::fprintf(stderr, "passes %lld cands %lld edges %lld conf_over %lld comp_max %lld mean_max %.1f in_big(>32) %lld\n",
                 (long long)passes, (long long)cands, (long long)conf_edges, (long long)conf_over, (long long)comp_max,
                 passes ? double(comp_sum_max) / passes : 0.0, (long long)comp_big);
    std::fprintf(stderr, "verified %lld bad %lld\n", (long long)verified, (long long)verify_bad);
    std::fprintf(stderr, "why: hit %lld overflow %lld nconf>CAPC %lld comp-diff %lld conflict %lld\n", (long long)why_hit,
                 (long long)why_over, (long long)why_nconf, (long long)why_diff, (long long)why_conf);
  }
};
inline Printer printer;
}  // namespace emu_stats
#endif

#ifndef TSL_PROF
#define TSL_PROF 0
#endif
#ifndef TSL_DEBUG_REASONS
#define TSL_DEBUG_REASONS 0
#endif
constexpr int SH_WORDS = 1024;   // CTA-shared int64 scalars
constexpr int MAXB = 32;         // jobs per evaluation batch
constexpr int EV_FIELDS = 12;    // swap-event fields (rollback copies)
constexpr int RC_FIELDS = 6;

TSL_HD int popc32(unsigned v) {
#ifdef __CUDA_ARCH__
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}
TSL_HD int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
TSL_HD int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
TSL_HD int nbits(uint64_t v) {  // bits needed to hold v (0 -> 0)
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

// transfer_duration, plan.cpp:22-28 (bandwidth / setup validated on the host).
TSL_HD int64_t duration(int64_t size, const GroupConfig& c) {
  return (size + c.bw - 1) / c.bw + c.setup;
}

// Storage accesses of `s` are s_acc[s_off[s] .. s_off[s+1]) in ascending
// access id, which is also (start, id) order: starts (and ends) never
// decrease with the access id, before or after recomputation shifts.

// ----------------------------------------------------------------------------
// Feasible-region queries (swap_planner.cpp:26-72, 315-337)
// ----------------------------------------------------------------------------
// A stream is a run of intervals sorted by start AND end, lifted by `sh`.
// Only the bound the sweep direction needs is searched; the other side ends
// the stream lazily (starts are sorted, so a forward sweep stops at the
// first start >= the window end; ends are sorted, so a reverse sweep stops
// at the first end <= the window begin). The head interval is cached.
struct Stream {
  const int64_t* s;
  const int64_t* e;
  const int32_t* ix;  // indirection (storage accesses) or null
  int32_t i, n;       // forward: next index i of n; reverse: remaining [0, i)
  int64_t sh;
  int64_t hs, he;     // cached head (lifted)
  bool live;
};
TSL_HD int32_t sidx(const Stream& q, int32_t k) { return q.ix ? q.ix[k] : k; }

TSL_HD void stream_load(Stream& q, bool fwd, int64_t b, int64_t e) {
  if (fwd) {
    q.live = q.i < q.n;
    if (q.live) {
      const int32_t k = sidx(q, q.i);
      q.hs = q.s[k] + q.sh;
      q.he = q.e[k] + q.sh;
      q.live = q.hs < e;
    }
  } else {
    q.live = q.i > 0;
    if (q.live) {
      const int32_t k = sidx(q, q.i - 1);
      q.hs = q.s[k] + q.sh;
      q.he = q.e[k] + q.sh;
      q.live = q.he > b;
    }
  }
}

// Bucketed time index over a sorted run: first[b] = first k with
// key(k) >= b << shift, for b in [0, TI_NB]. A lookup is one index load plus
// a short forward scan instead of ~log2(n) dependent probes.
constexpr int TI_NB = 256;

struct TIndex {
  const int32_t* first;  // [nb + 1] or null
  int32_t shift;
  int32_t nb;            // bucket count (TI_NB, or the job's finer ti_nb)
};

// First index k in [0, n) with key(k) > v (strict) or key(k) >= v, for
// nondecreasing keys key(k) = arr[ix ? ix[k] : k]. One code path for every
// caller (lanes searching different streams stay converged): the optional
// time index narrows [lo, hi) with two independent loads, then a binary
// search finishes.
TSL_HD_FORCE int32_t search_keys(const int64_t* arr, const int32_t* ix, int32_t n, int64_t v, bool strict,
                                    const TIndex* ti = nullptr) {
  int32_t lo = 0, hi = n;
  if (ti && ti->first && v >= 0) {
    // all k before first[b] have key < (b << shift) <= v; from first[b + 1]
    // on, key >= (b + 1) << shift > v
    int64_t bk = v >> ti->shift;
    if (bk > ti->nb) bk = ti->nb;
    lo = ti->first[bk];
    if (bk < ti->nb) hi = imin(hi, ti->first[bk + 1]);
    if (lo > hi) lo = hi;
  }
  while (lo < hi) {
    const int32_t m = (lo + hi) >> 1;
    const int64_t x = arr[ix ? ix[m] : m];
    if (strict ? x > v : x >= v) hi = m; else lo = m + 1;
  }
  return lo;
}

TSL_HD int tindex_shift(int64_t max_key, int32_t nb = TI_NB) {
  int sh = 0;
  while (max_key > 0 && (max_key >> sh) >= nb) ++sh;
  return sh;
}

// Builds first[0..nb] for keys[0, n) (nondecreasing, >= 0); CTA-collective
// (kWarp: warp-collective).
template <class X, bool kWarp = false>
TSL_HD void build_tindex(X& x, const int64_t* keys, int32_t n, int32_t* first, int shift, int32_t nb) {
  const int32_t t0 = kWarp ? x.lane : x.tid, dt = kWarp ? X::W : x.nthr;
  for (int32_t k = t0; k <= n; k += dt) {
    // buckets b with key(k-1) < (b << shift) <= key(k) get first[b] = k
    int64_t lo = k == 0 ? 0 : (keys[k - 1] >> shift) + 1;
    if (k > 0 && keys[k - 1] < 0) lo = 0;
    int64_t hi = k == n ? nb : (keys[k] < 0 ? -1 : (keys[k] >> shift));
    if (k < n && keys[k] >= 0 && (keys[k] & ((int64_t(1) << shift) - 1)) != 0) hi = keys[k] >> shift;
    if (hi > nb) hi = nb;
    for (int64_t b = lo; b <= hi; ++b) first[b] = k;
  }
  if constexpr (kWarp) x.wsync();
  else x.sync();
}

// Positions a stream on the intervals that intersect [b, e) (lifted).
// (s0, eN) are the run's first start and last end, loaded once per query.
TSL_HD void stream_open(Stream& q, int32_t n, bool fwd, int64_t b, int64_t e, int64_t s0, int64_t eN) {
  q.n = n;
  const int64_t L = b - q.sh, H = e - q.sh;
  if (n == 0 || eN <= L || s0 >= H) {
    q.i = fwd ? n : 0;
    q.live = false;
    return;
  }
  if (fwd) q.i = search_keys(q.e, q.ix, n, L, true);  // first e > L
  else q.i = search_keys(q.s, q.ix, n, H, false);     // first s >= H
  stream_load(q, fwd, b, e);
}

// A sorted set of swap intervals (pairwise disjoint at shift 0, so ends are
// sorted too): the pass-start busy structure, this pass's commits, or a
// speculative candidate's own commits.
struct Src {
  const int64_t* s;
  const int64_t* e;
  int32_t n;
  TIndex is, ie;  // optional time indexes over starts / ends
};

struct FitQuery {
  int32_t store;
  int64_t b, e, d;   // window [b, e], duration d
  bool has_extra;    // busy_intervals' `extra` (lifted like the others)
  int64_t xs, xe;
};

constexpr int64_t NONE = INT64_MIN;

// busy_intervals (swap_planner.cpp:39-50) restricted to [b, e) + the
// feasible_regions sweep + place_earliest / place_latest. Returns the
// placement start, or NONE when no region of length >= d exists.
// Forward sweep (earliest) stops at the first maximal free interval of length
// >= d; the reverse sweep (latest) enumerates the same maximal free intervals
// from the right.
//
// Streams sit in fixed slots (source t in {src0, src1, storage accesses} x
// lift k in {-P, 0, +P}, plus the <= 3 lifted copies of `extra`), and every
// loop over slots is unrolled, so the merge state stays in registers: the
// sweep is a chain of dependent global loads only, never local memory.
struct NoWarp {
  static constexpr bool kWarp = false;
  TSL_HD int lane() const { return 0; }
  TSL_HD int64_t shfl(int64_t v, int) const { return v; }
};

// Lane helper of a warp-redundant caller (fit's stream openings in parallel).
template <class X>
struct WarpOf {
  static constexpr bool kWarp = X::W > 1;
  X& x;
  TSL_HD int lane() const { return x.lane; }
  TSL_HD int64_t shfl(int64_t v, int src) const { return x.shfl(v, src); }
};

template <class CLK, class WP = NoWarp>
TSL_HD_FORCE int64_t fit(const JobDev& J, const JobState& st, const FitQuery& q, bool latest, const Src* src,
                            int nsrc, int64_t* swept, CLK clk, int64_t* prof, WP wp = WP{}) {
  if (q.e <= q.b) return NONE;
  int64_t tp0 = prof ? clk() : 0;
  const bool fwd = !latest;
  const int64_t P = imax(1, st.period);
  const int32_t a0 = J.s_off[q.store], na = J.s_off[q.store + 1] - a0;
  const int64_t* SS[3] = {nsrc > 0 ? src[0].s : nullptr, nsrc > 1 ? src[1].s : nullptr, J.a_start};
  const int64_t* SE[3] = {nsrc > 0 ? src[0].e : nullptr, nsrc > 1 ? src[1].e : nullptr, J.a_end};
  const int32_t* IX[3] = {nullptr, nullptr, J.s_acc + a0};
  const int32_t SN[3] = {nsrc > 0 ? src[0].n : 0, nsrc > 1 ? src[1].n : 0, na};
  const TIndex NOI{nullptr, 0, 0};
  const TIndex TIS[3] = {nsrc > 0 ? src[0].is : NOI, nsrc > 1 ? src[1].is : NOI, NOI};
  const TIndex TIE[3] = {nsrc > 0 ? src[0].ie : NOI, nsrc > 1 ? src[1].ie : NOI, NOI};
  int64_t S0[3], EN[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const bool any = SN[t] > 0;
    S0[t] = any ? SS[t][IX[t] ? IX[t][0] : 0] : 0;
    EN[t] = any ? SE[t][IX[t] ? IX[t][SN[t] - 1] : SN[t] - 1] : 0;
  }
  if (prof) { int64_t t = clk(); prof[0] += t - tp0; tp0 = t; }
  int32_t I[9];
  int64_t HS[9], HE[9];
  bool LIVE[9];
  // opens stream z = (source t, lift k): the first interval that can touch
  // the window, found by one search
  auto open = [&](int z, int32_t& oi, int64_t& ohs, int64_t& ohe, bool& olive) {
    const int t = z / 3, k = z % 3;
    const int64_t sh = (k - 1) * P;
    const int32_t n = SN[t];
    const int64_t L = q.b - sh, H = q.e - sh;
    olive = false;
    oi = 0;
    ohs = ohe = 0;
    if (n == 0 || EN[t] <= L || S0[t] >= H) return;
    int64_t tq = prof ? clk() : 0;
    int32_t i;
    if (fwd) i = search_keys(SE[t], IX[t], n, L, true, &TIE[t]);
    else i = search_keys(SS[t], IX[t], n, H, false, &TIS[t]);
    if (prof) { prof[3 + t] += clk() - tq; prof[6 + t] += 1; }
    oi = i;
    const int32_t h = fwd ? i : i - 1;
    if (h >= 0 && h < n) {
      const int32_t k2 = IX[t] ? IX[t][h] : h;
      ohs = SS[t][k2] + sh;
      ohe = SE[t][k2] + sh;
      olive = fwd ? ohs < q.e : ohe > q.b;
    }
  };
  if constexpr (WP::kWarp) {
    // warp-redundant caller: lane z opens stream z, the searches overlap
    int32_t mi = 0;
    int64_t mhs = 0, mhe = 0;
    bool ml = false;
    if (wp.lane() < 9) open(wp.lane(), mi, mhs, mhe, ml);
#pragma unroll
    for (int z = 0; z < 9; ++z) {
      I[z] = int32_t(wp.shfl(mi, z));
      HS[z] = wp.shfl(mhs, z);
      HE[z] = wp.shfl(mhe, z);
      LIVE[z] = wp.shfl(ml ? 1 : 0, z) != 0;
    }
    if (prof) { int64_t t = clk(); prof[1] += t - tp0; tp0 = t; }
  } else {
#pragma unroll
    for (int z = 0; z < 9; ++z) open(z, I[z], HS[z], HE[z], LIVE[z]);
  }
  // lifted copies of `extra`, ascending
  int64_t XS[3], XE[3];
  int nex = 0;
#pragma unroll
  for (int k = -1; k <= 1; ++k) {
    const int64_t sh = k * P;
    XS[k + 1] = XE[k + 1] = 0;
    if (q.has_extra && q.xe > q.xs && q.xe + sh > q.b && q.xs + sh < q.e) {
      if (nex == 0) { XS[0] = q.xs + sh; XE[0] = q.xe + sh; }
      else if (nex == 1) { XS[1] = q.xs + sh; XE[1] = q.xe + sh; }
      else { XS[2] = q.xs + sh; XE[2] = q.xe + sh; }
      ++nex;
    }
  }
  int xi = fwd ? 0 : nex;  // extra cursor
  if (prof) { int64_t t = clk(); prof[1] += t - tp0; tp0 = t; }
  int64_t n_swept = 0;
  int64_t result = NONE;
  if (fwd) {
    int64_t cursor = q.b;
    bool found = false;
    for (;;) {
      int best = -1;
      int64_t bs = 0, be = 0;
#pragma unroll
      for (int z = 0; z < 9; ++z)
        if (LIVE[z] && (best < 0 || HS[z] < bs)) { best = z; bs = HS[z]; be = HE[z]; }
      if (xi < nex) {
        const int64_t xs = xi == 0 ? XS[0] : (xi == 1 ? XS[1] : XS[2]);
        if (best < 0 || xs < bs) { best = 9; bs = xs; be = xi == 0 ? XE[0] : (xi == 1 ? XE[1] : XE[2]); }
      }
      if (best < 0) break;
      if (best == 9) {
        ++xi;
      } else {
#pragma unroll
        for (int z = 0; z < 9; ++z) {
          if (z != best) continue;
          const int t = z / 3;
          const int64_t sh = (z % 3 - 1) * P;
          const int32_t i = ++I[z];
          LIVE[z] = i < SN[t];
          if (LIVE[z]) {
            const int32_t k2 = IX[t] ? IX[t][i] : i;
            HS[z] = SS[t][k2] + sh;
            HE[z] = SE[t][k2] + sh;
            LIVE[z] = HS[z] < q.e;
          }
        }
      }
      if (be <= bs) continue;  // lift_into drops empty intervals
      ++n_swept;
      const int64_t cs = imax(bs, q.b), ce = imin(be, q.e);
      if (ce <= cs) continue;
      if (cs > cursor && cs - cursor >= q.d) { found = true; break; }
      cursor = imax(cursor, ce);
    }
    if (found || (q.e > cursor && q.e - cursor >= q.d)) result = cursor;
  } else {
    int64_t cur = q.e;
    bool found = false;
    for (;;) {
      int best = -1;
      int64_t bs = 0, be = 0;
#pragma unroll
      for (int z = 0; z < 9; ++z)
        if (LIVE[z] && (best < 0 || HE[z] > be)) { best = z; bs = HS[z]; be = HE[z]; }
      if (xi > 0) {
        const int64_t xe = xi == 1 ? XE[0] : (xi == 2 ? XE[1] : XE[2]);
        if (best < 0 || xe > be) { best = 9; be = xe; bs = xi == 1 ? XS[0] : (xi == 2 ? XS[1] : XS[2]); }
      }
      if (best < 0) break;
      if (best == 9) {
        --xi;
      } else {
#pragma unroll
        for (int z = 0; z < 9; ++z) {
          if (z != best) continue;
          const int t = z / 3;
          const int64_t sh = (z % 3 - 1) * P;
          const int32_t i = --I[z];
          LIVE[z] = i > 0;
          if (LIVE[z]) {
            const int32_t k2 = IX[t] ? IX[t][i - 1] : i - 1;
            HS[z] = SS[t][k2] + sh;
            HE[z] = SE[t][k2] + sh;
            LIVE[z] = HE[z] > q.b;
          }
        }
      }
      if (be <= bs) continue;
      ++n_swept;
      const int64_t cs = imax(bs, q.b), ce = imin(be, q.e);
      if (ce <= cs) continue;
      if (cur > ce && cur - ce >= q.d) { found = true; break; }
      cur = imin(cur, cs);
    }
    if (found || (cur > q.b && cur - q.b >= q.d)) result = cur - q.d;
  }
  if (swept) *swept += n_swept;
  if (prof) { prof[2] += clk() - tp0; prof[9] += n_swept; }
  return result;
}

struct NoClock {
  TSL_HD int64_t operator()() const { return 0; }
};

// ----------------------------------------------------------------------------
// Plan mutation helpers
// ----------------------------------------------------------------------------

// anchor, swap_planner.cpp:76-93: the access with the greatest end <= t, ties
// to the larger id; ends never decrease with the id, so it is the last one.
TSL_HD_FORCE void anchor(const JobDev& J, const JobState& st, int64_t t, bool wrapped, int64_t& trig,
                   int64_t& delta) {
  if (wrapped && st.period > 0) t = ((t % st.period) + st.period) % st.period;
  const TIndex ti{J.ai_e, st.ai_shift, J.ti_nb};
  const int32_t lo = search_keys(J.a_end, nullptr, J.A, t, true, &ti);
  if (lo == 0) { trig = -1; delta = t; }
  else { trig = lo - 1; delta = t - J.a_end[lo - 1]; }
}

// Last storage access with end <= t (skipping `skip`), or -1.
TSL_HD_FORCE int32_t preceding_access(const JobDev& J, int32_t store, int64_t t, int64_t skip) {
  const int32_t a0 = J.s_off[store], a1 = J.s_off[store + 1];
  int32_t lo = a0, hi = a1;  // first position with end > t
  while (lo < hi) {
    int32_t m = (lo + hi) >> 1;
    if (J.a_end[J.s_acc[m]] <= t) lo = m + 1; else hi = m;
  }
  for (int32_t k = lo - 1; k >= a0; --k)
    if (J.s_acc[k] != skip) return J.s_acc[k];
  return -1;
}

// One committed (or speculatively scored) out/in pair, with its anchors and
// the release flag it sets already resolved (make_event, swap_planner.cpp:95-113;
// flag_release_before, :115-122).
struct PairRec {
  int64_t os, oe, o_earl, o_late, otrig, odelta;
  int64_t is, ie, i_earl, i_late, itrig, idelta;
  int64_t serves;
  int32_t store, pre;
  int32_t wraps, pad;
  int64_t pad2;
};

struct PairSpec {
  int32_t store;
  int64_t os, oe, o_earl, o_late;
  int64_t is, ie, i_earl, i_late;
  bool wraps;
  int64_t serves;
  bool in_at_iter_start;  // schedule_wrapped_swap's forced anchor (swap_planner.cpp:448-452)
};

TSL_HD PairRec resolve_pair(const JobDev& J, const JobState& st, const PairSpec& p) {
  PairRec r;
  r.os = p.os; r.oe = p.oe; r.o_earl = p.o_earl; r.o_late = p.o_late;
  r.is = p.is; r.ie = p.ie; r.i_earl = p.i_earl; r.i_late = p.i_late;
  r.serves = p.serves; r.store = p.store; r.wraps = p.wraps ? 1 : 0; r.pad = 0;
  anchor(J, st, p.os, p.wraps, r.otrig, r.odelta);
  if (p.in_at_iter_start) { r.itrig = -1; r.idelta = p.is - st.period; }
  else anchor(J, st, p.is, p.wraps, r.itrig, r.idelta);
  r.pre = preceding_access(J, p.store, p.os, -2);
  return r;
}

// resolve_pair with its three searches on three lanes (warp-collective).
template <class X>
TSL_HD PairRec resolve_pair_warp(X& x, const JobDev& J, const JobState& st, const PairSpec& p) {
  if constexpr (X::W == 1) {
    return resolve_pair(J, st, p);
  } else {
    PairRec r;
    r.os = p.os; r.oe = p.oe; r.o_earl = p.o_earl; r.o_late = p.o_late;
    r.is = p.is; r.ie = p.ie; r.i_earl = p.i_earl; r.i_late = p.i_late;
    r.serves = p.serves; r.store = p.store; r.wraps = p.wraps ? 1 : 0; r.pad = 0;
    // lanes 0 and 1 anchor the swap-out and swap-in through the same call
    int64_t trig = 0, delta = 0;
    if (x.lane < 2) anchor(J, st, x.lane ? p.is : p.os, p.wraps, trig, delta);
    r.otrig = x.shfl(trig, 0); r.odelta = x.shfl(delta, 0);
    if (p.in_at_iter_start) { r.itrig = -1; r.idelta = p.is - st.period; }
    else { r.itrig = x.shfl(trig, 1); r.idelta = x.shfl(delta, 1); }
    r.pre = preceding_access(J, p.store, p.os, -2);
    return r;
  }
}

// This pass's committed intervals of one job ("pend"): s/e[0, pend_n), the
// prefix [0, pend_sorted) sorted by start, every commit since (taken verbatim
// from the speculation or re-scored) appended unsorted; ts/te are the merge
// target, tmp 2 * cap scratch words. The arrays sit in the sort scratch of
// shared memory when the pass's bound fits there, else in the job's global
// buffers.
struct PendBuf {
  int64_t *s, *e, *ts, *te, *tmp;
  int32_t cap;
};

// Before a re-score the (short) unsorted suffix is ranked and merged in with
// binary searches. Warp-collective.
template <class X>
TSL_HD void pend_sort(X& x, PendBuf& pb, JobState& st, bool pingpong = true) {
  const int32_t n = st.pend_n, p = st.pend_sorted;
  if (p >= n) return;
  const int32_t k = n - p;
  int64_t* ts = pb.tmp;      // sorted suffix
  int64_t* te = pb.tmp + k;
  x.wsync();
  for (int32_t i = x.lane; i < k; i += X::W) {
    const int64_t si = pb.s[p + i];
    int32_t r = 0;
    for (int32_t t = 0; t < k; ++t) {
      const int64_t sj = pb.s[p + t];
      r += (sj < si || (sj == si && t < i)) ? 1 : 0;
    }
    ts[r] = si;
    te[r] = pb.e[p + i];
  }
  x.wsync();
  // merge prefix [0, p) and sorted suffix ts[0, k) into the merge target,
  // prefix first on equal starts, then the two buffers swap roles
  if (k <= X::W) {
    // a few new entries (the usual case: the verbatim commits since the last
    // re-score): scatter, no dependent search. Prefix entry i moves past the
    // new entries that start strictly before it; new entry r lands after every
    // prefix entry that starts at or before it.
    const int64_t my_s = x.lane < k ? ts[x.lane] : 0, my_e = x.lane < k ? te[x.lane] : 0;
    int32_t before = 0;
    for (int32_t c0 = 0; c0 < p; c0 += X::W) {
      const int32_t i = c0 + x.lane;
      const bool valid = i < p;
      const int64_t si = valid ? pb.s[i] : 0, ei = valid ? pb.e[i] : 0;
      int32_t lt = 0;
      for (int32_t r = 0; r < k; ++r) {
        const int64_t v = x.shfl(my_s, r);
        lt += (valid && v < si) ? 1 : 0;
        const int32_t le = popc32(x.wballot(valid && si <= v));
        if (x.lane == r) before += le;
      }
      if (valid) { pb.ts[i + lt] = si; pb.te[i + lt] = ei; }
    }
    if (x.lane < k) { pb.ts[x.lane + before] = my_s; pb.te[x.lane + before] = my_e; }
  } else {
    // one contiguous output range per lane (merge-path split)
    const int32_t per = (n + X::W - 1) / X::W;
    const int32_t d0 = imin(n, int64_t(x.lane) * per), d1 = imin(n, int64_t(d0) + per);
    int32_t lo = imax(0, d0 - k), hi = imin(d0, p);
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (pb.s[mid] <= ts[d0 - mid - 1]) lo = mid + 1; else hi = mid;
    }
    int32_t i = lo, r = d0 - lo;
    for (int32_t d = d0; d < d1; ++d) {
      if (i < p && (r >= k || pb.s[i] <= ts[r])) { pb.ts[d] = pb.s[i]; pb.te[d] = pb.e[i]; ++i; }
      else { pb.ts[d] = ts[r]; pb.te[d] = te[r]; ++r; }
    }
  }
  x.wsync();
  if (pingpong) {
    int64_t* os = pb.s;
    int64_t* oe = pb.e;
    pb.s = pb.ts; pb.e = pb.te;  // every lane holds its own copy of pb
    pb.ts = os; pb.te = oe;
  } else {  // a caller that rebuilds its PendBuf from the job's arrays
    for (int32_t d = x.lane; d < n; d += X::W) { pb.s[d] = pb.ts[d]; pb.e[d] = pb.te[d]; }
  }
  x.wsync();
  st.pend_sorted = n;
  x.wsync();
}

// Re-scoring context (one warp, warp-redundant): busy = pass-start structure
// + every interval committed earlier in this pass (sorted by pend_sort at the
// re-score's start); pairs are recorded into the candidate's pool slot.
template <class X>
struct ReCtx {
  static constexpr bool kParallelGaps = true;
  using XT = X;
  X& x;
  const JobDev& J;
  JobState& st;
  const PendBuf& pb;
  const GroupConfig& cfg;
  GroupStats* gs;
  PairRec* out;
  int32_t nout, cap;
  bool overflow;
  int64_t* dbg = nullptr;  // development cycle counters (thread 0 only)
  // component speculation records the placement window of every successful
  // query (as SpecCtx does) for the later validity checks
  int64_t* win = nullptr;  // (lo, hi) pairs
  int32_t nwin = 0, cap_win = 0;
  TSL_HD void record(int64_t r, int64_t d) {
    if (!win || r == NONE) return;
    if (nwin >= cap_win) { overflow = true; return; }
    if (x.lane == 0) { win[2 * nwin] = r; win[2 * nwin + 1] = r + d; }
    ++nwin;
  }
  // a query made by one lane on its own (gap pairs in parallel)
  TSL_HD int64_t query_lane(const FitQuery& q, bool latest) {
    Src src[2] = {{J.bz_s, J.bz_e, st.bz_n, {J.bzi_s, st.bzi_shift, J.ti_nb}, {J.bzi_e, st.bzi_shift, J.ti_nb}},
                   {pb.s, pb.e, st.pend_sorted, {nullptr, 0, 0}, {nullptr, 0, 0}}};
    int64_t sw = 0;
    const int64_t r = fit(J, st, q, latest, src, 2, &sw, NoClock{}, nullptr);
    if (x.lane == 0) { gs->fit_queries += 1; gs->busy_intervals += sw; }
    return r;
  }
  TSL_HD int64_t query(const FitQuery& q, bool latest) {
    const int64_t c0 = x.clock();
    Src src[2] = {{J.bz_s, J.bz_e, st.bz_n, {J.bzi_s, st.bzi_shift, J.ti_nb}, {J.bzi_e, st.bzi_shift, J.ti_nb}},
                   {pb.s, pb.e, st.pend_sorted, {nullptr, 0, 0}, {nullptr, 0, 0}}};
    int64_t sw = 0;
#if TSL_PROF
    // development profile (TSL_PROF builds only): per-source search cycles
    // summed over the lanes that opened them, the rest from lane 0
    int64_t lp[10] = {};
    auto clk = [] { return int64_t(clock64()); };
    int64_t r = fit(J, st, q, latest, src, 2, &sw, clk, lp, WarpOf<X>{x});
    for (int k = 0; k < 10; ++k) {
      int64_t v = lp[k];
      if (k >= 3 && k <= 8)
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (x.lane == 0) gs->prof[k] += v;
    }
    if (x.lane == 0) gs->prof[10] += 1;
#else
    int64_t r = fit(J, st, q, latest, src, 2, &sw, NoClock{}, nullptr, WarpOf<X>{x});
#endif
    record(r, q.d);
    gs->fit_queries += 1;
    gs->busy_intervals += sw;
    if (dbg && x.tid == 0) { dbg[0] += x.clock() - c0; dbg[1] += 1; }
    return r;
  }
  // No later query of the same schedule can see this commit (the swap-in
  // query gets the swap-out as `extra`; gap windows are disjoint from the
  // main pair and from each other inside [0, P]), so the intervals are only
  // appended, unsorted, for the next re-score's pend_sort.
  TSL_HD bool commit(const PairSpec& p) {
    const int64_t c0 = x.clock();
    const int32_t pn = st.pend_n;
    if (nout >= cap || pn + 2 > pb.cap) { overflow = true; return false; }
    const PairRec r = resolve_pair_warp(x, J, st, p);
    if (dbg && x.tid == 0) { dbg[2] += x.clock() - c0; }
    x.wsync();
    if (x.lane == 0) {
      out[nout] = r;
      pb.s[pn] = r.os; pb.e[pn] = r.oe;
      pb.s[pn + 1] = r.is; pb.e[pn + 1] = r.ie;
    }
    st.pend_n = pn + 2;
    ++nout;
    x.wsync();
    if (dbg && x.tid == 0) { dbg[3] += x.clock() - c0; }
    return true;
  }
};

constexpr int GS_PCAP = 160;    // gsh slots: per-job reserved pair slots of a pass (<= 128 jobs)
constexpr int GS_POFF = 300;    // gsh slots: per-job pend buffer offsets in shared scratch
constexpr int GS_WK = 440;      // gsh slot: window-index bucket shift + 1 (0: no window index this pass)
constexpr int GS_NB = 441;      // gsh slot: bucket count of this pass's indexes
constexpr int GS_PPOOL = 442;   // gsh slot: pair-pool bump counter of the pass
constexpr int GS_WPOOL = 443;   // gsh slot: window-pool bump counter of the pass
constexpr int GS_CCHG = 444;    // gsh slot: component union-find round changed something
constexpr int GS_CRUN = 445;    // gsh slot: next component run to process
constexpr int GS_NRUN = 446;    // gsh slot: component runs of >= 2 members
constexpr int GS_QTOT = 448;    // gsh slots [448, 456): phase B prefix quarters' totals
static_assert(MAXB * 16 + GS_POFF + 128 < SH_WORDS - 1, "gsh slots overlap the clock word (NF == 16)");
static_assert(MAXB * 16 + 456 < SH_WORDS - 1, "gsh slots overlap the clock word (NF == 16)");
constexpr int CAPC = 7;         // conflict list entries per candidate
constexpr int CB_NB = 1024;     // time buckets of the conflict index
constexpr int CB_GRID_MAX = 160;  // passes with at most this many candidates check all pairs directly

// Speculative context (one thread, one candidate): busy = the pass-start
// structure. The schedule's own commits never reach its later queries (the
// swap-in query gets the swap-out as `extra`; gap windows lie right of the
// main pair and of each other inside [0, P], lifted copies included), so no
// private interval list is kept. Pairs and the placement window of every
// successful query are recorded for validation at commit time.
struct SpecCtx {
  static constexpr bool kParallelGaps = false;
  using XT = void;
  const JobDev& J;
  const JobState& st;
  const GroupConfig& cfg;
  GroupStats* gs;
  PairRec* pairs;
  int32_t npairs, cap_pairs;
  int64_t* win;  // (lo, hi) pairs
  int32_t nwin, cap_win;
  bool overflow;
  TSL_HD int64_t query(const FitQuery& q, bool latest) {
    Src src[1] = {{J.bz_s, J.bz_e, st.bz_n, {J.bzi_s, st.bzi_shift, J.ti_nb}, {J.bzi_e, st.bzi_shift, J.ti_nb}}};
    int64_t sw = 0;
    int64_t r = fit(J, st, q, latest, src, 1, &sw, NoClock{}, nullptr);
    gs->fit_queries += 1;
    gs->busy_intervals += sw;
    if (r != NONE) {
      // Adding busy intervals only removes free space, so a failed query
      // stays failed, and a found placement [r, r+d) moves only if a new
      // interval (any lifted copy) intersects it: regions left of it were
      // already shorter than d (earliest-fit) or its region only shrinks to a
      // length still >= d, and symmetrically for latest-fit.
      if (nwin >= cap_win) { overflow = true; return r; }
      win[2 * nwin] = r;
      win[2 * nwin + 1] = r + q.d;
      ++nwin;
    }
    return r;
  }
  TSL_HD bool commit(const PairSpec& p) {
    if (npairs >= cap_pairs) { overflow = true; return false; }
    pairs[npairs++] = resolve_pair(J, st, p);
    return true;
  }
};

// try_gap_pair, swap_planner.cpp:126-152.
template <class C>
TSL_HD bool try_gap_pair(C& c, int32_t store, int64_t lo, int64_t hi, int64_t serves) {
  const int64_t d = duration(c.J.t_size[store], c.cfg);
  if (hi - lo < 2 * d) return false;
  const int64_t os = c.query(FitQuery{store, lo, hi, d, false, 0, 0}, false);
  if (os == NONE) return false;
  // the busy list is the one filtered for [lo, hi) plus the out interval; the
  // in-regions re-clip to [out.end, hi], where that out interval is empty.
  const int64_t is = c.query(FitQuery{store, os + d, hi, d, false, 0, 0}, true);
  if (is == NONE) return false;
  return c.commit(PairSpec{store, os, os + d, lo, hi, is, is + d, os + d, hi, false, serves, false});
}

// The gap pairs of one schedule are independent of each other: gap k's window
// [end of access k, start of access k+1) lies inside [0, P], the windows are
// disjoint, and a commit inside one window (also inside [0, P]) cannot reach
// another window through its -P/+P lifted copies. A warp therefore places
// every gap at once (one lane per gap, against the state before any gap
// commit) and then commits the successful ones in order -- exactly what the
// reference's sequential loop (swap_planner.cpp:389-395) produces.
template <class C>
TSL_HD void gap_pairs_parallel(C& c, int32_t store, int32_t fk, int32_t a1, int64_t d) {
  const JobDev& J = c.J;
  auto& x = c.x;
  using X = typename C::XT;
  const int64_t g0 = x.clock();
  for (int32_t k0 = fk; k0 + 1 < a1; k0 += X::W) {
    const int32_t k = k0 + x.lane;
    bool ok = false;
    int64_t lo = 0, hi = 0, os = NONE, is = NONE, serves = -1;
    if (k + 1 < a1) {
      const int32_t a = J.s_acc[k], b = J.s_acc[k + 1];
      if (J.a_type[b] == ACC_TUA) {
        lo = J.a_end[a];
        hi = J.a_start[b];
        serves = b;
        if (hi - lo >= 2 * d) {
          os = c.query_lane(FitQuery{store, lo, hi, d, false, 0, 0}, false);
          if (os != NONE) {
            is = c.query_lane(FitQuery{store, os + d, hi, d, false, 0, 0}, true);
            ok = is != NONE;
          }
        }
      }
    }
    if (c.win) {  // both placements of every lane whose queries succeeded (ordered by lane)
      const int32_t nw = (os != NONE ? 1 : 0) + (is != NONE ? 1 : 0);
      int32_t tot = 0;
      const int32_t ex = x.wexcl(nw, &tot);
      if (c.nwin + tot > c.cap_win) { c.overflow = true; return; }
      if (os != NONE) { c.win[2 * (c.nwin + ex)] = os; c.win[2 * (c.nwin + ex) + 1] = os + d; }
      if (is != NONE) { c.win[2 * (c.nwin + ex + 1)] = is; c.win[2 * (c.nwin + ex + 1) + 1] = is + d; }
      c.nwin += tot;
      x.wsync();
    }
    const unsigned okm = x.wballot(ok);
    for (int t = 0; t < X::W; ++t) {
      if (!(okm >> t & 1u)) continue;
      const int64_t tlo = x.shfl(lo, t), thi = x.shfl(hi, t), tos = x.shfl(os, t), tis = x.shfl(is, t);
      const int64_t tsv = x.shfl(serves, t);
      if (!c.commit(PairSpec{store, tos, tos + d, tlo, thi, tis, tis + d, tos + d, thi, false, tsv, false})) return;
    }
    if (c.dbg && x.tid == 0) c.dbg[6] += x.clock() - g0;  // cyc[18]: gap pairs
  }
}

// schedule_swap, swap_planner.cpp:339-399, single shot: a failed swap-in
// placement leaves the next retry with the same swap-out region, the same
// first access and the same swap-in window, so the reference's retry loop
// (swap_planner.cpp:503-513) can never succeed after the first failure.
template <class C>
TSL_HD bool schedule_swap(C& c, int32_t store, int64_t earliest, int64_t latest) {
  const JobDev& J = c.J;
  const int64_t d = duration(J.t_size[store], c.cfg);
  const int64_t os = c.query(FitQuery{store, earliest, latest, d, false, 0, 0}, false);
  if (os == NONE) return false;
  const int64_t oe = os + d;
  const int32_t a0 = J.s_off[store], a1 = J.s_off[store + 1];
  int32_t fk = -1;
  for (int32_t k = a0; k < a1; ++k) {
    int32_t a = J.s_acc[k];
    if (J.a_type[a] == ACC_TUA && J.a_start[a] >= oe) { fk = k; break; }
  }
  c.gs->candidate_accesses += a1 - a0;
  if (fk < 0) return false;
  const int32_t fa = J.s_acc[fk];
  const int64_t fs = J.a_start[fa];
  const int64_t is = c.query(FitQuery{store, oe, fs, d, true, os, oe}, true);
  if (is == NONE) return false;
  if (!c.commit(PairSpec{store, os, oe, earliest, latest, is, is + d, oe, fs, false, fa, false})) return false;
  // Greedily keep the tensor offloaded between its remaining uses.
  if constexpr (C::kParallelGaps) {
    gap_pairs_parallel(c, store, fk, a1, d);
  } else {
    for (int32_t k = fk; k + 1 < a1; ++k) {
      int32_t a = J.s_acc[k], b = J.s_acc[k + 1];
      if (J.a_type[b] != ACC_TUA) continue;
      try_gap_pair(c, store, J.a_end[a], J.a_start[b], b);
    }
  }
  return true;
}

// schedule_wrapped_swap, swap_planner.cpp:401-459.
template <class C>
TSL_HD bool schedule_wrapped_swap(C& c, int32_t param) {
  const JobDev& J = c.J;
  if (J.t_upd[param] < 0) return false;
  const int64_t d = duration(J.t_size[param], c.cfg);
  const int64_t period = c.st.period;
  const int32_t ut = J.t_utga[param];
  const int64_t tga_end = ut >= 0 ? J.a_end[ut] : -1;
  if (tga_end < 0) return false;
  const int64_t os = c.query(FitQuery{param, tga_end, period, d, false, 0, 0}, false);
  if (os == NONE) return false;
  const int32_t fa = J.t_wfirst[param];
  if (fa < 0) return false;
  const int64_t in_lo = period, in_hi = period + J.a_start[fa];
  const int64_t is = c.query(FitQuery{param, in_lo, in_hi, d, true, os, os + d}, true);
  if (is == NONE) return false;
  return c.commit(PairSpec{param, os, os + d, tga_end, period, is, is + d, in_lo, in_hi, true, fa, true});
}

// swap_window, swap_planner.cpp:290-313.
TSL_HD bool swap_window(const JobDev& J, int32_t store, int64_t peak_time, int64_t& earliest, int64_t& latest) {
  latest = peak_time;
  earliest = -1;
  bool has_tga = false;
  for (int32_t k = J.s_off[store]; k < J.s_off[store + 1]; ++k) {
    int32_t a = J.s_acc[k];
    if (J.a_type[a] == ACC_TGA) { has_tga = true; earliest = imax(earliest, J.a_end[a]); }
    if (J.a_start[a] < latest) earliest = imax(earliest, J.a_end[a]);
  }
  if (!has_tga && J.t_kind[store] == K_INTERIM) return false;
  if (earliest < 0) earliest = 0;
  return true;
}

// Which branch swap_pass takes for a candidate (swap_planner.cpp:489-513):
// 1 wrapped, 2 normal (window in earliest/latest), 0 skip, -1 error.
TSL_HD int candidate_kind(const JobDev& J, const JobState& st, int32_t s, int64_t& earliest, int64_t& latest) {
  if (J.t_kind[s] == K_PARAM && J.t_upd[s] >= 0) return 1;
  if (J.s_off[s + 1] - J.s_off[s] <= 1) return 0;
  if (!swap_window(J, s, st.peak_time, earliest, latest)) return -1;
  return latest > earliest ? 2 : 0;
}

// ----------------------------------------------------------------------------
// Stage 1: timeline builder (generate_access_sequence + activity_analysis +
// CSR by storage), one job, whole CTA.
// ----------------------------------------------------------------------------
template <class X>
TSL_HD void build_sequence(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  int64_t* lat = g.x_fp;    // [O] latencies in topo order -> inclusive ends
  int64_t* cnt = g.x_time;  // [O] accesses per op -> inclusive offsets
  for (int32_t k = x.tid; k < J.O; k += x.nthr) {
    int32_t o = J.topo[k];
    lat[k] = J.o_lat[o];
    cnt[k] = (J.o_in_off[o + 1] - J.o_in_off[o]) + (J.o_out_off[o + 1] - J.o_out_off[o]);
  }
  x.sync();
  x.scan(lat, J.O);
  x.scan(cnt, J.O);
  for (int32_t k = x.tid; k < J.O; k += x.nthr) {
    int32_t o = J.topo[k];
    int64_t end = lat[k], start = end - J.o_lat[o];
    int32_t a = int32_t(cnt[k] - ((J.o_in_off[o + 1] - J.o_in_off[o]) + (J.o_out_off[o + 1] - J.o_out_off[o])));
    for (int32_t i = J.o_in_off[o]; i < J.o_in_off[o + 1]; ++i, ++a) {
      int32_t t = J.o_in[i];
      J.a_tensor[a] = t; J.a_store[a] = J.t_store[t]; J.a_type[a] = ACC_TUA;
      J.a_start[a] = start; J.a_end[a] = end;
    }
    for (int32_t i = J.o_out_off[o]; i < J.o_out_off[o + 1]; ++i, ++a) {
      int32_t t = J.o_out[i];
      J.a_tensor[a] = t; J.a_store[a] = J.t_store[t]; J.a_type[a] = ACC_TGA;
      J.a_start[a] = start; J.a_end[a] = end;
    }
  }
  // activity analysis: last access of every tensor id (st_evcnt as scratch)
  for (int32_t t = x.tid; t < J.T; t += x.nthr) J.st_evcnt[t] = -1;
  if (x.tid == 0) { st.period = J.O > 0 ? lat[J.O - 1] : 0; }
  x.sync();
  for (int32_t a = x.tid; a < J.A; a += x.nthr) x.amax32(&J.st_evcnt[J.a_tensor[a]], a);
  x.sync();
  // CSR by storage: stable sort of (storage, access id)
  const int ab = nbits(uint64_t(J.A > 0 ? J.A - 1 : 0));
  for (int32_t a = x.tid; a < J.A; a += x.nthr) {
    int32_t t = J.a_tensor[a];
    uint8_t f = (J.st_evcnt[t] == a && J.t_kind[t] == K_INTERIM) ? 1 : 0;
    J.a_base[a] = f;
    J.a_flag[a] = f;
    g.k_key[a] = (uint64_t(J.a_store[a]) << ab) | uint64_t(a);
    g.k_val[a] = a;
  }
  x.sync();
  x.sort(g.k_key, g.k_val, J.A, ab + nbits(uint64_t(J.T)));
  for (int32_t m = x.tid; m < J.A; m += x.nthr) {
    int32_t a = g.k_val[m];
    J.s_acc[m] = a;
    int32_t cur = J.a_store[a];
    int32_t prev = m == 0 ? -1 : J.a_store[g.k_val[m - 1]];
    for (int32_t s = prev + 1; s <= cur; ++s) J.s_off[s] = m;
    if (m == J.A - 1)
      for (int32_t s = cur + 1; s <= J.T; ++s) J.s_off[s] = J.A;
  }
  if (J.A == 0)
    for (int32_t s = x.tid; s <= J.T; s += x.nthr) J.s_off[s] = 0;
  x.sync();
  for (int32_t t = x.tid; t < J.T; t += x.nthr) {
    int32_t wf = -1, ut = -1;
    const int32_t u = J.t_upd[t];
    if (u >= 0) {
      for (int32_t k = J.s_off[t]; k < J.s_off[t + 1]; ++k) {
        int32_t a = J.s_acc[k];
        if (wf < 0 && J.a_tensor[a] == t && J.a_type[a] == ACC_TUA) wf = a;
        if (J.a_tensor[a] == u && J.a_type[a] == ACC_TGA) ut = a;
      }
    }
    J.t_wfirst[t] = wf;
    J.t_utga[t] = ut;
    J.st_evcnt[t] = 0;
    J.swapped[t] = 0;
    J.in_peak[t] = 0;
  }
  if (x.tid == 0) {
    st.S = 0; st.R = 0; st.n_peak = 0; st.n_curve = 0;
    g.ec_ok = 0; g.ec_S0 = -1;
    st.next_id = 0; st.peak = 0; st.peak_time = 0; st.lua = -1; st.has_lua = 0;
    st.dirty = 1; st.n_events = 0; st.son = 0; st.bz_n = 0; st.bzi_shift = 0;
  }
  x.sync();
  build_anchor_index(x, g, j);
  build_busy_index(x, g, j);
}

// The timeline builder of one job; an execution context may route it
// elsewhere (the CUDA build runs it on every CTA of a cooperative launch).
template <class X>
TSL_HD void seq_batch(X& x, GroupDev& g, int j) {
  build_sequence(x, g, j);
}

// ----------------------------------------------------------------------------
// Stage 2: footprint evaluator for jobs [jb, je) (analyze_job, peak.cpp:246-250)
// ----------------------------------------------------------------------------
// Shared scalar layout per batch job b: sh[b*16 + field].
enum { F_BASE = 0, F_N, F_REL, F_INIT, F_OFF, F_MAXFP, F_PPOS, F_LUA, F_ERR, F_NPEAK, NF = 16 };

// ----------------------------------------------------------------------------
// Incremental timeline order (one-job big builds; GroupDev.ec_*)
// ----------------------------------------------------------------------------
// The timeline sort key (time, frees first, storage rank, type rank) as an
// int64 time and a 32-bit low word. The evaluator's two sorts -- timeline
// order and (storage, timeline) grouping -- are replaced by merges: the
// accesses and every access's potential release (the "base") are sorted once
// per access-time configuration, a release is active iff its access is
// flagged and not owned by a swap-out, and the swap events keep their orders
// from the previous evaluation (a swap pass only appends events), so each
// evaluation sorts only the pass's new events. Ties follow the full sort's
// slot order: swap events (plan order), recomputes, accesses, releases.
TSL_HD uint32_t ev_lo(int type, int32_t rank) {
  const bool fr = type == EV_REL || type == EV_SOUT;
  return (uint32_t(fr ? 0 : 1) << 30) | (uint32_t(rank) << 2) | uint32_t(fr ? type - EV_SOUT : type);
}
TSL_HD uint32_t lo_rank(uint32_t lo) { return (lo >> 2) & 0xffffff; }
TSL_HD uint32_t lo_cls(uint32_t lo) { return ((lo >> 30) << 2) | (lo & 3); }  // class bit, type rank
// timeline order of (time, low word)
TSL_HD bool tl_less(int64_t ta, uint32_t la, int64_t tb, uint32_t lb) { return ta < tb || (ta == tb && la < lb); }
// storage-grouped order: (rank, time, class, type rank)
TSL_HD bool gr_less(int64_t ta, uint32_t la, int64_t tb, uint32_t lb) {
  const uint32_t ra = lo_rank(la), rb = lo_rank(lb);
  if (ra != rb) return ra < rb;
  if (ta != tb) return ta < tb;
  return lo_cls(la) < lo_cls(lb);
}
TSL_HD uint64_t tl_key(int64_t dt, uint32_t lo, int rbits) {
  return (uint64_t(dt) << (rbits + 3)) | (uint64_t(lo >> 30) << (rbits + 2)) | (uint64_t(lo_rank(lo)) << 2) | (lo & 3);
}
TSL_HD uint64_t gr_key(int64_t dt, uint32_t lo, int tbits) {
  return (uint64_t(lo_rank(lo)) << (tbits + 3)) | (uint64_t(dt) << 3) | lo_cls(lo);
}

// Merge-path merge of two sorted slot lists, each with a payload, over every
// thread of x (less is a strict total order on slots). No barrier.
template <class X, class Less>
TSL_HD void merge_slots(X& x, const int32_t* a, const int32_t* ap, int64_t n1, const int32_t* b, const int32_t* bp,
                        int64_t n2, int32_t* out, int32_t* outp, Less less) {
  const int64_t n = n1 + n2;
  const int64_t per = (n + x.nthr - 1) / x.nthr;
  const int64_t d0 = imin(n, int64_t(x.tid) * per), d1 = imin(n, d0 + per);
  if (d0 >= d1) return;
  int64_t lo = imax(0, d0 - n2), hi = imin(d0, n1);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (less(a[mid], b[d0 - mid - 1])) lo = mid + 1; else hi = mid;
  }
  int64_t i = lo, k = d0 - lo;
  for (int64_t d = d0; d < d1; ++d) {
    if (i < n1 && (k >= n2 || less(a[i], b[k]))) { out[d] = a[i]; outp[d] = ap[i]; ++i; }
    else { out[d] = b[k]; outp[d] = bp[k]; ++k; }
  }
}

// New D entries ordered by counting (each entry's rank = the entries before
// it) while there are few of them; a radix sort above this.
constexpr int64_t INC_COUNT_MAX = 8192;

// Timeline positions (E_x_order) and the storage-grouped order (E_x_seq2,
// E_x_key2, and the slots in that order in k_val) of job j's events, from the cached base and D orders. Needs the
// emitted events: times in x_time, D low words in ec_dl, accesses at slot
// acc0 + a and releases at acc0 + A + a.
//
// Positions: an ordered D entry k with base insertion point ins (the base
// entries ordering before it) lands at k + #active base entries before ins; an
// active base entry p lands at #active base entries before p + #D entries
// with ins <= p. One scan of (active, D count) per base entry gives both; the
// grouped order is the same construction over the grouped base. D entries
// keep their insertion points across evaluations (the base does not move).
template <class X>
TSL_HD void inc_order(X& x, GroupDev& g, int j, int64_t n, int rbits, int64_t acc0) {
  const JobDev& J = g.jobs[j];
  const JobState& st = g.st[j];
  int64_t* gsh = x.sh + MAXB * NF;  // [5..8] reductions
  const int32_t A = J.A;
  const int64_t NB = 2 * int64_t(A);
  uint64_t* const kk = g.k_key;
  int32_t* const kv = g.k_val;
  const int64_t* const xt = g.x_time;
  int64_t* const bt = g.ec_bt;
  uint32_t* const bl = g.ec_bl;
  int32_t* const bs = g.ec_bs;
  int64_t* const gt = g.ec_gt;
  uint32_t* const gl = g.ec_gl;
  int32_t* const gb = g.ec_gb;      // base slot of each grouped entry
  int32_t* const ginv = g.ec_ginv;  // base position -> grouped position
  int32_t* const posb = g.ec_posb;  // grouped position -> merged timeline position
  int64_t* const sc = g.ec_sc;
  int64_t* const sc2 = g.ec_sc + (NB + 1);
  uint32_t* const dl = g.ec_dl;
  int32_t* const posd = g.ec_posd;
  const uint8_t* const a_flag = J.a_flag;
  const uint8_t* const a_owned = J.a_owned;
  const int32_t* const a_store = J.a_store;
  const int32_t* const t_rank = J.t_rank;
  auto base_time = [&](int32_t i) -> int64_t {
    const int32_t a = i < A ? i : i - A;
    return (i < A && J.a_type[a] == ACC_TGA) ? J.a_start[a] : J.a_end[a];
  };
  auto base_lo = [&](int32_t i) -> uint32_t {
    const int32_t a = i < A ? i : i - A;
    const int type = i >= A ? EV_REL : (J.a_type[a] == ACC_TGA ? EV_TGA : EV_TUA);
    return ev_lo(type, t_rank[a_store[a]]);
  };
  auto active = [&](int32_t i) -> int64_t { return i < A ? 1 : ((a_flag[i - A] && !a_owned[i - A]) ? 1 : 0); };
  int64_t ic0 = x.clock();
  auto itick = [&](int k) { const int64_t c = x.clock(); if (x.tid == 0) g.stats.sprof[k] += c - ic0; ic0 = c; };
  // 1. the base, once per access-time configuration
  if (!g.ec_ok) {
    if (x.tid == 0) { gsh[5] = INT64_MAX; gsh[6] = INT64_MIN; }
    x.sync();
    {
      int64_t mn = INT64_MAX, mx = INT64_MIN;
      for (int64_t i = x.tid; i < NB; i += x.nthr) { const int64_t t = base_time(int32_t(i)); mn = imin(mn, t); mx = imax(mx, t); }
      if (mn != INT64_MAX) { x.amin(&gsh[5], mn); x.amax(&gsh[6], mx); }
    }
    x.sync();
    const int64_t tmin = gsh[5];
    const int tb = nbits(uint64_t(gsh[6] - gsh[5]));
    if (tb + rbits + 3 > 63) {
      if (x.tid == 0 && !g.err.code) { g.err.code = E_CAPACITY; g.err.job = j; g.err.tensor = NB; g.err.tick = tb + rbits + 3; }
      x.sync();
      return;
    }
    for (int64_t i = x.tid; i < NB; i += x.nthr) {
      kk[i] = tl_key(base_time(int32_t(i)) - tmin, base_lo(int32_t(i)), rbits);
      kv[i] = int32_t(i);
    }
    x.sort(kk, kv, int32_t(NB), tb + rbits + 3);  // stable: ties keep accesses, then releases, by access
    for (int64_t p = x.tid; p < NB; p += x.nthr) {
      const int32_t i = kv[p];
      const uint32_t lo = base_lo(i);
      bs[p] = i; bt[p] = base_time(i); bl[p] = lo;
      kk[p] = lo_rank(lo);
      kv[p] = int32_t(p);
    }
    x.sort(kk, kv, int32_t(NB), rbits);
    for (int64_t q = x.tid; q < NB; q += x.nthr) {
      const int32_t p = kv[q];
      const int32_t i = bs[p];
      gb[q] = i; gt[q] = bt[p]; gl[q] = bl[p]; ginv[p] = int32_t(q);
      const int32_t a = i < A ? i : i - A;
      const int32_t s = a_store[a];
      g.ec_gbst[q] = s;
      g.ec_gbt[q] = i >= A ? int8_t(EV_REL)
                  : J.a_type[a] == ACC_TGA ? int8_t(EV_TGA | (J.a_tensor[a] != s ? 8 : 0)) : int8_t(EV_TUA);
      const uint8_t act = uint8_t(active(i));
      g.ec_act[p] = act;
      g.ec_act[NB + q] = act;
      if (i >= A) { g.ec_ract[a] = act; g.ec_rpos[a] = p; g.ec_rpos[A + a] = int32_t(q); }
    }
    x.sync();
    if (x.tid == 0) { g.ec_ok = 1; g.ec_S0 = -1; }
    x.sync();
    itick(0);
  }
  // 2. D (swap events, recomputes): the new entries ordered, with their base
  // insertion points, merged with the cached orders
  const int64_t nD = int64_t(st.S) + st.R;
  const bool keep = g.ec_S0 >= 0 && st.R == 0 && st.S >= g.ec_S0;
  const int64_t n0 = keep ? g.ec_S0 : 0, nn = nD - n0;
  const int cur = g.ec_cur;
  const int64_t dcap = g.ec_dcap;
  const int32_t* const dord0 = g.ec_dord + cur * dcap;
  const int32_t* const dins0 = g.ec_dins + cur * dcap;
  const int32_t* const dgrp0 = g.ec_dgrp + cur * dcap;
  const int32_t* const gins0 = g.ec_gins + cur * dcap;
  int32_t* const dord = g.ec_dord + (1 - cur) * dcap;
  int32_t* const dins = g.ec_dins + (1 - cur) * dcap;
  int32_t* const dgrp = g.ec_dgrp + (1 - cur) * dcap;
  int32_t* const gins = g.ec_gins + (1 - cur) * dcap;
  // new-entry scratch: ranks, then the ordered lists with their insertion points
  int32_t* const rk_t = kv;
  int32_t* const rk_g = kv + nn;
  int32_t* const nw_t = g.ec_nw;
  int32_t* const nw_ti = g.ec_nw + nn;
  int32_t* const nw_g = g.ec_nw + 2 * nn;
  int32_t* const nw_gi = g.ec_nw + 3 * nn;
  auto d_tl = [&](int32_t u, int32_t v) { return xt[u] != xt[v] || dl[u] != dl[v] ? tl_less(xt[u], dl[u], xt[v], dl[v]) : u < v; };
  auto d_gr = [&](int32_t u, int32_t v) { return xt[u] != xt[v] || dl[u] != dl[v] ? gr_less(xt[u], dl[u], xt[v], dl[v]) : u < v; };
  auto ins_tl = [&](int32_t u) -> int32_t {  // base entries ordering before D slot u (D first on ties)
    const int64_t t = xt[u];
    const uint32_t l = dl[u];
    int64_t lo = 0, hi = NB;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (tl_less(bt[mid], bl[mid], t, l)) lo = mid + 1; else hi = mid;
    }
    return int32_t(lo);
  };
  auto ins_gr = [&](int32_t u) -> int32_t {
    const int64_t t = xt[u];
    const uint32_t l = dl[u];
    int64_t lo = 0, hi = NB;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (gr_less(gt[mid], gl[mid], t, l)) lo = mid + 1; else hi = mid;
    }
    return int32_t(lo);
  };
  itick(7);
  if (nn <= INC_COUNT_MAX) {
    for (int64_t i = x.tid; i < 2 * nn; i += x.nthr) kv[i] = 0;
    x.sync();
    itick(8);
    // pairs (u, v-slice) over the threads; one atomic per (u, slice)
    const int64_t L = nn > 0 ? imax(1, x.nthr / nn) : 1;
    const int64_t ss = (nn + L - 1) / L;
    for (int64_t w = x.tid; w < nn * L; w += x.nthr) {
      const int64_t iu = w % nn, sl = w / nn;
      const int32_t u = int32_t(n0 + iu);
      const int64_t t = xt[u];
      const uint32_t l = dl[u];
      int32_t ct = 0, cg = 0;
      const int64_t v1 = imin(nn, (sl + 1) * ss);
      const int64_t* __restrict__ r_xt = xt;
      const uint32_t* __restrict__ r_dl = dl;
#pragma unroll 4
      for (int64_t iv = sl * ss; iv < v1; ++iv) {
        const int32_t v = int32_t(n0 + iv);
        const int64_t tv = r_xt[v];
        const uint32_t lv = r_dl[v];
        const bool same = tv == t && lv == l;
        ct += (same ? v < u : tl_less(tv, lv, t, l)) ? 1 : 0;
        cg += (same ? v < u : gr_less(tv, lv, t, l)) ? 1 : 0;
      }
      if (ct) x.aadd32(&rk_t[iu], ct);
      if (cg) x.aadd32(&rk_g[iu], cg);
    }
    x.sync();
    itick(9);
    for (int64_t iu = x.tid; iu < nn; iu += x.nthr) {
      const int32_t u = int32_t(n0 + iu);
      nw_t[rk_t[iu]] = u; nw_ti[rk_t[iu]] = ins_tl(u);
      nw_g[rk_g[iu]] = u; nw_gi[rk_g[iu]] = ins_gr(u);
    }
    x.sync();
    itick(10);
  } else {
    if (x.tid == 0) { gsh[7] = INT64_MAX; gsh[8] = INT64_MIN; }
    x.sync();
    {
      int64_t mn = INT64_MAX, mx = INT64_MIN;
      for (int64_t i = n0 + x.tid; i < nD; i += x.nthr) { mn = imin(mn, xt[i]); mx = imax(mx, xt[i]); }
      if (mn != INT64_MAX) { x.amin(&gsh[7], mn); x.amax(&gsh[8], mx); }
    }
    x.sync();
    const int64_t tmin_n = gsh[7];
    const int tbn = nbits(uint64_t(gsh[8] - gsh[7]));
    for (int64_t i = x.tid; i < nn; i += x.nthr) {
      kk[i] = tl_key(xt[n0 + i] - tmin_n, dl[n0 + i], rbits);
      kv[i] = int32_t(n0 + i);
    }
    x.sort(kk, kv, int32_t(nn), tbn + rbits + 3);
    for (int64_t i = x.tid; i < nn; i += x.nthr) { nw_t[i] = kv[i]; nw_ti[i] = ins_tl(kv[i]); }
    x.sync();
    for (int64_t i = x.tid; i < nn; i += x.nthr) {
      kk[i] = gr_key(xt[n0 + i] - tmin_n, dl[n0 + i], tbn);
      kv[i] = int32_t(n0 + i);
    }
    x.sort(kk, kv, int32_t(nn), tbn + rbits + 3);
    for (int64_t i = x.tid; i < nn; i += x.nthr) { nw_g[i] = kv[i]; nw_gi[i] = ins_gr(kv[i]); }
  }
  // (the scan arrays' initial values: active base entries)
  {
    // activity of the base entries, kept across evaluations in both orders:
    // only releases whose activity changed since the last evaluation are
    // rewritten, then both scan inputs expand from the bytes (coalesced).
    // (restrict-qualified views and unrolled strides: several iterations'
    // loads in flight -- these loops are latency-bound at 8 warps per SM)
    const uint8_t* __restrict__ r_flag = a_flag;
    const uint8_t* __restrict__ r_own = a_owned;
    uint8_t* __restrict__ r_ract = g.ec_ract;
    uint8_t* __restrict__ r_act = g.ec_act;
    const int32_t* __restrict__ r_rpos = g.ec_rpos;
#pragma unroll 4
    for (int32_t a = x.tid; a < A; a += x.nthr) {
      const uint8_t now = (r_flag[a] && !r_own[a]) ? 1 : 0;
      if (now != r_ract[a]) {
        r_ract[a] = now;
        r_act[r_rpos[a]] = now;
        r_act[NB + r_rpos[A + a]] = now;
      }
    }
  }
  x.sync();
  {
    const uint8_t* __restrict__ r_act = g.ec_act;
    int64_t* __restrict__ r_sc = sc;
    int64_t* __restrict__ r_sc2 = sc2;
#pragma unroll 4
    for (int64_t i = x.tid; i < NB; i += x.nthr) {
      r_sc[i] = r_act[i];
      r_sc2[i] = r_act[NB + i];
    }
  }
  if (x.tid == 0) { sc[NB] = 0; sc2[NB] = 0; }
  x.sync();
  itick(1);
  merge_slots(x, dord0, dins0, n0, nw_t, nw_ti, nn, dord, dins, d_tl);
  merge_slots(x, dgrp0, gins0, n0, nw_g, nw_gi, nn, dgrp, gins, d_gr);
  x.sync();
  itick(2);
  // 3. D insertion counts, then one scan per order
  for (int64_t k = x.tid; k < nD; k += x.nthr) {
    x.aadd(&sc[dins[k]], int64_t(1) << 32);
    x.aadd(&sc2[gins[k]], int64_t(1) << 32);
  }
  x.sync();
  itick(3);
  x.scan(sc, int32_t(NB + 1));
  x.scan(sc2, int32_t(NB + 1));
  itick(4);
  constexpr int64_t LOW = 0xffffffffLL;
  {
    const int64_t* __restrict__ r_sc = sc;
    const int32_t* __restrict__ r_bs = bs;
    const int32_t* __restrict__ r_ginv = ginv;
    int32_t* __restrict__ r_ord = g.x_order;
    int32_t* __restrict__ r_posb = posb;
#pragma unroll 4
    for (int64_t p = x.tid; p < NB; p += x.nthr) {
      const int64_t e = p > 0 ? r_sc[p - 1] : 0;
      const int64_t c = r_sc[p];
      const int32_t b = r_bs[p], gi = r_ginv[p];
      if (!((c - e) & LOW)) continue;  // inactive release
      const int64_t pos = (e & LOW) + (c >> 32);
      r_ord[pos] = int32_t(acc0 + b);
      r_posb[gi] = int32_t(pos);
    }
  }
  for (int64_t k = x.tid; k < nD; k += x.nthr) {
    const int64_t e = dins[k] > 0 ? sc[dins[k] - 1] : 0;
    const int64_t pos = k + (e & LOW);
    g.x_order[pos] = dord[k];
    posd[dord[k]] = int32_t(pos);
  }
  x.sync();
  itick(5);
  {
    const int64_t* __restrict__ r_sc = sc2;
    const int32_t* __restrict__ r_posb = posb;
    const uint32_t* __restrict__ r_gl = gl;
    const int32_t* __restrict__ r_gb = gb;
    const int8_t* __restrict__ r_gbt = g.ec_gbt;
    const int32_t* __restrict__ r_gbst = g.ec_gbst;
    int32_t* __restrict__ r_seq = g.x_seq2;
    uint64_t* __restrict__ r_key = g.x_key2;
    int32_t* __restrict__ r_kv = kv;
    int8_t* __restrict__ r_gty = g.ec_gty;
    int32_t* __restrict__ r_gst = g.ec_gst;
#pragma unroll 4
    for (int64_t q = x.tid; q < NB; q += x.nthr) {
      const int64_t e = q > 0 ? r_sc[q - 1] : 0;
      const int64_t c = r_sc[q];
      const int32_t pb = r_posb[q], b = r_gb[q], st0 = r_gbst[q];
      const uint32_t l = r_gl[q];
      const int8_t ty = r_gbt[q];
      if (!((c - e) & LOW)) continue;
      const int64_t gpos = (e & LOW) + (c >> 32);
      r_seq[gpos] = pb;
      r_key[gpos] = lo_rank(l);
      r_kv[gpos] = int32_t(acc0 + b);
      r_gty[gpos] = ty;
      r_gst[gpos] = st0;
    }
  }
  for (int64_t r = x.tid; r < nD; r += x.nthr) {
    const int64_t e = gins[r] > 0 ? sc2[gins[r] - 1] : 0;
    const int64_t gpos = r + (e & LOW);
    const int32_t u = dgrp[r];
    g.x_seq2[gpos] = posd[u];
    g.x_key2[gpos] = lo_rank(dl[u]);
    kv[gpos] = u;
    g.ec_gty[gpos] = g.x_type[u];
    g.ec_gst[gpos] = g.x_store[u];
  }
  x.sync();
  itick(6);
  if (x.tid == 0) {
    g.ec_cur = 1 - cur;
    g.ec_S0 = st.R == 0 ? st.S : -1;
    g.stats.sort_elems += 2 * nn;
  }
  (void)n;
  x.sync();
}


template <class X>
TSL_HD bool evaluate(X& x, GroupDev& g, int jb, int je) {
  // The scratch pointers live in the group struct in global memory; local
  // copies keep every store below from forcing a reload of the pointer.
  uint64_t* const E_k_key = g.k_key;
  int32_t* const E_k_val = g.k_val;
  int64_t* const E_x_time = g.x_time;
  int64_t* const E_x_fp = g.x_fp;
  int32_t* const E_x_store = g.x_store;
  int32_t* const E_x_aid = g.x_aid;
  int8_t* const E_x_type = g.x_type;
  int8_t* const E_x_job = g.x_job;
  uint8_t* const E_x_state = g.x_state;
  int32_t* const E_x_seq2 = g.x_seq2;
  uint64_t* const E_x_key2 = g.x_key2;
  int32_t* const E_x_order = g.x_order;
  int64_t* sh = x.sh;
  const int nb = je - jb;
  int64_t et0 = x.clock(), et1;
  auto etick = [&](int k) { et1 = x.clock(); if (x.tid == 0) g.stats.cyc[20 + k] += et1 - et0; et0 = et1; };
  int64_t* gsh = sh + MAXB * NF;  // [0]=tmin [1]=tmax [2]=n_total [3]=bits info [4]=fail
  if (x.tid == 0) {
    for (int b = 0; b < nb; ++b) {
      int64_t* f = sh + b * NF;
      f[F_REL] = 0; f[F_INIT] = 0; f[F_MAXFP] = INT64_MIN; f[F_PPOS] = INT64_MAX;
      f[F_LUA] = -1; f[F_ERR] = INT64_MAX; f[F_NPEAK] = 0;
    }
    gsh[0] = INT64_MAX; gsh[1] = INT64_MIN; gsh[4] = 0;
  }
  // 0. initial residency (peak.cpp:176-190) and release-ownership scratch
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    const int8_t* const t_kind = J.t_kind;
    const int32_t* const t_store = J.t_store;
    uint8_t* const res_init = J.res_init;
    uint8_t* const a_owned = J.a_owned;
    const int32_t T = J.T, A = J.A;
    for (int32_t t = x.tid; t < T; t += x.nthr) {
      int8_t k = t_kind[t];
      res_init[t] = (t_store[t] == t && (k == K_PARAM || k == K_INPUT || k == K_OUTPUT)) ? 1 : 0;
    }
    for (int32_t a = x.tid; a < A; a += x.nthr) a_owned[a] = 0;
  }
  x.sync();
  // 1. wrapped swap-ins leave the initial set; swap-outs own releases; time range
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    const JobState& st = g.st[jb + b];
    int64_t lmin = INT64_MAX, lmax = INT64_MIN;
    if (x.tid == 0 && J.A > 0) { lmin = J.a_start[0]; lmax = J.a_end[J.A - 1]; }
    const int32_t* const L_t_store = J.t_store;
    const int32_t* const L_ev_tensor = J.ev_tensor;
    const int64_t* const L_ev_end = J.ev_end;
    const int64_t* const L_ev_start = J.ev_start;
    const int64_t* const L_ev_trig = J.ev_trig;
    const int8_t* const L_ev_dir = J.ev_dir;
    const int8_t* const L_ev_wraps = J.ev_wraps;
    uint8_t* const L_res_init = J.res_init;
    uint8_t* const L_a_owned = J.a_owned;
    const int64_t* const L_a_end = J.a_end;
    const int64_t* const L_a_start = J.a_start;
    const int32_t* const L_s_off = J.s_off;
    const int32_t* const L_s_acc = J.s_acc;
    const int32_t L_A = J.A;
    for (int32_t i = x.tid; i < st.S; i += x.nthr) {
      const int32_t s = L_t_store[L_ev_tensor[i]];
      int64_t when = L_ev_end[i];
      if (L_ev_dir[i] == 1) {
        if (L_ev_wraps[i]) {
          L_res_init[s] = 0;
          if (st.period > 0) when = ((when % st.period) + st.period) % st.period;
        }
      } else {
        const int64_t tr = L_ev_trig[i];
        if (tr != -1) {
          if (tr < 0 || tr >= L_A) {
            x.amax(&gsh[4], 1);
          } else {
            when = imax(when, L_a_end[tr]);
          }
        }
        // peak.cpp:107-130: a flagged access a loses its release when a
        // swap-out of its storage starts in [a.end, next access start).
        // With m = the last storage access start <= t, that is m < a.end <= t.
        const int64_t t0 = L_ev_start[i];
        const int32_t k0 = L_s_off[s], k1 = L_s_off[s + 1];
        int32_t lo = k0, hi = k1;
        while (lo < hi) {
          int32_t md = (lo + hi) >> 1;
          if (L_a_start[L_s_acc[md]] <= t0) lo = md + 1; else hi = md;
        }
        if (lo > k0) {
          const int64_t m = L_a_start[L_s_acc[lo - 1]];
          int32_t l2 = k0, h2 = k1;  // first position with end > m
          while (l2 < h2) {
            int32_t md = (l2 + h2) >> 1;
            if (L_a_end[L_s_acc[md]] <= m) l2 = md + 1; else h2 = md;
          }
          for (int32_t k = l2; k < k1; ++k) {
            int32_t a = L_s_acc[k];
            if (L_a_end[a] > t0) break;
            L_a_owned[a] = 1;
          }
        }
      }
      lmin = imin(lmin, when);
      lmax = imax(lmax, when);
    }
    for (int32_t r = x.tid; r < st.R; r += x.nthr) {
      const int64_t tg = J.rc_target[r];
      if (tg < 0 || tg >= J.A) { x.amax(&gsh[4], 1); continue; }
      int64_t when = J.a_start[tg] - J.rc_lat[r];
      lmin = imin(lmin, when);
      lmax = imax(lmax, when);
    }
    x.ramin(&gsh[0], lmin);  // (identity values are harmless; a grid context reduces per warp first)
    x.ramax(&gsh[1], lmax);
  }
  x.sync();
  if (gsh[4]) {  // unknown access id in a caller plan (access.cpp:8-10)
    if (x.tid == 0) {
      for (int b = 0; b < nb && !g.err.code; ++b) {
        const JobDev& J = g.jobs[jb + b];
        const JobState& st = g.st[jb + b];
        for (int32_t i = 0; i < st.S; ++i)
          if (J.ev_dir[i] == 0 && J.ev_trig[i] != -1 && (J.ev_trig[i] < 0 || J.ev_trig[i] >= J.A)) {
            g.err.code = E_UNKNOWN_ACCESS; g.err.job = jb + b; g.err.tensor = J.ev_trig[i]; g.err.tick = 0;
            break;
          }
        for (int32_t r = 0; r < st.R && !g.err.code; ++r)
          if (J.rc_target[r] < 0 || J.rc_target[r] >= J.A) {
            g.err.code = E_UNKNOWN_ACCESS; g.err.job = jb + b; g.err.tensor = J.rc_target[r]; g.err.tick = 0;
          }
      }
    }
    x.sync();
    return false;
  }
  // 2. initial footprint; releases counted per contiguous access chunk of
  // each thread and scanned over (job, thread), so release slots are numbered
  // in access order (the scan's per-job totals are the release counts).
  // (one-job big builds order the timeline incrementally, inc_order: events
  // keep fixed slots -- a release at acc0 + A + a -- so only the count is
  // needed, and no sort keys)
  const bool inc = g.ec_bt != nullptr && nb == 1 && g.n_jobs == 1;
  int64_t* rcnt = E_x_fp;  // [nb * nthr] release counts -> offsets (free until step 7)
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    int64_t fp = 0;
    for (int32_t t = x.tid; t < J.T; t += x.nthr) if (J.res_init[t]) fp += J.t_size[t];
    x.radd(&sh[b * NF + F_INIT], fp);
    if (inc) {
      const uint8_t* __restrict__ r_flag = J.a_flag;
      const uint8_t* __restrict__ r_own = J.a_owned;
      int64_t c = 0;
#pragma unroll 4
      for (int32_t a = x.tid; a < J.A; a += x.nthr) c += (r_flag[a] && !r_own[a]) ? 1 : 0;
      x.radd(&sh[b * NF + F_REL], c);
      continue;
    }
    const int32_t ch = (J.A + x.nthr - 1) / x.nthr;
    const int32_t a0 = imin(J.A, int64_t(x.tid) * ch), a1 = imin(J.A, int64_t(a0) + ch);
    int64_t c = 0;
    for (int32_t a = a0; a < a1; ++a) c += (J.a_flag[a] && !J.a_owned[a]) ? 1 : 0;
    rcnt[int64_t(b) * x.nthr + x.tid] = c;
  }
  if (inc) x.sync();
  else x.scan(rcnt, nb * x.nthr);  // inclusive; barriers on both sides
  // 3. bases and key geometry
  if (x.tid == 0) {
    int64_t base = 0, maxT = 1;
    for (int b = 0; b < nb; ++b) {
      const JobDev& J = g.jobs[jb + b];
      const JobState& st = g.st[jb + b];
      int64_t* f = sh + b * NF;
      if (!inc) f[F_REL] = rcnt[int64_t(b + 1) * x.nthr - 1] - (b > 0 ? rcnt[int64_t(b) * x.nthr - 1] : 0);
      f[F_BASE] = base;
      f[F_N] = J.A + f[F_REL] + st.S + st.R;
      base += f[F_N];
      maxT = imax(maxT, J.T);
    }
    gsh[2] = base;
    int64_t tmin = gsh[0], tmax = gsh[1];
    if (tmin > tmax) { tmin = 0; tmax = 0; }
    gsh[0] = tmin;
    const int jbits = nbits(uint64_t(nb - 1)), tbits = nbits(uint64_t(tmax - tmin));
    const int rbits = nbits(uint64_t(maxT - 1));
    gsh[3] = (int64_t(jbits) << 48) | (int64_t(tbits) << 32) | (int64_t(rbits) << 16);
    if (base > g.ecap || jbits + tbits + 1 + rbits + 2 > 63) {
      g.err.code = E_CAPACITY; g.err.job = jb; g.err.tensor = base; g.err.tick = jbits + tbits + rbits + 3;
    }
  }
  x.sync();
  if (g.err.code) return false;
  const int jbits = int(gsh[3] >> 48), tbits = int((gsh[3] >> 32) & 0xffff);
  const int rbits = int((gsh[3] >> 16) & 0xffff);
  const int64_t tmin = gsh[0];
  const int64_t n = gsh[2];
  // Timeline key (sort_timeline, peak.cpp:44-62) without its last field: the
  // reference's final tie (accesses, then swap events in plan order, then
  // recomputes; access ids within each) is the slot order below -- swap
  // events, recomputes, accesses, releases (in access order) -- and the radix
  // sort is stable.
  auto key = [&](int b, int64_t time, int type, int32_t srank) -> uint64_t {
    const bool fr = type == EV_REL || type == EV_SOUT;
    uint64_t k = uint64_t(b);
    k = (k << tbits) | uint64_t(time - tmin);
    k = (k << 1) | (fr ? 0u : 1u);
    k = (k << rbits) | uint64_t(srank);
    // type rank within the free / non-free class: TGA < TUA < SIN and
    // SOUT < REL (the class bit above already orders frees first), 2 bits
    k = (k << 2) | uint64_t(fr ? type - EV_SOUT : type);
    return k;
  };
  etick(0);
  uint32_t* const E_dl = g.ec_dl;
  // 4. emit events (build_timeline, peak.cpp:66-174); release slots from the
  // step-2 scan.
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    const JobState& st = g.st[jb + b];
    int64_t* f = sh + b * NF;
    const int64_t base = f[F_BASE];
    const int64_t acc0 = base + st.S + st.R;  // first access slot
    if (inc) {  // fixed slots: a coalesced strided walk
      const int32_t* __restrict__ a_store = J.a_store;
      const int32_t* __restrict__ a_tensor = J.a_tensor;
      const uint8_t* __restrict__ a_flag = J.a_flag;
      const uint8_t* __restrict__ a_owned = J.a_owned;
      const int8_t* __restrict__ a_type = J.a_type;
      const int64_t* __restrict__ a_start = J.a_start;
      const int64_t* __restrict__ a_end = J.a_end;
      int64_t* __restrict__ r_time = E_x_time + acc0;
      int8_t* __restrict__ r_type = E_x_type + acc0;
      int32_t* __restrict__ r_store = E_x_store + acc0;
      int32_t* __restrict__ r_aid = E_x_aid + acc0;
      int8_t* __restrict__ r_job = E_x_job + acc0;
      const int32_t A = J.A;
#pragma unroll 4
      for (int32_t a = x.tid; a < A; a += x.nthr) {
        const int32_t s = a_store[a];
        const bool flagged = a_flag[a] != 0;
        const bool owned = a_owned[a] != 0;
        const bool tga = a_type[a] == ACC_TGA;
        const int64_t te = a_end[a];
        const int64_t ts = a_start[a];
        r_time[a] = tga ? ts : te;
        r_type[a] = tga ? int8_t(EV_TGA | (a_tensor[a] != s ? 8 : 0)) : int8_t(EV_TUA | (flagged ? 16 : 0));
        r_store[a] = s; r_aid[a] = a; r_job[a] = int8_t(b);
        if (flagged && !owned) {
          r_time[A + a] = te; r_type[A + a] = EV_REL; r_store[A + a] = s; r_aid[A + a] = a; r_job[A + a] = int8_t(b);
        }
      }
    } else {
    const int32_t ch = (J.A + x.nthr - 1) / x.nthr;
    const int32_t a0 = imin(J.A, int64_t(x.tid) * ch), a1 = imin(J.A, int64_t(a0) + ch);
    const int64_t idx = int64_t(b) * x.nthr + x.tid;
    int64_t rel = (idx > 0 ? rcnt[idx - 1] : 0) - (b > 0 ? rcnt[int64_t(b) * x.nthr - 1] : 0);
    {
      const int32_t* const a_store = J.a_store;
      const int32_t* const a_tensor = J.a_tensor;
      const uint8_t* const a_flag = J.a_flag;
      const uint8_t* const a_owned = J.a_owned;
      const int8_t* const a_type = J.a_type;
      const int64_t* const a_start = J.a_start;
      const int64_t* const a_end = J.a_end;
      const int32_t* const t_rank = J.t_rank;
      const int32_t A = J.A;
      for (int32_t a = a0; a < a1; ++a) {
        const int32_t s = a_store[a];
        const int64_t slot = acc0 + a;
        const bool flagged = a_flag[a] != 0;
        const int32_t rk = t_rank[s];
        const int64_t te = a_end[a];
        if (a_type[a] == ACC_TGA) {
          const int64_t ts = a_start[a];
          E_x_time[slot] = ts;
          E_x_type[slot] = int8_t(EV_TGA | (a_tensor[a] != s ? 8 : 0));
          if (!inc) E_k_key[slot] = key(b, ts, EV_TGA, rk);
        } else {
          E_x_time[slot] = te;
          E_x_type[slot] = int8_t(EV_TUA | (flagged ? 16 : 0));
          if (!inc) E_k_key[slot] = key(b, te, EV_TUA, rk);
        }
        E_x_store[slot] = s; E_x_aid[slot] = a; E_x_job[slot] = int8_t(b);
        if (!inc) E_k_val[slot] = int32_t(slot);
        if (flagged && !a_owned[a]) {
          const int64_t rs = inc ? acc0 + A + a : acc0 + A + rel++;
          E_x_time[rs] = te; E_x_type[rs] = EV_REL; E_x_store[rs] = s; E_x_aid[rs] = a;
          E_x_job[rs] = int8_t(b);
          if (!inc) { E_k_val[rs] = int32_t(rs); E_k_key[rs] = key(b, te, EV_REL, rk); }
        }
      }
    }
    }
    for (int32_t i = x.tid; i < st.S; i += x.nthr) {
      const int32_t s = J.t_store[J.ev_tensor[i]];
      const int64_t slot = base + i;
      int64_t when = J.ev_end[i];
      int type;
      if (J.ev_dir[i] == 0) {
        type = EV_SOUT;
        if (J.ev_trig[i] != -1) when = imax(when, J.a_end[J.ev_trig[i]]);
      } else {
        type = EV_SIN;
        if (J.ev_wraps[i] && st.period > 0) when = ((when % st.period) + st.period) % st.period;
      }
      E_x_time[slot] = when; E_x_type[slot] = int8_t(type); E_x_store[slot] = s; E_x_aid[slot] = -1;
      E_x_job[slot] = int8_t(b); E_k_val[slot] = int32_t(slot);
      E_k_key[slot] = key(b, when, type, J.t_rank[s]);
      if (inc) E_dl[slot] = ev_lo(type, J.t_rank[s]);
    }
    for (int32_t r = x.tid; r < st.R; r += x.nthr) {
      const int32_t s = J.t_store[J.rc_tensor[r]];
      const int64_t slot = base + st.S + r;
      const int64_t when = J.a_start[J.rc_target[r]] - J.rc_lat[r];
      E_x_time[slot] = when; E_x_type[slot] = EV_TGA; E_x_store[slot] = s; E_x_aid[slot] = -1;
      E_x_job[slot] = int8_t(b); E_k_val[slot] = int32_t(slot);
      E_k_key[slot] = key(b, when, EV_TGA, J.t_rank[s]);
      if (inc) E_dl[slot] = ev_lo(EV_TGA, J.t_rank[s]);
    }
  }
  x.sync();
  etick(1);
  if (inc) {
    // 5-6. timeline order and (storage, timeline) grouping by merges
    inc_order(x, g, jb, n, rbits, sh[F_BASE] + g.st[jb].S + g.st[jb].R);
    if (g.err.code) return false;
    etick(2);
  } else {
  // 5. timeline order (sort_timeline, peak.cpp:44-62)
  x.sort(E_k_key, E_k_val, int32_t(n), jbits + tbits + 1 + rbits + 2);
  etick(2);
  // 6. group sorted positions by (job, storage), keeping timeline order
  for (int64_t m = x.tid; m < n; m += x.nthr) {
    const int32_t slot = E_k_val[m];
    E_x_order[m] = slot;
    const int b = E_x_job[slot];
    E_x_key2[m] = (uint64_t(b) << rbits) | uint64_t(g.jobs[jb + b].t_rank[E_x_store[slot]]);
    E_x_seq2[m] = int32_t(m);
  }
  x.sync();
  x.sort(E_x_key2, E_x_seq2, int32_t(n), jbits + rbits);
  for (int64_t m = x.tid; m < n; m += x.nthr) E_k_val[m] = E_x_order[E_x_seq2[m]];
  x.sync();
  etick(3);
  }
  const int32_t* const E_gslot = E_k_val;  // slots in (job, storage)-grouped order
  // 7. per-storage residency automaton (analyze_peak's switch, peak.cpp:206-230),
  // in parallel: in (job, storage)-grouped order, the residency before an
  // event is set by the previous state-changing event of its storage (TGA
  // and swap-in make it resident, release and swap-out evict); a max-scan
  // gives that index, and since a storage's events are contiguous it belongs
  // to the same storage iff its group key matches.
  {
    int64_t* chg = reinterpret_cast<int64_t*>(E_k_key);  // free after sort 1
    {
      // (restrict-qualified views and unrolled strides keep several
      // iterations' loads in flight: these loops are latency-bound)
      const int32_t* __restrict__ r_gs = E_gslot;
      const int8_t* __restrict__ r_type = E_x_type;
      int64_t* __restrict__ r_chg = chg;
      if (inc) {  // (types already laid out in grouped order)
        const int8_t* __restrict__ r_gty = g.ec_gty;
#pragma unroll 4
        for (int64_t m = x.tid; m < n; m += x.nthr) r_chg[m] = (r_gty[m] & 7) == EV_TUA ? -1 : m;
      } else {
#pragma unroll 4
        for (int64_t m = x.tid; m < n; m += x.nthr) r_chg[m] = (r_type[r_gs[m]] & 7) == EV_TUA ? -1 : m;
      }
    }
    x.sync();
    x.scan_max(chg, int32_t(n));
    if (nb == 1) {  // one job: no per-event job lookup
      const uint8_t* __restrict__ c_res = g.jobs[jb].res_init;
      const int64_t* __restrict__ c_size = g.jobs[jb].t_size;
      const int32_t* __restrict__ r_seq = E_x_seq2;
      const int32_t* __restrict__ r_gs = E_gslot;
      const int32_t* __restrict__ r_store = E_x_store;
      const int8_t* __restrict__ r_type = E_x_type;
      const int64_t* __restrict__ r_chg = chg;
      const uint64_t* __restrict__ r_key = E_x_key2;
      int64_t* __restrict__ r_fp = E_x_fp;
      uint8_t* __restrict__ r_state = E_x_state;
      const int8_t* __restrict__ r_gty = inc ? g.ec_gty : nullptr;  // (grouped-order types / storages)
      const int32_t* __restrict__ r_gst = inc ? g.ec_gst : nullptr;
#pragma unroll 2
      for (int64_t m = x.tid; m < n; m += x.nthr) {
        const int32_t pos = r_seq[m];
        const int64_t prev = m > 0 ? r_chg[m - 1] : -1;
        int32_t s;
        int tyf;
        if (r_gty) { s = r_gst[m]; tyf = r_gty[m]; }
        else { const int32_t slot = r_gs[m]; s = r_store[slot]; tyf = r_type[slot]; }
        const int ty = tyf & 7;
        uint8_t res;
        if (prev >= 0 && r_key[prev] == r_key[m]) {
          const int pt = (r_gty ? r_gty[prev] : r_type[r_gs[prev]]) & 7;
          res = (pt == EV_TGA || pt == EV_SIN) ? 1 : 0;
        } else {
          res = c_res[s];
        }
        const int64_t size = c_size[s];
        int64_t eff = 0;
        int errc = 0;
        switch (ty) {
          case EV_TGA:
            if (!res) { eff = (tyf & 8) ? 0 : size; res = 1; }
            break;
          case EV_TUA: break;
          case EV_REL:
          case EV_SOUT:
            if (!res) errc = E_DOUBLE_RELEASE;
            eff = -size; res = 0;
            break;
          default:  // EV_SIN
            if (res) errc = E_SWAPIN_RESIDENT;
            eff = size; res = 1;
            break;
        }
        r_fp[pos] = eff;
        r_state[pos] = res;
        if (errc) x.amin(&sh[F_ERR], (int64_t(pos) << 3) | errc);
      }
    } else {
    int cb = -1;
    const uint8_t* c_res = nullptr;
    const int64_t* c_size = nullptr;
    for (int64_t m = x.tid; m < n; m += x.nthr) {
      const int32_t pos = E_x_seq2[m];
      const int32_t slot = E_gslot[m];
      const int b = E_x_job[slot];
      if (b != cb) {  // job arrays cached in registers (the byte stores below alias the struct)
        cb = b;
        c_res = g.jobs[jb + b].res_init;
        c_size = g.jobs[jb + b].t_size;
      }
      const int32_t s = E_x_store[slot];
      const int ty = E_x_type[slot] & 7;
      const int64_t prev = m > 0 ? chg[m - 1] : -1;  // last state change strictly before m
      uint8_t res;
      if (prev >= 0 && E_x_key2[prev] == E_x_key2[m]) {
        const int pt = E_x_type[E_gslot[prev]] & 7;
        res = (pt == EV_TGA || pt == EV_SIN) ? 1 : 0;
      } else {
        res = c_res[s];
      }
      const int64_t size = c_size[s];
      int64_t eff = 0;
      int errc = 0;
      switch (ty) {
        case EV_TGA:
          if (!res) { eff = (E_x_type[slot] & 8) ? 0 : size; res = 1; }
          break;
        case EV_TUA: break;
        case EV_REL:
        case EV_SOUT:
          if (!res) errc = E_DOUBLE_RELEASE;
          eff = -size; res = 0;
          break;
        default:  // EV_SIN
          if (res) errc = E_SWAPIN_RESIDENT;
          eff = size; res = 1;
          break;
      }
      E_x_fp[pos] = eff;
      E_x_state[pos] = res;
      if (errc) x.amin(&sh[b * NF + F_ERR], (int64_t(pos) << 3) | errc);
    }
    }
    x.sync();
  }
  etick(4);
  // 8. footprint curve: inclusive scan of the effective deltas
  x.scan(E_x_fp, int32_t(n));
  if (x.tid == 0) {
    for (int b = 0; b < nb; ++b) {
      int64_t* f = sh + b * NF;
      f[F_OFF] = f[F_INIT] - (f[F_BASE] > 0 ? E_x_fp[f[F_BASE] - 1] : 0);
    }
  }
  x.sync();
  if (nb == 1) {  // one job: the offset fix-up fused with the maximum, no job lookup
    const int64_t off = sh[F_OFF];
    int64_t* __restrict__ r_fp = E_x_fp;
    int64_t cmx = INT64_MIN, neg = INT64_MAX;
#pragma unroll 4
    for (int64_t m = x.tid; m < n; m += x.nthr) {
      const int64_t fp = r_fp[m] + off;
      r_fp[m] = fp;
      cmx = imax(cmx, fp);
      if (fp < 0 && neg == INT64_MAX) neg = m;
    }
    if (neg != INT64_MAX) x.amin(&sh[F_ERR], (neg << 3) | E_NEG_FOOTPRINT);
    x.ramax(&sh[F_MAXFP], cmx);
  } else {
    // offset fix-up fused with the per-job maximum: jobs occupy contiguous
    // position ranges, so each thread folds its strided elements locally and
    // issues one atomic per job it touched.
    int cb = -1;
    int64_t cmx = INT64_MIN;
    for (int64_t m = x.tid; m < n; m += x.nthr) {
      const int b = E_x_job[E_x_order[m]];
      int64_t* f = sh + b * NF;
      const int64_t fp = E_x_fp[m] + f[F_OFF];
      E_x_fp[m] = fp;  // own element only: no cross-thread hazard after the scan
      if (fp < 0) x.amin(&f[F_ERR], (int64_t(m) << 3) | E_NEG_FOOTPRINT);
      if (b != cb) {
        if (cb >= 0) x.amax(&sh[cb * NF + F_MAXFP], cmx);
        cb = b;
        cmx = fp;
      } else {
        cmx = imax(cmx, fp);
      }
    }
    if (nb == 1) x.ramax(&sh[F_MAXFP], cb >= 0 ? cmx : INT64_MIN);
    else if (cb >= 0) x.amax(&sh[cb * NF + F_MAXFP], cmx);
  }
  x.sync();
  etick(5);
  // 9. first strict maximum (analyze_peak, peak.cpp:236-241)
  if (nb == 1) {  // each thread's first match is its only candidate
    const int64_t mx = sh[F_MAXFP];
    if (mx > sh[F_INIT]) {
      const int64_t* __restrict__ r_fp = E_x_fp;
      for (int64_t m = x.tid; m < n; m += x.nthr)
        if (r_fp[m] == mx) { x.amin(&sh[F_PPOS], m); break; }
    }
  } else
  for (int64_t m = x.tid; m < n; m += x.nthr) {
    const int b = E_x_job[E_x_order[m]];
    int64_t* f = sh + b * NF;
    if (f[F_MAXFP] > f[F_INIT] && E_x_fp[m] == f[F_MAXFP]) x.amin(&f[F_PPOS], m);
  }
  x.sync();
  // 10. last_input_access at the peak; residency at the peak
  if (nb == 1) {  // one job: only positions up to the peak matter
    const int64_t pp = sh[F_PPOS];
    int64_t cl = -1;
    if (pp != INT64_MAX) {
      const int32_t* __restrict__ r_ord = E_x_order;
      const int8_t* __restrict__ r_type = E_x_type;
#pragma unroll 4
      for (int64_t m = x.tid; m <= pp; m += x.nthr) {
        const int ty = r_type[r_ord[m]];
        if ((ty & 7) == EV_TUA && !(ty & 16)) cl = m;
      }
    }
    x.ramax(&sh[F_LUA], cl);
  } else {
    int cb = -1;
    int64_t cl = -1;
    for (int64_t m = x.tid; m < n; m += x.nthr) {
      const int32_t slot = E_x_order[m];
      const int b = E_x_job[slot];
      const int64_t pp = sh[b * NF + F_PPOS];
      if (b != cb) {
        if (cl >= 0) x.amax(&sh[cb * NF + F_LUA], cl);
        cb = b;
        cl = -1;
      }
      if (pp != INT64_MAX && m <= pp && (E_x_type[slot] & 7) == EV_TUA && !(E_x_type[slot] & 16)) cl = m;
    }
    if (nb == 1) x.ramax(&sh[F_LUA], cl);
    else if (cl >= 0) x.amax(&sh[cb * NF + F_LUA], cl);
  }
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    uint8_t* const in_peak = J.in_peak;
    const uint8_t* const res_init = J.res_init;
    const int32_t T = J.T;
    for (int32_t t = x.tid; t < T; t += x.nthr) in_peak[t] = res_init[t];
  }
  x.sync();
  // A storage's residency at the peak is its state after its last event at or
  // before the peak position: within a (job, storage) group positions ascend,
  // so that event is the one whose successor leaves the group or the prefix.
  if (nb == 1) {
    const int64_t pp = sh[F_PPOS];
    if (pp != INT64_MAX) {
      const int32_t* __restrict__ r_seq = E_x_seq2;
      const int32_t* __restrict__ r_gs = E_gslot;
      const uint64_t* __restrict__ r_key = E_x_key2;
      const int32_t* __restrict__ r_store = E_x_store;
      const uint8_t* __restrict__ r_state = E_x_state;
      uint8_t* __restrict__ r_peak = g.jobs[jb].in_peak;
#pragma unroll 4
      for (int64_t m = x.tid; m < n; m += x.nthr) {
        const int32_t pos = r_seq[m];
        if (pos > pp) continue;
        if (m + 1 < n && r_key[m + 1] == r_key[m] && r_seq[m + 1] <= pp) continue;
        r_peak[inc ? g.ec_gst[m] : r_store[r_gs[m]]] = r_state[pos];
      }
    }
  } else
  for (int64_t m = x.tid; m < n; m += x.nthr) {
    const int32_t pos = E_x_seq2[m];
    const int32_t slot = E_gslot[m];
    const int b = E_x_job[slot];
    const int64_t pp = sh[b * NF + F_PPOS];
    if (pp == INT64_MAX || pos > pp) continue;
    if (m + 1 < n && E_x_key2[m + 1] == E_x_key2[m] && E_x_seq2[m + 1] <= pp) continue;
    g.jobs[jb + b].in_peak[E_x_store[slot]] = E_x_state[pos];
  }
  x.sync();
  etick(6);
  // 11. report + curve
  for (int b = 0; b < nb; ++b) {
    const JobDev& J = g.jobs[jb + b];
    int64_t* f = sh + b * NF;
    // the peak storages, unordered: the next swap pass's candidates
    int32_t* const pk_list = J.pk_list;
    for (int32_t t = x.tid; t < J.T; t += x.nthr)
      if (J.in_peak[t]) pk_list[x.aadd(&f[F_NPEAK], 1)] = t;
    const int64_t base = f[F_BASE], nn = f[F_N];
    if (x.tid == 0) { J.curve_t[0] = 0; J.curve_b[0] = f[F_INIT]; }
    {
      const int64_t* __restrict__ r_time = E_x_time;
      const int32_t* __restrict__ r_ord = E_x_order + base;
      const int64_t* __restrict__ r_fp = E_x_fp + base;
      int64_t* __restrict__ r_ct = J.curve_t + 1;
      int64_t* __restrict__ r_cb = J.curve_b + 1;
#pragma unroll 4
      for (int64_t m = x.tid; m < nn; m += x.nthr) {
        r_ct[m] = r_time[r_ord[m]];
        r_cb[m] = r_fp[m];
      }
    }
  }
  x.sync();
  if (x.tid == 0) {
    for (int b = 0; b < nb; ++b) {
      int64_t* f = sh + b * NF;
      if (f[F_ERR] != INT64_MAX && !g.err.code) {
        const int64_t pos = f[F_ERR] >> 3;
        const int32_t slot = E_x_order[pos];
        g.err.code = int32_t(f[F_ERR] & 7);
        g.err.job = jb + b;
        g.err.tensor = E_x_store[slot];
        g.err.tick = E_x_time[slot];
      }
      JobState& st = g.st[jb + b];
      const bool up = f[F_PPOS] != INT64_MAX;
      st.peak = up ? f[F_MAXFP] : f[F_INIT];
      st.peak_time = up ? E_x_time[E_x_order[f[F_PPOS]]] : 0;
      st.has_lua = (up && f[F_LUA] >= 0) ? 1 : 0;
      st.lua = st.has_lua ? E_x_aid[E_x_order[f[F_LUA]]] : -1;
      st.n_peak = int32_t(f[F_NPEAK]);
      st.n_curve = int32_t(f[F_N] + 1);
      st.n_events = f[F_N];
      st.dirty = 0;
    }
    g.stats.evaluations += nb;
    g.stats.timeline_events += n;
    g.stats.sort_elems += 2 * n;
  }
  x.sync();
  return g.err.code == 0;
}

// One evaluation batch; an execution context may route it elsewhere (the
// CUDA build runs it on every CTA of a cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD bool eval_batch(X& x, GroupDev& g, int jb, int je) {
  return evaluate(x, g, jb, je);
}

// Evaluate every job in [j0, j1) whose plan changed (or all when force),
// in batches that fit the sort capacity.
template <class X>
TSL_HD bool refresh(X& x, GroupDev& g, int j0, int j1, bool force) {
  int j = j0;
  while (j < j1) {
    while (j < j1 && !force && !g.st[j].dirty) ++j;
    if (j >= j1) break;
    int e = j;
    int64_t tot = 0;
    // (the release-slot scan needs nthr scratch words per batched job)
    while (e < j1 && e - j < MAXB && int64_t(e - j + 1) * x.nthr <= g.ecap && (force || g.st[e].dirty || e == j)) {
      const int64_t need = int64_t(g.jobs[e].A) * 2 + g.st[e].S + g.st[e].R;
      if (e > j && tot + need > g.ecap) break;
      tot += need;
      ++e;
    }
    if (!eval_batch(x, g, j, e)) return false;
    j = e;
  }
  return true;
}

// ----------------------------------------------------------------------------
// Stage 3+4: swap pass (swap_planner.cpp:461-520), speculate -> validate ->
// commit in order.
//
//  A. every candidate is scored by one thread against the pass-start busy set
//     plus its own commits (SpecCtx), recording its pairs and the effective
//     windows of its successful queries;
//  B. for every candidate, the earlier candidates of the same job whose
//     speculative intervals (lifted by -P/0/+P) touch one of its windows;
//  C. one warp per job (one warp overall when a swap ratio < 1 couples the
//     jobs through SwapBudget) walks the candidates in the reference order and
//     decides: a candidate none of whose conflicting predecessors committed as
//     speculated, and whose windows no re-scored commit touches, keeps its
//     speculative result; any other candidate is re-scored against the real
//     state (ReCtx), exactly like the sequential reference. Event slots and
//     ids are assigned here, in order;
//  D. all threads write the committed events, flags and counters;
//  E. one block sort rebuilds every job's sorted busy structure.
// ----------------------------------------------------------------------------
enum { CI_P0 = 0, CI_NP, CI_W0, CI_NW, CI_STATUS, CI_NCONF, CI_CONF, CI_STATE = CI_CONF + CAPC, CI_EV0, CI_ID0,
       CI_STRIDE = 16 };
enum { CS_FAIL = 0, CS_OK = 1, CS_OVERFLOW = 2, CS_SKIP = 3, CS_ERROR = 4 };

TSL_HD bool hits(int64_t s, int64_t e, int64_t wl, int64_t wh, int64_t P) {
  for (int k = -1; k <= 1; ++k) {
    const int64_t sh = k * P;
    if (s + sh < wh && wl < e + sh) return true;
  }
  return false;
}

// Time indexes over the sorted busy structure (starts and ends) of job j.
template <class X>
TSL_HD void build_busy_index(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  const int32_t n = st.S;
  const int sh = tindex_shift(n ? imax(J.bz_e[n - 1], 0) : 0, J.ti_nb);
  x.sync();
  if (x.tid == 0) st.bzi_shift = sh;
  build_tindex(x, J.bz_s, n, J.bzi_s, sh, J.ti_nb);
  build_tindex(x, J.bz_e, n, J.bzi_e, sh, J.ti_nb);
}

template <class X>
TSL_HD void build_anchor_index(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  const int sh = tindex_shift(J.A ? imax(J.a_end[J.A - 1], 0) : 0, J.ti_nb);
  x.sync();
  if (x.tid == 0) st.ai_shift = sh;
  build_tindex(x, J.a_end, J.A, J.ai_e, sh, J.ti_nb);
}

// Sorted busy structure of every job rebuilt from the plan: block sorts of
// (job, start) keys over batches of jobs that fit one sort tile.
template <class X>
TSL_HD void rebuild_busy(X& x, GroupDev& g) {
  int64_t* gsh = x.sh + MAXB * NF;
  if (g.n_jobs == 1 && g.st[0].bz_n == g.st[0].S_pass && g.st[0].S >= g.st[0].S_pass) {
    // One job whose busy structure was not folded into during the pass: it
    // still holds the pass-start events sorted by (start, event), so only the
    // pass's new events are sorted and merged in (old first on equal starts,
    // the full sort's tie order).
    const JobDev& J = g.jobs[0];
    JobState& st = g.st[0];
    const int32_t S0 = st.S_pass, nn = st.S - S0;
    if (x.tid == 0) gsh[14] = 0;
    x.sync();
    {
      int64_t mx = 0;
      for (int32_t i = x.tid; i < nn; i += x.nthr) mx = imax(mx, J.ev_start[S0 + i]);
      x.ramax(&gsh[14], mx);
    }
    x.sync();
    const int tbits = nbits(uint64_t(gsh[14]));
    for (int32_t i = x.tid; i < nn; i += x.nthr) { g.k_key[i] = uint64_t(J.ev_start[S0 + i]); g.k_val[i] = S0 + i; }
    x.sort(g.k_key, g.k_val, nn, tbits);
    int64_t* const ms = J.bk_bz;  // (the fold / rollback buffer: idle here)
    int64_t* const me = J.bk_bz + J.Scap;
    {
      const int64_t* const bs = J.bz_s;
      const int64_t* const be = J.bz_e;
      const int32_t* const nv = g.k_val;
      const int64_t n = int64_t(S0) + nn;
      const int64_t per = (n + x.nthr - 1) / x.nthr;
      const int64_t d0 = imin(n, int64_t(x.tid) * per), d1 = imin(n, d0 + per);
      if (d0 < d1) {
        int64_t lo = imax(0, d0 - nn), hi = imin(d0, S0);
        while (lo < hi) {  // old entries before the d0-th output
          const int64_t mid = (lo + hi) >> 1;
          if (bs[mid] <= J.ev_start[nv[d0 - mid - 1]]) lo = mid + 1; else hi = mid;
        }
        int64_t i = lo, k = d0 - lo;
        for (int64_t d = d0; d < d1; ++d) {
          if (i < S0 && (k >= nn || bs[i] <= J.ev_start[nv[k]])) { ms[d] = bs[i]; me[d] = be[i]; ++i; }
          else { ms[d] = J.ev_start[nv[k]]; me[d] = J.ev_end[nv[k]]; ++k; }
        }
      }
      x.sync();
      for (int64_t d = x.tid; d < n; d += x.nthr) { J.bz_s[d] = ms[d]; J.bz_e[d] = me[d]; }
    }
    if (x.tid == 0) st.bz_n = st.S;
    x.sync();
    build_busy_index(x, g, 0);
    return;
  }
  int j0 = 0;
  while (j0 < g.n_jobs) {
    if (x.tid == 0) {
      int64_t off = 0;
      int j1 = j0;
      while (j1 < g.n_jobs && (j1 == j0 || off + g.st[j1].S <= g.ecap)) { gsh[16 + j1] = off; off += g.st[j1].S; ++j1; }
      gsh[15] = off;
      gsh[13] = j1;
      gsh[14] = 0;
    }
    x.sync();
    const int j1 = int(gsh[13]);
    const int64_t n = gsh[15];
    if (n > g.ecap) {
      if (x.tid == 0) { g.err.code = E_CAPACITY; g.err.job = j0; g.err.tensor = n; g.err.tick = 3; }
      x.sync();
      return;
    }
    for (int j = j0; j < j1; ++j) {
      const JobDev& J = g.jobs[j];
      int64_t mx = 0;
      for (int32_t i = x.tid; i < g.st[j].S; i += x.nthr) mx = imax(mx, J.ev_start[i]);
      x.ramax(&gsh[14], mx);
    }
    x.sync();
    const int jbits = nbits(uint64_t(j1 - j0 - 1));
    const int tbits = nbits(uint64_t(gsh[14]));
    for (int j = j0; j < j1; ++j) {
      const JobDev& J = g.jobs[j];
      const int64_t base = gsh[16 + j];
      for (int32_t i = x.tid; i < g.st[j].S; i += x.nthr) {
        g.k_key[base + i] = (uint64_t(j - j0) << tbits) | uint64_t(J.ev_start[i]);
        g.k_val[base + i] = (j << 24) | i;
      }
    }
    x.sync();
    x.sort(g.k_key, g.k_val, int32_t(n), jbits + tbits);
    for (int64_t m = x.tid; m < n; m += x.nthr) {
      const int j = g.k_val[m] >> 24;
      const int32_t i = g.k_val[m] & 0xffffff;
      const JobDev& J = g.jobs[j];
      const int64_t pos = m - gsh[16 + j];
      J.bz_s[pos] = J.ev_start[i];
      J.bz_e[pos] = J.ev_end[i];
    }
    for (int j = j0 + x.tid; j < j1; j += x.nthr) g.st[j].bz_n = g.st[j].S;
    x.sync();
    for (int j = j0; j < j1; ++j) build_busy_index(x, g, j);
    j0 = j1;
  }
}

// The end-of-pass rebuild; an execution context may route it elsewhere (the
// CUDA build runs it on every CTA of a cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD void rebuild_batch(X& x, GroupDev& g) {
  rebuild_busy(x, g);
}

// Folds the pass's sorted commit list into the job's busy structure (warp-
// collective, the job's deciding warp only): queries see the same union of
// intervals, later pend merges start from an empty list. Both lists are
// disjoint at shift 0, so starts and ends stay sorted; busy elements go first
// on equal starts. Each lane merges one contiguous output range (merge-path
// split) into the job's merge buffers, copied back; the time indexes are
// rebuilt. Folding happens once
// the list passes max(1024, busy / 128) intervals (a fold is linear in the
// busy structure, a re-score's pend merge linear in the list).
constexpr int32_t PEND_MERGE = 1024;

template <class X>
TSL_HD void merge_pend_into_busy(X& x, GroupDev& g, int j, const PendBuf& pb) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  const int32_t n1 = st.bz_n, n2 = st.pend_n, n = n1 + n2;
  const int64_t* bs = J.bz_s;
  const int64_t* be = J.bz_e;
  int64_t* ms = J.bk_bz;             // the recompute rollback copy of the busy
  int64_t* me = J.bk_bz + J.Scap;    // structure: idle during a swap pass
  x.wsync();
  {
    // a cooperative launch folds on its worker CTAs
    const int64_t mx = imax(n1 ? J.bz_e[n1 - 1] : 0, n2 ? pb.e[n2 - 1] : 0);
    const int sh = tindex_shift(imax(mx, 0), J.ti_nb);
    if (x.fold_hook(bs, be, n1, pb.s, pb.e, n2, ms, me, J.bz_s, J.bz_e, J.bzi_s, J.bzi_e, sh, J.ti_nb)) {
      x.wsync();
      st.bz_n = n;
      st.pend_n = 0;
      st.pend_sorted = 0;
      st.bzi_shift = sh;
      x.wsync();
      return;
    }
  }
  const int32_t per = (n + X::W - 1) / X::W;
  const int32_t d0 = imin(n, int64_t(x.lane) * per), d1 = imin(n, int64_t(d0) + per);
  int32_t lo = imax(0, d0 - n2), hi = imin(d0, n1);  // busy elements among the first d0 outputs
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (bs[mid] <= pb.s[d0 - mid - 1]) lo = mid + 1; else hi = mid;
  }
  int32_t i = lo, k = d0 - lo;
  for (int32_t d = d0; d < d1; ++d) {
    if (i < n1 && (k >= n2 || bs[i] <= pb.s[k])) { ms[d] = bs[i]; me[d] = be[i]; ++i; }
    else { ms[d] = pb.s[k]; me[d] = pb.e[k]; ++k; }
  }
  x.wsync();
  for (int32_t d = x.lane; d < n; d += X::W) { J.bz_s[d] = ms[d]; J.bz_e[d] = me[d]; }
  x.wsync();
  const int sh = tindex_shift(n ? imax(J.bz_e[n - 1], 0) : 0, J.ti_nb);
  x.wsync();
  st.bz_n = n;
  st.pend_n = 0;
  st.pend_sorted = 0;
  st.bzi_shift = sh;
  x.wsync();
  build_tindex<X, true>(x, J.bz_s, n, J.bzi_s, sh, J.ti_nb);
  build_tindex<X, true>(x, J.bz_e, n, J.bzi_e, sh, J.ti_nb);
}

// Appends the intervals of the candidates taken verbatim (speculation kept)
// since the last append, up to candidate m, to the job's pend list, 32
// candidates at a time (a warp prefix sum places them in plan order).
// Warp-collective; false on overflow.
template <class X>
TSL_HD bool pend_append(X& x, GroupDev& g, int j, int64_t m, const int32_t* cand, const int32_t* cinfo, PendBuf& pb,
                        ErrInfo& lerr) {
  JobState& st = g.st[j];
  for (int64_t q0 = st.pend_upto; q0 < m; q0 += X::W) {
    const int64_t q = q0 + x.lane;
    const int32_t* cq = cinfo + q * CI_STRIDE;
    const int32_t nq = (q < m && cq[CI_STATE] == 1 && (cand[q] >> 24) == j) ? cq[CI_NP] : 0;
    int32_t tot = 0;
    const int32_t ex = x.wexcl(2 * nq, &tot);
    const int32_t pn = st.pend_n;
    if (pn + tot > pb.cap) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = pb.cap; return false; }
    x.wsync();
    if (nq) {
      const PairRec* pr = g.pr_pool + cq[CI_P0];
      for (int32_t p = 0; p < nq; ++p) {
        const int32_t o = pn + ex + 2 * p;
        pb.s[o] = pr[p].os; pb.e[o] = pr[p].oe;
        pb.s[o + 1] = pr[p].is; pb.e[o + 1] = pr[p].ie;
      }
    }
    st.pend_n = pn + tot;
    x.wsync();
  }
  x.wsync();
  st.pend_upto = int32_t(m);  // callers never move backwards (m >= pend_upto)
  x.wsync();
  return true;
}

// Re-scores candidate m of job j exactly against the real state: pass-start
// busy structure + every interval committed before it in this pass (pend,
// brought up to date lazily) -- the sequential reference semantics. Returns
// the number of pairs committed (0: failed); -1 on error.
template <class X>
TSL_HD int32_t rescore_candidate(X& x, GroupDev& g, int j, int32_t s, int64_t m, int32_t* cand, int32_t* cinfo,
                                 PendBuf& pb, GroupStats& ls, ErrInfo& lerr) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  int32_t* ci = cinfo + m * CI_STRIDE;
  ls.rescored += 1;
  const int64_t rc0 = x.clock();
  if (!pend_append(x, g, j, m, cand, cinfo, pb, lerr)) return -1;
  const int64_t rc1 = x.clock();
  pend_sort(x, pb, st);
  if (st.pend_n >= x.fold_threshold(st.bz_n)) {
    const int64_t f0 = x.clock();
    merge_pend_into_busy(x, g, j, pb);
    if (x.tid == 0) g.stats.cyc[19] += x.clock() - f0;
  }
  const int64_t rc2 = x.clock();
  int64_t earliest = 0, latest = 0;
  const int kind = candidate_kind(J, st, s, earliest, latest);
  const int32_t capp = kind == 1 ? 1 : imax(1, J.s_off[s + 1] - J.s_off[s]);
#if TSL_EMU_STATS
  const std::vector<PairRec> spec(g.pr_pool + ci[CI_P0], g.pr_pool + ci[CI_P0] + ((ci[CI_STATUS] & 0xf) == CS_OK ? ci[CI_NP] : 0));
  const int spec_status = ci[CI_STATUS] & 0xf;
#endif
  ReCtx<X> c{x, J, st, pb, g.cfg, &ls, g.pr_pool + ci[CI_P0], 0, capp, false};
  c.dbg = &g.stats.cyc[12];
  const bool ok = kind == 1 ? schedule_wrapped_swap(c, s) : schedule_swap(c, s, earliest, latest);
#if TSL_EMU_STATS
  {
    emu_stats::n_rescore++;
    const int np = ok ? c.nout : 0;
    if (spec_status != CS_OK) emu_stats::spec_not_ok++;
    if (kind == 1) emu_stats::wrapped++;
    emu_stats::spec_pairs += spec.size();
    emu_stats::new_pairs += np;
    int kept = 0;
    for (int p = 0; p < np; ++p)
      for (const PairRec& r : spec)
        if (r.os == c.out[p].os && r.is == c.out[p].is) { ++kept; break; }
    emu_stats::kept_pairs += kept;
    const bool main_same = np > 0 && !spec.empty() && spec[0].os == c.out[0].os && spec[0].is == c.out[0].is;
    const bool main_out_same = np > 0 && !spec.empty() && spec[0].os == c.out[0].os;
    if (main_same) emu_stats::main_same++;
    else if (main_out_same) emu_stats::main_in_only++;
    if (np == 0 && !spec.empty()) emu_stats::now_fail++;
    if (np > 0 && spec.empty()) emu_stats::now_ok++;
    if (np > 1 || spec.size() > 1) emu_stats::with_gaps++;
  }
#endif
  if (x.tid == 0) {
    const int64_t rc3 = x.clock();
    g.stats.cyc[10] += rc3 - rc0;
    g.stats.cyc[16] += rc1 - rc0;
    g.stats.cyc[11] += rc2 - rc1;
    g.stats.cyc[17] += rc3 - rc2;
  }
  if (c.overflow) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; lerr.tick = 5; return -1; }
  return ok ? c.nout : 0;
}

// In-order decisions of one uncoupled job's candidates [m0, m1), 32 at a
// time. A candidate needs individual attention only if it has a conflicting
// earlier candidate (nconf > 0), overflowed, or was hit by a re-scored
// commit (status bit CS_HIT, set right after each re-score); every other
// candidate keeps its speculative result, so a warp ballot finds the next
// attention candidate and everything before it is decided in bulk (a warp
// prefix sum assigns event slots and ids in plan order).
constexpr int32_t CS_HIT = 16;
constexpr int64_t COMP_MIN_CANDIDATES = 64;
constexpr int32_t CS_DIFF = 32;  // decided by a re-score whose result differs from the speculation
constexpr int32_t CS_BRK = 64;   // an earlier member of the candidate's component has CS_DIFF

#if TSL_EMU_STATS
// Emulation-only check (TSL_VERIFY=1): the speculation a candidate is about to
// be decided with equals an exact re-score against the real state.
template <class X>
void emu_verify(X& x, GroupDev& g, int j, int64_t m, int32_t* cand, int32_t* cinfo, PendBuf& pb, int32_t S,
                int64_t id, const int32_t* cprev, int64_t cw0) {
  static const bool on = std::getenv("TSL_VERIFY") != nullptr;
  if (!on) return;
  JobState& st = g.st[j];
  const JobDev& J = g.jobs[j];
  int32_t* ci = cinfo + m * CI_STRIDE;
  ErrInfo lerr{};
  st.S = S;
  st.next_id = id;
  pend_append(x, g, j, m, cand, cinfo, pb, lerr);
  pend_sort(x, pb, st);
  if (st.pend_n >= x.fold_threshold(st.bz_n)) merge_pend_into_busy(x, g, j, pb);
  const int32_t pn0 = st.pend_n;
  const int32_t s = cand[m] & 0xffffff;
  int64_t earliest = 0, latest = 0;
  const int kind = candidate_kind(J, st, s, earliest, latest);
  const int32_t capp = kind == 1 ? 1 : imax(1, J.s_off[s + 1] - J.s_off[s]);
  static std::vector<PairRec> scratch(1 << 20);
  GroupStats ls{};
  ReCtx<X> c{x, J, st, pb, g.cfg, &ls, scratch.data(), 0, capp, false};
  const bool ok = kind == 1 ? schedule_wrapped_swap(c, s) : schedule_swap(c, s, earliest, latest);
  st.pend_n = pn0;
  st.pend_sorted = pn0;
  const int32_t np_spec = (ci[CI_STATUS] & 0xf) == CS_OK ? ci[CI_NP] : 0;
  const int32_t np_ex = ok ? c.nout : 0;
  bool bad = np_spec != np_ex;
  const PairRec* pr = g.pr_pool + ci[CI_P0];
  for (int32_t q = 0; !bad && q < np_ex; ++q)
    bad = pr[q].os != c.out[q].os || pr[q].oe != c.out[q].oe || pr[q].is != c.out[q].is || pr[q].ie != c.out[q].ie;
  if (bad) {
    ++emu_stats::verify_bad;
    if (emu_stats::verify_bad <= 5)
      std::fprintf(stderr, "VERIFY m=%lld status=%x nconf=%d prev=%d np spec %d exact %d spec.os %lld ex.os %lld\n",
                   (long long)m, ci[CI_STATUS], ci[CI_NCONF], cprev ? cprev[m - cw0] : -9, np_spec, np_ex,
                   np_spec ? (long long)pr[0].os : -1LL, np_ex ? (long long)c.out[0].os : -1LL);
  }
  ++emu_stats::verified;
}
#endif


template <class X>
TSL_HD bool decide_chunked(X& x, GroupDev& g, int j, int64_t m0, int64_t m1, int32_t* cand, int32_t* cinfo,
                           int64_t* chull, PendBuf& pb, GroupStats& ls, ErrInfo& lerr, bool fold_end,
                           const int32_t* cprev = nullptr, int64_t cw0 = 0) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  int32_t S = st.S;
  int64_t id = st.next_id;
  int64_t son = st.son;
  bool changed = false;
  const int64_t P = imax(1, st.period);
  int64_t m = m0;
  const int64_t dc0 = x.clock();
  int64_t dcb = 0, dca = 0, dch = 0, dcn = 0;
  while (m < m1) {
    const int64_t db0 = x.clock();
    const int64_t c = m + x.lane;
    const bool in = c < m1;
    int32_t status = in ? cinfo[c * CI_STRIDE + CI_STATUS] : CS_SKIP;
    const int32_t nconf = in ? cinfo[c * CI_STRIDE + CI_NCONF] : 0;
    // component speculation: a member whose component predecessor (decided
    // in an earlier chunk) was re-scored needs attention
    const int32_t pv = (in && cprev) ? cprev[c - cw0] : -1;
    const bool brk = pv >= 0 && pv < m && (cinfo[int64_t(pv) * CI_STRIDE + CI_STATUS] & (CS_DIFF | CS_BRK));
    const bool attn = in && (status & 0xf) != CS_SKIP &&
                      ((status & CS_HIT) || nconf > 0 || (status & 0xf) == CS_OVERFLOW || (status & 0xf) == CS_ERROR ||
                       cinfo[c * CI_STRIDE + CI_P0] < 0 || brk);
    const unsigned amask = x.wballot(attn);
    const int f = amask ? x.ffs(amask) - 1 : X::W;
    const int64_t nbulk = imin(int64_t(f), m1 - m);
    // bulk: candidates [m, m + nbulk) keep their speculation
    const bool take = x.lane < nbulk && (status & 0xf) == CS_OK;
    const int32_t np = take ? cinfo[c * CI_STRIDE + CI_NP] : 0;
    int32_t tot = 0;
    const int32_t ex = x.wexcl(2 * np, &tot);
    const int32_t ntake = popc32(x.wballot(take));
#if TSL_EMU_STATS
    if (x.lane < nbulk && (status & 0xf) == CS_FAIL) emu_verify(x, g, j, c, cand, cinfo, pb, S, id, cprev, cw0);
    if (take) emu_verify(x, g, j, c, cand, cinfo, pb, S, id, cprev, cw0);
#endif
    if (S + tot > J.Scap) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; return changed; }
    x.wsync();
    if (x.lane < nbulk) {
      int32_t* ci = cinfo + c * CI_STRIDE;
      ci[CI_STATE] = take ? 1 : 0;
      if (take) {
        ci[CI_EV0] = S + ex;
        ci[CI_ID0] = int32_t(id + ex);
        J.swapped[cand[c] & 0xffffff] = 1;
      }
    }
    x.wsync();
    S += tot;
    id += tot;
    son += ntake;
    changed = changed || ntake > 0;
    m += nbulk;
    dcb += x.clock() - db0;
    if (nbulk == X::W || m >= m1) continue;
    // attention candidate m
    const int64_t da0 = x.clock();
    ++dcn;
    int32_t* ci = cinfo + m * CI_STRIDE;
    const int32_t st_m = ci[CI_STATUS];
    const int32_t s = cand[m] & 0xffffff;
    if ((st_m & 0xf) == CS_ERROR) { lerr.code = E_NO_TGA; lerr.job = j; lerr.tensor = s; lerr.tick = 0; return changed; }
    if (ci[CI_P0] < 0) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = g.pr_cap; lerr.tick = 4; return changed; }
    bool valid = !(st_m & CS_HIT) && (st_m & 0xf) != CS_OVERFLOW && ci[CI_NCONF] <= CAPC;
    // a component member's speculation assumed every earlier member's: once
    // one of them decided differently (DIFF), the rest of the component is
    // re-scored in order (BRK carries that down the chain)
    bool pbrk = false;
    if (cprev) {
      const int32_t pvm = cprev[m - cw0];
      pbrk = pvm >= 0 && (cinfo[int64_t(pvm) * CI_STRIDE + CI_STATUS] & (CS_DIFF | CS_BRK));
      if (pbrk) valid = false;
    }
    {
      bool bad = false;
      for (int32_t k = x.lane; valid && k < ci[CI_NCONF]; k += X::W)
        bad = bad || cinfo[int64_t(ci[CI_CONF + k]) * CI_STRIDE + CI_STATE] == 1;
      valid = valid && !x.wany(bad);
    }
    int32_t npm = 0;
    int32_t state = 0;
    dca += x.clock() - da0;
#if TSL_EMU_STATS
    if (!valid) {
      if (st_m & CS_HIT) emu_stats::why_hit++;
      else if ((st_m & 0xf) == CS_OVERFLOW) emu_stats::why_over++;
      else if (ci[CI_NCONF] > CAPC) emu_stats::why_nconf++;
      else if (cprev && cprev[m - cw0] >= 0 && (cinfo[int64_t(cprev[m - cw0]) * CI_STRIDE + CI_STATUS] & (CS_DIFF | CS_BRK))) emu_stats::why_diff++;
      else emu_stats::why_conf++;
    }
#endif
    if (valid) {
#if TSL_EMU_STATS
      emu_verify(x, g, j, m, cand, cinfo, pb, S, id, cprev, cw0);
#endif
      if ((st_m & 0xf) == CS_OK) { npm = ci[CI_NP]; state = 1; }
    } else {
      // the real state needs this pass's commits so far
      x.wsync();
      st.S = S; st.next_id = id;
      x.wsync();
      // component speculation: later members of m's component assumed m's
      // speculated commits; keep them (to compare) unless there are none
      int64_t* keep = g.wbuf + int64_t(x.warp) * 4 * g.wcap + 2 * g.wcap;
      const int32_t np_old = (cprev && (st_m & 0xf) == CS_OK && ci[CI_P0] >= 0) ? ci[CI_NP] : 0;
      if (np_old > 0) {
        const PairRec* pr = g.pr_pool + ci[CI_P0];
        for (int32_t q = x.lane; q < np_old; q += X::W) {
          keep[4 * q] = pr[q].os; keep[4 * q + 1] = pr[q].oe; keep[4 * q + 2] = pr[q].is; keep[4 * q + 3] = pr[q].ie;
        }
        x.wsync();
      }
      npm = rescore_candidate(x, g, j, s, m, cand, cinfo, pb, ls, lerr);
      if (npm < 0) return changed;
      if (cprev) {
        // the chain stays intact only if the re-score commits exactly the
        // speculated intervals (a speculated failure: nothing)
        bool diff = npm != np_old || (st_m & 0xf) == CS_OVERFLOW;
        if (!diff && npm > 0) {
          const PairRec* pr = g.pr_pool + ci[CI_P0];
          bool d = false;
          for (int32_t q = x.lane; q < npm; q += X::W)
            d = d || keep[4 * q] != pr[q].os || keep[4 * q + 1] != pr[q].oe || keep[4 * q + 2] != pr[q].is ||
                keep[4 * q + 3] != pr[q].ie;
          diff = x.wany(d);
        }
        x.wsync();
        if (x.lane == 0) ci[CI_STATUS] |= (diff ? CS_DIFF : 0) | (pbrk ? CS_BRK : 0);
        x.wsync();
      }
      if (npm > 0) {
        const int64_t dh0 = x.clock();
        state = 2;
        // later candidates whose placements the new intervals hit must be
        // re-examined individually
        const PairRec* pr = g.pr_pool + ci[CI_P0];
        int64_t lo = INT64_MAX, hi = INT64_MIN;
        for (int32_t p = 0; p < npm; ++p) {
          lo = imin(lo, imin(pr[p].os, pr[p].is));
          hi = imax(hi, imax(pr[p].oe, pr[p].ie));
        }
        x.wsync();
        const int64_t wk = x.sh[MAXB * 16 + GS_WK];
        if (wk > 0) {
          // window index (large passes): only candidates whose placement
          // windows share a bucket with a lifted copy of a new interval
          const int shb = int(wk - 1);
          const int64_t NB = x.sh[MAXB * 16 + GS_NB];
          auto bucket = [&](int64_t t) -> int64_t { return t < 0 ? -1 : imin(t >> shb, NB - 1); };
          const int32_t* wk_cnt = g.cb_idx + 2 * (NB + 2);
          const int32_t* wk_ent = g.cb_ent + g.cb_cap;
          for (int32_t p = 0; p < npm; ++p)
            for (int h = 0; h < 2; ++h) {
              const int64_t s0 = h ? pr[p].is : pr[p].os, e0 = h ? pr[p].ie : pr[p].oe;
              for (int k = -1; k <= 1; ++k) {
                const int64_t ls = s0 + k * P, le = e0 + k * P;
                if (le <= 0) continue;
                for (int64_t b = imax(0, bucket(ls)); b <= bucket(le - 1) && b >= 0; ++b)
                  for (int32_t e = wk_cnt[b] + x.lane; e < wk_cnt[b + 1]; e += X::W) {
                    const int64_t q = wk_ent[e];
                    if (q <= m || q >= m1) continue;
                    int32_t* cq = cinfo + q * CI_STRIDE;
                    if ((cq[CI_STATUS] & 0xf) == CS_SKIP || (cq[CI_STATUS] & CS_HIT)) continue;
                    const int64_t* wv = g.w_pool + 2 * int64_t(cq[CI_W0]);
                    bool hit = false;
                    for (int32_t w = 0; w < cq[CI_NW] && !hit; ++w) hit = hits(s0, e0, wv[2 * w], wv[2 * w + 1], P);
                    if (hit) x.aor32(&cq[CI_STATUS], CS_HIT);  // lanes may reach q through several buckets
                  }
              }
            }
        } else {
          for (int64_t q = m + 1 + x.lane; q < m1; q += X::W) {
            int32_t* cq = cinfo + q * CI_STRIDE;
            if ((cq[CI_STATUS] & 0xf) == CS_SKIP || cq[CI_NW] == 0) continue;
            if (!hits(lo, hi, chull[q * 4], chull[q * 4 + 1], P)) continue;
            const int64_t* wv = g.w_pool + 2 * int64_t(cq[CI_W0]);
            bool hit = false;
            for (int32_t p = 0; p < npm && !hit; ++p)
              for (int32_t w = 0; w < cq[CI_NW] && !hit; ++w)
                hit = hits(pr[p].os, pr[p].oe, wv[2 * w], wv[2 * w + 1], P) ||
                      hits(pr[p].is, pr[p].ie, wv[2 * w], wv[2 * w + 1], P);
            if (hit) cq[CI_STATUS] |= CS_HIT;
          }
        }
        x.wsync();
        dch += x.clock() - dh0;
      }
    }
    if (state) {
      if (S + 2 * npm > J.Scap) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; return changed; }
      x.wsync();
      ci[CI_STATE] = state;
      ci[CI_NP] = npm;
      ci[CI_EV0] = S;
      ci[CI_ID0] = int32_t(id);
      J.swapped[s] = 1;
      x.wsync();
      S += 2 * npm;
      id += 2 * npm;
      son += 1;
      changed = true;
    } else {
      x.wsync();
      ci[CI_STATE] = 0;
      x.wsync();
    }
    ++m;
  }
  x.wsync();
  st.S = S;
  st.next_id = id;
  st.son = son;
  if (changed) st.dirty = 1;
  x.wsync();
  if (fold_end && m0 < m1) {
    // a later speculation window follows: this window's commits join the
    // busy structure its speculation is taken against
    const int64_t f0 = x.clock();
    if (!pend_append(x, g, j, m1, cand, cinfo, pb, lerr)) return changed;
    pend_sort(x, pb, st);
    if (st.pend_n > 0) merge_pend_into_busy(x, g, j, pb);
    if (x.tid == 0) g.stats.cyc[19] += x.clock() - f0;
  }
  if (x.lane == 0) {  // development cycle counters
    x.aadd(&g.stats.cyc[27], x.clock() - dc0);
    x.aadd(&g.stats.cyc[28], dcb);
    x.aadd(&g.stats.cyc[29], dca);
    x.aadd(&g.stats.cyc[30], dch);
    x.aadd(&g.stats.cyc[31], dcn);
  }
  return changed;
}

// Phase B of a speculation window [w0, w1): for every candidate, the earlier
// candidates of its job whose speculative pair intervals (lifted by -P/0/+P)
// touch one of its placement windows (ci[CI_CONF..], count ci[CI_NCONF]),
// and the window index phase C's hit marking uses. With `comp` (component
// speculation), conflicts inside a component are not recorded: a member's
// speculation already includes its component predecessors' commits.
template <class X>
TSL_HD void find_conflicts(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo,
                           const int64_t* chull, bool coupled, const int32_t* comp) {
  int64_t* gsh = x.sh + MAXB * NF;
  const int64_t wn = w1 - w0;
#if TSL_PROF
  int64_t pc0 = clock64();
  auto ptick = [&](int k) { if (x.tid == 0) { const int64_t t = clock64(); g.stats.prof[k] += t - pc0; pc0 = t; } };
#else
  auto ptick = [](int) {};
#endif
  // ---- B. conflicts with earlier speculative commits of the same job ----
  // Small passes: one thread per (candidate, earlier candidate) pair. Large
  // passes: every speculative pair interval goes into a time-bucketed index;
  // a candidate then checks only the buckets its placement windows (lifted
  // by -P/0/+P) touch, against entries of earlier candidates of its job.
  if (wn <= CB_GRID_MAX) {
    // one warp per candidate, its lanes over the earlier candidates
    const int32_t gw = x.tid / X::W, ngw = x.nthr / X::W;  // warps of the context (the grid's, cooperatively)
    for (int32_t m = int32_t(w0) + gw; m < int32_t(w1); m += ngw) {
      int32_t* ci = cinfo + int64_t(m) * CI_STRIDE;
      if (ci[CI_NW] == 0) continue;
      const int jm = cand[m] >> 24;
      const int64_t P = imax(1, g.st[jm].period);
      for (int32_t i = int32_t(w0) + x.lane; i < m; i += X::W) {
        const int32_t* cj = cinfo + int64_t(i) * CI_STRIDE;
        if (cj[CI_STATUS] != CS_OK || (cand[i] >> 24) != jm) continue;
        if (comp && comp[i - w0] == comp[m - w0]) continue;  // same component: consistent by construction
        if (!hits(chull[i * 4 + 2], chull[i * 4 + 3], chull[m * 4], chull[m * 4 + 1], P)) continue;
        const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
        const PairRec* pr = g.pr_pool + cj[CI_P0];
        bool conf = false;
        for (int32_t p = 0; p < cj[CI_NP] && !conf; ++p)
          for (int32_t w = 0; w < ci[CI_NW] && !conf; ++w)
            conf = hits(pr[p].os, pr[p].oe, wv[2 * w], wv[2 * w + 1], P) ||
                   hits(pr[p].is, pr[p].ie, wv[2 * w], wv[2 * w + 1], P);
        if (conf) {
          const int32_t k = x.aadd32(&ci[CI_NCONF], 1);
          if (k < CAPC) ci[CI_CONF + k] = int32_t(i);
        }
      }
    }
  } else {
    // bucket count: 1024, or the group's larger tables (big launches:
    // weight tensors with hundreds of gap pairs would crowd 1024 buckets)
    const int32_t NB = g.cb_nb > CB_NB ? g.cb_nb : CB_NB;
    int32_t* bk_cnt = g.cb_idx;             // [NB + 1] counts -> offsets
    int32_t* bk_cur = bk_cnt + (NB + 2);    // [NB] fill cursors
    int32_t* bk_ent = g.cb_ent;             // [cb_cap] candidate of each entry
    // the same buckets over every candidate's placement windows: phase C's
    // hit marking visits only the candidates whose windows share a bucket
    // with a re-scored commit
    int32_t* wk_cnt = g.cb_idx + 2 * (NB + 2);
    int32_t* wk_cur = wk_cnt + (NB + 2);
    int32_t* wk_ent = g.cb_ent + g.cb_cap;
    // bucket width: the largest interval end in the pass (ints are >= 0)
    if (x.tid == 0) { gsh[14] = 0; gsh[GS_NB] = NB; }
    for (int32_t k = x.tid; k < NB + 1; k += x.nthr) { bk_cnt[k] = 0; wk_cnt[k] = 0; }
    x.sync();
    ptick(0);
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      const int32_t* ci = cinfo + m * CI_STRIDE;
      if (ci[CI_STATUS] == CS_OK) x.amax(&gsh[14], chull[m * 4 + 3]);
      if (ci[CI_NW]) x.amax(&gsh[14], chull[m * 4 + 1]);
    }
    x.sync();
    ptick(1);
    int shb = 0;
    while ((gsh[14] >> shb) >= NB) ++shb;
    auto bucket = [&](int64_t t) -> int64_t { return t < 0 ? -1 : imin(t >> shb, int64_t(NB) - 1); };
    // count
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      const int32_t* ci = cinfo + m * CI_STRIDE;
      if (ci[CI_STATUS] != CS_OK) continue;
      const PairRec* pr = g.pr_pool + ci[CI_P0];
      for (int32_t p = 0; p < ci[CI_NP]; ++p)
        for (int h = 0; h < 2; ++h) {
          const int64_t s0 = h ? pr[p].is : pr[p].os, e0 = h ? pr[p].ie : pr[p].oe;
          for (int64_t q = imax(0, bucket(s0)); q <= bucket(e0 - 1) && q >= 0; ++q) x.aadd32(&bk_cnt[q + 1], 1);
        }
    }
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      const int32_t* ci = cinfo + m * CI_STRIDE;
      const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
      for (int32_t w = 0; w < ci[CI_NW]; ++w)
        for (int64_t q = imax(0, bucket(wv[2 * w])); q <= bucket(wv[2 * w + 1] - 1) && q >= 0; ++q)
          x.aadd32(&wk_cnt[q + 1], 1);
    }
    x.sync();
    ptick(2);
    // prefix over the bucket counts (the block scan's scratch holds the
    // candidate records here): 4 warps per table, each scanning its quarter
    // 32 consecutive buckets at a time (coalesced, a warp prefix sum carrying
    // the running total), then the quarters' totals are added in
    constexpr int QW = 4;
    if constexpr (X::GRID) {  // the grid's coalesced scans (a handful of barriers, no serial rows)
      x.scan32(bk_cnt + 1, NB);
      x.scan32(wk_cnt + 1, NB);
      if (x.tid == 0) {
        gsh[15] = bk_cnt[NB];
        gsh[GS_WK] = wk_cnt[NB] <= g.cb_cap ? shb + 1 : 0;
      }
    } else {
    if (X::W > 1 && x.tid < 2 * QW * X::W) {
      const int tab = x.tid / (QW * X::W), q = (x.tid / X::W) % QW;
      const int PER = NB / QW;
      int32_t* c = (tab ? wk_cnt : bk_cnt) + 1 + q * PER;
      int32_t run = 0;
      constexpr int U = 8;  // loads of 8 rows in flight before their scans
      for (int k = 0; k < PER; k += U * X::W) {
        int32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = (k + u * X::W < PER) ? c[k + u * X::W + x.lane] : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k + u * X::W >= PER) break;
          int32_t tot = 0;
          const int32_t ex = x.wexcl(v[u], &tot);
          c[k + u * X::W + x.lane] = run + ex + v[u];
          run += tot;
        }
      }
      if (x.lane == 0) gsh[GS_QTOT + tab * QW + q] = run;
    }
    if (X::W == 1 && x.tid == 0) {  // one-thread context
      for (int tab = 0; tab < 2; ++tab) {
        int32_t* c = (tab ? wk_cnt : bk_cnt) + 1;
        int32_t off = 0;
        for (int k = 0; k < NB; ++k) { off += c[k]; c[k] = off; }
        gsh[GS_QTOT + tab * QW] = off;
        for (int q = 1; q < QW; ++q) gsh[GS_QTOT + tab * QW + q] = 0;
      }
    }
    x.sync();
    ptick(3);
    if (X::W > 1 && x.tid < 2 * QW * X::W) {
      const int tab = x.tid / (QW * X::W), q = (x.tid / X::W) % QW;
      const int PER = NB / QW;
      int64_t add = 0;
      for (int r = 0; r < q; ++r) add += gsh[GS_QTOT + tab * QW + r];
      int32_t* c = (tab ? wk_cnt : bk_cnt) + 1 + q * PER;
      if (add) {
#pragma unroll 8
        for (int k = x.lane; k < PER; k += X::W) c[k] += int32_t(add);
      }
    }
    if (x.tid == 0) {
      int64_t tb = 0, tw = 0;
      for (int q = 0; q < QW; ++q) { tb += gsh[GS_QTOT + q]; tw += gsh[GS_QTOT + QW + q]; }
      gsh[15] = tb;
      gsh[GS_WK] = tw <= g.cb_cap ? shb + 1 : 0;
    }
    }
    x.sync();
    ptick(4);
    const bool fits = gsh[15] <= g.cb_cap;
    for (int32_t k = x.tid; k < NB; k += x.nthr) { bk_cur[k] = bk_cnt[k]; wk_cur[k] = wk_cnt[k]; }
    x.sync();
    ptick(5);
    if (gsh[GS_WK]) {
      for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
        const int32_t* ci = cinfo + m * CI_STRIDE;
        const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
        for (int32_t w = 0; w < ci[CI_NW]; ++w)
          for (int64_t q = imax(0, bucket(wv[2 * w])); q <= bucket(wv[2 * w + 1] - 1) && q >= 0; ++q)
            wk_ent[x.aadd32(&wk_cur[q], 1)] = int32_t(m);
      }
    }
    if (fits) {
      for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
        const int32_t* ci = cinfo + m * CI_STRIDE;
        if (ci[CI_STATUS] != CS_OK) continue;
        const PairRec* pr = g.pr_pool + ci[CI_P0];
        for (int32_t p = 0; p < ci[CI_NP]; ++p)
          for (int h = 0; h < 2; ++h) {
            const int64_t s0 = h ? pr[p].is : pr[p].os, e0 = h ? pr[p].ie : pr[p].oe;
            for (int64_t q = imax(0, bucket(s0)); q <= bucket(e0 - 1) && q >= 0; ++q)
              bk_ent[x.aadd32(&bk_cur[q], 1)] = int32_t(m);
          }
      }
    }
    x.sync();
    ptick(6);
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      int32_t* ci = cinfo + m * CI_STRIDE;
#if TSL_PROF
      if (g.grid_conf == 2) {
        int64_t* dbg = g.wbuf + 8 * g.wcap + (m - w0) * 6;
        dbg[0] = -7; dbg[1] = ci[CI_NW]; dbg[2] = ci[CI_STATUS]; dbg[3] = x.tid; dbg[4] = x.nthr; dbg[5] = w1;
      }
#endif
      if (ci[CI_NW] == 0) continue;
      const int j = cand[m] >> 24;
      const int64_t P = imax(1, g.st[j].period);
      const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
      const int64_t m0 = imax(w0, coupled ? 0 : gsh[16 + j]);
      int32_t nconf = 0;
      int64_t npass = 0, nlate = 0;
      auto consider = [&](int64_t i) {
        if (i >= m) ++nlate;
        if (i >= m || i < m0 || (cand[i] >> 24) != j) return;
        ++npass;
        if (comp && comp[i - w0] == comp[m - w0]) return;
        for (int32_t k = 0; k < imin(nconf, CAPC); ++k)
          if (ci[CI_CONF + k] == i) return;
        const int32_t* cj = cinfo + i * CI_STRIDE;
        const PairRec* pr = g.pr_pool + cj[CI_P0];
        bool conf = false;
        for (int32_t p = 0; p < cj[CI_NP] && !conf; ++p)
          for (int32_t w = 0; w < ci[CI_NW] && !conf; ++w)
            conf = hits(pr[p].os, pr[p].oe, wv[2 * w], wv[2 * w + 1], P) ||
                   hits(pr[p].is, pr[p].ie, wv[2 * w], wv[2 * w + 1], P);
        if (conf) {
          if (nconf < CAPC) ci[CI_CONF + nconf] = int32_t(i);
          ++nconf;
        }
      };
      int64_t nexam = 0;
      if (!fits || nconf > CAPC) {
        for (int64_t i = m0; i < m; ++i) {
          if (cinfo[i * CI_STRIDE + CI_STATUS] != CS_OK) continue;
          consider(i);
        }
      } else {
        for (int32_t w = 0; w < ci[CI_NW]; ++w)
          for (int k = -1; k <= 1; ++k) {
            const int64_t lo = wv[2 * w] - k * P, hi = wv[2 * w + 1] - k * P;  // raw coordinates
            if (hi <= 0) continue;
            for (int64_t q = imax(0, bucket(lo)); q <= bucket(hi - 1) && q >= 0; ++q)
              for (int32_t e = bk_cnt[q]; e < bk_cnt[q + 1]; ++e) { consider(bk_ent[e]); ++nexam; }
          }
      }
#if TSL_PROF
      if (g.grid_conf == 2) {
        int64_t* dbg = g.wbuf + 8 * g.wcap + (m - w0) * 6;
        dbg[0] = nexam; dbg[1] = fits; dbg[2] = shb; dbg[3] = ci[CI_NW]; dbg[4] = npass; dbg[5] = nlate;
      }
#endif
      ci[CI_NCONF] = nconf;
    }
  }
  x.sync();  // (a grid context returns only when every CTA has written its lists)
  ptick(7);
}

// Component runs [r] of a window (x_order / x_seq2 / c_comp from
// component_speculation), taken in turn by warps through *run_ctr: each
// member is re-speculated in order against the pass-start state plus the
// run's earlier results (private sorted list in wb: 6 * cap words).
// Warp-collective; any number of warps on any number of CTAs.
template <class X>
TSL_HD void comp_runs(X& x, GroupDev& g, int64_t w0, const int32_t* cand, int32_t* cinfo, int64_t* chull,
                      int64_t* run_ctr, int64_t nruns, int64_t* wb, int64_t cap) {
  const int64_t wn = g.c_wn;
  GroupStats ls{};
  const volatile int32_t* par = g.c_comp;
  for (;;) {
    int64_t r = 0;
    if (x.lane == 0) r = x.aadd(run_ctr, 1);
    r = x.shfl(r, 0);
    if (r >= nruns) break;
    const int32_t p0 = g.x_order[r];
    const int32_t root = par[g.x_seq2[p0]];
    const int j = cand[w0 + g.x_seq2[p0]] >> 24;
    const JobDev& J = g.jobs[j];
    JobState lst = g.st[j];  // this warp's view: pass-start busy + the component's commits
    lst.pend_n = 0;
    lst.pend_sorted = 0;
    PendBuf pl{wb, wb + cap, wb + 2 * cap, wb + 3 * cap, wb + 4 * cap, int32_t(imin(cap, INT32_MAX))};
    const int64_t P = imax(1, lst.period);
    bool broken = false;
    const int64_t rc0 = x.clock();
    int64_t p = p0;
    for (; p < wn && par[g.x_seq2[p]] == root; ++p) {
      const int64_t m = w0 + g.x_seq2[p];
      int32_t* ci = cinfo + m * CI_STRIDE;
      const int32_t stm = ci[CI_STATUS] & 0xf;
      if (stm == CS_SKIP || stm == CS_ERROR || ci[CI_P0] < 0) continue;
      if (broken) {  // an earlier member overflowed: the walk re-scores the rest
        x.wsync();
        if (x.lane == 0) ci[CI_STATUS] = CS_OVERFLOW;
        x.wsync();
        continue;
      }
      // phase-A result still valid against the component's commits so far?
      bool valid = stm != CS_OVERFLOW;
      if (valid && lst.pend_n > 0) {
        const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
        const int32_t nw = ci[CI_NW];
        bool hit = false;
        for (int32_t e = x.lane; e < lst.pend_n && !hit; e += X::W)
          for (int32_t w = 0; w < nw && !hit; ++w) hit = hits(pl.s[e], pl.e[e], wv[2 * w], wv[2 * w + 1], P);
        valid = !x.wany(hit);
      }
      if (valid) {
        if (stm == CS_OK) {  // its pairs join the component's commits
          const PairRec* pr = g.pr_pool + ci[CI_P0];
          const int32_t np = ci[CI_NP];
          if (lst.pend_n + 2 * np > pl.cap) { broken = true; continue; }
          for (int32_t q = x.lane; q < np; q += X::W) {
            const int32_t o = lst.pend_n + 2 * q;
            pl.s[o] = pr[q].os; pl.e[o] = pr[q].oe;
            pl.s[o + 1] = pr[q].is; pl.e[o + 1] = pr[q].ie;
          }
          x.wsync();
          lst.pend_n += 2 * np;
          x.wsync();
        }
        continue;
      }
      ls.comp_rescored += 1;
      pend_sort(x, pl, lst);
      const int32_t s = cand[m] & 0xffffff;
      int64_t earliest = 0, latest = 0;
      const int kind = candidate_kind(J, lst, s, earliest, latest);
      const int32_t capp = kind == 1 ? 1 : imax(1, J.s_off[s + 1] - J.s_off[s]);
      ReCtx<X> c{x, J, lst, pl, g.cfg, &ls, g.pr_pool + ci[CI_P0], 0, capp, false};
      c.win = g.w_pool + 2 * int64_t(ci[CI_W0]);
      c.cap_win = 2 * capp + 2;
      const bool ok = kind == 1 ? schedule_wrapped_swap(c, s) : schedule_swap(c, s, earliest, latest);
      x.wsync();
      if (c.overflow) {
        broken = true;
        if (x.lane == 0) ci[CI_STATUS] = CS_OVERFLOW;
        x.wsync();
        continue;
      }
      if (x.lane == 0) {
        ci[CI_STATUS] = ok ? CS_OK : CS_FAIL;
        ci[CI_NP] = ok ? c.nout : 0;
        ci[CI_NW] = c.nwin;
        int64_t* hl = chull + m * 4;
        hl[0] = INT64_MAX; hl[1] = INT64_MIN; hl[2] = INT64_MAX; hl[3] = INT64_MIN;
        for (int32_t w = 0; w < c.nwin; ++w) { hl[0] = imin(hl[0], c.win[2 * w]); hl[1] = imax(hl[1], c.win[2 * w + 1]); }
        for (int32_t q = 0; ok && q < c.nout; ++q) {
          hl[2] = imin(hl[2], imin(c.out[q].os, c.out[q].is));
          hl[3] = imax(hl[3], imax(c.out[q].oe, c.out[q].ie));
        }
      }
      if (!ok) {  // a failed schedule commits nothing (ReCtx appended nothing)
        x.wsync();
        continue;
      }
      x.wsync();
    }
    if (x.lane == 0) {  // run statistics (stageprof)
      const int64_t rc = x.clock() - rc0;
      x.amax(&g.stats.sprof[21], p - p0);
      x.amax(&g.stats.sprof[22], rc);
      x.aadd(&g.stats.sprof[17], p - p0);
      x.aadd(&g.stats.sprof[18], 1);
      x.aadd(&g.stats.sprof[20], rc);
    }
  }
  if (x.lane == 0) {
    x.aadd(&g.stats.comp_rescored, ls.comp_rescored);
    x.aadd(&g.stats.fit_queries, ls.fit_queries);
    x.aadd(&g.stats.busy_intervals, ls.busy_intervals);
  }
}

// The run processing of component_speculation; an execution context may
// route it elsewhere (the CUDA build spreads it over every CTA of a
// cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD void comp_dispatch(X& x, GroupDev& g, int64_t w0, const int32_t* cand, int32_t* cinfo, int64_t* chull,
                          int64_t nruns) {
  int64_t* gsh = x.sh + MAXB * NF;
  if (X::W > 1 && g.c_wscratch) {  // a grid context: every warp of the launch, each with its own list
    comp_runs(x, g, w0, cand, cinfo, chull, &gsh[GS_CRUN], nruns, g.c_wscratch + int64_t(x.tid / X::W) * 6 * g.c_wscap,
              g.c_wscap);
    return;
  }
  const int64_t cap = (g.wcap * 4) / 6;
  comp_runs(x, g, w0, cand, cinfo, chull, &gsh[GS_CRUN], nruns, g.wbuf + int64_t(x.warp) * 4 * g.wcap, cap);
}

// ---- A2. component speculation (uncoupled swap passes) ----
// Phase B's conflict edges group a window's candidates into components; the
// members of a component (in the candidate order, typically tensors of one
// layer and micro-batch packing into the same channel gaps) are speculated
// again IN ORDER by one warp, against the pass-start state plus the results
// of their earlier component members, so a member's speculation no longer
// conflicts with its own component. A member whose phase-A result survives its
// predecessors' commits keeps it (same validity argument as phase C). The
// grouping only affects speed: phase B is then re-run across components, and
// the in-order walk accepts a member only while every earlier member of its
// component committed its speculation unchanged (CS_DIFF breaks the chain).
template <class X>
TSL_HD void component_speculation(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo,
                                  int64_t* chull) {
  const int64_t wn = w1 - w0;
  volatile int32_t* par = g.c_comp;      // [wn] union-find parent -> root (window-relative)
  int32_t* prv = g.c_comp + g.c_cap;     // [wn] previous member (candidate index) or -1
  int64_t* gsh = x.sh + MAXB * NF;
  for (int64_t i = x.tid; i < wn; i += x.nthr) par[i] = int32_t(i);
  x.sync();
  // hook the larger root under the smaller one (atomic min) until no conflict
  // edge joins two components; a lost race is redone by the next round
  for (int round = 0; round < 64; ++round) {
    if (x.tid == 0) gsh[GS_CCHG] = 0;
    x.sync();
    int64_t chg = 0;
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      const int32_t* ci = cinfo + m * CI_STRIDE;
      const int32_t nc = imin(ci[CI_NCONF], CAPC);
      for (int k = 0; k < nc; ++k) {
        int32_t a = int32_t(m - w0), b = ci[CI_CONF + k] - int32_t(w0);
        while (par[a] != a) a = par[a];
        while (par[b] != b) b = par[b];
        if (a != b) { x.amin32(const_cast<int32_t*>(&par[imax(a, b)]), int32_t(imin(a, b))); chg = 1; }
      }
    }
    if (chg) x.amax(&gsh[GS_CCHG], 1);
    x.sync();
    for (int64_t i = x.tid; i < wn; i += x.nthr) {
      int32_t r = par[i];
      while (par[r] != r) r = par[r];
      par[i] = r;
    }
    x.sync();
    const bool again = gsh[GS_CCHG] != 0;
    x.sync();  // (every thread has read the flag before the next round resets it)
    if (x.tid == 0) g.stats.sprof[23] += 1;  // union-find rounds (stageprof)
    if (!again) break;
  }
  // members of each component in candidate order: sort (root, index)
  const int rb = nbits(uint64_t(wn));
  for (int64_t i = x.tid; i < wn; i += x.nthr) {
    g.x_key2[i] = (uint64_t(par[i]) << rb) | uint64_t(i);
    g.x_seq2[i] = int32_t(i);
  }
  if (x.tid == 0) { gsh[GS_NRUN] = 0; gsh[GS_CRUN] = 0; g.c_wn = wn; }
  x.sync();
  x.sort(g.x_key2, g.x_seq2, int32_t(wn), 2 * rb);
  for (int64_t p = x.tid; p < wn; p += x.nthr) {
    const int32_t i = g.x_seq2[p];
    const bool first = p == 0 || par[g.x_seq2[p - 1]] != par[i];
    prv[i] = first ? -1 : int32_t(w0 + g.x_seq2[p - 1]);
    if (first && p + 1 < wn && par[g.x_seq2[p + 1]] == par[i]) {  // a run of >= 2 members
      const int64_t r = x.aadd(&gsh[GS_NRUN], 1);
      g.x_order[r] = int32_t(p);
    }
  }
  x.sync();
  const int64_t nruns = gsh[GS_NRUN];
  if (x.tid == 0) { g.stats.sprof[21] = 0; g.stats.sprof[22] = 0; }
  x.sync();
  // one warp per run (taken in turn): on every CTA of a cooperative launch
  comp_dispatch(x, g, w0, cand, cinfo, chull, nruns);
  x.sync();
  if (x.tid == 0) {
    const volatile int64_t* sp = g.stats.sprof;
    g.stats.sprof[16] += sp[21];
    g.stats.sprof[19] += sp[22];
  }
  for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) cinfo[m * CI_STRIDE + CI_NCONF] = 0;
  x.sync();
}

// Phase A2 of a window; an execution context may route it elsewhere (the
// CUDA build runs it on every CTA of a cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD void comp_batch(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo,
                       int64_t* chull) {
  component_speculation(x, g, w0, w1, cand, cinfo, chull);
}

// Phase B of a window; an execution context may route it elsewhere (the CUDA
// build runs it on every CTA of a cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD void conflicts_batch(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo,
                            const int64_t* chull, bool coupled, const int32_t* comp) {
  find_conflicts(x, g, w0, w1, cand, cinfo, chull, coupled, comp);
}

// ---- A. speculative scoring of the window [w0, w1), one thread per
// candidate (pool counters GS_PPOOL / GS_WPOOL / GS_PCAP + j in x's scalars).
// No trailing barrier.
template <class X>
TSL_HD void spec_phase(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo, int64_t* chull) {
  int64_t* gsh = x.sh + MAXB * NF;
  {
    GroupStats ls{};
    for (int64_t m = w0 + x.tid; m < w1; m += x.nthr) {
      const int j = cand[m] >> 24;
      const int32_t s = cand[m] & 0xffffff;
      const JobDev& J = g.jobs[j];
      const JobState& st = g.st[j];
      int32_t* ci = cinfo + m * CI_STRIDE;
      int64_t* hl = chull + m * 4;
      ci[CI_NP] = 0; ci[CI_NW] = 0; ci[CI_NCONF] = 0; ci[CI_STATE] = 0; ci[CI_EV0] = 0; ci[CI_ID0] = 0;
      ci[CI_P0] = -1;
      hl[0] = INT64_MAX; hl[1] = INT64_MIN; hl[2] = INT64_MAX; hl[3] = INT64_MIN;
      if (J.swapped[s]) { ci[CI_STATUS] = CS_SKIP; continue; }
      int64_t earliest = 0, latest = 0;
      const int kind = candidate_kind(J, st, s, earliest, latest);
      if (kind == 0) { ci[CI_STATUS] = CS_SKIP; continue; }
      if (kind < 0) { ci[CI_STATUS] = CS_ERROR; continue; }
      const int32_t capp = kind == 1 ? 1 : imax(1, J.s_off[s + 1] - J.s_off[s]);
      const int32_t capw = 2 * capp + 2;
      const int64_t p0 = x.aadd(&gsh[GS_PPOOL], capp);
      const int64_t wp0 = x.aadd(&gsh[GS_WPOOL], capw);
      x.aadd(&gsh[GS_PCAP + j], capp);
      if (p0 + capp > g.pr_cap || wp0 + capw > g.w_cap) { ci[CI_STATUS] = CS_OVERFLOW; continue; }
      ci[CI_P0] = int32_t(p0);
      SpecCtx c{J, st, g.cfg, &ls, g.pr_pool + p0, 0, capp, g.w_pool + 2 * wp0, 0, capw, false};
      const bool ok = kind == 1 ? schedule_wrapped_swap(c, s) : schedule_swap(c, s, earliest, latest);
      ci[CI_STATUS] = c.overflow ? CS_OVERFLOW : (ok ? CS_OK : CS_FAIL);
      ci[CI_NP] = c.npairs;
      ci[CI_W0] = int32_t(wp0);
      ci[CI_NW] = c.nwin;
      for (int32_t w = 0; w < c.nwin; ++w) {
        hl[0] = imin(hl[0], c.win[2 * w]);
        hl[1] = imax(hl[1], c.win[2 * w + 1]);
      }
      for (int32_t p = 0; p < c.npairs; ++p) {
        hl[2] = imin(hl[2], imin(c.pairs[p].os, c.pairs[p].is));
        hl[3] = imax(hl[3], imax(c.pairs[p].oe, c.pairs[p].ie));
      }
    }
    if (ls.fit_queries | ls.busy_intervals | ls.candidate_accesses) {  // (idle grid threads skip the atomics)
      x.aadd(&g.stats.fit_queries, ls.fit_queries);
      x.aadd(&g.stats.busy_intervals, ls.busy_intervals);
      x.aadd(&g.stats.candidate_accesses, ls.candidate_accesses);
    }
  }
}

// Phase A of a window; an execution context may route it elsewhere (the CUDA
// build runs it on every CTA of a cooperative launch, tsl_kernel.cu).
template <class X>
TSL_HD void spec_batch(X& x, GroupDev& g, int64_t w0, int64_t w1, const int32_t* cand, int32_t* cinfo, int64_t* chull) {
  spec_phase(x, g, w0, w1, cand, cinfo, chull);
}

template <class X>
TSL_HD bool swap_pass(X& x, GroupDev& g) {
  int64_t* sh = x.sh;
  int64_t pc0 = x.clock();
  auto ptick = [&](int k) { const int64_t c = x.clock(); if (x.tid == 0) g.stats.sprof[k] += c - pc0; pc0 = c; };
  int64_t* gsh = sh + MAXB * NF;  // [9]=maxT [10]=changed [11]=cursor [12]=maxsize [13..14] pools [16..] segments
  if (x.tid == 0) {
    int64_t maxT = 1;
    for (int j = 0; j < g.n_jobs; ++j) maxT = imax(maxT, g.jobs[j].T);
    gsh[9] = maxT; gsh[10] = 0; gsh[11] = 0; gsh[12] = 1; gsh[GS_PPOOL] = 0; gsh[GS_WPOOL] = 0; gsh[GS_WK] = 0;
    for (int j = 0; j < g.n_jobs; ++j) {
      JobState& st = g.st[j];
      st.bz_n = st.S; st.S_pass = st.S; st.pend_n = 0; st.pend_sorted = 0;
      gsh[GS_PCAP + j] = 0;
    }
  }
  x.sync();
  for (int j = 0; j < g.n_jobs; ++j) {  // (the evaluator lists each job's peak storages)
    const JobDev& J = g.jobs[j];
    int64_t mx = 1;
    for (int32_t i = x.tid; i < g.st[j].n_peak; i += x.nthr) mx = imax(mx, J.t_size[J.pk_list[i]]);
    x.amax(&gsh[12], mx);
  }
  x.sync();
  ptick(11);
  const int jbits = nbits(uint64_t(g.n_jobs - 1));
  const int rbits = nbits(uint64_t(gsh[9] - 1));
  const int sbits = nbits(uint64_t(gsh[12]));
  const uint64_t smax = (sbits >= 63) ? (~0ull >> 1) : ((1ull << sbits) - 1);
  const bool coupled = g.coupled != 0;
  // candidates: every job's peak tensors (the report stays stale for the whole
  // pass), ordered (size desc, job id, storage id) -- swap_planner.cpp:469-481
  for (int j = 0; j < g.n_jobs; ++j) {
    const JobDev& J = g.jobs[j];
    for (int32_t i = x.tid; i < g.st[j].n_peak; i += x.nthr) {
      const int32_t t = J.pk_list[i];
      const int64_t slot = x.aadd(&gsh[11], 1);
      if (slot >= g.ecap) continue;
      const uint64_t inv = smax - uint64_t(J.t_size[t]);
      uint64_t k;
      if (coupled) k = (((inv << jbits) | uint64_t(J.rank)) << rbits) | uint64_t(J.t_rank[t]);
      else k = (((uint64_t(j) << sbits) | inv) << rbits) | uint64_t(J.t_rank[t]);
      g.k_key[slot] = k;
      g.k_val[slot] = (j << 24) | t;  // the host guarantees T < 2^24 and <= 128 jobs
    }
  }
  x.sync();
  const int64_t nc = gsh[11];
  if (nc > g.ecap) {
    if (x.tid == 0) { g.err.code = E_CAPACITY; g.err.job = -1; g.err.tensor = nc; g.err.tick = 1; }
    x.sync();
    return false;
  }
  ptick(12);
  x.sort(g.k_key, g.k_val, int32_t(nc), jbits + sbits + rbits);
  ptick(13);
  // component speculation (phase A2): spec_comp 2 always, 1 for passes of
  // at least COMP_MIN_CANDIDATES candidates (below that -- C1's ~40 -- the
  // extra phase costs more than the few re-scores it saves), 0 never
  const bool comp_on = !coupled && (g.spec_comp == 2 || (g.spec_comp == 1 && nc >= COMP_MIN_CANDIDATES));
  // Candidate records live in shared memory when they fit (the sort scratch
  // is free until phase E): the in-order decisions read them back-to-back.
  int32_t* cand = g.k_val;
  int32_t* cinfo = g.c_info;
  int64_t* chull = g.c_hull;
  size_t rec_bytes = 0;  // shared scratch taken by the candidate records
  {
    const size_t need = size_t(nc) * (sizeof(int64_t) * 4 + sizeof(int32_t) * (CI_STRIDE + 2)) + 64;
    // (component speculation sorts in that scratch, and a cooperative
    // launch's grid phases read the records from every SM: records stay in HBM)
    if (need <= x.tmp_bytes && !comp_on && !(g.coop && g.grid_conf)) {
      chull = reinterpret_cast<int64_t*>(x.tmp);
      cinfo = reinterpret_cast<int32_t*>(chull + 4 * nc);
      cand = cinfo + CI_STRIDE * nc;
      rec_bytes = (need + 15) & ~size_t(15);
    }
  }
  if (cand != g.k_val)
    for (int64_t m = x.tid; m < nc; m += x.nthr) cand[m] = g.k_val[m];
  // segment starts: first candidate of each job (candidates are job-major
  // when uncoupled)
  for (int j = x.tid; j <= g.n_jobs; j += x.nthr) gsh[16 + j] = nc;
  x.sync();
  if (!coupled)
    for (int64_t m = x.tid; m < nc; m += x.nthr) x.amin(&gsh[16 + (cand[m] >> 24)], m);
  x.sync();
  if (x.tid == 0) {
    g.stats.candidates += nc;
    g.stats.sort_elems += nc;
    if (!coupled)
      for (int j = g.n_jobs - 1; j >= 0; --j) gsh[16 + j] = imin(gsh[16 + j], gsh[16 + j + 1]);
  }
  x.sync();
  ptick(14);
  int64_t t0 = x.clock(), t1;
  auto tick = [&](int k) { t1 = x.clock(); if (x.tid == 0) g.stats.cyc[k] += t1 - t0; t0 = t1; };
  // Speculation windows: phases A-C run on consecutive windows of the
  // candidate order [w0, w1). A window's speculation is taken against the
  // state after every earlier window (their commits are folded into the busy
  // structure at the end of each window's decisions), so it only has to
  // survive the commits of its own window -- the validity argument of
  // phase A holds unchanged relative to the window start. Coupled groups (one
  // global walk) use one window.
  const int64_t WIN = (coupled || g.spec_window <= 0) ? nc : int64_t(g.spec_window);
  for (int64_t w0 = 0; w0 < nc;) {
  const int64_t w1 = imin(nc, w0 + WIN);
  const int64_t wn = w1 - w0;
  if (x.tid == 0) {
    gsh[GS_WK] = 0;
    for (int j = 0; j < g.n_jobs; ++j) {
      gsh[GS_PCAP + j] = 0;
      JobState& st = g.st[j];
      st.pend_n = 0; st.pend_sorted = 0;
      st.pend_upto = coupled ? 0 : int32_t(imax(gsh[16 + j], w0));
    }
  }
  x.sync();
  // ---- A. speculative scoring, one thread per candidate ----
  spec_batch(x, g, w0, w1, cand, cinfo, chull);
  x.sync();
  if (x.tid == 0) g.stats.sprof[15] += x.clock() - t0;
  tick(5);
  // ---- B. conflicts with earlier speculative commits of the same job ----
  conflicts_batch(x, g, w0, w1, cand, cinfo, chull, coupled, nullptr);
  const bool use_comp = comp_on && wn > 1;
  if (use_comp) {
    x.sync();
    tick(6);
    comp_batch(x, g, w0, w1, cand, cinfo, chull);
    tick(5);
    // conflicts across components (a member's speculation includes its own
    // component's earlier results)
    conflicts_batch(x, g, w0, w1, cand, cinfo, chull, coupled, g.c_comp);
  }
  x.sync();
  tick(6);
#if TSL_EMU_STATS
  {  // conflict components of this window (union-find over the conflict lists)
    std::vector<int64_t> par(wn);
    for (int64_t i = 0; i < wn; ++i) par[i] = i;
    auto find = [&](int64_t a) { while (par[a] != a) a = par[a] = par[par[a]]; return a; };
    int64_t over = 0, edges = 0;
    for (int64_t m = w0; m < w1; ++m) {
      const int32_t* ci = cinfo + m * CI_STRIDE;
      if ((ci[CI_STATUS] & 0xf) == CS_SKIP) continue;
      if (ci[CI_NCONF] > CAPC) ++over;
      for (int k = 0; k < imin(ci[CI_NCONF], CAPC); ++k) {
        ++edges;
        par[find(m - w0)] = find(ci[CI_CONF + k] - w0);
      }
    }
    std::vector<int64_t> sz(wn, 0);
    for (int64_t i = 0; i < wn; ++i) sz[find(i)]++;
    int64_t mx = 0, big = 0, ncomp = 0;
    for (int64_t i = 0; i < wn; ++i)
      if (sz[i]) { ++ncomp; mx = imax(mx, sz[i]); if (sz[i] > 32) big += sz[i]; }
    emu_stats::passes++;
    emu_stats::comp_max = imax(emu_stats::comp_max, mx);
    emu_stats::comp_sum_max += mx;
    emu_stats::comp_big += big;
    emu_stats::conf_over += over;
    emu_stats::conf_edges += edges;
    emu_stats::cands += wn;
  }
#endif
  // ---- C. in-order decisions ----
  const int nseg = coupled ? 1 : g.n_jobs;
  if (!coupled) {
    // pend buffers: a job commits at most 2 intervals per reserved pair slot;
    // when every job's bound fits the free sort scratch they all live there
    if (x.tid == 0) {
      int64_t off = 0;
      for (int j = 0; j < g.n_jobs; ++j) {
        gsh[GS_POFF + j] = off;
        off += 6 * (2 * gsh[GS_PCAP + j] + 2);
      }
      // (a cooperative launch's workers fold pend lists: keep them in HBM)
      gsh[GS_POFF - 1] = (g.coop == nullptr &&
                          int64_t(rec_bytes) + off * int64_t(sizeof(int64_t)) <= int64_t(x.tmp_bytes)) ? 1 : 0;
    }
    x.sync();
    const bool pend_shared = gsh[GS_POFF - 1] != 0;
    for (int seg = x.warp; seg < nseg; seg += x.nwarp) {
      GroupStats ls{};
      ErrInfo lerr{};
      const JobDev& Jg = g.jobs[seg];
      PendBuf pb{Jg.pd_s, Jg.pd_e, Jg.pd_ts, Jg.pd_te, g.wbuf + int64_t(x.warp) * 4 * g.wcap, Jg.Scap};
      if (pend_shared) {
        const int32_t cap = int32_t(2 * gsh[GS_PCAP + seg] + 2);
        int64_t* b = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(x.tmp) + rec_bytes) + gsh[GS_POFF + seg];
        pb = PendBuf{b, b + cap, b + 2 * cap, b + 3 * cap, b + 4 * cap, cap};
      }
      const bool ch = decide_chunked(x, g, seg, imax(w0, gsh[16 + seg]), imin(w1, gsh[16 + seg + 1]), cand, cinfo,
                                     chull, pb, ls, lerr, w1 < nc, use_comp ? g.c_comp + g.c_cap : nullptr, w0);
      x.wsync();
      if (x.lane == 0) {
        if (ch) gsh[10] = 1;
        if (lerr.code) x.errset(g, lerr);
        x.aadd(&g.stats.fit_queries, ls.fit_queries);
        x.aadd(&g.stats.busy_intervals, ls.busy_intervals);
        x.aadd(&g.stats.candidate_accesses, ls.candidate_accesses);
        x.aadd(&g.stats.rescored, ls.rescored);
#if TSL_PROF
        for (int k = 0; k < 16; ++k) x.aadd(&g.stats.prof[k], ls.prof[k]);
#endif
      }
    }
  }
  for (int seg = x.warp; coupled && seg < nseg; seg += x.nwarp) {
    GroupStats ls{};
    ErrInfo lerr{};
    const int64_t m0 = coupled ? 0 : gsh[16 + seg];
    const int64_t m1 = coupled ? nc : gsh[16 + seg + 1];
    int64_t* wtmp = g.wbuf + int64_t(x.warp) * 4 * g.wcap;
    int32_t ndev = 0;
    int64_t dev_lo = INT64_MAX, dev_hi = INT64_MIN;  // hull of re-scored commits (raw)
    bool changed = false;
    for (int64_t m = m0; m < m1; ++m) {
      int32_t* ci = cinfo + m * CI_STRIDE;
      const int32_t status = ci[CI_STATUS];
      if (status == CS_SKIP) continue;
      const int j = cand[m] >> 24;
      const int32_t s = cand[m] & 0xffffff;
      const JobDev& J = g.jobs[j];
      JobState& st = g.st[j];
      if (coupled && g.total_swapped != 0) {  // SwapBudget::allows, swap_planner.cpp:268-276
        const double lhs = double(st.son + 1) / double(g.total_swapped + 1);
        if (!(lhs <= J.ratio)) continue;
      }
      if (status == CS_ERROR) { lerr.code = E_NO_TGA; lerr.job = j; lerr.tensor = s; lerr.tick = 0; break; }
      if (ci[CI_P0] < 0) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = g.pr_cap; lerr.tick = 4; break; }
      const int64_t P = imax(1, st.period);
      bool valid = status != CS_OVERFLOW && ci[CI_NCONF] <= CAPC;
      for (int32_t k = 0; valid && k < ci[CI_NCONF]; ++k)
        if (cinfo[int64_t(ci[CI_CONF + k]) * CI_STRIDE + CI_STATE] == 1) valid = false;
      if (valid && ndev && ci[CI_NW] && hits(dev_lo, dev_hi, chull[m * 4], chull[m * 4 + 1], P)) {
        const int64_t* wv = g.w_pool + 2 * int64_t(ci[CI_W0]);
        for (int32_t d = 0; d < ndev && valid; ++d) {
          const int64_t dm = g.dev_list[m0 + d];
          if ((cand[dm] >> 24) != j) continue;
          const int32_t* cd = cinfo + dm * CI_STRIDE;
          const PairRec* pr = g.pr_pool + cd[CI_P0];
          for (int32_t p = 0; p < cd[CI_NP] && valid; ++p)
            for (int32_t w = 0; w < ci[CI_NW] && valid; ++w)
              if (hits(pr[p].os, pr[p].oe, wv[2 * w], wv[2 * w + 1], P) ||
                  hits(pr[p].is, pr[p].ie, wv[2 * w], wv[2 * w + 1], P))
                valid = false;
        }
      }
      int32_t np = 0;
      int32_t state = 0;
      if (valid) {
        if (status == CS_OK) { np = ci[CI_NP]; state = 1; }
      } else {
        ls.rescored += 1;
        const int64_t rc0 = x.clock();
        PendBuf pbj{J.pd_s, J.pd_e, J.pd_ts, J.pd_te, wtmp, J.Scap};
        // bring this pass's pend list up to date: intervals of every candidate
        // of this job committed since the last re-score (lanes in parallel)
        for (int64_t q = st.pend_upto; q < m; ++q) {
          const int32_t* cq = cinfo + q * CI_STRIDE;
          if (cq[CI_STATE] != 1 || (cand[q] >> 24) != j) continue;
          const int32_t nq = cq[CI_NP];
          const int32_t pn = st.pend_n;
          if (pn + 2 * nq > J.Scap) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; break; }
          const PairRec* pr = g.pr_pool + cq[CI_P0];
          x.wsync();
          for (int32_t p = x.lane; p < nq; p += X::W) {
            pbj.s[pn + 2 * p] = pr[p].os; pbj.e[pn + 2 * p] = pr[p].oe;
            pbj.s[pn + 2 * p + 1] = pr[p].is; pbj.e[pn + 2 * p + 1] = pr[p].ie;
          }
          st.pend_n = pn + 2 * nq;
          x.wsync();
        }
        if (lerr.code) break;
        x.wsync();
        st.pend_upto = int32_t(m);
        x.wsync();
        const int64_t ps0 = x.clock();
        pend_sort(x, pbj, st, false);
        if (x.tid == 0) g.stats.cyc[11] += x.clock() - ps0;
        int64_t earliest = 0, latest = 0;
        const int kind = candidate_kind(J, st, s, earliest, latest);
        const int32_t capp = kind == 1 ? 1 : imax(1, J.s_off[s + 1] - J.s_off[s]);
        ReCtx<X> c{x, J, st, pbj, g.cfg, &ls, g.pr_pool + ci[CI_P0], 0, capp, false};
        c.dbg = &g.stats.cyc[12];
        const bool ok = kind == 1 ? schedule_wrapped_swap(c, s) : schedule_swap(c, s, earliest, latest);
        if (x.tid == 0) g.stats.cyc[10] += x.clock() - rc0;
        if (c.overflow) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; lerr.tick = 5; break; }
        if (ok) {
          np = c.nout;
          state = 2;
          int64_t lo = dev_lo, hi = dev_hi;
          for (int32_t p = 0; p < np; ++p) {
            lo = imin(lo, imin(c.out[p].os, c.out[p].is));
            hi = imax(hi, imax(c.out[p].oe, c.out[p].ie));
          }
          dev_lo = lo;
          dev_hi = hi;
          x.wsync();
          g.dev_list[m0 + ndev] = m;
          ci[CI_NP] = np;
          ++ndev;
          x.wsync();
        }
      }
      if (state) {  // SwapBudget::record + event slots/ids in plan order
        const int64_t son = st.son, tot = g.total_swapped;
        const int32_t S = st.S;
        const int64_t id = st.next_id;
        if (S + 2 * np > J.Scap) { lerr.code = E_CAPACITY; lerr.job = j; lerr.tensor = J.Scap; break; }
        x.wsync();
        ci[CI_STATE] = state;
        ci[CI_EV0] = S;
        ci[CI_ID0] = int32_t(id);
        J.swapped[s] = 1;
        st.son = son + 1;
        if (coupled) g.total_swapped = tot + 1;
        st.S = S + 2 * np;
        st.next_id = id + 2 * np;
        st.dirty = 1;
        changed = true;
        x.wsync();
      }
    }
    x.wsync();
    if (x.lane == 0) {
      if (changed) gsh[10] = 1;
      if (lerr.code) x.errset(g, lerr);
      x.aadd(&g.stats.fit_queries, ls.fit_queries);
      x.aadd(&g.stats.busy_intervals, ls.busy_intervals);
      x.aadd(&g.stats.candidate_accesses, ls.candidate_accesses);
      x.aadd(&g.stats.rescored, ls.rescored);
    }
  }
  x.sync();
  tick(7);
  if (g.err.code) return false;
  w0 = w1;
  }
  // ---- D. write the committed events (make_event + pair links + flags) ----
  for (int64_t m = x.tid; m < nc; m += x.nthr) {
    const int32_t* ci = cinfo + m * CI_STRIDE;
    if (!ci[CI_STATE]) continue;
    const int j = cand[m] >> 24;
    const JobDev& J = g.jobs[j];
    const PairRec* pr = g.pr_pool + ci[CI_P0];
    const int32_t np = ci[CI_NP];
    for (int32_t p = 0; p < np; ++p) {
      const PairRec& r = pr[p];
      const int32_t i0 = ci[CI_EV0] + 2 * p, i1 = i0 + 1;
      const int64_t id0 = int64_t(ci[CI_ID0]) + 2 * p, id1 = id0 + 1;
      J.ev_id[i0] = id0; J.ev_tensor[i0] = r.store; J.ev_dir[i0] = 0; J.ev_wraps[i0] = int8_t(r.wraps);
      J.ev_trig[i0] = r.otrig; J.ev_delta[i0] = r.odelta; J.ev_start[i0] = r.os; J.ev_end[i0] = r.oe;
      J.ev_earl[i0] = r.o_earl; J.ev_late[i0] = r.o_late; J.ev_pair[i0] = id1; J.ev_serves[i0] = -1;
      J.ev_id[i1] = id1; J.ev_tensor[i1] = r.store; J.ev_dir[i1] = 1; J.ev_wraps[i1] = int8_t(r.wraps);
      J.ev_trig[i1] = r.itrig; J.ev_delta[i1] = r.idelta; J.ev_start[i1] = r.is; J.ev_end[i1] = r.ie;
      J.ev_earl[i1] = r.i_earl; J.ev_late[i1] = r.i_late; J.ev_pair[i1] = id0; J.ev_serves[i1] = r.serves;
      if (r.pre >= 0) J.a_flag[r.pre] = 1;
    }
    x.aadd32(&J.st_evcnt[cand[m] & 0xffffff], 2 * np);
  }
  x.sync();
  tick(8);
  // ---- E. sorted busy structure for the next pass ----
  if (gsh[10]) rebuild_batch(x, g);
  tick(9);
  return gsh[10] != 0;
}

// ----------------------------------------------------------------------------
// revalidate_swap_events + rebuild_release_flags (swap_planner.cpp:171-266)
// ----------------------------------------------------------------------------
TSL_HD bool ovl_mod(int64_t s1, int64_t e1, int64_t s2, int64_t e2, int64_t P) {
  for (int k = -1; k <= 1; ++k) {
    const int64_t sh = k * P;
    if (s1 + sh < e2 && s2 < e1 + sh) return true;
  }
  return false;
}

template <class X>
TSL_HD void rebuild_flags(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  const JobState& st = g.st[j];
  for (int32_t a = x.tid; a < J.A; a += x.nthr) J.a_flag[a] = J.a_base[a];
  x.sync();
  for (int32_t i = x.tid; i < st.S; i += x.nthr) {
    if (J.ev_dir[i] != 0) continue;
    int32_t p = preceding_access(J, J.t_store[J.ev_tensor[i]], J.ev_start[i], -2);
    if (p >= 0) J.a_flag[p] = 1;
  }
  for (int32_t r = x.tid; r < st.R; r += x.nthr) {
    const int64_t tg = J.rc_target[r];
    int32_t p = preceding_access(J, J.t_store[J.rc_tensor[r]], J.a_start[tg], tg);
    if (p >= 0) J.a_flag[p] = 1;
  }
  x.sync();
}

// Rebuilds the sorted busy structure, per-storage counts and next_event_id.
template <class X>
TSL_HD void rebuild_index(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  int64_t* gsh = x.sh + MAXB * NF;
  if (x.tid == 0) { gsh[20] = INT64_MAX; gsh[21] = INT64_MIN; gsh[22] = 0; }
  for (int32_t t = x.tid; t < J.T; t += x.nthr) J.st_evcnt[t] = 0;
  x.sync();
  int64_t mn = INT64_MAX, mx = INT64_MIN, mid = -1;
  for (int32_t i = x.tid; i < st.S; i += x.nthr) {
    mn = imin(mn, J.ev_start[i]);
    mx = imax(mx, J.ev_start[i]);
    mid = imax(mid, J.ev_id[i]);
    x.aadd32(&J.st_evcnt[J.ev_tensor[i]], 1);
  }
  for (int32_t r = x.tid; r < st.R; r += x.nthr) mid = imax(mid, J.rc_id[r]);
  if (mn != INT64_MAX) { x.amin(&gsh[20], mn); x.amax(&gsh[21], mx); }
  x.amax(&gsh[22], mid + 1);
  x.sync();
  const int64_t lo = gsh[20];
  const int bits = st.S > 0 ? nbits(uint64_t(gsh[21] - lo)) : 0;
  const int ib = nbits(uint64_t(st.S > 0 ? st.S - 1 : 0));
  for (int32_t i = x.tid; i < st.S; i += x.nthr) {
    g.k_key[i] = (uint64_t(J.ev_start[i] - lo) << ib) | uint64_t(i);
    g.k_val[i] = i;
  }
  x.sync();
  x.sort(g.k_key, g.k_val, st.S, bits + ib);
  for (int32_t m = x.tid; m < st.S; m += x.nthr) {
    const int32_t i = g.k_val[m];
    J.bz_s[m] = J.ev_start[i];
    J.bz_e[m] = J.ev_end[i];
  }
  if (x.tid == 0) st.next_id = gsh[22];
  x.sync();
  build_busy_index(x, g, j);
}

template <class X>
TSL_HD bool revalidate(X& x, GroupDev& g, int j) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  const int64_t P = imax(1, st.period);
  int64_t* gsh = x.sh + MAXB * NF;
  if (x.tid == 0) gsh[23] = 0;
  x.sync();
  // re-derive absolute times from the (trigger, delta) anchors
  for (int32_t i = x.tid; i < st.S; i += x.nthr) {
    const int64_t tr = J.ev_trig[i];
    if (tr != -1 && (tr < 0 || tr >= J.A)) { x.amax(&gsh[23], 1); continue; }
    const int64_t base = tr == -1 ? 0 : J.a_end[tr];
    const int64_t d = duration(J.t_size[J.t_store[J.ev_tensor[i]]], g.cfg);
    int64_t s = base + J.ev_delta[i];
    if (J.ev_wraps[i] && J.ev_dir[i] == 1) s += P;
    J.ev_start[i] = s;
    J.ev_end[i] = s + d;
    J.ev_drop[i] = 0;
  }
  x.sync();
  if (gsh[23]) {
    if (x.tid == 0) { g.err.code = E_UNKNOWN_ACCESS; g.err.job = j; g.err.tensor = -1; g.err.tick = 0; }
    x.sync();
    return false;
  }
  // keep pairs in event order against an accumulating kept set (bz_* reused)
  if (x.warp == 0) {
    int32_t nk = 0;
    for (int32_t i = 0; i < st.S; ++i) {
      if (J.ev_dir[i] != 0) continue;
      int32_t in = -1;
      if (J.ev_pair[i] >= 0) {
        if (i + 1 < st.S && J.ev_id[i + 1] == J.ev_pair[i]) in = i + 1;
        else
          for (int32_t k = 0; k < st.S; ++k)
            if (J.ev_id[k] == J.ev_pair[i]) { in = k; break; }
      }
      bool ok = in >= 0 && J.ev_end[i] <= J.ev_start[in];
      if (ok && J.ev_serves[in] >= 0) {
        int64_t deadline = J.a_start[J.ev_serves[in]];
        if (J.ev_wraps[in]) deadline += P;
        ok = J.ev_end[in] <= deadline;
      }
      if (ok) {
        const int32_t s = J.t_store[J.ev_tensor[i]];
        bool bad = false;
        for (int32_t k = J.s_off[s] + x.lane; k < J.s_off[s + 1]; k += X::W) {
          const int32_t a = J.s_acc[k];
          if (ovl_mod(J.ev_start[i], J.ev_end[i], J.a_start[a], J.a_end[a], P) ||
              ovl_mod(J.ev_start[in], J.ev_end[in], J.a_start[a], J.a_end[a], P))
            bad = true;
        }
        for (int32_t k = x.lane; k < nk; k += X::W) {
          if (ovl_mod(J.ev_start[i], J.ev_end[i], J.bz_s[k], J.bz_e[k], P) ||
              ovl_mod(J.ev_start[in], J.ev_end[in], J.bz_s[k], J.bz_e[k], P))
            bad = true;
        }
        ok = !x.wany(bad);
      }
      if (!ok) {
        J.ev_drop[i] = 1;
        if (in >= 0) J.ev_drop[in] = 1;
      } else {
        x.wsync();
        J.bz_s[nk] = J.ev_start[i]; J.bz_e[nk] = J.ev_end[i];
        J.bz_s[nk + 1] = J.ev_start[in]; J.bz_e[nk + 1] = J.ev_end[in];
        nk += 2;
      }
      x.wsync();
    }
    x.wsync();  // every lane is past its last read of st.S before lane 0 rewrites it
    // stable compaction (lane 0; pairs are rare to drop)
    if (x.lane == 0) {
      int32_t w = 0;
      for (int32_t i = 0; i < st.S; ++i) {
        if (J.ev_drop[i]) continue;
        if (w != i) {
          J.ev_id[w] = J.ev_id[i]; J.ev_tensor[w] = J.ev_tensor[i]; J.ev_dir[w] = J.ev_dir[i];
          J.ev_wraps[w] = J.ev_wraps[i]; J.ev_trig[w] = J.ev_trig[i]; J.ev_delta[w] = J.ev_delta[i];
          J.ev_start[w] = J.ev_start[i]; J.ev_end[w] = J.ev_end[i]; J.ev_earl[w] = J.ev_earl[i];
          J.ev_late[w] = J.ev_late[i]; J.ev_pair[w] = J.ev_pair[i]; J.ev_serves[w] = J.ev_serves[i];
        }
        ++w;
      }
      st.S = w;
    }
  }
  x.sync();
  rebuild_flags(x, g, j);
  rebuild_index(x, g, j);
  return true;
}

// ----------------------------------------------------------------------------
// Recompute pass (recompute_planner.cpp:50-153)
// ----------------------------------------------------------------------------
template <class X>
TSL_HD void backup_job(X& x, GroupDev& g, int j, bool restore, int32_t S, int32_t R, int64_t nc) {
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  int64_t* E[EV_FIELDS] = {J.ev_id, nullptr, nullptr, nullptr, J.ev_trig, J.ev_delta,
                           J.ev_start, J.ev_end, J.ev_earl, J.ev_late, J.ev_pair, J.ev_serves};
  (void)st;
  auto cp64 = [&](int64_t* live, int64_t* bk, int64_t n) {
    for (int64_t i = x.tid; i < n; i += x.nthr) { if (restore) live[i] = bk[i]; else bk[i] = live[i]; }
  };
  auto cp8 = [&](uint8_t* live, uint8_t* bk, int64_t n) {
    for (int64_t i = x.tid; i < n; i += x.nthr) { if (restore) live[i] = bk[i]; else bk[i] = live[i]; }
  };
  cp64(J.a_start, J.bk_a_start, J.A);
  cp64(J.a_end, J.bk_a_end, J.A);
  cp8(J.a_flag, J.bk_flag, J.A);
  cp8(J.in_peak, J.bk_in_peak, J.T);
  for (int f = 0; f < EV_FIELDS; ++f)
    if (E[f]) cp64(E[f], J.bk_ev + int64_t(f) * J.Scap, S);
  for (int32_t i = x.tid; i < S; i += x.nthr) {  // narrow fields packed into word 1..3
    int64_t* b1 = J.bk_ev + 1LL * J.Scap;
    int64_t* b2 = J.bk_ev + 2LL * J.Scap;
    if (restore) {
      J.ev_tensor[i] = int32_t(b1[i]);
      J.ev_dir[i] = int8_t(b2[i] & 0xff);
      J.ev_wraps[i] = int8_t(b2[i] >> 8);
    } else {
      b1[i] = J.ev_tensor[i];
      b2[i] = int64_t(uint8_t(J.ev_dir[i])) | (int64_t(uint8_t(J.ev_wraps[i])) << 8);
    }
  }
  cp64(J.rc_id, J.bk_rc, R);
  cp64(J.rc_target, J.bk_rc + 2LL * J.Rcap, R);
  cp64(J.rc_lat, J.bk_rc + 4LL * J.Rcap, R);
  cp64(J.rc_saving, J.bk_rc + 5LL * J.Rcap, R);
  for (int32_t r = x.tid; r < R; r += x.nthr) {
    int64_t* b1 = J.bk_rc + 1LL * J.Rcap;
    int64_t* b3 = J.bk_rc + 3LL * J.Rcap;
    if (restore) { J.rc_tensor[r] = int32_t(b1[r]); J.rc_regen[r] = int32_t(b3[r]); }
    else { b1[r] = J.rc_tensor[r]; b3[r] = J.rc_regen[r]; }
  }
  cp64(J.bz_s, J.bk_bz, S);
  cp64(J.bz_e, J.bk_bz + J.Scap, S);
  for (int32_t t = x.tid; t < J.T; t += x.nthr) {
    if (restore) J.st_evcnt[t] = J.bk_evcnt[t]; else J.bk_evcnt[t] = J.st_evcnt[t];
  }
  cp64(J.curve_t, J.bk_curve, nc);
  cp64(J.curve_b, J.bk_curve + (J.Ecap + 1), nc);
  x.sync();
}

template <class X>
TSL_HD bool recompute_pass(X& x, GroupDev& g) {
  int64_t* gsh = x.sh + MAXB * NF;
  int64_t merged = 0;
  for (int j = 0; j < g.n_jobs; ++j) merged += g.st[j].peak;
  if (merged < g.cfg.budget) return false;  // strict (recompute_planner.cpp:54)
  // candidates (recompute_planner.cpp:56-110): one thread per (job, tensor)
  if (x.tid == 0) gsh[24] = 0;
  x.sync();
  for (int j = 0; j < g.n_jobs; ++j) {
    const JobDev& J = g.jobs[j];
    const JobState& st = g.st[j];
    for (int32_t i = x.tid; i < st.n_peak; i += x.nthr) {
      const int32_t t = J.pk_list[i];
      if (J.t_kind[t] != K_INTERIM) continue;
      if (J.st_evcnt[t] > 0) continue;  // storage_has_swap
      bool rec = false;
      for (int32_t r = 0; r < st.R; ++r) if (J.rc_tensor[r] == t) rec = true;
      if (rec) continue;
      const int32_t p = J.t_prod[t];
      if (p < 0) continue;
      bool resident = true;
      for (int32_t i = J.o_in_off[p]; i < J.o_in_off[p + 1] && resident; ++i) {
        const int32_t s = J.t_store[J.o_in[i]];
        if (J.st_evcnt[s] > 0) resident = false;
        for (int32_t k = J.s_off[s]; k < J.s_off[s + 1] && resident; ++k)
          if (J.a_flag[J.s_acc[k]]) resident = false;
      }
      if (!resident) continue;
      const int64_t lat = J.o_lat[p];
      if (lat <= 0) continue;
      int32_t target = -1, preceding = -1;
      for (int32_t k = J.s_off[t]; k < J.s_off[t + 1]; ++k) {
        const int32_t a = J.s_acc[k];
        if (J.a_type[a] == ACC_TUA && J.a_start[a] > st.peak_time) { target = a; break; }
        preceding = a;
      }
      if (target < 0 || preceding < 0) continue;
      if (J.a_end[preceding] > st.peak_time) continue;
      const int64_t slot = x.aadd(&gsh[24], 1);
      if (slot >= g.ecap) continue;
      g.x_time[slot] = (int64_t(j) << 32) | t;   // candidate identity
      g.x_fp[slot] = target;
    }
  }
  x.sync();
  const int64_t nc = imin(gsh[24], g.ecap);
  if (nc == 0) return false;
  // argmax (msps desc, job id asc, tensor id asc) -- recompute_planner.cpp:113-119
  if (x.tid == 0) {
    int64_t best = -1;
    double bv = 0;
    for (int64_t c = 0; c < nc; ++c) {
      const int j = int(g.x_time[c] >> 32);
      const int32_t t = int32_t(g.x_time[c] & 0xffffffff);
      const JobDev& J = g.jobs[j];
      const double v = double(J.t_size[t]) / double(J.o_lat[J.t_prod[t]]);
      bool better = best < 0;
      if (!better) {
        const int bj = int(g.x_time[best] >> 32);
        const int32_t bt = int32_t(g.x_time[best] & 0xffffffff);
        if (v != bv) better = v > bv;
        else if (J.rank != g.jobs[bj].rank) better = J.rank < g.jobs[bj].rank;
        else better = J.t_rank[t] < g.jobs[bj].t_rank[bt];
      }
      if (better) { best = c; bv = v; }
    }
    gsh[25] = g.x_time[best];
    gsh[26] = g.x_fp[best];
  }
  x.sync();
  const int j = int(gsh[25] >> 32);
  const int32_t t = int32_t(gsh[25] & 0xffffffff);
  const int32_t target = int32_t(gsh[26]);
  const JobDev& J = g.jobs[j];
  JobState& st = g.st[j];
  // backup (recompute_planner.cpp:123)
  const JobState saved = st;
  backup_job(x, g, j, false, saved.S, saved.R, saved.n_curve);
  if (st.R + 1 > J.Rcap) {
    if (x.tid == 0) { g.err.code = E_CAPACITY; g.err.job = j; g.err.tensor = J.Rcap; g.err.tick = 2; }
    x.sync();
    return false;
  }
  const int32_t p = J.t_prod[t];
  const int64_t lat = J.o_lat[p];
  const int64_t pivot = J.a_start[target];
  x.sync();
  if (x.tid == 0) {
    const int32_t r = st.R;
    J.rc_id[r] = st.next_id; J.rc_tensor[r] = t; J.rc_target[r] = target; J.rc_regen[r] = p;
    J.rc_lat[r] = lat; J.rc_saving[r] = J.t_size[t];
    st.R = r + 1;
    st.next_id += 1;
    st.period += lat;
    g.ec_ok = 0; g.ec_S0 = -1;  // access times shift: the incremental base is stale
  }
  for (int32_t a = x.tid; a < J.A; a += x.nthr)
    if (J.a_start[a] >= pivot) { J.a_start[a] += lat; J.a_end[a] += lat; }
  x.sync();
  build_anchor_index(x, g, j);
  if (!revalidate(x, g, j)) return false;
  if (x.tid == 0) st.dirty = 1;
  x.sync();
  if (!eval_batch(x, g, j, j + 1)) return false;
  if (st.peak > saved.peak) {  // rollback (recompute_planner.cpp:148-151)
    backup_job(x, g, j, true, saved.S, saved.R, saved.n_curve);
    if (x.tid == 0) { st = saved; g.ec_ok = 0; g.ec_S0 = -1; gsh[27] = 0; }
    x.sync();
    for (int32_t t = x.tid; t < J.T; t += x.nthr)  // the restored report's peak list
      if (J.in_peak[t]) J.pk_list[x.aadd(&gsh[27], 1)] = t;
    x.sync();
    build_anchor_index(x, g, j);
    build_busy_index(x, g, j);
    return false;
  }
  return true;
}

// ----------------------------------------------------------------------------
// build_plan (orchestrator.cpp:8-70) for one group
// ----------------------------------------------------------------------------
// Clears the group's mutable header so a prepared plan can be relaunched
// over resident inputs (every other piece of state is rebuilt from them).
template <class X>
TSL_HD void reset_group(X& x, GroupDev& g) {
  if (x.tid == 0) {
    g.n_hist = 0;
    g.final_merged = 0;
    g.within_budget = 0;
    g.total_swapped = 0;
    g.loop_iters = 0;
    g.err = ErrInfo{};
    g.stats = GroupStats{};
    g.ec_ok = 0; g.ec_S0 = -1;
  }
  x.sync();
}

template <class X>
TSL_HD void plan_group(X& x, GroupDev& g) {
  reset_group(x, g);
  int64_t c0 = x.clock(), c1;
  const int64_t cstart = c0;
  auto lap = [&](int k) { c1 = x.clock(); if (x.tid == 0) g.stats.cyc[k] += c1 - c0; c0 = c1; };
  for (int j = 0; j < g.n_jobs; ++j) seq_batch(x, g, j);
  lap(0);
  if (!refresh(x, g, 0, g.n_jobs, true)) return;  // make_job_context's refresh
  lap(1);
  bool swap_ok = true, rc_ok = true;
  int iter = 0;
  while (swap_ok || rc_ok) {
    c0 = x.clock();
    if (!refresh(x, g, 0, g.n_jobs, false)) return;  // only jobs whose plan changed
    lap(1);
    int64_t merged = 0;
    for (int j = 0; j < g.n_jobs; ++j) merged += g.st[j].peak;
    if (x.tid == 0) {
      if (g.n_hist < g.hist_cap) g.hist[g.n_hist] = merged;
      g.n_hist += 1;
    }
    x.sync();
    const int nh = g.n_hist;
    // stall rule: mean per-job peak barely moved over the last 3 rounds
    if (iter > g.cfg.stall_min_iters && nh > 3 && nh <= g.hist_cap) {
      const double nj = double(g.n_jobs);
      const double before = double(g.hist[nh - 4]) / nj;
      const double now = double(g.hist[nh - 1]) / nj;
      if (before > 0 && (before - now) / before < g.cfg.stall_eps) break;
    }
    if (swap_ok) {
      c0 = x.clock();
      swap_ok = swap_pass(x, g);
      lap(2);
    } else if (merged >= g.cfg.budget) {
      c0 = x.clock();
      rc_ok = recompute_pass(x, g);
      lap(3);
    } else {
      rc_ok = false;
    }
    if (g.err.code) return;
    ++iter;
  }
  if (!refresh(x, g, 0, g.n_jobs, false)) return;
  if (x.tid == 0) {
    int64_t merged = 0;
    for (int j = 0; j < g.n_jobs; ++j) merged += g.st[j].peak;
    g.final_merged = merged;
    g.within_budget = merged <= g.cfg.budget;
    g.loop_iters = iter;
    g.stats.loop_iterations = iter;
    g.stats.cyc[4] = x.clock() - cstart;
  }
  x.sync();
}

// analyze_job on a caller-supplied plan: timeline builder + one evaluation.
template <class X>
TSL_HD void analyze_group(X& x, GroupDev& g) {
  reset_group(x, g);
  for (int j = 0; j < g.n_jobs; ++j) {
    // keep the caller's plan (events/flags were uploaded into the job arrays)
    const JobState keep = g.st[j];
    seq_batch(x, g, j);
    const JobDev& J = g.jobs[j];
    for (int32_t a = x.tid; a < J.A; a += x.nthr) J.a_flag[a] = J.a_inflag[a];
    if (x.tid == 0) {
      JobState& st = g.st[j];
      st.S = keep.S; st.R = keep.R; st.next_id = keep.next_id; st.dirty = 1;
    }
    x.sync();
  }
  refresh(x, g, 0, g.n_jobs, true);
}

}  // namespace tsl
