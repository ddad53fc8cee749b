// Device-visible plain-old-data layout of one planning group (one CTA).
//
// The host (tsl_host.cpp) packs every group into one staging buffer with
// absolute device addresses already resolved, uploads it with one H2D copy,
// and launches one CTA per group (tsl_plan_kernel, tsl_kernel.cu). Everything
// here is integer SoA: tensor / op / access ids are dense int32 indices, and
// every std::string ordering of the reference (tensor ids, job ids) is carried
// as a precomputed lexicographic rank.
#pragma once
#include <stdint.h>

namespace tsl {

struct PairRec;

// AccessType (access.hpp:11): TGA = generating access, TUA = using access.
enum : int8_t { ACC_TGA = 0, ACC_TUA = 1 };
// TimelineEventType (peak.hpp:33-39), same order == same type rank.
enum : int { EV_TGA = 0, EV_TUA = 1, EV_SIN = 2, EV_SOUT = 3, EV_REL = 4 };
// TensorKind (types.hpp:21).
enum : int8_t { K_INPUT = 0, K_INTERIM = 1, K_PARAM = 2, K_UPD = 3, K_OUTPUT = 4 };

// Device error codes; the host turns them into the reference's
// ValidationError texts.
enum : int32_t {
  E_OK = 0,
  E_DOUBLE_RELEASE = 1,   // peak.cpp:220-222 "double release of tensor X"
  E_SWAPIN_RESIDENT = 2,  // peak.cpp:226-227 "swap-in of resident tensor X"
  E_NEG_FOOTPRINT = 3,    // peak.cpp:232-234 "negative footprint at tick T"
  E_NO_TGA = 4,           // swap_planner.cpp:309-310 "tensor X has no TGA in sequence"
  E_UNKNOWN_ACCESS = 5,   // access.cpp:8-10 "unknown access id N in job J"
  E_CAPACITY = 6,         // a compiled capacity was exceeded
  E_INTERNAL = 7
};

struct ErrInfo {
  int32_t code;
  int32_t job;     // job index in the group
  int64_t tensor;  // tensor index / access id, per code
  int64_t tick;
};

// Everything the planner knows and mutates about one job.
struct JobDev {
  // ---- sizes and identity ----
  int32_t A, T, O;   // accesses, tensors, ops
  int32_t rank;      // job-id rank inside the group (std::string order)
  double ratio;      // SwapBudget max ratio (config.max_swap_ratio(job))
  int32_t Scap, Rcap, Ecap;  // swap-event / recompute-event / timeline capacities
  int32_t ti_nb;             // buckets of the time indexes (TI_NB; finer for jobs above one sort tile)

  // ---- static graph (host-packed) ----
  const int32_t* topo;       // [O] op indices in topological order (graph.cpp:245-282)
  const int64_t* o_lat;      // [O] latency ticks
  const int32_t* o_in_off;   // [O+1]
  const int32_t* o_in;       // tensor indices, op.inputs order
  const int32_t* o_out_off;  // [O+1]
  const int32_t* o_out;      // tensor indices, op.outputs order
  const int64_t* t_size;     // [T]
  const int8_t* t_kind;      // [T]
  const int32_t* t_rank;     // [T] lexicographic rank of the tensor id
  const int32_t* t_store;    // [T] storage root (graph.cpp:159-163)
  const int32_t* t_upd;      // [T] param -> its updated version, else -1
  const int32_t* t_prod;     // [T] producer op, else -1
  const uint8_t* a_inflag;   // [A] caller plan release flags (tsl_analyze_job only)

  // ---- derived on the device by the timeline builder ----
  int32_t* a_tensor;  // [A]
  int32_t* a_store;   // [A]
  int8_t* a_type;     // [A]
  int64_t* a_start;   // [A] (shifted by recomputation)
  int64_t* a_end;     // [A]
  uint8_t* a_base;    // [A] activity-analysis release flags (access.cpp:61-78)
  uint8_t* a_flag;    // [A] current plan release flags
  uint8_t* a_owned;   // [A] scratch: release owned by a swap-out (peak.cpp:107-130)
  int32_t* s_off;     // [T+1] CSR by storage
  int32_t* s_acc;     // [A]   access ids of each storage, ascending (== (start, id) order)
  int32_t* t_wfirst;  // [T] first TUA whose tensor id is exactly the param (swap_planner.cpp:426-431)
  int32_t* t_utga;    // [T] last TGA access of the param's updated version (:412-415)

  // ---- plan: swap events in plan order (plan.hpp:18-32) ----
  int64_t* ev_id;
  int32_t* ev_tensor;
  int8_t* ev_dir;  // 0 out, 1 in
  int8_t* ev_wraps;
  int64_t* ev_trig;
  int64_t* ev_delta;
  int64_t* ev_start;
  int64_t* ev_end;
  int64_t* ev_earl;
  int64_t* ev_late;
  int64_t* ev_pair;
  int64_t* ev_serves;
  // busy structure: the job's swap intervals sorted by start (disjoint at shift 0)
  int64_t* bz_s;
  int64_t* bz_e;
  int64_t* pd_s;   // [Scap] this pass's committed intervals
  int64_t* pd_e;
  int64_t* pd_ts;  // [Scap] merge scratch
  int64_t* pd_te;
  int32_t* bzi_s;     // [ti_nb+1] time index over bz_s
  int32_t* bzi_e;     // [ti_nb+1] time index over bz_e
  int32_t* ai_e;      // [ti_nb+1] time index over a_end (anchor)
  int32_t* st_evcnt;  // [T] swap events per storage (storage_has_swap)
  uint8_t* swapped;   // [T] SwapBudget::swapped_storages for this job
  // recompute events (plan.hpp:34-42)
  int64_t* rc_id;
  int32_t* rc_tensor;
  int64_t* rc_target;
  int32_t* rc_regen;
  int64_t* rc_lat;
  int64_t* rc_saving;

  // ---- report (PeakReport, peak.hpp:47-56) ----
  uint8_t* in_peak;   // [T] storage resident at the peak
  int32_t* pk_list;   // [T] the storages resident at the peak, unordered (JobState.n_peak entries)
  uint8_t* ev_drop;   // [Scap] scratch for revalidation
  uint8_t* res_init;  // [T] scratch: initial residency (peak.cpp:176-190)
  int64_t* curve_t;   // [Ecap+1]
  int64_t* curve_b;   // [Ecap+1]

  // ---- recompute rollback copies (recompute_planner.cpp:123, 148-151) ----
  int64_t* bk_a_start;
  int64_t* bk_a_end;
  uint8_t* bk_flag;
  uint8_t* bk_in_peak;
  int64_t* bk_ev;      // 12 * Scap int64 words (all swap-event fields)
  int64_t* bk_rc;      // 6 * Rcap words
  int64_t* bk_bz;      // 2 * Scap
  int32_t* bk_evcnt;   // [T]
  int64_t* bk_curve;   // 2 * (Ecap+1)
};

// Mutable per-job scalars (kept apart so a rollback is one struct copy).
struct JobState {
  int32_t S, R;        // swap / recompute event counts
  int32_t n_peak;      // |peak_tensors|
  int32_t n_curve;     // footprint curve points
  int64_t period;      // iteration_period (shifted by recomputation)
  int64_t next_id;     // SchedulingPlan::next_event_id (plan.cpp:15-20)
  int64_t peak, peak_time, lua;
  int32_t has_lua;
  int32_t dirty;       // plan changed since the last evaluation
  int64_t n_events;    // timeline events of the last evaluation
  int64_t son;         // SwapBudget::swapped_out_count[job] (swap_planner.cpp:278-282)
  int32_t bz_n;        // events reflected in the sorted busy structure
  int32_t pend_n;      // this pass's commits not yet merged into it
  int32_t pend_sorted; // pend_[0, pend_sorted) is sorted by start
  int32_t pend_upto;   // candidates before this index are in the pend list
  int32_t bzi_shift;   // bucket shift of the busy-structure time index
  int32_t ai_shift;    // bucket shift of the access-end (anchor) time index
  int32_t S_pass;      // S at the start of the current swap pass
  int32_t pad_st;
};

struct GroupConfig {
  int64_t bw, setup, budget;
  double stall_eps;
  int32_t stall_min_iters;
};

// Device-side counters for the roofline (SURVEY §8(d) byte formula).
struct GroupStats {
  int64_t evaluations;       // analyze_job evaluations
  int64_t timeline_events;   // sum of timeline events over evaluations
  int64_t candidates;        // swap candidates visited
  int64_t candidate_accesses;// storage accesses read by the scorer
  int64_t busy_intervals;    // busy intervals swept by feasible-region queries
  int64_t fit_queries;
  int64_t loop_iterations;
  int64_t sort_elems;        // elements through block sorts
  int64_t rescored;          // swap candidates re-scored after speculation
  int64_t cyc[32];           // SM cycles per stage (thread 0): seq, eval, swap, rc, total, spec, conflict, sweep, merge
  int64_t prof[16];          // development profile of re-score queries (TSL_PROF builds)
  int64_t comp_rescored;     // candidates re-speculated inside their conflict component
  int64_t sprof[24];         // SM cycles (thread 0): [0..6] incremental timeline order, [11..14] swap-pass prologue
};

// Control block of a cooperative launch (one group above one sort tile,
// one CTA per SM): CTA 0 plans; the other CTAs wait for block-wide radix-sort
// passes it publishes (epoch), run their share, and meet at grid barriers.
struct CoopCtl {
  int32_t epoch;      // task generation (CTA 0 bumps it per task)
  int32_t type;       // COOP_PASS / COOP_EXIT
  int32_t bar_count;  // grid barrier arrivals
  int32_t bar_gen;    // grid barrier generation
  int32_t exited;     // workers that saw COOP_EXIT
  int32_t grid;       // CTAs of the launch
  const uint64_t* ks; // pass input / output
  const int32_t* vs;
  uint64_t* kd;
  int32_t* vd;
  int32_t n, sh, nb, pad;
  int32_t* tile_hist; // [tiles * 256] digit counts per tile
  int32_t jb, je;     // COOP_EVAL: the job batch
  int64_t* gsh;       // [SH_WORDS] grid-shared scalars of a cooperative evaluation
  int64_t* cta_part;  // [1024] per-CTA partials of grid scans
  // COOP_FOLD (workers only, while one warp of CTA 0 waits): merge the sorted
  // lists a (busy) and b (pend) into m, copy m back over a, rebuild a's index
  const int64_t *fa_s, *fa_e, *fb_s, *fb_e;
  int64_t *fm_s, *fm_e, *fo_s, *fo_e;
  int32_t* fi_s;
  int32_t* fi_e;
  int32_t fn1, fn2, fshift, fdone, fnb, fpad;
  int32_t wbar_count, wbar_gen;  // barrier of the worker CTAs
  // COOP_COMP: component runs of a speculation window, taken by every warp
  int64_t cw0, cnruns, crun;     // window start, runs, next run (atomic)
  const int32_t* ccand;
  int32_t* ccinfo;
  int64_t* cchull;
  int32_t cdone, cpad;           // worker CTAs done
  // COOP_CONF / COOP_SPEC: phase B / phase A of the window [cw0, cw1) on the grid
  int64_t cw1;
  const int32_t* ccomp;
  int32_t ccoupled;
  int32_t abort;                 // a spin timed out: every CTA leaves (the group reports E_INTERNAL)
};
enum : int32_t { COOP_PASS = 1, COOP_EVAL = 2, COOP_FOLD = 3, COOP_REBUILD = 4, COOP_COMP = 5, COOP_CONF = 6, COOP_SPEC = 7,
                 COOP_A2 = 8, COOP_SEQ = 10,
                 COOP_EXIT = 9 };

struct GroupDev {
  int32_t n_jobs;
  int32_t coupled;      // some job has ratio < 1: swap passes run globally in order
  int32_t hist_cap;
  int32_t n_hist;
  GroupConfig cfg;
  JobDev* jobs;         // [n_jobs]
  JobState* st;         // [n_jobs]
  int64_t* hist;        // merged_peak_history
  int64_t final_merged;
  int32_t within_budget;
  int32_t spec_window;  // candidates per speculation window of a swap pass (0: the whole pass)
  int64_t total_swapped;  // SwapBudget::total_swapped
  int32_t loop_iters;
  int32_t pad2;
  ErrInfo err;
  GroupStats stats;
  // timeline / sort scratch, capacity ecap (global memory)
  int32_t ecap;
  int32_t pad1;
  uint64_t* k_key;   // [ecap]
  int32_t* k_val;    // [ecap]
  int64_t* x_time;   // [ecap] event time
  int64_t* x_fp;     // [ecap] footprint after the event (sorted order)
  int32_t* x_store;  // [ecap]
  int32_t* x_aid;    // [ecap]
  int8_t* x_type;    // [ecap] type | 8 if the TGA delta is 0 (aliased) | 16 if a flagged TUA
  int8_t* x_job;     // [ecap]
  uint8_t* x_state;  // [ecap] residency after the event (per-position)
  int32_t* x_seq2;   // [ecap] positions grouped by (job, storage)
  uint64_t* x_key2;  // [ecap]
  int32_t* x_order;  // [ecap] sorted position -> slot
  // speculative swap pass scratch (tsl_plan.cuh swap_pass)
  CoopCtl* coop;     // cooperative launch control (one group above one tile), else null
  uint64_t* bs_key;  // [ecap] ping-pong of the block-wide radix sort (jobs above one sort tile), else null
  int32_t* bs_val;   // [ecap]
  int32_t* c_info;   // [candidates * 16]
  int64_t* c_hull;   // [candidates * 4]
  int64_t* dev_list; // [candidates]
  PairRec* pr_pool;  // [pr_cap]
  int64_t* w_pool;   // [2 * w_cap]
  int64_t pr_cap, w_cap;
  int64_t* wbuf;     // [NT/32 warps * 4 * wcap] re-scoring gather scratch
  int64_t wcap;
  int32_t cb_nb;     // time buckets of the conflict / window indexes (1024; more for big passes)
  int32_t* cb_idx;   // [2 * CB_NB + 4] conflict-index bucket offsets / cursors
  int32_t* cb_ent;   // [cb_cap] conflict-index entries
  int64_t cb_cap;
  int32_t* c_comp;   // [2 * c_cap] component speculation: union-find roots, previous members
  int64_t c_cap;
  int32_t spec_comp; // component speculation on (uncoupled swap passes)
  int32_t grid_conf; // cooperative launches run phase B on the whole grid
  int64_t c_wn;      // candidates of the window being processed
  int64_t* c_wscratch;  // cooperative launches: per-warp run lists (6 * c_wscap words per warp of the grid)
  int64_t c_wscap;
  // Incremental timeline order (tsl_plan.cuh inc_order; one-job big builds,
  // null otherwise). The "base" is every access event plus one potential
  // release per access (2A entries), sorted once per access-time
  // configuration; swap passes only append events, so the swap events'
  // timeline and storage-grouped orders are kept across evaluations and
  // only each pass's new events are sorted and merged in.
  int32_t ec_ok;       // base valid (access times unchanged since it was built)
  int32_t ec_S0;       // swap events [0, ec_S0) are in the cached D orders (-1: none)
  int32_t ec_cur;      // current half of the D ping-pong buffers
  int32_t ec_pad;
  int64_t ec_dcap;     // D capacity (Scap + Rcap)
  int64_t* ec_bt;      // [2A] base in timeline order: time
  uint32_t* ec_bl;     // [2A] key low word: non-free << 30 | storage rank << 2 | type rank
  int32_t* ec_bs;      // [2A] base slot: a (access a), A + a (release of a)
  int64_t* ec_gt;      // [2A] base in (storage rank, timeline) order: time
  uint32_t* ec_gl;     // [2A] key low word
  int32_t* ec_gb;      // [2A] base slot
  int32_t* ec_ginv;    // [2A] base position -> grouped position
  int32_t* ec_posb;    // [2A] merged timeline position of each grouped base entry
  int64_t* ec_sc;      // [2 x (2A + 1)] active base entries + D insertions, per order (scan scratch)
  int32_t* ec_dord;    // [2 * dcap] D slots in timeline order (ping-pong)
  int32_t* ec_dins;    // [2 * dcap] their base insertion points
  int32_t* ec_dgrp;    // [2 * dcap] D slots in storage-grouped order (ping-pong)
  int32_t* ec_gins;    // [2 * dcap] their grouped-base insertion points
  int32_t* ec_nw;      // [4 * dcap] an evaluation's new D entries, ordered, with insertion points
  int32_t* ec_posd;    // [dcap] merged timeline position of each D slot
  uint32_t* ec_dl;     // [dcap] key low word of each D slot
  int8_t* ec_gbt;      // [2A] grouped base entry: event type (| 8: an aliased TGA)
  int32_t* ec_gbst;    // [2A] grouped base entry: storage
  uint8_t* ec_act;     // [2 x 2A] activity of each base entry, timeline then grouped order
  uint8_t* ec_ract;    // [A] activity of access a's release as last recorded
  int32_t* ec_rpos;    // [2 x A] positions of access a's release entry in the two orders
  int8_t* ec_gty;      // [ecap] an evaluation's events in grouped order: type
  int32_t* ec_gst;     // [ecap] storage
};

}  // namespace tsl
