/*
 * tensile_b200.h -- C-ABI of the B200-native TENSILE scheduling-plan generator.
 *
 * This is the drop-in boundary for the reference's hot path
 *   memsched::build_plan            (/root/reference/proj/include/memsched/orchestrator.hpp:26-28,
 *                                    src/orchestrator.cpp:8-70)
 *   memsched::analyze_job           (peak.hpp:77-78, src/peak.cpp:246-250)
 *   memsched::save_plans            (plan.hpp:57, src/plan.cpp:30-65)
 *   memsched::PeakReport::to_json   (peak.hpp:55, src/peak.cpp:258-272)
 * Everything is plain C: pointers, sizes, int status codes. Inputs are
 * caller-owned and copied at call time; results are library-owned and freed by
 * tsl_result_destroy. Errors return a nonzero status and leave a message in
 * tsl_last_error() (thread-local), mirroring the reference's ValidationError
 * texts where the reference throws.
 *
 * A graph is passed exactly as the reference's ComputeGraph holds it
 * (graph.hpp:14-54): tensors (id, size, kind) and operators (id, kind, inputs,
 * outputs, phase) with the per-op latency table (the reference's
 * std::map<OpId, Tick>, orchestrator.hpp:26-28) flattened to one entry per op.
 */
#ifndef TENSILE_B200_H
#define TENSILE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define TSL_OK 0
#define TSL_ERR_VALIDATION 1 /* reference would throw memsched::ValidationError */
#define TSL_ERR_CUDA 2       /* CUDA runtime / launch failure                    */
#define TSL_ERR_INTERNAL 3   /* invariant broken inside the library              */
#define TSL_ERR_ARGUMENT 4   /* NULL pointer / bad size at the C boundary        */
#define TSL_ERR_CAPACITY 5   /* input exceeds a compiled device capacity         */

/* TensorKind (types.hpp:21) and OpPhase (types.hpp:22), same order. */
enum tsl_tensor_kind {
  TSL_KIND_INPUT = 0,
  TSL_KIND_INTERIM = 1,
  TSL_KIND_PARAMETER = 2,
  TSL_KIND_UPDATED_PARAMETER = 3,
  TSL_KIND_OUTPUT = 4
};
enum tsl_op_phase { TSL_PHASE_FORWARD_BACKWARD = 0, TSL_PHASE_OPTIMIZE = 1 };

/* An op with no latency entry (generate_access_sequence throws
 * "missing latency entry for op X", access.cpp:35-36). */
#define TSL_LATENCY_MISSING INT64_MIN

/* PlannerConfig (config.hpp:9-18). The max_swap_ratios map is the arrays
 * max_swap_ratio_jobs/max_swap_ratio_values (n_max_swap_ratios entries, unique
 * job ids, any order; they need to live only for the call that takes the
 * config). Like PlannerConfig::validate, every entry is checked, including
 * entries naming no job of the build; a job without an entry gets 1.0. */
typedef struct tsl_config {
  int64_t pcie_bandwidth;      /* bytes per tick, > 0          */
  int64_t transfer_setup;      /* ticks, >= 0                  */
  int64_t memory_budget;       /* bytes, >= 0                  */
  double ewma_alpha;           /* [0,1], default 0.3           */
  double replan_threshold;     /* > 0, default 0.2             */
  double stall_epsilon;        /* (0,1), default 0.0005        */
  int32_t stall_min_iters;     /* default 100                  */
  double cold_start_gpu_usage; /* default 0.5                  */
  int32_t n_max_swap_ratios;                /* entries of the map, default 0 */
  const char* const* max_swap_ratio_jobs;   /* [n_max_swap_ratios] job ids   */
  const double* max_swap_ratio_values;      /* [n_max_swap_ratios], (0,1]    */
} tsl_config;

/* Fills the reference defaults (config.hpp:10-18). */
void tsl_config_default(tsl_config* cfg);

/* One job: ComputeGraph + latency table. */
typedef struct tsl_job_desc {
  const char* job_id;
  int32_t n_tensors;
  const char* const* tensor_ids; /* [n_tensors]                      */
  const int64_t* tensor_sizes;   /* [n_tensors], > 0                 */
  const int8_t* tensor_kinds;    /* [n_tensors], tsl_tensor_kind     */
  int32_t n_ops;
  const char* const* op_ids;     /* [n_ops]                          */
  const char* const* op_kinds;   /* [n_ops]; "update" marks updates  */
  const int8_t* op_phases;       /* [n_ops], tsl_op_phase            */
  const int32_t* op_in_offsets;  /* [n_ops+1] CSR into op_inputs     */
  const int32_t* op_inputs;      /* tensor indices, op.inputs order  */
  const int32_t* op_out_offsets; /* [n_ops+1] CSR into op_outputs    */
  const int32_t* op_outputs;     /* tensor indices, op.outputs order */
  const int64_t* op_latencies;   /* [n_ops] ticks or TSL_LATENCY_MISSING */
} tsl_job_desc;

/* Read-only view of one job's plan + peak report inside a result. All arrays
 * are owned by the result. Swap events are in plan order (the reference's
 * SchedulingPlan::swap_events vector, plan.hpp:46-53). */
typedef struct tsl_job_view {
  const char* job_id;
  int64_t version;
  /* SwapEvent (plan.hpp:18-32); tensor = index of the storage tensor */
  int32_t n_swap;
  const int64_t* ev_id;
  const int32_t* ev_tensor;
  const int8_t* ev_dir; /* 0 = out, 1 = in */
  const int64_t* ev_trigger;
  const int64_t* ev_delta;
  const int64_t* ev_start;
  const int64_t* ev_end;
  const int64_t* ev_earliest;
  const int64_t* ev_latest;
  const int8_t* ev_wraps;
  const int64_t* ev_pair;
  const int64_t* ev_serves;
  /* RecomputeEvent (plan.hpp:34-42) */
  int32_t n_recompute;
  const int64_t* rc_id;
  const int32_t* rc_tensor;
  const int64_t* rc_target;
  const int32_t* rc_regen_op;
  const int64_t* rc_latency;
  const int64_t* rc_saving;
  /* release_flags (std::set<AccessId>, ascending) */
  int32_t n_release;
  const int64_t* release_flags;
  /* PeakReport (peak.hpp:47-56) */
  int64_t memory_peak;
  int64_t peak_time;
  int8_t has_last_input_access;
  int64_t last_input_access;
  int32_t n_peak_tensors;
  const int32_t* peak_tensors; /* tensor indices, std::set<string> order */
  int32_t n_curve;
  const int64_t* curve_time;
  const int64_t* curve_bytes;
  /* working access sequence after planning (recomputation shifts it) */
  int64_t iteration_period;
  int32_t n_accesses;
} tsl_job_view;

/* Device-side counters of one build, for the roofline. */
typedef struct tsl_stats {
  double kernel_ms;          /* device time of the planning kernel(s)       */
  double total_ms;           /* host wall time of tsl_build_plan            */
  int64_t n_accesses;        /* sum of |AccessSequence| over jobs           */
  int64_t loop_iterations;   /* orchestrator loop iterations                */
  int64_t evaluations;       /* analyze_job evaluations performed           */
  int64_t timeline_events;   /* sum of timeline events over evaluations     */
  int64_t candidates;        /* swap candidates visited                     */
  int64_t candidate_accesses;/* sum of storage accesses read by the scorer  */
  int64_t busy_intervals;    /* channel intervals scanned by gap searches   */
  int64_t algorithmic_bytes; /* SURVEY §8(d) byte formula over the build    */
  int64_t kernel_launches;   /* device kernels launched by this call        */
  /* SM clock cycles spent per stage inside the planning CTA (thread 0):
   * timeline builder, evaluator, swap passes, recompute passes, whole CTA */
  int64_t cyc_sequence, cyc_evaluate, cyc_swap, cyc_recompute, cyc_total;
  int64_t rescored;          /* speculative swap candidates re-scored in order */
  /* inside the swap passes: speculation, conflicts, in-order sweep, merge */
  int64_t cyc_spec, cyc_conflict, cyc_sweep, cyc_merge;
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by this call     */
  double prep_ms;               /* host validation + packing before the H2D  */
  int64_t cyc_rescore;          /* part of cyc_sweep spent re-scoring (job 0's warp) */
  int64_t cyc_apply;            /* part of cyc_merge spent writing committed events */
  int64_t debug[4];             /* development counters */
  int64_t cyc_pendsort;
  int64_t fitprof[9];
  int64_t evalprof[7];  /* evaluator phases: prep, emit, sort1, group, automaton, scan.., peak..report */
  int64_t queryprof[16];  /* development profile of re-score queries (zero unless built with TSL_PROF) */
  int64_t comp_rescored;  /* candidates re-speculated inside their conflict component (phase A2) */
  int64_t stageprof[24];  /* SM cycles: [0..6] incremental timeline order phases, [7..10] its new-entry ordering,
                             [11..14] swap-pass prologue (peak sizes, candidates, sort, rest), [15] phase A,
                             [16..20] component runs: sum of per-pass longest run, members, runs,
                             sum of per-pass slowest run cycles, run cycles, [23] union-find rounds */
} tsl_stats;

typedef struct tsl_ctx tsl_ctx;
typedef struct tsl_result tsl_result;
typedef struct tsl_plan tsl_plan;

const char* tsl_last_error(void);

/* Device context: CUDA device, streams, device workspace (grown on demand). */
int tsl_create(int device, tsl_ctx** out);
int tsl_destroy(tsl_ctx* ctx);

/* memsched::build_plan(jobs, config) -- orchestrator.cpp:8-70. */
int tsl_build_plan(tsl_ctx* ctx, const tsl_job_desc* jobs, int32_t n_jobs,
                   const tsl_config* cfg, tsl_result** out);

/* Several independent build_plan calls ("job groups", e.g. the 8 workload
 * shards of one GPU, or every arrival/departure replan of a scenario) planned
 * by ONE device launch, one CTA per group. group_offsets[n_groups+1]
 * partitions jobs[]. cfgs holds n_cfgs configs: 1 (shared by every group) or
 * n_groups (one per group, e.g. a per-set memory budget). out[g] receives
 * each group's result. */
int tsl_build_plan_groups(tsl_ctx* ctx, const tsl_job_desc* jobs,
                          const int32_t* group_offsets, int32_t n_groups,
                          const tsl_config* cfgs, int32_t n_cfgs, tsl_result** out);

/* The same call split in three so inputs can stay resident in HBM between
 * device-only runs (bench.py's device-timed `value`):
 *   tsl_plan_prepare  validate + pack + one H2D copy      (no kernel)
 *   tsl_plan_run      `repeats` kernel launches on the context stream, timed
 *                     with CUDA events; *kernel_ms = mean per launch
 *   tsl_plan_collect  one D2H copy + results; out[n_groups]
 * tsl_build_plan_groups == prepare + run(1) + collect. */
int tsl_plan_prepare(tsl_ctx* ctx, const tsl_job_desc* jobs, const int32_t* group_offsets,
                     int32_t n_groups, const tsl_config* cfgs, int32_t n_cfgs, tsl_plan** out);
int tsl_plan_run(tsl_plan* plan, int32_t repeats, double* kernel_ms);
/* Enqueue one launch on `stream` (a cudaStream_t, NULL = the context stream)
 * without synchronising -- for callers that time with their own events. */
int tsl_plan_launch_async(tsl_plan* plan, void* stream);
int tsl_plan_collect(tsl_plan* plan, tsl_result** out);
void tsl_plan_destroy(tsl_plan* plan);

/* A caller-supplied plan for one job (SchedulingPlan, plan.hpp:46-53), used by
 * tsl_analyze_job. ev_tensor / rc_tensor / rc_regen_op index the job's
 * tensor / op tables. */
typedef struct tsl_plan_desc {
  int32_t n_swap;
  const int64_t* ev_id;
  const int32_t* ev_tensor;
  const int8_t* ev_dir;
  const int64_t* ev_trigger;
  const int64_t* ev_delta;
  const int64_t* ev_start;
  const int64_t* ev_end;
  const int8_t* ev_wraps;
  const int64_t* ev_pair;
  const int64_t* ev_serves;
  int32_t n_recompute;
  const int64_t* rc_id;
  const int32_t* rc_tensor;
  const int64_t* rc_target;
  const int32_t* rc_regen_op;
  const int64_t* rc_latency;
  const int64_t* rc_saving;
  int32_t n_release;
  const int64_t* release_flags;
  int64_t version;
} tsl_plan_desc;

/* memsched::analyze_job(seq, plan, catalog) -- peak.cpp:246-250 -- where seq
 * is the job's activity-analysed access sequence (make_job_context,
 * swap_planner.cpp:156-169). The result holds one job: the given plan and its
 * PeakReport. */
int tsl_analyze_job(tsl_ctx* ctx, const tsl_job_desc* job, const tsl_plan_desc* plan,
                    tsl_result** out);

/* ---- plan executor (north-star item 5; reference analogue: the scheduled
 * mode of memsched::simulate, simulator.cpp:112-569) --------------------------
 * Replays job `job` of a build_plan result on the device: ops are timed spin
 * kernels on a compute stream (1 tick = tick_ns of device time), swaps are
 * real pinned-host cudaMemcpyAsync on ONE copy stream (the reference's single
 * FIFO channel) fired at trigger end + delta, and a device-side allocator
 * counts footprint and high-water mark. A swapped-out device slot is
 * poisoned, so reads after a late or missing swap-in are caught. */
typedef struct tsl_exec_config {
  int64_t tick_ns;        /* device ns per planner tick (default 1000)      */
  int32_t iterations;     /* iterations replayed, 1..8 (default 3)           */
  int64_t bytes_per_unit; /* device/host bytes per planner byte (default 16) */
  int32_t vanilla;        /* 1: replay without the scheduler -- release at last
                             use (activity analysis), no swaps, no recomputation
                             (the reference's vanilla mode, the MSR/EOR/CBR base) */
  int32_t mempool;        /* 1: every storage lives in memory of a private CUDA
                             memory pool, allocated (cudaMallocAsync) when it
                             becomes resident and freed (cudaFreeAsync) when it is
                             released or swapped out, issued in the replay's planned
                             order; the report carries the pool's high-water marks.
                             Single-job replays (tsl_execute_plan) only. */
} tsl_exec_config;

typedef struct tsl_exec_report {
  int64_t predicted_peak;      /* PeakReport::memory_peak of the plan         */
  int64_t hwm;                 /* executor allocator high-water mark (units)  */
  int64_t final_footprint;     /* allocator footprint after the last iteration */
  int32_t iterations;
  double iteration_ms[8];      /* device-timed length of each iteration       */
  double planned_iteration_ms; /* iteration_period x tick_ns                  */
  int32_t swap_outs, swap_ins; /* completed transfers                         */
  int64_t bytes_d2h, bytes_h2d;
  int32_t verify_errors;       /* inputs whose data did not survive a swap    */
  int32_t violations;          /* reads of absent inputs / bad releases       */
  int32_t kernels;             /* kernels launched by the replay              */
  double total_ms;             /* host wall time of the call                  */
  int64_t pool_used_hwm;       /* mempool: cudaMemPoolAttrUsedMemHigh (bytes)  */
  int64_t pool_reserved_hwm;   /* mempool: cudaMemPoolAttrReservedMemHigh      */
  int64_t pool_allocs;         /* mempool: cudaMallocAsync calls               */
} tsl_exec_report;

void tsl_exec_config_default(tsl_exec_config* cfg);
/* cfg: the planner config the plan was built with (transfer durations). */
int tsl_execute_plan(tsl_ctx* ctx, const tsl_result* r, int32_t job, const tsl_config* cfg,
                     const tsl_exec_config* ex, tsl_exec_report* out);

/* Replays EVERY job of a build result together, as the reference's scheduled
 * simulation co-schedules them (simulator.cpp:112-569, SimConfig over several
 * SimJobs): one compute stream per job, all jobs' swaps on ONE copy stream
 * (the FIFO channel) in planned-arrival order, one device allocator counter
 * over all jobs. per_job[k] (k in tsl_result_n_jobs order) gets each job's own
 * counters; *merged gets the global high-water mark against the merged
 * predicted peak (sum of the jobs' peaks), summed swaps/bytes/errors and the
 * slowest job's iteration times. Replaces simulate()'s scheduled mode for a
 * multi-job SimConfig (simulator.hpp:84-87). */
int tsl_execute_plans(tsl_ctx* ctx, const tsl_result* r, const tsl_config* cfg, const tsl_exec_config* ex,
                      tsl_exec_report* per_job, tsl_exec_report* merged);

/* Result accessors. Jobs are ordered by job id (std::map<JobId,...>). */
int32_t tsl_result_n_jobs(const tsl_result* r);
int tsl_result_job(const tsl_result* r, int32_t i, tsl_job_view* out);
int32_t tsl_result_history(const tsl_result* r, const int64_t** merged_peak_history);
int64_t tsl_result_final_merged_peak(const tsl_result* r);
int32_t tsl_result_within_budget(const tsl_result* r);
const char* tsl_result_diagnostic(const tsl_result* r);
int tsl_result_stats(const tsl_result* r, tsl_stats* out);
/* save_plans(result.plans) byte-for-byte (plan.cpp:30-65). Caller frees with tsl_free. */
char* tsl_result_save_plans(const tsl_result* r);
/* PeakReport::to_json of job i (peak.cpp:258-272). Caller frees with tsl_free. */
char* tsl_result_report_json(const tsl_result* r, int32_t i);
void tsl_result_destroy(tsl_result* r);
void tsl_free(void* p);

/* PlannerConfig::validate (config.hpp:25-35) alone. */
int tsl_validate_config(const tsl_config* cfg);
/* SchedulingPlan::version of one job in a result (Orchestrator::rebuild
 * numbers its plans, orchestrator.cpp:104-108). */
int tsl_result_set_version(tsl_result* result, const char* job_id, int64_t version);

/* ---- Planning session: memsched::Orchestrator (orchestrator.hpp:30-60;
 * orchestrator.cpp:89-159) -- the replan lifecycle around the device planner.
 * Jobs arrive (add_job, op_latencies = current estimates or NULL) and depart
 * (remove_job); rebuild = one build_plan over the active set with per-job
 * plan versions; replan_if_needed = EWMA correction + drift-triggered rebuild
 * (result NULL when no replan). Every rebuild's wall time is recorded. ---- */
typedef struct tsl_session tsl_session;
int tsl_session_create(tsl_ctx* ctx, const tsl_config* cfg, tsl_session** out);
void tsl_session_destroy(tsl_session* session);
int tsl_session_add_job(tsl_session* session, const tsl_job_desc* job);
int tsl_session_remove_job(tsl_session* session, const char* job_id);
int tsl_session_set_latencies(tsl_session* session, const char* job_id, const int64_t* op_latencies);
int tsl_session_rebuild(tsl_session* session, tsl_result** out);
int tsl_session_replan_if_needed(tsl_session* session, int32_t n, const char* const* job_ids,
                                 const int64_t* const* observed_op_ticks, tsl_result** out);
int32_t tsl_session_replan_count(const tsl_session* session);
int32_t tsl_session_rebuild_times(const tsl_session* session, const double** ms);
int32_t tsl_session_n_jobs(const tsl_session* session);
int tsl_session_latencies(const tsl_session* session, const char* job_id, int64_t* out_op_latencies);

/* ---- Cold-start latency predictor: LatencyPredictor (latency.hpp:45-66,
 * latency.cpp:11-149) and predict_latencies (orchestrator.cpp:72-87). ---- */
typedef struct tsl_predictor tsl_predictor;
/* LatencyPredictor::fit: sample k = (op_kinds[k], values[value_offsets[k] ..
 * value_offsets[k+1]) = input dims, attributes, gpu usage, labels[k]). */
int tsl_latency_fit(int32_t n_samples, const char* const* op_kinds, const int32_t* value_offsets,
                    const double* values, const double* labels, tsl_predictor** out);
int tsl_latency_from_json(const char* document, tsl_predictor** out);
char* tsl_latency_to_json(const tsl_predictor* predictor);  /* free with tsl_free */
int tsl_latency_predict(const tsl_predictor* predictor, const char* op_kind, const double* values,
                        int32_t n_values, double* out);
int tsl_latency_r2(const tsl_predictor* predictor, const char* op_kind, double* out);
/* every op's predicted latency (ticks, op order); op attributes as CSR (NULL: none) */
int tsl_predict_latencies(const tsl_predictor* predictor, const tsl_job_desc* job, const int32_t* op_attr_offsets,
                          const double* op_attrs, double gpu_usage, int64_t* out_op_latencies);
void tsl_latency_destroy(tsl_predictor* predictor);

/* ---- Tick-level executor model (the reference's simulate, simulator.hpp:84-87;
 * simulator.cpp:26-582): vanilla / scheduled / passive modes, one FIFO
 * transfer channel, LRU eviction under the budget in passive mode. ---- */
typedef struct tsl_sim tsl_sim;
enum { TSL_SIM_VANILLA = 0, TSL_SIM_SCHEDULED = 1, TSL_SIM_PASSIVE = 2 };
typedef struct tsl_sim_config {      /* SimConfig (simulator.hpp:16-27) */
  int32_t mode;                      /* TSL_SIM_*                        */
  int32_t iterations;                /* >= 1                             */
  int64_t ticks_per_iteration_limit; /* default 10,000,000               */
  int64_t memory_budget;             /* enforced in passive mode only    */
  int64_t pcie_bandwidth;
  int64_t transfer_setup;
  int32_t n_slowdown;                /* gpu_slowdown_curve entries       */
  const int32_t* slowdown_jobs;      /* concurrent jobs ...              */
  const double* slowdown_mult;       /* ... -> multiplier (>= 1)         */
} tsl_sim_config;
/* SimController::on_iteration_end (simulator.hpp:73-79): called at each job's
 * iteration boundary with the ticks of the ops it ran (op order, -1 = not
 * run); new plans are installed with tsl_sim_set_plan from inside the
 * callback and take effect at each affected job's next boundary. Nonzero
 * return aborts the run with that status. */
typedef int (*tsl_sim_controller_fn)(void* user, tsl_sim* sim, int32_t job, int32_t iteration,
                                     const int64_t* observed_op_ticks);
/* memsched::simulate(jobs, plans, config, controller): jobs carry their TRUE
 * latencies in op_latencies; plans[k] may have no events (vanilla/passive
 * runs read only release_flags). */
int tsl_simulate(const tsl_job_desc* jobs, const int64_t* launch_ticks, int32_t n_jobs,
                 const tsl_plan_desc* plans, const tsl_sim_config* cfg,
                 tsl_sim_controller_fn controller, void* user, tsl_sim** out);
int tsl_sim_set_plan(tsl_sim* sim, int32_t job, const tsl_plan_desc* plan);
int64_t tsl_sim_peak(const tsl_sim* sim);
/* SimulationTrace as JSON (peak, blocked_ticks, passive_swap_count, per job:
 * peak, iteration_times, plan_versions, footprint_curve; transfers,
 * safety_violations, passive_events) / SimulationTrace::to_csv. Free with tsl_free. */
char* tsl_sim_trace_json(const tsl_sim* sim);
char* tsl_sim_trace_csv(const tsl_sim* sim);
void tsl_sim_destroy(tsl_sim* sim);
/* activity_analysis (access.cpp:61-78): the release-at-last-use flags (the
 * last access of every Interim tensor id), ascending; the vanilla / passive
 * modes' plans (scenario.cpp:180-194). out may be null to query *n_out. */
int tsl_base_release_flags(const tsl_job_desc* job, int64_t* out_flags, int32_t cap, int32_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* TENSILE_B200_H */
