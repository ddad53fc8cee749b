// Plan executor: device-side state and launch helpers (tsl_exec.cu); the
// host driver is tsl_execute_plan in tsl_host.cpp.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsl {

// Allocator counters shared by every job of a multi-job replay.
struct ExecAcct {
  int64_t footprint;
  int64_t hwm;
};

struct ExecDevice {
  ExecAcct* acct;         // the replay's global counters (every job's allocations)
  uint64_t tick_ns;
  uint8_t* pool;          // device pool: one slot per storage
  const int64_t* slot_off;
  uint8_t** addr;         // mempool mode: each storage's current allocation (else null)
  int32_t* resident;      // [T] allocator residency flags
  int32_t* version;       // [T] data version (tag) of each storage
  int32_t* out_pending;   // [T] swap-outs of the storage not yet complete this iteration
  uint64_t* op_end_ns;    // [iterations * steps]
  uint64_t* iter_start_ns;// [iterations + 1]
  uint64_t xfer_start_ns; // channel: start of the transfer in flight
  int64_t footprint;      // allocator bytes (units) in use
  int64_t hwm;            // allocator high-water mark
  int32_t violations;     // releases of non-resident storages / reads of absent inputs
  int32_t verify_errors;  // inputs whose data tag did not match
  int32_t n_out, n_in;    // completed swap-outs / swap-ins
};

struct ExecOp {
  int32_t index;          // step index within the iteration (op_end_ns slot = base + index)
  int32_t pad;
  int64_t ticks;
  int64_t start;          // planned start tick within the iteration
  int32_t n_in, n_out, n_rel;
  const int32_t* ins;     // input storages
  const int32_t* outs;    // written storages
  const int64_t* out_size;// accounted size (0: in-place update, not allocated)
  const int32_t* rel;     // storages released at the op's end (if no swap-out pends)
  const int64_t* rel_size;
};

cudaError_t exec_launch_op(ExecDevice* d, const ExecOp* op, int base, int iter, cudaStream_t s);
cudaError_t exec_launch_delay(ExecDevice* d, int32_t anchor_op, int iter, int64_t delta, cudaStream_t s);
cudaError_t exec_launch_done(ExecDevice* d, int32_t st, int64_t size, int64_t dur, int dir, cudaStream_t s);
cudaError_t exec_launch_init(ExecDevice* d, const int32_t* st, const int64_t* sz, int n, cudaStream_t s);
cudaError_t exec_launch_host_tag(ExecDevice* d, int32_t st, uint8_t* host_slot, cudaStream_t s);
cudaError_t exec_launch_iter_begin(ExecDevice* d, const int32_t* outs_per_iter, int32_t T, int iter,
                                   cudaStream_t s);

}  // namespace tsl
