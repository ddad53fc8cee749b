// Plan executor: replays a scheduling plan on the device with real
// pinned-host cudaMemcpyAsync swaps, to check the planner's predicted memory
// peak against the executor allocator's high-water mark.
//
// Reference analogue: the scheduled mode of the discrete-event simulator
// (/root/reference/proj/src/simulator.cpp:112-569): one compute stream per job
// (ops back to back, outputs allocated at op start, releases at op end unless
// a pending swap-out owns them), ONE FIFO transfer channel (here: one copy
// stream), swaps fired at trigger end + delta (iteration start + delta for
// anchor -1), swap-outs free at completion, swap-ins allocate at completion
// (simulator.cpp:325-342, 438-470, 486-497), an op waits for the swap-ins that
// serve it. Here time is real: a tick is `tick_ns` of device time (%globaltimer),
// ops are spin kernels, transfers move real bytes between a device pool slot
// and a pinned host slot and then hold the channel for the planned duration.
// Allocation, release and swap accounting run on the device (atomics on one
// footprint counter), so the high-water mark reflects the real interleaving.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsl_exec.h"

namespace tsl {

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void count_add(int64_t* fp, int64_t* hwm, int64_t size) {
  const unsigned long long f = atomicAdd(reinterpret_cast<unsigned long long*>(fp), (unsigned long long)size) + size;
  atomicMax(reinterpret_cast<long long*>(hwm), (long long)f);
}

// Allocation / release on the job's counters and the replay's global ones.
__device__ __forceinline__ void acct_add(ExecDevice* d, int32_t s, int64_t size) {
  if (atomicExch(&d->resident[s], 1) == 0) {
    count_add(&d->footprint, &d->hwm, size);
    if (d->acct) count_add(&d->acct->footprint, &d->acct->hwm, size);
  }
}

__device__ __forceinline__ void acct_sub(ExecDevice* d, int32_t s, int64_t size) {
  if (atomicExch(&d->resident[s], 0) == 1) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&d->footprint), (unsigned long long)(-size));
    if (d->acct) atomicAdd(reinterpret_cast<unsigned long long*>(&d->acct->footprint), (unsigned long long)(-size));
  } else {
    atomicAdd(&d->violations, 1);  // release of a non-resident storage
  }
}

// Where a storage's data lives: its fixed slot, or (mempool mode) the
// allocation the host made for its current residency.
__device__ __forceinline__ uint8_t* slot_of(ExecDevice* d, int32_t s) {
  return d->addr ? d->addr[s] : d->pool + d->slot_off[s];
}

__device__ __forceinline__ uint64_t tag_of(int32_t s, int32_t version) {
  return 0x5453'4c00'0000'0000ull ^ (uint64_t(uint32_t(s)) << 20) ^ uint64_t(uint32_t(version));
}

// One op (or recompute regeneration): allocate outputs, verify inputs, run
// for `ticks` of device time, tag outputs, release, timestamp the end.
__global__ void exec_op(ExecDevice* d, const ExecOp* op, int base, int iter) {
  if (threadIdx.x != 0) return;
  // start at the planned offset into the iteration, never earlier (a late
  // swap-in still delays the op through the stream wait)
  const uint64_t planned = d->iter_start_ns[iter] + uint64_t(op->start) * d->tick_ns;
  // allocations land half a tick after their planned instant, frees exactly
  // on it: the reference processes a tick's frees before its allocations
  // (simulator.cpp:47-52, peak.cpp:51-62)
  while (gtimer() < planned + d->tick_ns / 2) {
  }
  const uint64_t t0 = gtimer();
  for (int k = 0; k < op->n_in; ++k) {
    const int32_t s = op->ins[k];
    if (!d->resident[s]) { atomicAdd(&d->violations, 1); continue; }
    const uint64_t* slot = reinterpret_cast<const uint64_t*>(slot_of(d, s));
    if (*slot != tag_of(s, d->version[s])) atomicAdd(&d->verify_errors, 1);
  }
  for (int k = 0; k < op->n_out; ++k)
    if (op->out_size[k] > 0) acct_add(d, op->outs[k], op->out_size[k]);
  // run until the planned end (absorbs launch overhead); a genuinely late
  // start still gets its full duration only when it began after that end
  const uint64_t until = planned + uint64_t(op->ticks) * d->tick_ns;
  while (gtimer() < until) {
  }
  for (int k = 0; k < op->n_out; ++k) {
    const int32_t s = op->outs[k];
    d->version[s] += 1;
    *reinterpret_cast<uint64_t*>(slot_of(d, s)) = tag_of(s, d->version[s]);
  }
  // a pending swap-out of the storage owns its eviction (simulator.cpp:461-470)
  for (int k = 0; k < op->n_rel; ++k)
    if (d->out_pending[op->rel[k]] == 0 && d->resident[op->rel[k]]) acct_sub(d, op->rel[k], op->rel_size[k]);
  d->op_end_ns[base + op->index] = gtimer();
  __threadfence_system();
}

// Channel wait: hold the copy stream until anchor + delta ticks.
__global__ void exec_delay(ExecDevice* d, int32_t anchor_slot, int iter, int64_t delta_ticks) {
  if (threadIdx.x != 0) return;
  const uint64_t base = anchor_slot >= 0 ? d->op_end_ns[anchor_slot] : d->iter_start_ns[iter];
  const uint64_t until = base + uint64_t(delta_ticks > 0 ? delta_ticks : 0) * d->tick_ns;
  d->xfer_start_ns = gtimer();
  while (gtimer() < until) {
  }
  if (gtimer() > d->xfer_start_ns) d->xfer_start_ns = gtimer();
}

// After the bytes moved: hold the channel for the planned transfer duration,
// then account the storage (swap-out frees and poisons the device slot so
// only a correct swap-in can restore it; swap-in allocates).
__global__ void exec_xfer_done(ExecDevice* d, int32_t s, int64_t size, int64_t dur_ticks, int dir) {
  if (threadIdx.x != 0) return;
  const uint64_t until = d->xfer_start_ns + uint64_t(dur_ticks) * d->tick_ns + (dir == 1 ? d->tick_ns / 2 : 0);
  while (gtimer() < until) {
  }
  if (dir == 0) {
    atomicSub(&d->out_pending[s], 1);
    if (d->resident[s]) acct_sub(d, s, size);
    *reinterpret_cast<uint64_t*>(slot_of(d, s)) = 0xdeaddeaddeaddeadull;
    d->n_out += 1;
  } else {
    acct_add(d, s, size);
    d->n_in += 1;
  }
}

// Iteration start: arm the per-storage pending swap-out counts and stamp the
// iteration start (the anchor of iteration-start swap events).
__global__ void exec_iter_begin(ExecDevice* d, const int32_t* outs_per_iter, int32_t T, int iter) {
  for (int32_t s = threadIdx.x; s < T; s += blockDim.x) d->out_pending[s] = outs_per_iter[s];
  if (threadIdx.x == 0) d->iter_start_ns[iter] = gtimer();
}

// Initial residency (simulator.cpp:247-269): tag and account.
__global__ void exec_init(ExecDevice* d, const int32_t* st, const int64_t* sz, int n) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < n; ++k) {
    acct_add(d, st[k], sz[k]);
    *reinterpret_cast<uint64_t*>(slot_of(d, st[k])) = tag_of(st[k], d->version[st[k]]);
  }
}

// Tags of storages that start on the host (wrapped swap-ins): the host slot
// must hold the tag the first swap-in restores.
__global__ void exec_host_tag(ExecDevice* d, int32_t s, uint8_t* host_slot) {
  if (threadIdx.x != 0) return;
  *reinterpret_cast<uint64_t*>(host_slot) = tag_of(s, d->version[s]);
}

cudaError_t exec_launch_op(ExecDevice* d, const ExecOp* op, int base, int iter, cudaStream_t s) {
  exec_op<<<1, 32, 0, s>>>(d, op, base, iter);
  return cudaGetLastError();
}
cudaError_t exec_launch_iter_begin(ExecDevice* d, const int32_t* outs_per_iter, int32_t T, int iter,
                                   cudaStream_t s) {
  exec_iter_begin<<<1, 256, 0, s>>>(d, outs_per_iter, T, iter);
  return cudaGetLastError();
}
cudaError_t exec_launch_delay(ExecDevice* d, int32_t anchor_op, int iter, int64_t delta, cudaStream_t s) {
  exec_delay<<<1, 32, 0, s>>>(d, anchor_op, iter, delta);
  return cudaGetLastError();
}
cudaError_t exec_launch_done(ExecDevice* d, int32_t st, int64_t size, int64_t dur, int dir, cudaStream_t s) {
  exec_xfer_done<<<1, 32, 0, s>>>(d, st, size, dur, dir);
  return cudaGetLastError();
}
cudaError_t exec_launch_init(ExecDevice* d, const int32_t* st, const int64_t* sz, int n, cudaStream_t s) {
  exec_init<<<1, 32, 0, s>>>(d, st, sz, n);
  return cudaGetLastError();
}
cudaError_t exec_launch_host_tag(ExecDevice* d, int32_t st, uint8_t* host_slot, cudaStream_t s) {
  exec_host_tag<<<1, 32, 0, s>>>(d, st, host_slot);
  return cudaGetLastError();
}

}  // namespace tsl
