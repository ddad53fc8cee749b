// Host-side view of the planning kernel (tsl_kernel.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "tsl_types.h"

namespace tsl {
constexpr int NT = 256;         // threads per planning CTA
constexpr int SORT_IPT = 24;    // largest block-sort tile: NT * SORT_IPT keys
constexpr int SORT_CAP = NT * SORT_IPT;
constexpr int TI_NB_HOST = 256;  // == TI_NB in tsl_plan.cuh
constexpr size_t PAIRREC_BYTES = 16 * 8;  // sizeof(PairRec), checked in tsl_kernel.cu
// Smallest supported block-sort tile (items per thread) covering n keys.
int sort_ipt_for(int64_t n);
constexpr int RES_MAX_JOBS = 16;  // groups up to this many jobs may keep job arrays in shared memory
constexpr size_t RES_FULL_MAX = size_t(64) << 10;  // ... when all of them fit in this many bytes
// Dynamic shared memory of a launch; res_bytes > 0 adds the JobDev copies and
// the resident job arrays (build mode, <= RES_MAX_JOBS jobs per group).
// Launches whose largest job exceeds one sort tile ("big") sort in global
// memory with a small shared digit table instead of resident job arrays.
constexpr size_t BIG_AUX_BYTES = (4 * 256 + NT) * sizeof(int32_t);
size_t kernel_smem_bytes(int max_jobs, int ipt, size_t res_bytes, bool big = false);
// Shared-memory bytes that would hold every resident array of the job.
size_t resident_bytes_for(int32_t A, int32_t T, int32_t Scap);
// coop: a single group above one sort tile runs as a cooperative launch of one
// CTA per SM (CTA 0 plans; the others join its block-wide sorts).
cudaError_t launch_plan_kernel(GroupDev* d_groups, int n_groups, int mode, int max_jobs, int ipt, size_t res_bytes,
                               bool big, bool coop, cudaStream_t stream);
}  // namespace tsl
