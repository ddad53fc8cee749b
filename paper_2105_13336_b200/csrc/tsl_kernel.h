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
size_t kernel_smem_bytes(int max_jobs, int ipt);
cudaError_t launch_plan_kernel(GroupDev* d_groups, int n_groups, int mode, int max_jobs, int ipt,
                               cudaStream_t stream);
}  // namespace tsl
