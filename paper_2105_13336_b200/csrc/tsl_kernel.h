// Host-side view of the planning kernel (tsl_kernel.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "tsl_types.h"

namespace tsl {
constexpr int NT = 512;         // threads per planning CTA
constexpr int SORT_IPT = 24;    // largest block-sort tile: NT * SORT_IPT keys
constexpr int SORT_CAP = NT * SORT_IPT;
constexpr size_t PAIRREC_BYTES = 16 * 8;  // sizeof(PairRec), checked in tsl_kernel.cu
size_t kernel_smem_bytes();
cudaError_t launch_plan_kernel(GroupDev* d_groups, int n_groups, int mode, cudaStream_t stream);
}  // namespace tsl
