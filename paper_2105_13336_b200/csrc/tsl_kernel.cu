// The planning kernel: one CTA of NT threads runs memsched::build_plan for one
// group of jobs (tsl_plan.cuh), grid = groups. This file supplies the device
// execution context: CUB block radix sort / block scan in shared memory,
// warp votes and atomics.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "tsl_plan.cuh"
#include "tsl_kernel.h"

namespace tsl {

static_assert(sizeof(PairRec) == PAIRREC_BYTES, "PairRec layout");

template <int IPT>
using BRS = cub::BlockRadixSort<uint64_t, NT, IPT, int32_t>;
using BScan = cub::BlockScan<int64_t, NT>;

constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t TMP_BYTES =
    cmax(cmax(cmax(sizeof(typename BRS<1>::TempStorage), sizeof(typename BRS<2>::TempStorage)),
              cmax(sizeof(typename BRS<4>::TempStorage), sizeof(typename BRS<8>::TempStorage))),
         cmax(cmax(sizeof(typename BRS<16>::TempStorage), sizeof(typename BRS<SORT_IPT>::TempStorage)),
              sizeof(typename BScan::TempStorage)));

struct DevX {
  static constexpr int W = 32;
  int tid, nthr, lane, warp, nwarp;
  int64_t* sh;
  void* tmp;

  __device__ void sync() { __syncthreads(); }
  __device__ int64_t clock() { return (int64_t)clock64(); }
  __device__ void wsync() { __syncwarp(); }
  __device__ bool wany(bool p) { return __any_sync(0xffffffffu, p); }
  // warp exclusive prefix sum of v; *total = warp sum
  __device__ int32_t wexcl(int32_t v, int32_t* total) {
    int32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    *total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
  }
  __device__ int64_t aadd(int64_t* p, int64_t v) {
    return (int64_t)atomicAdd((unsigned long long*)p, (unsigned long long)v);
  }
  __device__ int32_t aadd32(int32_t* p, int32_t v) { return atomicAdd(p, v); }
  __device__ void amin(int64_t* p, int64_t v) { atomicMin((long long*)p, (long long)v); }
  __device__ void amax(int64_t* p, int64_t v) { atomicMax((long long*)p, (long long)v); }
  __device__ void amax32(int32_t* p, int32_t v) { atomicMax(p, v); }
  __device__ void errset(GroupDev& g, const ErrInfo& e) {
    if (atomicCAS(&g.err.code, 0, e.code) == 0) {
      g.err.job = e.job;
      g.err.tensor = e.tensor;
      g.err.tick = e.tick;
    }
  }

  template <int IPT>
  __device__ void sort_ipt(uint64_t* keys, int32_t* vals, int n, int bits) {
    uint64_t k[IPT];
    int32_t v[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int idx = tid * IPT + i;
      k[i] = idx < n ? keys[idx] : ~0ull;
      v[i] = idx < n ? vals[idx] : -1;
    }
    __syncthreads();
    BRS<IPT>(*reinterpret_cast<typename BRS<IPT>::TempStorage*>(tmp)).Sort(k, v, 0, bits);
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int idx = tid * IPT + i;
      if (idx < n) { keys[idx] = k[i]; vals[idx] = v[i]; }
    }
    __syncthreads();
  }

  // Stable sort of n (key, value) pairs on key bits [0, bits).
  __device__ void sort(uint64_t* keys, int32_t* vals, int n, int bits) {
    __syncthreads();
    if (n <= 1 || bits <= 0) return;
    if (n <= NT) sort_ipt<1>(keys, vals, n, bits);
    else if (n <= 2 * NT) sort_ipt<2>(keys, vals, n, bits);
    else if (n <= 4 * NT) sort_ipt<4>(keys, vals, n, bits);
    else if (n <= 8 * NT) sort_ipt<8>(keys, vals, n, bits);
    else if (n <= 16 * NT) sort_ipt<16>(keys, vals, n, bits);
    else if (n <= SORT_IPT * NT) sort_ipt<SORT_IPT>(keys, vals, n, bits);
    else __trap();  // callers check SORT_CAP first
  }

  // Inclusive scan of a[0, n) in place.
  __device__ void scan(int64_t* a, int n) {
    __syncthreads();
    const int chunk = (n + NT - 1) / NT;
    const int b = tid * chunk, e = min(n, b + chunk);
    int64_t s = 0;
    for (int i = b; i < e; ++i) s += a[i];
    int64_t off;
    BScan(*reinterpret_cast<typename BScan::TempStorage*>(tmp)).ExclusiveSum(s, off);
    for (int i = b; i < e; ++i) { off += a[i]; a[i] = off; }
    __syncthreads();
  }
};

}  // namespace tsl

extern "C" __global__ void __launch_bounds__(tsl::NT, 1) tsl_plan_kernel(tsl::GroupDev* groups, int mode) {
  extern __shared__ __align__(16) uint8_t smem[];
  tsl::DevX x;
  x.tid = threadIdx.x;
  x.nthr = blockDim.x;
  x.lane = threadIdx.x & 31;
  x.warp = threadIdx.x >> 5;
  x.nwarp = blockDim.x >> 5;
  x.sh = reinterpret_cast<int64_t*>(smem);
  x.tmp = smem + tsl::SH_WORDS * sizeof(int64_t);
  tsl::GroupDev& g = groups[blockIdx.x];
  if (mode == 0) tsl::plan_group(x, g);
  else tsl::analyze_group(x, g);
}

namespace tsl {
size_t kernel_smem_bytes() { return SH_WORDS * sizeof(int64_t) + TMP_BYTES; }

cudaError_t launch_plan_kernel(GroupDev* d_groups, int n_groups, int mode, cudaStream_t stream) {
  static bool attr_set = false;
  const size_t smem = kernel_smem_bytes();
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tsl_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  tsl_plan_kernel<<<n_groups, NT, smem, stream>>>(d_groups, mode);
  return cudaGetLastError();
}
}  // namespace tsl
