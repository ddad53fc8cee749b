// TEST INFRASTRUCTURE ONLY: runs tsl_plan.cuh's plan_group/analyze_group with a
// one-thread host context in place of tsl_plan_kernel (see cuda_runtime.h here).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <utility>
#include <vector>

#include "tsl_exec.h"
#include "tsl_kernel.h"
#include "tsl_plan.cuh"

namespace tsl {

struct HostX {
  static constexpr int W = 1;
  static constexpr bool GRID = false;
  int tid = 0, nthr = 1, lane = 0, warp = 0, nwarp = 1;
  int64_t* sh = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int sort_cap = 0;
  void sync() {}
  int32_t fold_threshold(int32_t bz_n) const { return std::max(PEND_MERGE, bz_n / 128); }
  bool fold_hook(const int64_t*, const int64_t*, int32_t, const int64_t*, const int64_t*, int32_t, int64_t*, int64_t*,
                 int64_t*, int64_t*, int32_t*, int32_t*, int, int32_t) { return false; }
  int64_t clock() { return 0; }
  void wsync() {}
  bool wany(bool p) { return p; }
  unsigned wballot(bool p) { return p ? 1u : 0u; }
  int64_t shfl(int64_t v, int) { return v; }
  int ffs(unsigned m) { return m ? __builtin_ffs(m) : 0; }
  int32_t wexcl(int32_t v, int32_t* total) { *total = v; return 0; }
  int64_t aadd(int64_t* p, int64_t v) { int64_t o = *p; *p += v; return o; }
  int32_t aadd32(int32_t* p, int32_t v) { int32_t o = *p; *p += v; return o; }
  void amin(int64_t* p, int64_t v) { if (v < *p) *p = v; }
  void amax(int64_t* p, int64_t v) { if (v > *p) *p = v; }
  void radd(int64_t* p, int64_t v) { *p += v; }
  void ramin(int64_t* p, int64_t v) { if (v < *p) *p = v; }
  void ramax(int64_t* p, int64_t v) { if (v > *p) *p = v; }
  void amax32(int32_t* p, int32_t v) { if (v > *p) *p = v; }
  void aor32(int32_t* p, int32_t v) { *p |= v; }
  void amin32(int32_t* p, int32_t v) { if (v < *p) *p = v; }
  void errset(GroupDev& g, const ErrInfo& e) { if (!g.err.code) g.err = e; }
  void sort(uint64_t* keys, int32_t* vals, int n, int bits) {
    if (n <= 1 || bits <= 0) return;
    const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    std::vector<std::pair<uint64_t, int32_t>> v(n);
    for (int i = 0; i < n; ++i) v[i] = {keys[i], vals[i]};
    std::stable_sort(v.begin(), v.end(), [&](const auto& a, const auto& b) { return (a.first & mask) < (b.first & mask); });
    for (int i = 0; i < n; ++i) { keys[i] = v[i].first; vals[i] = v[i].second; }
  }
  void scan(int64_t* a, int n) { for (int i = 1; i < n; ++i) a[i] += a[i - 1]; }
  void scan_max(int64_t* a, int n) { for (int i = 1; i < n; ++i) a[i] = std::max(a[i], a[i - 1]); }
};

int sort_ipt_for(int64_t n) {
  for (int ipt : {1, 2, 4, 8, 16}) if (n <= int64_t(NT) * ipt) return ipt;
  return SORT_IPT;
}
size_t kernel_smem_bytes(int, int, size_t, bool) { return SH_WORDS * sizeof(int64_t); }
size_t resident_bytes_for(int32_t, int32_t, int32_t) { return 0; }

cudaError_t launch_plan_kernel(GroupDev* groups, int n_groups, int mode, int, int ipt, size_t, bool, bool, cudaStream_t) {
  std::vector<int64_t> sh(SH_WORDS);
  std::vector<int64_t> tmp(96 * 1024 / 8);  // stands in for the shared sort scratch
  for (int gi = 0; gi < n_groups; ++gi) {
    HostX x;
    x.sh = sh.data();
    x.tmp = tmp.data();
    x.tmp_bytes = size_t(NT) * ipt * sizeof(int64_t);  // like the device tile
    x.sort_cap = NT * ipt;
    if (mode == 0) plan_group(x, groups[gi]);
    else analyze_group(x, groups[gi]);
  }
  return cudaSuccess;
}

// The plan executor needs a GPU: the emulation build reports an error.
cudaError_t exec_launch_op(ExecDevice*, const ExecOp*, int, int, cudaStream_t) { return 1; }
cudaError_t exec_launch_delay(ExecDevice*, int32_t, int, int64_t, cudaStream_t) { return 1; }
cudaError_t exec_launch_done(ExecDevice*, int32_t, int64_t, int64_t, int, cudaStream_t) { return 1; }
cudaError_t exec_launch_init(ExecDevice*, const int32_t*, const int64_t*, int, cudaStream_t) { return 1; }
cudaError_t exec_launch_host_tag(ExecDevice*, int32_t, uint8_t*, cudaStream_t) { return 1; }
cudaError_t exec_launch_iter_begin(ExecDevice*, const int32_t*, int32_t, int, cudaStream_t) { return 1; }

}  // namespace tsl
