// Dev tool: which global-load flavours hit L1 on sm_100a for a dependent chain.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_ca(const int* p) { int v; asm volatile("ld.global.ca.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ int ld_cg(const int* p) { int v; asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ int ld_last(const int* p) { int v; asm volatile("ld.global.L1::evict_last.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ int ld_nc_last(const int* p) { int v; asm volatile("ld.global.nc.L1::evict_last.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ int ld_gen(const int* p) { int v; asm volatile("ld.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }

template <int K>
__device__ long long chase(const int* a, int steps, int* sink) {
  int p = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    if (K == 0) p = a[p];
    if (K == 1) p = ld_ca(a + p);
    if (K == 2) p = ld_cg(a + p);
    if (K == 3) p = ld_last(a + p);
    if (K == 4) p = ld_nc_last(a + p);
    if (K == 5) p = ld_gen(a + p);
  }
  long long t1 = clock64();
  *sink += p;
  return t1 - t0;
}

__global__ void probe(const int* a, int steps, long long* out, int* sink) {
  if (threadIdx.x != 0) return;
  int s = 0;
  chase<0>(a, steps, &s); out[0] = chase<0>(a, steps, &s);
  chase<1>(a, steps, &s); out[1] = chase<1>(a, steps, &s);
  chase<2>(a, steps, &s); out[2] = chase<2>(a, steps, &s);
  chase<3>(a, steps, &s); out[3] = chase<3>(a, steps, &s);
  chase<4>(a, steps, &s); out[4] = chase<4>(a, steps, &s);
  chase<5>(a, steps, &s); out[5] = chase<5>(a, steps, &s);
  *sink = s;
}

int main() {
  const int steps = 4000;
  const char* names[] = {"plain a[p]", "ld.global.ca", "ld.global.cg", "ld.global.L1::evict_last",
                         "ld.global.nc.L1::evict_last", "generic ld"};
  for (int n : {256, 2048, 8192}) {
    std::vector<int> h(n), perm(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    uint64_t x = 88172645463325252ull;
    for (int i = n - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = x % (i + 1); std::swap(perm[i], perm[j]); }
    for (int i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
    int *d, *sink; long long* o;
    cudaMalloc(&d, n * 4); cudaMalloc(&o, 64); cudaMalloc(&sink, 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    probe<<<1, 32>>>(d, steps, o, sink);
    cudaDeviceSynchronize();
    long long r[6];
    cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
    printf("working set %d KB\n", n * 4 / 1024);
    for (int k = 0; k < 6; ++k) printf("  %-30s %6.1f cycles/load\n", names[k], double(r[k]) / steps);
  }
  return 0;
}
