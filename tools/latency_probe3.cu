// Dev tool: L1 hit latency vs dynamic shared memory / carveout on sm_100a.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase(const int* a, int steps, long long* out, int* sink) {
  extern __shared__ int dyn[];
  if (threadIdx.x == 0 && steps < 0) dyn[0] = 1;
  if (threadIdx.x != 0) return;
  int p = 0;
  for (int s = 0; s < steps; ++s) p = a[p];
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) p = a[p];
  long long t1 = clock64();
  *out = t1 - t0;
  *sink = p;
}

int main() {
  const int steps = 4000;
  for (int kb : {8, 32, 96}) {
    const int n = kb * 256;
    std::vector<int> h(n), perm(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    uint64_t x = 88172645463325252ull;
    for (int i = n - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = x % (i + 1); std::swap(perm[i], perm[j]); }
    for (int i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
    int *d, *sink; long long* o;
    cudaMalloc(&d, n * 4); cudaMalloc(&o, 8); cudaMalloc(&sink, 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int smem_kb : {0, 16, 64, 116, 200}) {
      for (int carve : {-1, 0, 25, 50, 100}) {
        cudaFuncSetAttribute(chase, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
        if (carve >= 0) cudaFuncSetAttribute(chase, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        else cudaFuncSetAttribute(chase, cudaFuncAttributePreferredSharedMemoryCarveout, -1);
        chase<<<1, 256, smem_kb * 1024>>>(d, steps, o, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long r = 0;
        cudaMemcpy(&r, o, 8, cudaMemcpyDeviceToHost);
        printf("set %3d KB  dyn smem %3d KB  carveout %4d  -> %6.1f cyc/load %s\n", kb, smem_kb, carve, double(r) / steps,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
    cudaFree(d);
  }
  return 0;
}
