// Microbenchmark (dev tool): dependent-load latency seen by one thread for
// the access patterns the planner uses.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(int32_t* next_host, int32_t* next_dev, int n, int steps, long long* out) {
  extern __shared__ int32_t snext[];
  // (b) the CTA writes a permutation chain into global memory itself
  for (int i = threadIdx.x; i < n; i += blockDim.x) { next_dev[i] = next_host[i]; snext[i] = next_host[i]; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int p; long long t0, t1;
  // (a) host-written global, first touch (cold L1)
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = next_host[p]; t1 = clock64(); out[0] = t1 - t0; out[8] = p;
  // (a') same again (warm)
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = next_host[p]; t1 = clock64(); out[1] = t1 - t0; out[8] += p;
  // (b) written by other threads of this CTA earlier in the kernel
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = next_dev[p]; t1 = clock64(); out[2] = t1 - t0; out[8] += p;
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = next_dev[p]; t1 = clock64(); out[3] = t1 - t0; out[8] += p;
  // (c) shared memory
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = snext[p]; t1 = clock64(); out[4] = t1 - t0; out[8] += p;
  // (d) host-written via __ldg
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = __ldg(&next_host[p]); t1 = clock64(); out[5] = t1 - t0; out[8] += p;
  // (e) store then reload own write (same thread), L1 write-through behaviour
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) { next_dev[n + (s & 7)] = p; p = next_dev[p] + (next_dev[n + (s & 7)] & 0); } t1 = clock64(); out[6] = t1 - t0; out[8] += p;
}

int main() {
  const int n = 8192, steps = 2000;
  std::vector<int32_t> h(n);
  // random single-cycle permutation over a 32 KB working set
  std::vector<int32_t> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  uint64_t x = 88172645463325252ull;
  for (int i = n - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = x % (i + 1); std::swap(perm[i], perm[j]); }
  for (int i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
  int32_t *dh, *dd; long long* dout;
  cudaMalloc(&dh, n * 4); cudaMalloc(&dd, (n + 64) * 4); cudaMalloc(&dout, 16 * 8);
  cudaMemcpy(dh, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 4);
  for (int it = 0; it < 2; ++it) {
    probe<<<1, 256, n * 4>>>(dh, dd, n, steps, dout);
    cudaDeviceSynchronize();
  }
  long long o[16];
  cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
  const char* names[] = {"host-written global, cold", "host-written global, warm", "CTA-written global, 1st",
                         "CTA-written global, 2nd", "shared memory", "__ldg host-written", "store+reload own"};
  for (int k = 0; k < 7; ++k) printf("%-28s %6.1f cycles/load\n", names[k], double(o[k]) / steps);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
