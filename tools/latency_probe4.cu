// Dev tool: does L1 serve data written by the CTA itself (sm_100a)?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(const int* hostw, int* devw, int* scratch, int n, int steps, long long* out) {
  extern __shared__ int dyn[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) devw[i] = hostw[i];  // other threads write
  __syncthreads();
  if (threadIdx.x != 0) return;
  int p; long long t0, t1;
  p = 0; for (int s = 0; s < steps; ++s) p = hostw[p];
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = hostw[p]; t1 = clock64(); out[0] = t1 - t0; out[9] = p;
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = devw[p]; t1 = clock64(); out[1] = t1 - t0; out[9] += p;
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) p = devw[p]; t1 = clock64(); out[2] = t1 - t0; out[9] += p;
  // interleave an unrelated store (different line) with every load
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) { scratch[(s & 15) * 32] = s; p = hostw[p]; } t1 = clock64(); out[3] = t1 - t0; out[9] += p;
  // store to the same line that is then loaded
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) { const int q = hostw[p]; devw[p] = q; p = devw[q]; } t1 = clock64(); out[4] = t1 - t0; out[9] += p;
  // after a __threadfence_block
  p = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) { p = hostw[p]; __threadfence_block(); } t1 = clock64(); out[5] = t1 - t0; out[9] += p;
  // int64 chain (8 B loads) for comparison
  const long long* h64 = reinterpret_cast<const long long*>(hostw);
  long long q = 0; t0 = clock64(); for (int s = 0; s < steps; ++s) q = h64[(q & ((n / 2) - 1))] >> 0; t1 = clock64(); out[6] = t1 - t0; out[9] += (int)q;
}

int main() {
  const int n = 2048, steps = 4000;  // 8 KB working set
  std::vector<int> h(n), perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  uint64_t x = 88172645463325252ull;
  for (int i = n - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = x % (i + 1); std::swap(perm[i], perm[j]); }
  for (int i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
  int *dh, *dd, *sc; long long* o;
  cudaMalloc(&dh, n * 4); cudaMalloc(&dd, n * 4); cudaMalloc(&sc, 4096 * 4); cudaMalloc(&o, 128);
  cudaMemcpy(dh, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 << 10);
  probe<<<1, 256, 48 << 10>>>(dh, dd, sc, n, steps, o);
  cudaDeviceSynchronize();
  long long r[10];
  cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
  const char* names[] = {"host-written", "CTA-written, 1st pass", "CTA-written, 2nd pass", "load + unrelated store",
                         "store then load same line", "load + threadfence_block", "int64 loads"};
  for (int k = 0; k < 7; ++k) printf("%-28s %6.1f cycles/step\n", names[k], double(r[k]) / steps);
  return 0;
}
