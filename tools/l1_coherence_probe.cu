// Dev probe: after the planner's grid barrier (volatile generation spin +
// __threadfence), do plain (L1-cached) loads of data another CTA wrote
// observe the new values? CTA 1 caches the array, CTA 0 rewrites it, CTA 1
// re-reads it -- many rounds, all CTAs of a cooperative launch.
#include <cstdio>
#include <cuda_runtime.h>

struct Bar { int count, gen; };

__device__ void grid_barrier(Bar* b, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile int* gen = &b->gen;
    const int g0 = *gen;
    __threadfence();
    if (atomicAdd(&b->count, 1) == G - 1) { b->count = 0; __threadfence(); atomicAdd(&b->gen, 1); }
    else while (*gen == g0) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

__global__ void probe(int* data, int n, Bar* bar, int rounds, int* errors, long long* sink) {
  const int G = gridDim.x;
  long long acc = 0;
  for (int r = 0; r < rounds; ++r) {
    // every CTA but the writer reads (caches) the array
    if (blockIdx.x != 0) for (int i = threadIdx.x; i < n; i += blockDim.x) acc += data[i];
    grid_barrier(bar, G);
    if (blockIdx.x == 0) for (int i = threadIdx.x; i < n; i += blockDim.x) data[i] = r * 7 + i;
    grid_barrier(bar, G);
    if (blockIdx.x != 0)
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (data[i] != r * 7 + i) atomicAdd(errors, 1);
    grid_barrier(bar, G);
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 4096, rounds = 2000, T = 256;
  int *data, *errors; Bar* bar; long long* sink;
  cudaMalloc(&data, n * sizeof(int)); cudaMemset(data, 0, n * sizeof(int));
  cudaMalloc(&errors, sizeof(int)); cudaMemset(errors, 0, sizeof(int));
  cudaMalloc(&bar, sizeof(Bar)); cudaMemset(bar, 0, sizeof(Bar));
  cudaMalloc(&sink, sms * T * sizeof(long long));
  int nn = n, rr = rounds;
  void* args[] = {&data, &nn, &bar, &rr, &errors, &sink};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, dim3(sms), dim3(T), args, 0, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  int h = -1;
  cudaMemcpy(&h, errors, sizeof(int), cudaMemcpyDeviceToHost);
  printf("launch %s sync %s grid %d rounds %d stale reads %d\n", cudaGetErrorString(e), cudaGetErrorString(e2), sms,
         rounds, h);
  return 0;
}
