// Floor of the mapped host step: host launches a kernel and spins on a
// completion word the kernel writes into pinned host memory. Modes:
//  0: every CTA __threadfence_system + counts itself, the last raises the word
//  1: every CTA __threadfence (device scope) + counts, last CTA fences system
//  2: as 1, and the last CTA copies the whole [rewards|dones] block (9 B/env)
//     from device memory to host before the system fence
//  3: as 0, and every CTA writes its 4 envs' results to host first
//  4: as 3 with a device-scope fence per CTA, the last CTA fences system
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mapped ubench_mapped.cu
#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <cstdio>

__global__ void k_flag(volatile int* done, const long long* act, unsigned* cnt, int ncta, int gen,
                       int mode, const uint4* dres, uint4* hres, int n16) {
  long long a = 0;
  if (threadIdx.x < 4) a = act[blockIdx.x * 4 + threadIdx.x];
  __syncthreads();
  if (mode >= 3 && threadIdx.x < 4) ((double*)hres)[blockIdx.x * 4 + threadIdx.x] = (double)a;
  __shared__ int last;
  if (threadIdx.x == 0) {
    if (mode == 0 || mode == 3) __threadfence_system(); else __threadfence();
    unsigned prev = atomicAdd(cnt, 1u);
    last = prev == (unsigned)(gen * ncta + ncta - 1);
  }
  __syncthreads();
  if (!last) return;
  if (mode == 2)
    for (int i = threadIdx.x; i < n16; i += blockDim.x) hres[i] = dres[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode != 0 && mode != 3) __threadfence_system();
    done[0] = gen + 1;
  }
}

int main() {
  int *h; long long* act; unsigned* cnt; uint4 *dres, *hres;
  cudaHostAlloc(&h, 64, cudaHostAllocMapped);
  cudaHostAlloc(&act, 1 << 20, cudaHostAllocMapped);
  cudaHostAlloc(&hres, 1 << 20, cudaHostAllocMapped);
  cudaMalloc(&dres, 1 << 20);
  cudaMalloc(&cnt, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int mode = 0; mode < 5; mode++)
  for (int ncta : {1, 148, 1036}) {
    cudaMemset(cnt, 0, 4); cudaDeviceSynchronize();
    volatile int* d = h; d[0] = 0;
    const int K = 2000, n16 = ncta * 4 * 9 / 16;
    double tl = 0, tw = 0;
    auto T = [] { return std::chrono::duration<double, std::micro>(
                     std::chrono::steady_clock::now().time_since_epoch()).count(); };
    for (int g = 0; g < K + 50; g++) {
      double t0 = T();
      k_flag<<<ncta, 128, 0, st>>>(d, act, cnt, ncta, g, mode, dres, hres, n16);
      double t1 = T();
      while (d[0] != g + 1) {}
      std::atomic_thread_fence(std::memory_order_acquire);
      double t2 = T();
      if (g >= 50) { tl += t1 - t0; tw += t2 - t1; }
    }
    cudaDeviceSynchronize();
    printf("mode=%d ncta=%4d: launch %.2f us, wait %.2f us\n", mode, ncta, tl / K, tw / K);
  }
  return 0;
}
