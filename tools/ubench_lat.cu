// Dependent-chain latency of the instructions on the step kernel's critical
// path (perf experiments only): one warp, clock64 around a chain of N ops.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/ubl tools/ubench_lat.cu
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int N = 1024;

__global__ void lat(long long* out, double* dsink, int* isink, double seed, int iseed) {
  __shared__ int sm[1024];
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) sm[k] = (k * 7 + 1) & 1023;
  __syncwarp();
  double x = seed, y = seed * 0.5;
  int v = iseed;
  long long t0, t1;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) x = x + y;
  t1 = clock64();
  out[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) x = x * y;
  t1 = clock64();
  out[1] = t1 - t0;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) x = fma(x, y, y);
  t1 = clock64();
  out[2] = t1 - t0;
  // IEEE reciprocal 1.0 / x
  t0 = clock64();
#pragma unroll 4
  for (int k = 0; k < N / 8; k++) x = 1.0 / (x + 1.5);
  t1 = clock64();
  out[3] = (t1 - t0) * 8;
  // IEEE division y / x
  t0 = clock64();
#pragma unroll 4
  for (int k = 0; k < N / 8; k++) x = (y + 3.0) / (x + 1.5);
  t1 = clock64();
  out[4] = (t1 - t0) * 8;
  // sqrt
  t0 = clock64();
#pragma unroll 4
  for (int k = 0; k < N / 8; k++) x = sqrt(x + 2.0);
  t1 = clock64();
  out[5] = (t1 - t0) * 8;
  // LDS pointer chase
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) v = sm[v];
  t1 = clock64();
  out[6] = t1 - t0;
  // SHFL chain
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64();
  out[7] = t1 - t0;
  // double -> int -> double
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) x = (double)(int)(x + 1.0);
  t1 = clock64();
  out[8] = t1 - t0;
  // DSETP + predicated DADD (the march's fp chain)
  double sx = seed, sy = seed + 0.25;
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) {
    if (sx < sy) sx += 0.7; else sy += 0.9;
  }
  t1 = clock64();
  out[9] = t1 - t0;
  // IADD chain
  t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; k++) v = v * 3 + 1;
  t1 = clock64();
  out[10] = t1 - t0;
  dsink[threadIdx.x] = x + sx + sy;
  isink[threadIdx.x] = v;
}

int main() {
  long long* out;
  double* ds;
  int* is;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&ds, 1024 * 8);
  cudaMalloc(&is, 1024 * 4);
  for (int rep = 0; rep < 2; rep++) lat<<<1, 32>>>(out, ds, is, 1.000001, 3);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"DADD", "DMUL", "DFMA", "1.0/x (IEEE)", "y/x (IEEE)", "sqrt (IEEE)",
                         "LDS chase", "SHFL chain", "F2I+I2F", "DSETP+DADD step", "IMAD"};
  for (int k = 0; k < 11; k++) printf("%-18s %7.1f cycles/op\n", names[k], (double)h[k] / N);
  return 0;
}
