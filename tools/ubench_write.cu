// Floor measurements for the one-wave C2 step shape (perf experiments only):
// how long do 4096 x 12288-byte frame writes take with the step kernel's
// launch shapes, with and without a compute phase in front, and what does a
// graph of K back-to-back launches cost per launch?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubw tools/ubench_write.cu && /tmp/ubw
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 4096, FB = 12288;

// G lanes per env, envs interleaved contiguously per CTA; each lane stores
// chunks l, l+G, ... of the env's frame (16-byte streaming stores);
// `spin` cycles of dependent work before the stores (a stand-in for the
// ray pass latency)
template <int G>
__global__ void __launch_bounds__(128) frames_kernel(uint4* __restrict__ out, int n, int spin,
                                                     int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  const int per_cta = 128 / G;
  const int epc = (n + gridDim.x - 1) / gridDim.x;
  if (grp >= epc) return;
  const int i = blockIdx.x * epc + grp;
  if (i >= n) return;
  uint32_t x = i * 2654435761u + lane;
  for (int k = 0; k < spin; k++) x = x * 1664525u + 1013904223u;
  uint4* f = out + (size_t)i * (FB / 16);
  for (int c = lane; c < FB / 16; c += G) __stcs(f + c, make_uint4(x, x + 1, x + 2, c));
  (void)per_cta;
}

__global__ void persistent_frames(uint4* __restrict__ out, size_t n16) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n16;
       k += (size_t)gridDim.x * blockDim.x)
    __stcs(out + k, make_uint4((uint32_t)k, 1, 2, 3));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int ring = 8;
  uint4* buf;
  CK(cudaMalloc(&buf, (size_t)ring * N * FB));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 200;
  auto run = [&](const char* name, auto launch) -> int {
    for (int w = 0; w < 5; w++) launch(w % ring);
    CK(cudaStreamSynchronize(st));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    for (int k_steps : {20, K}) {
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
      for (int k = 0; k < k_steps; k++) launch(k % ring);
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, st));
      CK(cudaStreamSynchronize(st));
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double us = 1e3 * best / k_steps;
      printf("%-44s K=%3d  %7.2f us/launch  %7.1f GB/s  %6.1f M env-steps/s\n", name, k_steps, us,
             (double)N * FB / (us * 1e-6) / 1e9, N / us);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
    return 0;
  };
  auto launch_ex = [&](const void* fn, int grid, void** args, int pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaLaunchKernelExC(&cfg, fn, args);
  };
  for (int pdl = 0; pdl < 2; pdl++) {
    for (int spin : {0, 2000, 8000}) {
      char name[128];
      snprintf(name, sizeof name, "G16 grid=%d spin=%d pdl=%d", 4 * sms, spin, pdl);
      run(name, [&](int r) {
        uint4* o = buf + (size_t)r * N * FB / 16;
        int n = N, sp = spin, p = pdl;
        void* args[] = {&o, &n, &sp, &p};
        launch_ex((const void*)frames_kernel<16>, 4 * sms, args, p);
      });
      snprintf(name, sizeof name, "G32 grid=%d spin=%d pdl=%d", 7 * sms, spin, pdl);
      run(name, [&](int r) {
        uint4* o = buf + (size_t)r * N * FB / 16;
        int n = N, sp = spin, p = pdl;
        void* args[] = {&o, &n, &sp, &p};
        launch_ex((const void*)frames_kernel<32>, 7 * sms, args, p);
      });
    }
  }
  run("persistent grid-stride 148x1024", [&](int r) {
    persistent_frames<<<sms, 1024, 0, st>>>(buf + (size_t)r * N * FB / 16, (size_t)N * FB / 16);
  });
  run("grid-stride 4x148x512", [&](int r) {
    persistent_frames<<<4 * sms, 512, 0, st>>>(buf + (size_t)r * N * FB / 16, (size_t)N * FB / 16);
  });
  return 0;
}
