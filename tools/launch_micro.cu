// launch_micro.cu — the GPU-side gap between back-to-back kernels on one
// stream (dev tool, 1 GPU): 148 CTAs x 512 threads, each CTA spins a fixed
// time; per launch = event time / launches; gap = per launch - spin. Varies
// the kernel-parameter size (a ~1.1 KB __grid_constant__ struct like
// LaneParams vs 16 B) and programmatic dependent launch (PDL).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_micro tools/launch_micro.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

struct Big {
  uint64_t w[140];  // 1120 B
  uint64_t spin_ns;
};
struct Small {
  uint64_t spin_ns;
  uint64_t* out;
};

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool PDL>
__device__ __forceinline__ void body(uint64_t spin_ns, uint64_t salt) {
  if (PDL) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  const uint64_t t0 = gt();
  while (gt() - t0 < spin_ns) {
  }
  if (salt == 0xdeadbeef) asm volatile("trap;");
}

template <bool PDL>
__global__ void __launch_bounds__(512, 1) k_big(const __grid_constant__ Big b) {
  body<PDL>(b.spin_ns, b.w[threadIdx.x & 127]);
}
template <bool PDL>
__global__ void __launch_bounds__(512, 1) k_small(const __grid_constant__ Small s) {
  body<PDL>(s.spin_ns, (uint64_t)s.out);
}

template <typename P>
cudaError_t launch(const void* fn, P& prm, bool pdl, cudaStream_t s) {
  void* args[] = {&prm};
  if (!pdl) return cudaLaunchKernel(fn, dim3(148), dim3(512), args, 0, s);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  Big big;
  memset(&big, 0, sizeof(big));
  Small small{0, nullptr};
  const uint64_t spins[] = {0, 5000, 20000, 50000};
  for (uint64_t sp : spins)
    for (int variant = 0; variant < 4; ++variant) {
      const bool pdl = variant & 1, isbig = variant & 2;
      big.spin_ns = small.spin_ns = sp;
      const void* fn = isbig ? (pdl ? (const void*)k_big<true> : (const void*)k_big<false>)
                             : (pdl ? (const void*)k_small<true> : (const void*)k_small<false>);
      const int n = 200;
      for (int w = 0; w < 20; ++w) CK(isbig ? launch(fn, big, pdl, s) : launch(fn, small, pdl, s));
      CK(cudaEventRecord(e0, s));
      for (int i = 0; i < n; ++i) CK(isbig ? launch(fn, big, pdl, s) : launch(fn, small, pdl, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double per = ms * 1e3 / n;
      printf("spin %6.1f us  params %-5s pdl %d : %8.2f us per launch, gap %6.2f us\n", sp / 1e3,
             isbig ? "1.1KB" : "16B", (int)pdl, per, per - sp / 1e3);
    }
  return 0;
}
