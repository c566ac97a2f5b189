// ll128_micro.cu — how fast can SMs push 128-byte LL128 lines to a peer GPU?
// (dev tool; 2 GPUs, one process, both GPUs push to each other at once, as
// phase A of the lane kernel does at 2x2 / 1x2).
//
// Each thread moves U granules per step: loads U x 16 B of its source
// (ld.global.cs, like load_x), then stores them to the peer with
//   weak     : st.global.v4 (16 B per lane, 512 B per warp instruction)
//   volatile : st.volatile.global.v4 in the LL128 line layout (lanes 0-6 data,
//              lane 7 the epoch; what lane_ll128.cuh line_store does)
//   relaxed  : st.relaxed.sys.global.v4 in the line layout
// and the "line" modes move 7/8 of the bytes as data (GB/s counts line bytes).
// Sizes: a phase-sized push (8, 16 MiB) and a long one (256 MiB).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ll128_micro tools/ll128_micro.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint4 ld_cs(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int MODE>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
  if (MODE == 0)
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if (MODE == 1)
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else
    asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// n16 = 16-byte units of the destination; warp w of CTA c handles steps
// (c * warps + w) + k * (grid warps); a step = U * 32 consecutive units.
template <int MODE, int U, bool LINE>
__global__ void __launch_bounds__(512, 1) k_push(const uint4* __restrict__ src, uint4* dst, int64_t n16, uint32_t ep) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t s = w0; s * U * 32 < n16; s += warps) {
    uint4 v[U];
    const int64_t base = s * U * 32;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      v[u] = (i < n16 && !(LINE && (lane & 7) == 7)) ? ld_cs(src + i) : make_uint4(ep, ep, ep, ep);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      if (i < n16) st16<MODE>(dst + i, v[u]);
    }
  }
}

typedef void (*kfn)(const uint4*, uint4*, int64_t, uint32_t);

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const int64_t maxb = 256ll << 20;
  char *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], maxb));
    CK(cudaMalloc(&b[d], maxb));
    CK(cudaMemset(a[d], 1, maxb));
    CK(cudaMemset(b[d], 0, maxb));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  struct K {
    const char* name;
    kfn f;
  } ks[] = {
      {"weak U1", k_push<0, 1, false>},       {"weak U2", k_push<0, 2, false>},
      {"weak U4", k_push<0, 4, false>},       {"weak U8", k_push<0, 8, false>},
      {"line-volatile U1", k_push<1, 1, true>}, {"line-volatile U2", k_push<1, 2, true>},
      {"line-volatile U4", k_push<1, 4, true>}, {"line-volatile U8", k_push<1, 8, true>},
      {"line-weak U2", k_push<0, 2, true>},     {"line-weak U4", k_push<0, 4, true>},
      {"line-relaxed U2", k_push<2, 2, true>},  {"line-relaxed U4", k_push<2, 4, true>},
  };
  const int64_t sizes[] = {8ll << 20, 16ll << 20, 256ll << 20};
  const int ctas[] = {148, 74};
  for (int64_t bytes : sizes)
    for (int C : ctas)
      for (const K& k : ks) {
        const int reps = bytes >= (256ll << 20) ? 5 : 50;
        float best = 1e30f, tot = 0;
        for (int r = 0; r < reps + 2; ++r) {
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(e0[d], st[d]));
            k.f<<<C, 512, 0, st[d]>>>((const uint4*)a[d], (uint4*)b[1 - d], bytes / 16, 7u + r);
            CK(cudaEventRecord(e1[d], st[d]));
          }
          float ms[2];
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(e1[d]));
            CK(cudaEventElapsedTime(&ms[d], e0[d], e1[d]));
          }
          const float t = ms[0] > ms[1] ? ms[0] : ms[1];
          if (r >= 2) {
            tot += t;
            if (t < best) best = t;
          }
        }
        printf("bi %4lld MiB ctas=%3d %-18s mean %7.1f GB/s  best %7.1f GB/s  (%.2f us)\n", (long long)(bytes >> 20), C,
               k.name, bytes / (tot / reps * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9, tot / reps * 1e3);
        fflush(stdout);
      }
  return 0;
}
