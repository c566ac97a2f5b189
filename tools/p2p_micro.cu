// p2p_micro.cu — NVLink peer-copy microbenchmark (dev tool, 2 GPUs, one process).
//
// Measures the bandwidth of the two data-movement primitives the lane
// allreduce can use, as a function of the number of CTAs:
//   ldst : 128-bit LDG / STG, unrolled, grid-stride
//   tma  : cp.async.bulk global->smem (mbarrier) then smem->global (bulk_group)
// modes: push (local src -> peer dst), pull (peer src -> local dst), local.
// "bi" runs the same kernel on both GPUs at once (each pushes/pulls to the
// other), which is what an allreduce does.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_micro tools/p2p_micro.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <int U>
__global__ void __launch_bounds__(512) k_ldst(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t i = i0 + u * stride;
      if (i < n) v[u] = __ldcg(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t i = i0 + u * stride;
      if (i < n) __stcg(dst + i, v[u]);
    }
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// per CTA: contiguous slice; one thread streams tiles through an S-stage ring
__global__ void k_tma(const char* src, char* dst, int64_t bytes, int tile, int stages) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * tile);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t per = (bytes / gridDim.x) & ~(int64_t)15;
  const char* s0 = src + per * blockIdx.x;
  char* d0 = dst + per * blockIdx.x;
  const int64_t nt = (per + tile - 1) / tile;
  // prologue: issue loads for the first `stages` tiles
  for (int64_t t = 0; t < nt + stages; ++t) {
    if (t >= stages) {  // consume tile t - stages
      const int64_t c = t - stages;
      const int s = (int)(c % stages);
      const uint32_t par = (uint32_t)((c / stages) & 1);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok) : "r"(sa(&full[s])), "r"(par) : "memory");
      const int64_t off = c * tile;
      const uint32_t b = (uint32_t)(per - off < tile ? per - off : tile);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d0 + off),
                   "r"(sa(sm + (size_t)s * tile)), "r"(b) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (t < nt) {
      const int s = (int)(t % stages);
      if (t >= stages) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
      const int64_t off = t * tile;
      const uint32_t b = (uint32_t)(per - off < tile ? per - off : tile);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(b) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)s * tile)), "l"(s0 + off), "r"(b), "r"(sa(&full[s])) : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 1024) << 20;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  char *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaMemset(b[d], 0, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  const char* modes[] = {"push", "pull", "local"};
  const int ctas[] = {8, 16, 32, 64, 96, 148};
  for (int bi = 0; bi < 2; ++bi)
    for (int eng = 0; eng < 3; ++eng)
      for (int m = 0; m < 3; ++m)
        for (int ci = 0; ci < 6; ++ci) {
          const int C = ctas[ci];
          int tile = eng == 2 ? 32768 : 49152, stages = 4;
          float ms[2] = {0, 0};
          for (int rep = 0; rep < 4; ++rep) {
            for (int d = 0; d <= bi; ++d) {
              CK(cudaSetDevice(d));
              const int o = 1 - d;
              const char* src = m == 1 ? a[o] : a[d];
              char* dst = m == 0 ? b[o] : b[d];
              CK(cudaEventRecord(e0[d], st[d]));
              if (eng == 0)
                k_ldst<8><<<C, 512, 0, st[d]>>>((const uint4*)src, (uint4*)dst, bytes / 16);
              else
                k_tma<<<C, 32, (size_t)stages * tile + 64, st[d]>>>(src, dst, bytes, tile, stages);
              CK(cudaEventRecord(e1[d], st[d]));
            }
            for (int d = 0; d <= bi; ++d) {
              CK(cudaSetDevice(d));
              CK(cudaEventSynchronize(e1[d]));
              CK(cudaEventElapsedTime(&ms[d], e0[d], e1[d]));
            }
          }
          float t = ms[0] > ms[1] ? ms[0] : ms[1];
          printf("%s %-5s %-5s ctas=%3d  %7.1f GB/s  (%.3f ms)\n", bi ? "bi " : "uni",
                 eng == 0 ? "ldst" : (eng == 1 ? "tma48" : "tma32"), modes[m], C, bytes / (t * 1e-3) / 1e9, t);
          fflush(stdout);
        }
  return 0;
}
