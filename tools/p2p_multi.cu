// p2p_multi.cu — multi-GPU NVLink traffic-pattern microbenchmark (dev tool).
//
// All n GPUs run concurrently (one stream each, one process). Each GPU moves
// `bytes` per run with 128-bit LDG/STG kernels:
//   ring-push  : to (d+1) % n
//   a2a-push   : 1/(n-1) to every other GPU (CTA c writes to peer c % (n-1))
//   a2a-pull   : 1/(n-1) from every other GPU
//   a2a-push-i : like a2a-push but every CTA interleaves all peers chunk by chunk
// Reported: per-GPU outbound GB/s (bytes / max time over GPUs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_multi tools/p2p_multi.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

struct Ptrs {
  uint4* p[8];
};

// Each CTA owns a contiguous slice of `n` granules; destination/source peer
// chosen per CTA (mode 0) or per 64 KiB block (mode 1, interleaved).
__global__ void __launch_bounds__(512) k_move(Ptrs remote, uint4* local, int npeer, int64_t n, int push,
                                              int interleave) {
  const int64_t per = n / gridDim.x;
  const int64_t base = per * blockIdx.x;
  const int64_t blk = 4096;  // granules = 64 KiB
  for (int64_t b0 = 0; b0 < per; b0 += blk) {
    const int peer = interleave ? (int)((blockIdx.x + b0 / blk) % npeer) : (int)(blockIdx.x % npeer);
    uint4* r = remote.p[peer] + base + b0;
    uint4* l = local + base + b0;
    const int64_t len = per - b0 < blk ? per - b0 : blk;
    for (int64_t i = threadIdx.x; i < len; i += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * blockDim.x < len) v[u] = __ldcg((push ? l : r) + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * blockDim.x < len) __stcg((push ? r : l) + i + u * blockDim.x, v[u]);
    }
  }
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n > 8) n = 8;
  const int64_t bytes = (int64_t)(argc > 1 ? atoll(argv[1]) : 1024) << 20;
  char *src[8], *dst[8];
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int o = 0; o < n; ++o)
      if (o != d) CK(cudaDeviceEnablePeerAccess(o, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    CK(cudaMemset(src[d], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  const char* names[] = {"ring-push", "ring-pull", "a2a-push", "a2a-pull", "a2a-push-i", "a2a-pull-i"};
  const int ctas[] = {16, 32, 64, 148};
  for (int pat = 0; pat < 6; ++pat)
    for (int ci = 0; ci < 4; ++ci) {
      float tmax = 0;
      for (int rep = 0; rep < 3; ++rep) {
        for (int d = 0; d < n; ++d) {
          CK(cudaSetDevice(d));
          Ptrs rp;
          int np = 0;
          if (pat < 2) {  // ring: push to next / pull from prev
            int o = pat == 0 ? (d + 1) % n : (d + n - 1) % n;
            rp.p[np++] = (uint4*)(pat == 0 ? dst[o] : src[o]);
          } else {
            for (int o = 1; o < n; ++o) {
              int peer = (d + o) % n;
              rp.p[np++] = (uint4*)((pat % 2 == 0) ? dst[peer] : src[peer]);
            }
          }
          uint4* loc = (uint4*)((pat % 2 == 0) ? src[d] : dst[d]);
          CK(cudaEventRecord(e0[d], st[d]));
          k_move<<<ctas[ci], 512, 0, st[d]>>>(rp, loc, np, bytes / 16, pat % 2 == 0, pat >= 4);
          CK(cudaEventRecord(e1[d], st[d]));
        }
        tmax = 0;
        for (int d = 0; d < n; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          if (ms > tmax) tmax = ms;
        }
      }
      printf("n=%d %-10s ctas=%3d  %7.1f GB/s per GPU  (%.3f ms)\n", n, names[pat], ctas[ci],
             bytes / (tmax * 1e-3) / 1e9, tmax);
      fflush(stdout);
    }
  return 0;
}
