// fence_micro.cu — cost of a release fence on B200 (dev tool, 2 GPUs, one process).
//
// Each of C CTAs on GPU 0: lane 0 of warp 0 repeats R times
//     [store `job` bytes to GPU 1 (its own slice, 128-bit st.global, whole warp)]
//     t0 = globaltimer; fence.acq_rel.{sys|gpu}; t1 = globaltimer
// while warps 1..W of the CTA keep streaming 128-bit stores to GPU 1 (background
// traffic, like the consumer warps of the lane kernel). Reported: mean fence time
// (ns) over all CTAs and repetitions, and the background store bandwidth.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fence_micro tools/fence_micro.cu
// tools/fence_micro   (prints one line per configuration)
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

__device__ __forceinline__ uint64_t now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// out[blockIdx] = total fence ns; bg[blockIdx] = background bytes stored
__global__ void k(uint4* peer, int64_t slice, int job, int reps, int sys, int bg_warps, volatile int* stop,
                  unsigned long long* out, unsigned long long* bgb) {
  uint4* base = peer + (int64_t)blockIdx.x * slice;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint4 v = make_uint4(blockIdx.x, threadIdx.x, 1, 2);
  if (warp == 0) {
    uint64_t acc = 0;
    const int per = job / 16;  // granules per job
    for (int r = 0; r < reps; ++r) {
      for (int i = lane; i < per; i += 32) __stcg(base + (r * per + i) % (slice / 2), v);
      __syncwarp();
      if (lane == 0) {
        const uint64_t t0 = now();
        if (sys)
          asm volatile("fence.acq_rel.sys;" ::: "memory");
        else
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        acc += now() - t0;
      }
      __syncwarp();
    }
    if (lane == 0) {
      out[blockIdx.x] = acc;
      if (blockIdx.x == 0) *stop = 1;
    }
    return;
  }
  if (warp > bg_warps) return;
  uint64_t n = 0;
  uint4* b2 = base + slice / 2;
  const int64_t span = slice / 2;
  for (int64_t i = (warp - 1) * 32 + lane;; i += bg_warps * 32) {
    __stcg(b2 + (i % span), v);
    n += 16;
    if ((i & 1023) < bg_warps * 32 && *stop) break;
  }
  atomicAdd(&bgb[blockIdx.x], (unsigned long long)n);
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  const int maxC = 148;
  const int64_t slice = 1 << 20;  // granules per CTA (16 MiB)
  uint4* peer;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&peer, (size_t)maxC * slice * 16));
  CK(cudaSetDevice(0));
  unsigned long long *out, *bgb;
  int* stop;
  CK(cudaMalloc(&out, maxC * 8));
  CK(cudaMalloc(&bgb, maxC * 8));
  CK(cudaMalloc(&stop, 4));
  unsigned long long h[maxC], hb[maxC];
  struct Cfg {
    int C, job, sys, bg;
  } cfgs[] = {{1, 0, 1, 0},       {1, 0, 0, 0},       {1, 32768, 1, 0},   {1, 32768, 0, 0},
              {148, 0, 1, 0},     {148, 0, 0, 0},     {148, 32768, 1, 0}, {148, 32768, 0, 0},
              {148, 4096, 1, 0},  {148, 32768, 1, 6}, {148, 32768, 0, 6}, {148, 4096, 1, 6},
              {16, 32768, 1, 6},  {32, 32768, 1, 0},  {64, 32768, 1, 0},  {1, 32768, 1, 6}};
  printf("C job_bytes scope bg_warps | mean_fence_us | bg_GBps\n");
  for (auto& c : cfgs) {
    const int reps = 200;
    CK(cudaMemset(out, 0, maxC * 8));
    CK(cudaMemset(bgb, 0, maxC * 8));
    CK(cudaMemset(stop, 0, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    k<<<c.C, 32 * (1 + 6)>>>(peer, slice, c.job, reps, c.sys, c.bg, stop, out, bgb);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaMemcpy(h, out, c.C * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb, bgb, c.C * 8, cudaMemcpyDeviceToHost));
    double tot = 0, bytes = 0;
    for (int i = 0; i < c.C; ++i) tot += h[i], bytes += hb[i];
    printf("%3d %6d %s %d | %8.3f | %7.1f\n", c.C, c.job, c.sys ? "sys" : "gpu", c.bg, tot / c.C / reps / 1e3,
           bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
