// ce_ag_micro.cu — can copy engines take the all-gather share of a push while
// SM kernels do the rest, chunk by chunk? (dev tool, 2 GPUs, one process;
// DESIGN §11 item 4). Both GPUs push `bytes` to each other at once:
//   sm     : one 148-CTA kernel of 128-bit stores moves everything
//   ce     : per-chunk cudaMemcpyPeerAsync, each behind a cuStreamWaitValue32
//            on a flag that is already set (the cost of the gating alone)
//   hybrid : the kernel moves a fraction f and, as it finishes its i-th share,
//            raises flag i (release at system scope); the copy-engine stream
//            waits on flag i, then copies chunk i of the rest — the copy
//            engines trail the kernel the way an all-gather trails the
//            reduction that produces its parts.
// GB/s = bytes per direction / time until both streams of both GPUs are done.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_ag_micro tools/ce_ag_micro.cu -lcuda
// ./ce_ag_micro [nchunks=256] [u = ce-only copies without waits]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                     \
    }                                                                               \
  } while (0)
#define CU(x)                                                                       \
  do {                                                                              \
    CUresult r = (x);                                                               \
    if (r != CUDA_SUCCESS) {                                                        \
      const char* m = nullptr;                                                      \
      cuGetErrorString(r, &m);                                                      \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, m ? m : "?");       \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

// The kernel's share is cut into `nchunks` pieces; CTAs claim pieces in order
// and, after the last CTA finishes piece i, flag[i] = epoch (so flag i rises
// roughly when the kernel is i/nchunks of the way through).
__global__ void __launch_bounds__(512) k_push_flags(const uint4* __restrict__ src, uint4* dst, int64_t n16,
                                                    int nchunks, uint32_t* flags, uint32_t* done, uint32_t epoch,
                                                    uint32_t arrivals) {
  const int64_t per = (n16 + nchunks - 1) / nchunks;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t a = c * per, b = (a + per < n16) ? a + per : n16;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += stride)
      __stcg(dst + i, __ldcs(src + i));
    if (flags) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        const uint32_t prev = atomicAdd(done + c, 1u);
        if (prev + 1 == arrivals) {  // last CTA of piece c in this launch (done[] counts all launches)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags + c), "r"(epoch) : "memory");
        }
      }
    }
  }
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  CU(cuInit(0));
  const int64_t bytes = 512ll << 20;
  const int nchunks = argc > 1 ? atoi(argv[1]) : 256;  // 256: 2 MiB per chunk of the whole message
  const bool gate = !(argc > 2 && argv[2][0] == 'u');   // "u": ce-only copies without the waits
  char *a[2], *b[2];
  uint32_t *flags[2], *done[2];
  cudaStream_t s1[2], s2[2];
  cudaEvent_t e0[2], e1[2], e2[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaMalloc(&flags[d], nchunks * sizeof(uint32_t)));
    CK(cudaMalloc(&done[d], nchunks * sizeof(uint32_t)));
    CK(cudaMemset(flags[d], 0, nchunks * sizeof(uint32_t)));
    CK(cudaMemset(done[d], 0, nchunks * sizeof(uint32_t)));
    CK(cudaStreamCreateWithFlags(&s1[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaEventCreate(&e2[d]));
  }
  uint32_t epoch = 0, flagged[2] = {0, 0};
  const double fracs[] = {1.0, 0.0, 0.75, 0.6, 0.5};
  for (double f : fracs) {
    // SM share [0, xs), CE share [xs, bytes) in nchunks pieces matched to the kernel's pieces
    const int64_t xs = ((int64_t)(bytes * f)) & ~(int64_t)(nchunks * 16 - 1);
    const int64_t ys = bytes - xs;
    const int64_t cper = ys / nchunks;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      ++epoch;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], s1[d]));
        CK(cudaStreamWaitEvent(s2[d], e0[d], 0));
        if (xs) {
          if (ys) ++flagged[d];
          k_push_flags<<<148, 512, 0, s1[d]>>>((const uint4*)a[d], (uint4*)b[1 - d], xs / 16, nchunks,
                                               ys ? flags[d] : nullptr, done[d], epoch, flagged[d] * 148u);
        }
        for (int c = 0; ys && c < nchunks; ++c) {
          // ce only: wait for a value every flag already holds (the gating's own cost)
          if (gate || xs)
            CU(cuStreamWaitValue32((CUstream)s2[d], (CUdeviceptr)(flags[d] + c), xs ? epoch : 0u,
                                   CU_STREAM_WAIT_VALUE_GEQ));
          const int64_t off = xs + c * cper;
          const int64_t len = (c == nchunks - 1) ? bytes - off : cper;
          CK(cudaMemcpyPeerAsync(b[1 - d] + off, 1 - d, a[d] + off, d, len, s2[d]));
        }
        CK(cudaEventRecord(e2[d], s2[d]));
        CK(cudaStreamWaitEvent(s1[d], e2[d], 0));
        CK(cudaEventRecord(e1[d], s1[d]));
      }
      float worst = 0;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        if (ms > worst) worst = ms;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    const char* mode = f == 1.0 ? "sm only" : (f == 0.0 ? (gate ? "ce only, gated copies" : "ce only, plain copies")
                                                           : "hybrid (ce trails sm)");
    printf("bi 512 MiB  %4d chunks  sm-fraction %.2f  %-22s: %7.1f GB/s per direction (%.3f ms)\n", nchunks, f, mode,
           bytes / (best * 1e-3) / 1e9, best);
    fflush(stdout);
  }
  // data check of the last run: b on each GPU equals the other GPU's a (memset 1)
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    unsigned char h[4];
    CK(cudaMemcpy(h, b[d] + bytes - 4, 4, cudaMemcpyDeviceToHost));
    if (h[0] != 1 || h[3] != 1) printf("GPU %d: destination not written\n", d);
  }
  return 0;
}
