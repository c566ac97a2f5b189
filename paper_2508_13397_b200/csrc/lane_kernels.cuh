// lane_kernels.cuh — sm_100a kernels of the k-split multi-lane allreduce.
//
// One persistent kernel per round runs all three phases of Alg. 2
// for every k-slice (§3.1.2, P L364-373):
//
//   A  phase-1 push   : GPU (a,h) stores group part g of its sendbuf into
//                       (a,g)'s phase-1 inbox S1 over NVLink        (P L243)
//   B  phase-1 reduce : (a,g) sums the G contributions in ascending h
//                       (fp32 accumulate, one rounding) and stores lane
//                       sub-part b of the result into (b,g)'s S2   (P L243, L246)
//   C  phase-2 reduce : (a,g) sums the N contributions to its sub-part in
//                       ascending b -> R (its lane result) and recvbuf (P L246)
//   D  phase-2 gather : (a,g) loads the other lane members' sub-parts from
//                       their R over NVLink -> own R and recvbuf   (P L246)
//   E  phase-3 gather : (a,g) loads group part h from (a,h)'s R over NVLink
//                       -> recvbuf                                  (P L248)
//
// Each CTA group l (one per k-slice; the paper's process l_r) has C CTAs;
// CTA j owns chunks j, j+C, ... of its slice on every rank and runs phase
// A for all its chunks, then B, C, D, E. A wait in phase X for chunk c only
// needs peers' phase < X for chunk c, which the peers' CTA j reaches without
// waiting on us: no cyclic wait as long as every CTA is resident (grid <=
// co-resident capacity; cooperative launch in emulated mode).
//
// Cross-GPU ordering: data stores -> __syncthreads -> one thread per peer
// st.release.sys(flag = epoch); the waiter ld.acquire.sys(flag) >= epoch ->
// __syncthreads -> data loads (L2-only .cg loads for data other GPUs wrote).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_plan.h"

namespace lane {

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release pattern for several flags: ONE fence.acq_rel.sys, then relaxed
// strong stores (PTX memory model: a fence.release-or-stronger followed by a
// strong write is a release pattern). st.release.sys per flag would emit a
// MEMBAR.SYS per flag.
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Programmatic dependent launch (PDL). The host launches every multi-GPU call
// with cudaLaunchAttributeProgrammaticStreamSerialization, so the next grid
// in the stream may be scheduled before this one has finished. Each kernel
// first waits until the previous grid in the stream has completed and its
// memory operations are visible (griddepcontrol.wait; a no-op for a launch
// without a programmatic dependency), so stream order is kept for every
// access, then allows the next grid to launch (launch_dependents): the next
// call's CTAs are dispatched onto SMs as this call's CTAs exit and wait there,
// instead of paying the launch latency after the last CTA is gone.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns();

// The launch's epoch (the generation of its flags, packets and inbox parity
// set), set once per CTA by launch_prologue; every device-side use reads it
// from here (cur_epoch()).
//  - eager launches: the host's counter (LaneParams::epoch); the first CTA of
//    each local rank also stores epoch + 1 as the rank's NEXT epoch in device
//    memory, so the device word always follows the host;
//  - CUDA graph launches (LaneParams::dev_epoch, sticky once a comm was
//    captured): a replayed graph carries the epoch it was captured with, so
//    the launch takes the NEXT epoch from device memory instead, and the last
//    CTA of the rank to arrive advances it (atomic arrival count,
//    acquire-release: every CTA read the word before the last one moves it).
//    Every launch therefore still gets epoch previous + 1 on every rank.
__shared__ uint32_t g_epoch;
__device__ __forceinline__ uint32_t cur_epoch() { return g_epoch; }

__device__ __noinline__ uint32_t epoch_from_device(const LaneParams& p, int rank, int per_rank) {
  uint32_t* const st = p.epoch_dev + (int64_t)rank * 16;
  uint32_t e, t;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(e) : "l"(st) : "memory");
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(st + 1) : "memory");
  if ((int)t == per_rank - 1) {  // the last CTA of this rank to read it: advance for the next launch
    st[1] = 0u;
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(st), "r"(e + 1u) : "memory");
  }
  return e;
}

// Zero the chunk-claim counters of the next launch's parity (lane_plan.h).
__device__ __noinline__ void claims_reset(const LaneParams& p, int rank) {
  const int par = (int)((cur_epoch() + 1u) & 1u);
  for (int l = threadIdx.x; l < p.k; l += blockDim.x) p.claims[claim_index(rank, par, l)] = 0u;
}

// Every kernel of a comm starts here (all threads): PDL wait (pdl_enter), the
// launch's epoch (g_epoch), then the first CTA of each local rank zeroes the
// next launch's chunk-claim counters. Returns the time the CTA began, before
// the wait (trace: how early PDL dispatched it).
__device__ __forceinline__ uint64_t launch_prologue(const LaneParams& p) {
  const uint64_t t = globaltimer_ns();
  pdl_enter();
  const int per_rank = p.k * p.C;
  const int rank = p.rank0 + (int)(blockIdx.x / per_rank);
  if (threadIdx.x == 0) {
    if (p.dev_epoch) {
      g_epoch = epoch_from_device(p, rank, per_rank);
    } else {
      g_epoch = p.epoch;
      if (p.epoch_dev != nullptr && blockIdx.x % per_rank == 0) p.epoch_dev[(int64_t)rank * 16] = p.epoch + 1u;
    }
  }
  __syncthreads();
  if (p.claims != nullptr && blockIdx.x % per_rank == 0) claims_reset(p, rank);
  return t;
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// data movement: 128-bit, L2-only loads (data written by other GPUs or by
// other launches is never served from a stale L1 line)
__device__ __forceinline__ uint4 ld_cg(const uint4* p) { return __ldcg(p); }
// sendbuf is read once: streaming
__device__ __forceinline__ uint4 ld_cs(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_cg(uint4* p, const uint4& v) { __stcg(p, v); }
__device__ __forceinline__ void st_cs(uint4* p, const uint4& v) { __stcs(p, v); }

// ------------------------------------------------------------------ element ops
// DT: 0 int32 (wrap-around, R#9), 1 float32, 2 bfloat16 (fp32 accumulate,
// RNE once per phase, R#8). Acc holds one 16-byte granule widened.
template <int DT>
struct Ops;

template <>
struct Ops<0> {
  struct Acc {
    uint32_t v[4];
  };
  static __device__ __forceinline__ void init(Acc& a, const uint4& x) {
    a.v[0] = x.x; a.v[1] = x.y; a.v[2] = x.z; a.v[3] = x.w;
  }
  static __device__ __forceinline__ void add(Acc& a, const uint4& x) {
    a.v[0] += x.x; a.v[1] += x.y; a.v[2] += x.z; a.v[3] += x.w;
  }
  static __device__ __forceinline__ uint4 narrow(const Acc& a) {
    return make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
  }
};

template <>
struct Ops<1> {
  struct Acc {
    float v[4];
  };
  static __device__ __forceinline__ void init(Acc& a, const uint4& x) {
    a.v[0] = __uint_as_float(x.x); a.v[1] = __uint_as_float(x.y);
    a.v[2] = __uint_as_float(x.z); a.v[3] = __uint_as_float(x.w);
  }
  static __device__ __forceinline__ void add(Acc& a, const uint4& x) {
    a.v[0] = __fadd_rn(a.v[0], __uint_as_float(x.x));
    a.v[1] = __fadd_rn(a.v[1], __uint_as_float(x.y));
    a.v[2] = __fadd_rn(a.v[2], __uint_as_float(x.z));
    a.v[3] = __fadd_rn(a.v[3], __uint_as_float(x.w));
  }
  static __device__ __forceinline__ uint4 narrow(const Acc& a) {
    return make_uint4(__float_as_uint(a.v[0]), __float_as_uint(a.v[1]),
                      __float_as_uint(a.v[2]), __float_as_uint(a.v[3]));
  }
};

template <>
struct Ops<2> {
  struct Acc {
    float v[8];
  };
  static __device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
  static __device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
  static __device__ __forceinline__ void init(Acc& a, const uint4& x) {
    a.v[0] = lo(x.x); a.v[1] = hi(x.x); a.v[2] = lo(x.y); a.v[3] = hi(x.y);
    a.v[4] = lo(x.z); a.v[5] = hi(x.z); a.v[6] = lo(x.w); a.v[7] = hi(x.w);
  }
  static __device__ __forceinline__ void add(Acc& a, const uint4& x) {
    a.v[0] = __fadd_rn(a.v[0], lo(x.x)); a.v[1] = __fadd_rn(a.v[1], hi(x.x));
    a.v[2] = __fadd_rn(a.v[2], lo(x.y)); a.v[3] = __fadd_rn(a.v[3], hi(x.y));
    a.v[4] = __fadd_rn(a.v[4], lo(x.z)); a.v[5] = __fadd_rn(a.v[5], hi(x.z));
    a.v[6] = __fadd_rn(a.v[6], lo(x.w)); a.v[7] = __fadd_rn(a.v[7], hi(x.w));
  }
  static __device__ __forceinline__ uint32_t pack(float l, float h) {
    __nv_bfloat162 b = __floats2bfloat162_rn(l, h);  // cvt.rn.bf16x2.f32: RNE
    return *reinterpret_cast<uint32_t*>(&b);
  }
  static __device__ __forceinline__ uint4 narrow(const Acc& a) {
    return make_uint4(pack(a.v[0], a.v[1]), pack(a.v[2], a.v[3]), pack(a.v[4], a.v[5]),
                      pack(a.v[6], a.v[7]));
  }
};

// ------------------------------------------------------------------ tail
// Only the message's last granule can be partial (tail_elems < q); only
// sendbuf reads and recvbuf writes ever touch it (scratch holds whole,
// zero-padded granules).
// (fully unrolled over the 8 halfwords with constant register indices: a
// byte-addressed view of a local uint4 would live on the stack)
__device__ __forceinline__ uint4 load_partial(const uint4* p, int nbytes) {
  const uint16_t* s = reinterpret_cast<const uint16_t*>(p);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (2 * i < nbytes) w[i >> 1] |= (uint32_t)s[i] << (16 * (i & 1));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void store_partial(uint4* p, const uint4& v, int nbytes) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint16_t* d = reinterpret_cast<uint16_t*>(p);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (2 * i < nbytes) d[i] = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
}

struct Msg {
  const uint4* send;  // rank's sendbuf, granule-indexed
  uint4* recv;        // rank's recvbuf, granule-indexed
  int64_t partial_g;  // granule index of a partial last granule, or -1
  int partial_bytes;
};

// The message's one partial granule: out of line (cold), so the unrolled
// halfword code does not compete for registers in the kernels' hot loops;
// arguments and result travel by value (registers), nothing by reference.
__device__ __noinline__ uint4 load_partial_cold(const uint4* p, int nbytes) { return load_partial(p, nbytes); }
__device__ __noinline__ void store_partial_cold(uint4* p, uint4 v, int nbytes) { store_partial(p, v, nbytes); }

__device__ __forceinline__ uint4 load_x(const Msg& m, int64_t gi) {
  if (gi == m.partial_g) return load_partial_cold(m.send + gi, m.partial_bytes);
  return ld_cs(m.send + gi);
}

__device__ __forceinline__ void store_out(const Msg& m, int64_t gi, const uint4& v) {
  if (gi == m.partial_g) {
    store_partial_cold(m.recv + gi, v, m.partial_bytes);
    return;
  }
  st_cs(m.recv + gi, v);
}

// ------------------------------------------------------------------ waits
// Threads t < n poll flag idx(t) (skipping `skip`) until >= epoch; returns
// false on timeout/abort (block-uniform).
template <class IdxF>
__device__ __forceinline__ bool wait_flags(const LaneParams& p, const uint32_t* flags, int n,
                                           int skip, IdxF idx) {
  int fail = 0;
  const int t = threadIdx.x;
  if (t < n && t != skip) {
    const uint32_t* f = flags + idx(t);
    if ((int32_t)(ld_acquire_sys(f) - cur_epoch()) < 0) {
      uint64_t t0 = globaltimer_ns();
      for (uint32_t it = 1;; ++it) {
        if ((int32_t)(ld_acquire_sys(f) - cur_epoch()) >= 0) break;
        if ((it & 63u) == 0) {
          if (*reinterpret_cast<volatile uint32_t*>(p.abort_flag)) {
            fail = 1;
            break;
          }
          if (globaltimer_ns() - t0 > p.timeout_ns) {
            atomicExch(p.abort_flag, 1u);
            *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_TIMEOUT);
            __threadfence_system();
            fail = 1;
            break;
          }
        }
      }
    }
  }
  return __syncthreads_or(fail) == 0;
}

// ------------------------------------------------------------------ kernel
struct ChunkGeo {
  int64_t id;   // chunk index within the round (flag / slot index)
  int64_t g0;   // message granule of the chunk's first granule
  int64_t len;  // granules
};

__device__ __forceinline__ uint4* s1_slot(const LaneParams& p, const RankMem& m, int slot,
                                          int64_t chunk) {
  return reinterpret_cast<uint4*>(m.s1) + ((int64_t)slot * p.cap + chunk) * p.sg;
}
__device__ __forceinline__ uint4* s2_slot(const LaneParams& p, const RankMem& m, int slot,
                                          int64_t chunk) {
  return reinterpret_cast<uint4*>(m.s2) + ((int64_t)slot * p.cap + chunk) * p.su;
}
__device__ __forceinline__ uint4* r_slot(const LaneParams& p, const RankMem& m, int64_t chunk) {
  return reinterpret_cast<uint4*>(m.r) + chunk * p.sg;
}

constexpr int kUnroll = 4;     // granules in flight per thread in copy phases
constexpr int kRedUnroll = 2;  // granules per thread in reduce phases
constexpr int kFanBatch = 4;   // sources loaded together in reduce phases

template <int DT>
__global__ void __launch_bounds__(512, 1) lane_allreduce_kernel(const __grid_constant__ LaneParams p) {
  launch_prologue(p);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int rank = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int j = (int)(blockIdx.x % p.C);
  const int G = p.G, N = p.N;
  const int a = rank / G, g = rank % G;
  const RankMem& me = p.rk[rank];
  const uint32_t ep = cur_epoch();
  const int tid = threadIdx.x, nthr = blockDim.x;

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(me.send);
  msg.recv = reinterpret_cast<uint4*>(me.recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sl = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  auto geo = [&](int64_t c) {
    ChunkGeo ch;
    ch.id = cb + c;
    ch.g0 = p.round_g0 + sl.start + c * p.cg;
    int64_t rest = sl.len - c * p.cg;
    ch.len = rest < p.cg ? rest : p.cg;
    return ch;
  };

  // ---------------- A: phase-1 push (intra-node reduce-scatter, send side)
  if (G > 1) {
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      for (int t = 1; t < G; ++t) {
        const int gd = (g + t) % G;  // destination GPU in the node
        const Span gp = rf_split(ch.len, G, gd);
        const RankMem& dm = p.rk[a * G + gd];
        uint4* dst = s1_slot(p, dm, g < gd ? g : g - 1, ch.id);
        const int64_t gbase = ch.g0 + gp.start;
        for (int64_t i0 = tid; i0 < gp.len; i0 += kUnroll * nthr) {
          uint4 v[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < gp.len) v[u] = load_x(msg, gbase + i);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < gp.len) st_cg(dst + i, v[u]);
          }
        }
      }
      __syncthreads();
      if (tid < G - 1) {
        const int gd = (g + 1 + tid) % G;
        st_release_sys(p.rk[a * G + gd].flags + f1_idx(p, g, ch.id), ep);
      }
    }
  }

  // ---------------- B: phase-1 reduce + phase-2 reduce-scatter push
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    if (G > 1 && !wait_flags(p, me.flags, G, g, [&](int h) { return f1_idx(p, h, ch.id); }))
      return;
    const Span gp = rf_split(ch.len, G, g);
    const int64_t gbase = ch.g0 + gp.start;
    const uint4* s1c = s1_slot(p, me, 0, ch.id);  // slot 0 of this chunk
    const int64_t s1stride = p.cap * p.sg;         // granules between slots
    for (int t = 1; t <= N; ++t) {
      const int b = (a + t) % N;  // remote sub-parts first, own sub-part last
      const Span up = rf_split(gp.len, N, b);
      uint4* dst = s2_slot(p, p.rk[b * G + g], a, ch.id);
      for (int64_t i0 = tid; i0 < up.len; i0 += kRedUnroll * nthr) {
        typename O::Acc acc[kRedUnroll];
        for (int h0 = 0; h0 < G; h0 += kFanBatch) {
          uint4 x[kRedUnroll][kFanBatch];
#pragma unroll
          for (int u = 0; u < kRedUnroll; ++u) {
            const int64_t ii = i0 + (int64_t)u * nthr;
#pragma unroll
            for (int hh = 0; hh < kFanBatch; ++hh) {
              const int h = h0 + hh;
              if (h < G && ii < up.len) {
                const int64_t gi = up.start + ii;
                x[u][hh] = (h == g) ? load_x(msg, gbase + gi)
                                    : ld_cg(s1c + (int64_t)(h < g ? h : h - 1) * s1stride + gi);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < kRedUnroll; ++u) {
#pragma unroll
            for (int hh = 0; hh < kFanBatch; ++hh) {
              const int h = h0 + hh;
              if (h < G && i0 + u * nthr < up.len) {
                if (h == 0)
                  O::init(acc[u], x[u][hh]);  // canonical order: h = 0, 1, ..., G-1
                else
                  O::add(acc[u], x[u][hh]);
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u)
          if (i0 + u * nthr < up.len) st_cg(dst + i0 + (int64_t)u * nthr, O::narrow(acc[u]));
      }
    }
    __syncthreads();
    if (tid < N - 1) {
      const int b = (a + 1 + tid) % N;
      st_release_sys(p.rk[b * G + g].flags + f2_idx(p, a, ch.id), ep);
    }
  }

  // ---------------- C: phase-2 reduce (lane reduce-scatter, owner side)
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    if (N > 1 && !wait_flags(p, me.flags, N, a, [&](int b) { return f2_idx(p, b, ch.id); }))
      return;
    const Span gp = rf_split(ch.len, G, g);
    const Span up = rf_split(gp.len, N, a);
    const uint4* s2c = s2_slot(p, me, 0, ch.id);
    const int64_t s2stride = p.cap * p.su;
    uint4* rdst = r_slot(p, me, ch.id) + up.start;
    const int64_t obase = ch.g0 + gp.start + up.start;
    for (int64_t i0 = tid; i0 < up.len; i0 += kRedUnroll * nthr) {
      typename O::Acc acc[kRedUnroll];
      for (int b0 = 0; b0 < N; b0 += kFanBatch) {
        uint4 x[kRedUnroll][kFanBatch];
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) {
          const int64_t ii = i0 + (int64_t)u * nthr;
#pragma unroll
          for (int bb = 0; bb < kFanBatch; ++bb)
            if (b0 + bb < N && ii < up.len) x[u][bb] = ld_cg(s2c + (int64_t)(b0 + bb) * s2stride + ii);
        }
#pragma unroll
        for (int u = 0; u < kRedUnroll; ++u) {
#pragma unroll
          for (int bb = 0; bb < kFanBatch; ++bb) {
            const int b = b0 + bb;
            if (b < N && i0 + u * nthr < up.len) {
              if (b == 0)
                O::init(acc[u], x[u][bb]);  // canonical order: b = 0, 1, ..., N-1
              else
                O::add(acc[u], x[u][bb]);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kRedUnroll; ++u) {
        const int64_t i = i0 + (int64_t)u * nthr;
        if (i < up.len) {
          const uint4 v = O::narrow(acc[u]);
          st_cg(rdst + i, v);
          store_out(msg, obase + i, v);
        }
      }
    }
    __syncthreads();
    if (N > 1) {
      if (tid < N - 1) {
        const int b = (a + 1 + tid) % N;
        st_release_sys(p.rk[b * G + g].flags + f3_idx(p, a, ch.id), ep);
      }
    } else if (tid < G - 1) {  // N == 1: R is complete, release phase 3
      const int h = (g + 1 + tid) % G;
      st_release_sys(p.rk[a * G + h].flags + f4_idx(p, g, ch.id), ep);
    }
  }

  // ---------------- D: phase-2 allgather (pull lane members' results)
  if (N > 1) {
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      if (!wait_flags(p, me.flags, N, a, [&](int b) { return f3_idx(p, b, ch.id); })) return;
      const Span gp = rf_split(ch.len, G, g);
      for (int t = 1; t < N; ++t) {
        const int b = (a + t) % N;
        const Span up = rf_split(gp.len, N, b);
        const uint4* src = r_slot(p, p.rk[b * G + g], ch.id) + up.start;
        uint4* rdst = r_slot(p, me, ch.id) + up.start;
        const int64_t obase = ch.g0 + gp.start + up.start;
        for (int64_t i0 = tid; i0 < up.len; i0 += kUnroll * nthr) {
          uint4 v[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < up.len) v[u] = ld_cg(src + i);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < up.len) {
              if (G > 1) st_cg(rdst + i, v[u]);
              store_out(msg, obase + i, v[u]);
            }
          }
        }
      }
      __syncthreads();
      if (tid < G - 1) {
        const int h = (g + 1 + tid) % G;
        st_release_sys(p.rk[a * G + h].flags + f4_idx(p, g, ch.id), ep);
      }
    }
  }

  // ---------------- E: phase-3 allgather (pull node peers' group parts)
  if (G > 1) {
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      if (!wait_flags(p, me.flags, G, g, [&](int h) { return f4_idx(p, h, ch.id); })) return;
      for (int t = 1; t < G; ++t) {
        const int h = (g + t) % G;
        const Span gp = rf_split(ch.len, G, h);
        const uint4* src = r_slot(p, p.rk[a * G + h], ch.id);
        const int64_t obase = ch.g0 + gp.start;
        for (int64_t i0 = tid; i0 < gp.len; i0 += kUnroll * nthr) {
          uint4 v[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < gp.len) v[u] = ld_cg(src + i);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            int64_t i = i0 + (int64_t)u * nthr;
            if (i < gp.len) store_out(msg, obase + i, v[u]);
          }
        }
      }
    }
  }
}

// P == 1: the allreduce of one rank is a copy (no-op when in place).
__global__ void __launch_bounds__(512) lane_copy_kernel(const uint4* __restrict__ src,
                                                        uint4* __restrict__ dst, int64_t ng,
                                                        int tail_bytes) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t full = tail_bytes ? ng - 1 : ng;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < full; i += stride)
    st_cs(dst + i, ld_cs(src + i));
  if (tail_bytes && blockIdx.x == 0 && threadIdx.x == 0)
    store_partial(dst + ng - 1, load_partial(src + ng - 1, tail_bytes), tail_bytes);
}

}  // namespace lane
