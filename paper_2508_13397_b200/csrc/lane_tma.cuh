// lane_tma.cuh — TMA bulk-copy engine for the multi-lane allreduce (sm_100a).
//
// Same protocol, partition, flags and canonical reduction order as
// lane_kernels.cuh (which documents phases A-E, Alg. 2 L218-251 and
// §3.1.2); only the data movement differs. Every phase of a chunk is
// a list of "jobs" (up to 16 sources in canonical order -> 1 or 2
// destinations, local or peer memory):
//
//   A(c, gd)  x[part gd]                     -> S1 of (a,gd)          release F1
//   B(c, b)   x[part g], S1[h] (h != g)      -> S2 of (b,g) (N>1)     release F2
//             (sum over h ascending)          -> R + recvbuf (N==1)   release F4
//   C(c)      S2[b], b = 0..N-1 (ascending)  -> R + recvbuf           release F3
//   D(c, b)   R of (b,g) [sub-part b]        -> R (G>1) + recvbuf     release F4 (last)
//   E(c, h)   R of (a,h) [part h]            -> recvbuf
//
// Warp specialisation inside a CTA (one CTA per SM, 4-stage smem ring):
//   warp 0, lane 0 : producer — acquires the job's flags, then streams its
//                    tiles into the ring with cp.async.bulk (global -> smem,
//                    completion on the stage's "full" mbarrier). Peer
//                    addresses are read straight over NVLink by the TMA unit.
//   warps 1..W     : consumers — reduce the tile's sources in shared memory
//                    (fp32 accumulate, canonical order, in place into slot 0);
//   consumer 0     : storer — cp.async.bulk smem -> global (local or peer),
//                    frees ring stages, and after a job completes
//                    (wait_group 0) releases its flags with st.release.sys.
//
// Schedule: CTA j of CTA group l owns chunks j, j+C, ... of slice l; at
// step s it runs A(c_s), B(c_{s-1}), C(c_{s-2}), D(c_{s-3}), E(c_{s-4}) — a
// wavefront, so every wait is on work the peer's CTA j did one step earlier
// and each step mixes push, pull and local traffic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_kernels.cuh"
#include "lane_plan.h"

namespace lane {
namespace tma {

constexpr int kStages = 4;
constexpr int kStageBytes = 48 * 1024;
constexpr int kStageGranules = kStageBytes / 16;
constexpr int kConsumerWarps = 7;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kMaxSrc = LANE_MAX_RANKS;
constexpr int kSmemBytes = kStages * kStageBytes + 2 * kStages * 8 + 16;

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_addr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// ------------------------------------------------------------------ jobs
struct Job {
  int nsrc, ndst, x_src, recv_dst;  // x_src / recv_dst: index or -1
  int nwait, nrel;
  int64_t len;  // granules
  int64_t m0;   // message granule of the job's first granule
  const uint4* src[kMaxSrc];
  uint4* dst[2];
  const uint32_t* wait[kMaxSrc];
  uint32_t* rel[kMaxSrc];
};

struct Ctx {
  const LaneParams* p;
  int rank, a, g, N, G;
  const RankMem* me;
  Msg msg;
};

__device__ __forceinline__ int njobs(const Ctx& x, int ph) {
  switch (ph) {
    case 0: return x.G - 1;
    case 1: return x.N;
    case 2: return x.N > 1 ? 1 : 0;
    case 3: return x.N - 1;
    default: return x.G - 1;
  }
}

// Job t of phase ph (0=A .. 4=E) for chunk ch.
__device__ void make_job(const Ctx& x, int ph, const ChunkGeo& ch, int t, Job& J) {
  const LaneParams& p = *x.p;
  const int a = x.a, g = x.g, N = x.N, G = x.G;
  J.nsrc = 1;
  J.ndst = 1;
  J.x_src = -1;
  J.recv_dst = -1;
  J.nwait = 0;
  J.nrel = 0;
  const Span gp = rf_split(ch.len, G, g);
  if (ph == 0) {  // A: push part gd of my sendbuf into (a,gd)'s S1
    const int gd = (g + 1 + t) % G;
    const Span pd = rf_split(ch.len, G, gd);
    const RankMem& dm = p.rk[a * G + gd];
    J.len = pd.len;
    J.m0 = ch.g0 + pd.start;
    J.src[0] = x.msg.send + J.m0;
    J.x_src = 0;
    J.dst[0] = s1_slot(p, dm, g < gd ? g : g - 1, ch.id);
    J.rel[J.nrel++] = dm.flags + f1_idx(p, g, ch.id);
  } else if (ph == 1) {  // B: reduce part g over the node, sub-part b
    const int b = (a + 1 + t) % N;  // own sub-part last
    const Span up = rf_split(gp.len, N, b);
    J.len = up.len;
    J.m0 = ch.g0 + gp.start + up.start;
    J.nsrc = G;
    for (int h = 0; h < G; ++h)
      J.src[h] = (h == g) ? x.msg.send + J.m0 : s1_slot(p, *x.me, h < g ? h : h - 1, ch.id) + up.start;
    J.x_src = g;
    if (t == 0)
      for (int h = 0; h < G; ++h)
        if (h != g) J.wait[J.nwait++] = x.me->flags + f1_idx(p, h, ch.id);
    if (N > 1) {
      const RankMem& dm = p.rk[b * G + g];
      J.dst[0] = s2_slot(p, dm, a, ch.id);
      J.rel[J.nrel++] = dm.flags + f2_idx(p, a, ch.id);
    } else {  // N == 1: the node sum is the final value of part g
      J.ndst = 2;
      J.dst[0] = r_slot(p, *x.me, ch.id) + up.start;
      J.dst[1] = x.msg.recv + J.m0;
      J.recv_dst = 1;
      for (int h = 0; h < G; ++h)
        if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    }
  } else if (ph == 2) {  // C: reduce my sub-part over the lane
    const Span up = rf_split(gp.len, N, a);
    J.len = up.len;
    J.m0 = ch.g0 + gp.start + up.start;
    J.nsrc = N;
    for (int b = 0; b < N; ++b) {
      J.src[b] = s2_slot(p, *x.me, b, ch.id);
      J.wait[J.nwait++] = x.me->flags + f2_idx(p, b, ch.id);
    }
    J.ndst = 2;
    J.dst[0] = r_slot(p, *x.me, ch.id) + up.start;
    J.dst[1] = x.msg.recv + J.m0;
    J.recv_dst = 1;
    for (int b = 0; b < N; ++b)
      if (b != a) J.rel[J.nrel++] = p.rk[b * G + g].flags + f3_idx(p, a, ch.id);
  } else if (ph == 3) {  // D: pull lane member b's sub-part
    const int b = (a + 1 + t) % N;
    const Span up = rf_split(gp.len, N, b);
    J.len = up.len;
    J.m0 = ch.g0 + gp.start + up.start;
    J.src[0] = r_slot(p, p.rk[b * G + g], ch.id) + up.start;
    J.wait[J.nwait++] = x.me->flags + f3_idx(p, b, ch.id);
    if (G > 1) {
      J.ndst = 2;
      J.dst[0] = r_slot(p, *x.me, ch.id) + up.start;
      J.dst[1] = x.msg.recv + J.m0;
      J.recv_dst = 1;
      if (t == N - 2)
        for (int h = 0; h < G; ++h)
          if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    } else {
      J.dst[0] = x.msg.recv + J.m0;
      J.recv_dst = 0;
    }
  } else {  // E: pull node peer h's part
    const int h = (g + 1 + t) % G;
    const Span ph_ = rf_split(ch.len, G, h);
    J.len = ph_.len;
    J.m0 = ch.g0 + ph_.start;
    J.src[0] = r_slot(p, p.rk[a * G + h], ch.id);
    J.wait[J.nwait++] = x.me->flags + f4_idx(p, h, ch.id);
    J.dst[0] = x.msg.recv + J.m0;
    J.recv_dst = 0;
  }
}

__device__ __forceinline__ int64_t tile_granules(int nsrc) {
  return (int64_t)(kStageGranules / nsrc);
}
__device__ __forceinline__ int64_t n_tiles(const Job& J) {
  const int64_t T = tile_granules(J.nsrc);
  return J.len > 0 ? (J.len + T - 1) / T : 1;  // empty jobs still take one (empty) tile
}

// Acquire-wait one flag (producer thread). false on timeout / abort.
__device__ bool wait_one(const LaneParams& p, const uint32_t* f) {
  if ((int32_t)(ld_acquire_sys(f) - p.epoch) >= 0) return true;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t it = 1;; ++it) {
    if ((int32_t)(ld_acquire_sys(f) - p.epoch) >= 0) return true;
    if ((it & 63u) == 0) {
      if (*reinterpret_cast<volatile uint32_t*>(p.abort_flag)) return false;
      if (globaltimer_ns() - t0 > p.timeout_ns) {
        atomicExch(p.abort_flag, 1u);
        *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_TIMEOUT);
        __threadfence_system();
        return false;
      }
    }
  }
}

// Iterate the CTA's jobs in wavefront order; f(job) returns false to stop.
template <class F>
__device__ __forceinline__ void for_each_job(const Ctx& x, int64_t j, int64_t nc, int C, int64_t cb,
                                             const Span& sl, F f) {
  const LaneParams& p = *x.p;
  const int64_t m = j < nc ? (nc - j + C - 1) / C : 0;  // my chunks
  for (int64_t s = 0; s < m + 4; ++s) {
    for (int ph = 0; ph < 5; ++ph) {
      const int64_t ci = s - ph;
      if (ci < 0 || ci >= m) continue;
      const int64_t c = j + ci * C;
      ChunkGeo ch;
      ch.id = cb + c;
      ch.g0 = p.round_g0 + sl.start + c * p.cg;
      const int64_t rest = sl.len - c * p.cg;
      ch.len = rest < p.cg ? rest : p.cg;
      const int nj = njobs(x, ph);
      for (int t = 0; t < nj; ++t) {
        Job J;
        make_job(x, ph, ch, t, J);
        if (!f(J)) return;
      }
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads, 1) lane_tma_kernel(const __grid_constant__ LaneParams p) {
  using O = Ops<DT>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  volatile int* abort_s = reinterpret_cast<volatile int*>(empty + kStages);

  const int per_rank = p.k * p.C;
  Ctx x;
  x.p = &p;
  x.rank = p.rank0 + (int)(blockIdx.x / per_rank);
  x.N = p.N;
  x.G = p.G;
  x.a = x.rank / p.G;
  x.g = x.rank % p.G;
  x.me = &p.rk[x.rank];
  x.msg.send = reinterpret_cast<const uint4*>(x.me->send);
  x.msg.recv = reinterpret_cast<uint4*>(x.me->recv);
  x.msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  x.msg.partial_bytes = p.tail_elems * (16 / p.q);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int64_t j = blockIdx.x % p.C;
  const Span sl = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    *abort_s = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid < 32) {
    // ------------------------------------------------ producer
    if (tid != 0) return;
    int64_t k = 0;  // global tile counter
    for_each_job(x, j, nc, p.C, cb, sl, [&](const Job& J) {
      for (int w = 0; w < J.nwait; ++w)
        if (!wait_one(p, J.wait[w])) {
          *abort_s = 1;
          return false;
        }
      if (J.nwait) fence_async_global();  // order the acquire before async-proxy reads
      const int64_t T = tile_granules(J.nsrc);
      const int64_t nt = n_tiles(J);
      for (int64_t t = 0; t < nt; ++t, ++k) {
        const int s = (int)(k % kStages);
        if (k >= kStages) {
          const uint32_t par = (uint32_t)(((k / kStages) - 1) & 1);
          uint32_t spins = 0;
          while (!mbar_try_wait(&empty[s], par)) {
            if ((++spins & 1023u) == 0 && *reinterpret_cast<volatile uint32_t*>(p.abort_flag)) {
              *abort_s = 1;
              return false;
            }
          }
        }
        const int64_t g0 = t * T;
        const int64_t tl = J.len - g0 < T ? J.len - g0 : T;  // may be 0 (empty job)
        const bool part = J.x_src >= 0 && x.msg.partial_g >= J.m0 + g0 && x.msg.partial_g < J.m0 + g0 + tl;
        uint4* stage = reinterpret_cast<uint4*>(smem + (size_t)s * kStageBytes);
        uint32_t tx = 0;
        for (int i = 0; i < J.nsrc; ++i) {
          int64_t cnt = tl;
          if (part && i == J.x_src) {  // the message's partial last granule: generic load
            const int64_t off = x.msg.partial_g - (J.m0 + g0);
            stage[i * T + off] = load_partial(J.src[i] + g0 + off, x.msg.partial_bytes);
            cnt = off;  // the partial granule is the last granule of the message
          }
          if (cnt > 0) tx += (uint32_t)(cnt * 16);
        }
        if (part) fence_async_smem();
        mbar_arrive_tx(&full[s], tx);
        for (int i = 0; i < J.nsrc; ++i) {
          int64_t cnt = tl;
          if (part && i == J.x_src) cnt = x.msg.partial_g - (J.m0 + g0);
          if (cnt > 0) bulk_load(stage + i * T, J.src[i] + g0, (uint32_t)(cnt * 16), &full[s]);
        }
      }
      return true;
    });
    return;
  }

  // -------------------------------------------------- consumers (+ storer)
  const int ct = tid - 32;
  const bool storer = ct == 0;
  int64_t k = 0;
  int64_t freed = -1;  // highest tile index whose stage was returned to the producer
  for_each_job(x, j, nc, p.C, cb, sl, [&](const Job& J) {
    const int64_t T = tile_granules(J.nsrc);
    const int64_t nt = n_tiles(J);
    for (int64_t t = 0; t < nt; ++t, ++k) {
      const int s = (int)(k % kStages);
      const uint32_t par = (uint32_t)((k / kStages) & 1);
      uint32_t spins = 0;
      while (!mbar_try_wait(&full[s], par)) {
        if ((++spins & 1023u) == 0 && *abort_s) return false;
      }
      const int64_t g0 = t * T;
      const int64_t tl = J.len - g0 < T ? J.len - g0 : T;
      uint4* stage = reinterpret_cast<uint4*>(smem + (size_t)s * kStageBytes);
      if (J.nsrc > 1) {  // canonical-order reduction, in place into slot 0
        for (int64_t i = ct; i < tl; i += kConsumers) {
          typename O::Acc acc;
          O::init(acc, stage[i]);
          for (int q = 1; q < J.nsrc; ++q) O::add(acc, stage[q * T + i]);
          stage[i] = O::narrow(acc);
        }
        fence_async_smem();
      }
      consumers_sync();
      if (storer) {
        const bool rpart = J.recv_dst >= 0 && x.msg.partial_g >= J.m0 + g0 && x.msg.partial_g < J.m0 + g0 + tl;
        for (int d = 0; d < J.ndst; ++d) {
          int64_t cnt = tl;
          if (rpart && d == J.recv_dst) {
            const int64_t off = x.msg.partial_g - (J.m0 + g0);
            store_partial(J.dst[d] + g0 + off, stage[off], x.msg.partial_bytes);
            cnt = off;
          }
          if (cnt > 0) bulk_store(J.dst[d] + g0, stage, (uint32_t)(cnt * 16));
        }
        bulk_commit();
        bulk_wait_read1();  // all store groups but this tile's have read their smem
        if (k - 1 > freed && k >= 1) {
          mbar_arrive(&empty[(k - 1) % kStages]);
          freed = k - 1;
        }
        if (t == nt - 1 && J.nrel > 0) {  // job complete: make it visible, then release
          bulk_wait_all();
          mbar_arrive(&empty[s]);
          freed = k;
          fence_async_global();
          __threadfence_system();
          for (int r = 0; r < J.nrel; ++r) st_release_sys(J.rel[r], p.epoch);
        }
      }
    }
    return true;
  });
  if (storer) bulk_wait_all();
}

}  // namespace tma
}  // namespace lane
