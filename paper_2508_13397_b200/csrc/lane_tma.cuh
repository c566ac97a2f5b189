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
//   warps 1..R     : releasers (lane 0) — take completed jobs' flag lists
//                    from a shared-memory ring, fence.acq_rel.sys, then
//                    relaxed .sys flag stores; R fences in flight at once.
//   warps R+1..    : consumers — reduce the tile's sources from shared memory
//                    (fp32 accumulate, canonical order) and store 128-bit
//                    st.global to every destination (or, from
//                    LANE_BULK_MIN_BYTES, cp.async.bulk smem -> global by
//                    consumer 0, the storer); the storer hands a finished
//                    job's flags to the releasers.
//
// Schedule: CTA j of CTA group l owns chunks j, j+C, ... of slice l. The
// producer issues jobs OUT OF ORDER: it takes the next job of any phase whose
// flags are already set (per chunk, phases stay in order A..E; phase A runs at
// most a small window of chunks ahead), so one lagging peer does not stall
// the ring. Consumers are driven entirely by per-stage tile descriptors.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_kernels.cuh"
#include "lane_plan.h"

namespace lane {
namespace tma {

#ifndef LANE_TMA_STAGES
#define LANE_TMA_STAGES 4
#endif
#ifndef LANE_TMA_STAGE_KB
#define LANE_TMA_STAGE_KB 48
#endif
#ifndef LANE_TMA_MIN_BLOCKS  // CTAs per SM the register budget is sized for
#define LANE_TMA_MIN_BLOCKS 1
#endif
constexpr int kStages = LANE_TMA_STAGES;
constexpr int kStageBytes = LANE_TMA_STAGE_KB * 1024;
constexpr int kStageGranules = kStageBytes / 16;
constexpr int kConsumerWarps = 6;
// A system-scope fence takes microseconds, and one thread can only wait for
// one at a time: kReleasers releaser warps (lane 0 each) publish completed
// jobs concurrently, each with its own fence.
constexpr int kReleasers = 4;
constexpr int kThreads = 32 * (1 + kReleasers + kConsumerWarps);  // producer, releasers, consumers
constexpr int kConsumerTid0 = 32 * (1 + kReleasers);
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kMaxSrc = LANE_MAX_RANKS;
constexpr int kRelSlots = 16;  // release records in flight between storer and releaser
constexpr int kJobCacheBytes = 5 * 576;  // producer's next job of every phase
constexpr int kProdStateBytes = 448;     // producer's per-phase cursors and claim ring (ProdState)
constexpr int kSmemBytes = kStages * kStageBytes + 2 * kStages * 8 + kStages * 320 + kRelSlots * 136 + 256 +
                           kJobCacheBytes + kProdStateBytes;

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
// wait until at most `newer` bulk groups are pending (0..2; larger: 2)
__device__ __forceinline__ void bulk_wait_upto(int64_t newer) {
  if (newer >= 2)
    asm volatile("cp.async.bulk.wait_group 2;" ::: "memory");
  else if (newer == 1)
    asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
  else
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
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
  int ph;                // 0..4 = phase A..E
  int nsrc, ndst;
  uint32_t x_mask;       // bit i: src[i] is a sendbuf (partial last granule possible)
  uint32_t recv_mask;    // bit d: dst[d] is a recvbuf
  int nwait, nrel;
  int entry;    // needs the start handshake first: writes a recvbuf or reads a peer's sendbuf
  int64_t len;  // granules
  int64_t m0;   // message granule of the job's first granule
  const uint4* src[kMaxSrc];
  uint4* dst[kMaxSrc];
  const uint32_t* wait[kMaxSrc];
  uint32_t* rel[kMaxSrc];
};

struct Ctx {
  const LaneParams* p;
  int rank, a, g, N, G;
  const RankMem* me;
  Msg msg;
};

// Jobs per chunk of each phase.
//  staged (default, unregistered buffers): A push, B reduce+push, C reduce,
//    D pull lane results, E pull node parts — through library scratch.
//    With G == 1 the own lane term is the sendbuf itself: B only sends the
//    N-1 remote sub-parts and C reads its own term from sendbuf.
//  direct (every rank's sendbuf/recvbuf addressable: emulated mode):
//    B reduces straight from the node's sendbufs, C stores the lane result
//    into every lane member's recvbuf, D is a zero-byte job that forwards
//    "part g complete" to the node, E pulls node peers' parts from their
//    recvbufs. No phase-1 or R staging.
//  direct-push (registered user buffers on real peers; all NVLink traffic is
//    stores, the faster direction on this fabric): A and B as staged, C stores
//    the lane result into every lane member's recvbuf, D pushes my completed
//    part g from my recvbuf into the node peers' recvbufs; no pull phase.
//  pull-all (registered user buffers; LANE_DIRECT=3): every job reads local or
//    peer memory and writes only this rank's memory, so a job's release
//    fence never waits behind stores in flight to other GPUs: B sums the
//    node's sendbufs into my S2 (slot b = sub-part b), C sums the lane
//    members' S2 slot a into my recvbuf, D pulls the lane members' results
//    from their recvbufs, E pulls the node peers' parts from theirs.
//  pull-push (registered user buffers; LANE_DIRECT=4): phase 1 as a pull, the
//    rest as direct-push: B reads the node peers' sendbufs straight over
//    NVLink (the start handshake already guarantees they are final), so there
//    is no A job, no S1 staging and no F1 hop on the chunk's critical path;
//    C and D push as in direct-push.
enum DirectMode { kStaged = 0, kDirectPull = 1, kDirectPush = 2, kPullAll = 3, kPullPush = 4 };

__device__ __forceinline__ int njobs(const Ctx& x, int ph) {
  const int dm = x.p->direct;
  if (dm == kPullAll) {
    switch (ph) {
      case 0: return 0;
      case 1: return x.G > 1 ? x.N : 0;
      case 2: return 1;
      case 3: return x.N - 1;
      default: return x.G - 1;
    }
  }
  switch (ph) {
    case 0: return (dm == kDirectPull || dm == kPullPush) ? 0 : x.G - 1;
    case 1: return x.G == 1 ? (dm == kDirectPull ? 0 : x.N - 1) : x.N;
    case 2: return x.N > 1 ? 1 : 0;
    case 3: return dm != kStaged ? ((x.N > 1 && x.G > 1) ? 1 : 0) : x.N - 1;
    default: return (dm == kDirectPush || dm == kPullPush) ? 0 : x.G - 1;
  }
}

__device__ __forceinline__ uint4* send_of(const RankMem& m) {
  return reinterpret_cast<uint4*>(const_cast<char*>(m.send));
}
__device__ __forceinline__ uint4* recv_of(const RankMem& m) { return reinterpret_cast<uint4*>(m.recv); }

// Job t of phase ph (0=A .. 4=E) for chunk ch.
__device__ void make_job_(const Ctx& x, int ph, const ChunkGeo& ch, int t, Job& J) {
  const LaneParams& p = *x.p;
  const int a = x.a, g = x.g, N = x.N, G = x.G;
  const bool direct = p.direct == kDirectPull;  // pull flavour (emulated mode)
  const bool push = p.direct == kDirectPush || p.direct == kPullPush;
  const bool pull1 = direct || p.direct == kPullPush;  // phase 1 reads the node's sendbufs
  J.ph = ph;
  J.nsrc = 1;
  J.ndst = 1;
  J.x_mask = 0;
  J.recv_mask = 0;
  J.nwait = 0;
  J.nrel = 0;
  const Span gp = rf_split(ch.len, G, g);
  if (p.direct == kPullAll) {
    if (ph == 1) {  // B: node sum (ascending h) of sub-part b of part g -> my S2 slot b
      const int b = (a + 1 + t) % N;  // own sub-part last
      const Span up = rf_split(gp.len, N, b);
      J.len = up.len;
      J.m0 = ch.g0 + gp.start + up.start;
      J.nsrc = G;
      for (int h = 0; h < G; ++h) J.src[h] = (h == g ? x.msg.send : send_of(p.rk[a * G + h])) + J.m0;
      J.x_mask = (1u << G) - 1;
      J.dst[0] = s2_slot(p, *x.me, b, ch.id);
      J.rel[J.nrel++] = p.rk[b * G + g].flags + f2_idx(p, a, ch.id);
    } else if (ph == 2) {  // C: lane sum (ascending b) of sub-part a -> my recvbuf
      const Span up = rf_split(gp.len, N, a);
      J.len = up.len;
      J.m0 = ch.g0 + gp.start + up.start;
      J.nsrc = N;
      for (int b = 0; b < N; ++b) {
        if (G == 1) {  // a one-GPU node's sum is its sendbuf
          J.src[b] = (b == a ? x.msg.send : send_of(p.rk[b * G + g])) + J.m0;
          J.x_mask |= 1u << b;
        } else {
          J.src[b] = s2_slot(p, p.rk[b * G + g], a, ch.id);
          J.wait[J.nwait++] = x.me->flags + f2_idx(p, b, ch.id);
        }
      }
      J.dst[0] = x.msg.recv + J.m0;
      J.recv_mask = 1;
      for (int b = 0; b < N; ++b)
        if (b != a) J.rel[J.nrel++] = p.rk[b * G + g].flags + f3_idx(p, a, ch.id);
      if (N == 1)  // part g of my recvbuf is complete
        for (int h = 0; h < G; ++h)
          if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    } else if (ph == 3) {  // D: pull lane member b's result sub-part -> my recvbuf
      const int b = (a + 1 + t) % N;
      const Span up = rf_split(gp.len, N, b);
      J.len = up.len;
      J.m0 = ch.g0 + gp.start + up.start;
      J.src[0] = recv_of(p.rk[b * G + g]) + J.m0;
      J.x_mask = 1;  // a user buffer: its partial last granule is loaded generically
      J.wait[J.nwait++] = x.me->flags + f3_idx(p, b, ch.id);
      J.dst[0] = x.msg.recv + J.m0;
      J.recv_mask = 1;
      if (t == N - 2)  // part g of my recvbuf complete (C's and every D's stores precede this)
        for (int h = 0; h < G; ++h)
          if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    } else {  // E: pull node peer h's part -> my recvbuf
      const int h = (g + 1 + t) % G;
      const Span ph_ = rf_split(ch.len, G, h);
      J.len = ph_.len;
      J.m0 = ch.g0 + ph_.start;
      J.src[0] = recv_of(p.rk[a * G + h]) + J.m0;
      J.x_mask = 1;
      J.wait[J.nwait++] = x.me->flags + f4_idx(p, h, ch.id);
      J.dst[0] = x.msg.recv + J.m0;
      J.recv_mask = 1;
    }
    return;
  }
  if (ph == 0) {  // A (staged): push part gd of my sendbuf into (a,gd)'s S1
    const int gd = (g + 1 + t) % G;
    const Span pd = rf_split(ch.len, G, gd);
    const RankMem& dm = p.rk[a * G + gd];
    J.len = pd.len;
    J.m0 = ch.g0 + pd.start;
    J.src[0] = x.msg.send + J.m0;
    J.x_mask = 1;
    J.dst[0] = s1_slot(p, dm, g < gd ? g : g - 1, ch.id);
    J.rel[J.nrel++] = dm.flags + f1_idx(p, g, ch.id);
  } else if (ph == 1) {  // B: reduce part g over the node (ascending h), sub-part b
    const int b = (a + 1 + t) % N;  // own sub-part last (absent when G == 1)
    const Span up = rf_split(gp.len, N, b);
    J.len = up.len;
    J.m0 = ch.g0 + gp.start + up.start;
    J.nsrc = G;
    for (int h = 0; h < G; ++h) {
      if (pull1) {
        J.src[h] = (h == g ? x.msg.send : send_of(p.rk[a * G + h])) + J.m0;
        J.x_mask |= 1u << h;
      } else {
        J.src[h] = (h == g) ? x.msg.send + J.m0 : s1_slot(p, *x.me, h < g ? h : h - 1, ch.id) + up.start;
      }
    }
    if (!pull1) {
      J.x_mask = 1u << g;
      if (t == 0)
        for (int h = 0; h < G; ++h)
          if (h != g) J.wait[J.nwait++] = x.me->flags + f1_idx(p, h, ch.id);
    }
    if (N > 1) {
      const RankMem& dm = p.rk[b * G + g];
      J.dst[0] = s2_slot(p, dm, a, ch.id);
      J.rel[J.nrel++] = dm.flags + f2_idx(p, a, ch.id);
    } else {  // N == 1: the node sum is the final value of part g
      if (push) {  // phase 3 by pushing part g into every node member's recvbuf
        J.ndst = G;
        for (int t2 = 0; t2 < G; ++t2) J.dst[t2] = recv_of(p.rk[a * G + (g + t2) % G]) + J.m0;
        J.recv_mask = (1u << G) - 1;
        return;  // completion is covered by the end-of-call handshake
      }
      if (direct) {
        J.dst[0] = x.msg.recv + J.m0;
        J.recv_mask = 1;
      } else {
        J.ndst = 2;
        J.dst[0] = r_slot(p, *x.me, ch.id) + up.start;
        J.dst[1] = x.msg.recv + J.m0;
        J.recv_mask = 2;
      }
      for (int h = 0; h < G; ++h)
        if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    }
  } else if (ph == 2) {  // C: reduce my sub-part over the lane (ascending b)
    const Span up = rf_split(gp.len, N, a);
    J.len = up.len;
    J.m0 = ch.g0 + gp.start + up.start;
    J.nsrc = N;
    for (int b = 0; b < N; ++b) {
      if (G == 1 && (b == a || direct)) {
        // T1 of a single-GPU node is its sendbuf (direct: read the lane member's sendbuf)
        J.src[b] = (b == a) ? x.msg.send + J.m0 : send_of(p.rk[b * G + g]) + J.m0;
        J.x_mask |= 1u << b;
      } else {
        J.src[b] = s2_slot(p, *x.me, b, ch.id);
        J.wait[J.nwait++] = x.me->flags + f2_idx(p, b, ch.id);
      }
    }
    if (direct || push) {  // lane allgather by pushing F into every lane member's recvbuf
      J.ndst = N;
      for (int t2 = 0; t2 < N; ++t2) {
        const int b = (a + t2) % N;  // own first
        J.dst[t2] = recv_of(p.rk[b * G + g]) + J.m0;
      }
      J.recv_mask = (1u << N) - 1;
    } else {
      J.ndst = 2;
      J.dst[0] = r_slot(p, *x.me, ch.id) + up.start;
      J.dst[1] = x.msg.recv + J.m0;
      J.recv_mask = 2;
    }
    for (int b = 0; b < N; ++b)
      if (b != a || push) J.rel[J.nrel++] = p.rk[b * G + g].flags + f3_idx(p, a, ch.id);
  } else if (ph == 3) {
    if (push) {  // D (push): part g of my recvbuf is complete -> store it into the node's recvbufs
      J.len = gp.len;
      J.m0 = ch.g0 + gp.start;
      J.src[0] = x.msg.recv + J.m0;
      J.x_mask = 1;  // a user buffer: its partial last granule is loaded generically
      for (int b = 0; b < N; ++b) J.wait[J.nwait++] = x.me->flags + f3_idx(p, b, ch.id);
      J.ndst = G - 1;
      for (int t2 = 1; t2 < G; ++t2) J.dst[t2 - 1] = recv_of(p.rk[a * G + (g + t2) % G]) + J.m0;
      J.recv_mask = (1u << (G - 1)) - 1;
      return;
    }
    if (direct) {  // D (direct): part g of my recvbuf is complete -> tell the node
      J.len = 0;
      J.m0 = ch.g0 + gp.start;
      J.src[0] = x.msg.recv + J.m0;
      J.dst[0] = x.msg.recv + J.m0;
      for (int b = 0; b < N; ++b)
        if (b != a) J.wait[J.nwait++] = x.me->flags + f3_idx(p, b, ch.id);
      for (int h = 0; h < G; ++h)
        if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
      return;
    }
    // D (staged): pull lane member b's sub-part
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
      J.recv_mask = 2;
      if (t == N - 2)  // R of part g complete (C's and every D's stores precede this)
        for (int h = 0; h < G; ++h)
          if (h != g) J.rel[J.nrel++] = p.rk[a * G + h].flags + f4_idx(p, g, ch.id);
    } else {
      J.dst[0] = x.msg.recv + J.m0;
      J.recv_mask = 1;
    }
  } else {  // E: pull node peer h's part (from its R, or its recvbuf when direct)
    const int h = (g + 1 + t) % G;
    const Span ph_ = rf_split(ch.len, G, h);
    J.len = ph_.len;
    J.m0 = ch.g0 + ph_.start;
    J.src[0] = direct ? recv_of(p.rk[a * G + h]) + J.m0 : r_slot(p, p.rk[a * G + h], ch.id);
    J.wait[J.nwait++] = x.me->flags + f4_idx(p, h, ch.id);
    J.dst[0] = x.msg.recv + J.m0;
    J.recv_mask = 1;
  }
}

// make_job_ plus J.entry. Jobs that only move data into peers' SCRATCH (S1,
// S2) may run before the start handshake: a peer reads its scratch of call e
// before it passes the end barrier of call e, which this rank passed before
// starting call e+1, and every scratch read is gated by its epoch flag. Jobs
// that write any recvbuf or read a peer's sendbuf wait for the handshake (the
// peer's kernel has started, so its stream's earlier work on those buffers is
// done, and its call signature matches ours).
__device__ void make_job(const Ctx& x, int ph, const ChunkGeo& ch, int t, Job& J) {
  make_job_(x, ph, ch, t, J);
  int e = J.recv_mask != 0;
  for (int i = 0; i < J.nsrc && !e; ++i)
    if ((J.x_mask >> i) & 1u) e = J.src[i] < x.msg.send || J.src[i] >= x.msg.send + x.p->ng;  // a peer's sendbuf
  J.entry = e;
}

__device__ __forceinline__ int64_t tile_granules(int nsrc) {
  return (int64_t)(kStageGranules / nsrc);
}

// Descriptor of one ring stage, written by the producer before it arrives on
// the stage's "full" barrier; consumers need nothing else.
struct TileDesc {
  int nsrc;            // 0 = end of the CTA's work
  int ndst, nrel, ph;
  uint32_t recv_mask;  // dsts that are recvbufs, when the tile holds the partial granule
  int64_t T;           // slot stride in granules
  int64_t tl;          // granules in this tile
  int64_t poff;        // granule offset of the message's partial last granule in the tile, or -1
  uint4* dst[kMaxSrc]; // already offset to the tile start
  uint32_t* rel[kMaxSrc];  // flags to release once this tile (the job's last) is stored
};

constexpr int kDescBytes = 320;
static_assert(sizeof(TileDesc) <= kDescBytes, "TileDesc must fit its smem slot");
static_assert(sizeof(Job) <= 576, "Job must fit its smem slot");

// A job's flag releases, handed from the storer to the releaser warp.
struct RelRec {
  int n;
  uint32_t* f[kMaxSrc];
};
static_assert(sizeof(RelRec) <= 136, "RelRec must fit its smem slot");

struct RelRing {
  volatile int tail;   // records published by the storer (record t lives in slot t % kRelSlots)
  int claim;           // next record index a releaser takes (shared-memory atomicAdd)
  volatile int done;   // storer finished (or aborted)
  int exited;          // releasers that left their loop
  unsigned long long fence_ns;  // trace: releasers' time in fences and flag stores
  volatile int busy[kRelSlots];  // 1 while the slot's record is published and not yet retired
};
static_assert(sizeof(RelRing) + 4 <= 256, "RelRing must fit its smem slot");

// Storer side, in two steps: reserve_release fills the record at the ring's
// tail (waiting until the releasers retired the slot) straight from the
// tile descriptor — shared memory to shared memory, no copy of the flag list
// in registers or on the stack — and commit_release hands it to the
// releasers. The storer holds at most one reserved record (the bulk-store
// path holds a job's release until its stores are done).
__device__ __forceinline__ void reserve_release(RelRing* ring, RelRec* rel_rec, uint32_t* const* rel, int nrel) {
  const int t = ring->tail;
  while (ring->busy[t % kRelSlots]) {
  }
  RelRec& r = rel_rec[t % kRelSlots];
  r.n = nrel;
  for (int i = 0; i < nrel; ++i) r.f[i] = rel[i];
}
__device__ __forceinline__ void commit_release(RelRing* ring) {
  const int t = ring->tail;
  __threadfence_block();
  ring->busy[t % kRelSlots] = 1;
  ring->tail = t + 1;
}
__device__ __forceinline__ void publish_release(RelRing* ring, RelRec* rel_rec, uint32_t* const* rel, int nrel) {
  reserve_release(ring, rel_rec, rel, nrel);
  commit_release(ring);
}

// The producer's per-phase cursors, in shared memory: they are indexed by the
// picked phase (a run-time value), which in registers would be a stack array.
constexpr int kClaimRing = 32;  // claimed chunks held by a CTA's producer (dynamic claims)

struct ProdState {
  int64_t cur[5];  // next chunk (ordinal among this CTA's chunks) per phase
  int64_t chunk[kClaimRing];  // dynamic claims: chunk of ordinal x at [x % kClaimRing]
  int64_t nclaimed;           // dynamic claims: ordinals claimed so far
  int nj[5];       // jobs per chunk per phase
  int prev[5];     // previous active phase
  int sub[5];      // next job within the chunk
  int wpos[5];     // flags of the cached job already seen set
  int have[5];     // cached job valid
};
static_assert(sizeof(ProdState) <= kProdStateBytes, "ProdState must fit its smem slot");

// Relaxed poll (no per-poll fence); a fence_acquire_sys() after the last
// observation completes the acquire pattern.
__device__ __forceinline__ bool flag_seen(const LaneParams& p, const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return (int32_t)(v - cur_epoch()) >= 0;
}
__device__ __forceinline__ void fence_acquire_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ bool flag_ready(const LaneParams& p, const uint32_t* f) {
  return (int32_t)(ld_acquire_sys(f) - cur_epoch()) >= 0;
}

// Blocking acquire-wait on one flag (single thread). false on timeout / abort.
__device__ bool wait_one(const LaneParams& p, const uint32_t* f) {
  if (flag_ready(p, f)) return true;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t it = 1;; ++it) {
    if (flag_ready(p, f)) return true;
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

__device__ __forceinline__ ChunkGeo chunk_geo(const LaneParams& p, int64_t cb, const Span& sl, int64_t c) {
  ChunkGeo ch;
  ch.id = cb + c;
  ch.g0 = p.round_g0 + sl.start + c * p.cg;
  const int64_t rest = sl.len - c * p.cg;
  ch.len = rest < p.cg ? rest : p.cg;
  return ch;
}

template <int DT, bool kLsuStore>
__global__ void __launch_bounds__(kThreads, LANE_TMA_MIN_BLOCKS) lane_tma_kernel(const __grid_constant__ LaneParams p) {
  const uint64_t t_entry = launch_prologue(p);
  using O = Ops<DT>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  TileDesc* desc = reinterpret_cast<TileDesc*>(empty + kStages);
  RelRec* rel_rec = reinterpret_cast<RelRec*>(desc + kStages);
  RelRing* ring = reinterpret_cast<RelRing*>(rel_rec + kRelSlots);
  volatile int* abort_s = reinterpret_cast<volatile int*>(reinterpret_cast<char*>(ring) + sizeof(RelRing));
  Job* jobs = reinterpret_cast<Job*>(smem + kSmemBytes - kJobCacheBytes - kProdStateBytes);  // producer only
  ProdState* ps = reinterpret_cast<ProdState*>(smem + kSmemBytes - kProdStateBytes);     // producer only

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
  const int64_t m = j < nc ? (nc - j + p.C - 1) / p.C : 0;  // my chunks: j, j+C, ...

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    *abort_s = 0;
    ring->tail = 0;
    ring->claim = 0;
    ring->done = 0;
    ring->exited = 0;
    ring->fence_ns = 0;
    for (int i = 0; i < kRelSlots; ++i) ring->busy[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid >= 32 && tid < kConsumerTid0) {
    // ================================================= releasers (lane 0 of warps 1..kReleasers)
    // Publish job-completion flags. The fence waits until the job's stores
    // (issued by every consumer before the storer's barrier, hence
    // happening-before this thread's acquire of the record) are visible
    // system-wide; doing it here keeps the consumer pipeline streaming, and
    // several releasers keep several fences in flight.
    const int nrw = p.releasers < 1 ? 1 : (p.releasers > kReleasers ? kReleasers : p.releasers);
    if (tid % 32 != 0 || tid / 32 - 1 >= nrw) return;
    const bool tr = p.trace != nullptr;
    uint64_t tr_fence = 0;
    for (;;) {
      // claim every published, unclaimed record [c0, c1) at once
      int c0, c1;
      for (;;) {
        c0 = *reinterpret_cast<volatile int*>(&ring->claim);
        c1 = ring->tail;
        if (c1 > c0) {
          if (atomicCAS(&ring->claim, c0, c1) == c0) break;
          continue;
        }
        if (ring->done && ring->tail <= *reinterpret_cast<volatile int*>(&ring->claim)) {
          c0 = c1 = -1;
          break;
        }
      }
      if (c0 < 0) break;
      __threadfence_block();  // acquire the records
      const uint64_t tw = tr ? globaltimer_ns() : 0;
      fence_acq_rel_sys();  // release pattern: one fence, then relaxed .sys flag stores
      for (int c = c0; c < c1; ++c) {
        const RelRec& r = rel_rec[c % kRelSlots];
        for (int i = 0; i < r.n; ++i) st_relaxed_sys(r.f[i], cur_epoch());
      }
      __threadfence_block();
      for (int c = c0; c < c1; ++c) ring->busy[c % kRelSlots] = 0;
      if (tr) tr_fence += globaltimer_ns() - tw;
    }
    if (tr) atomicAdd(&ring->fence_ns, (unsigned long long)tr_fence);
    if (atomicAdd(&ring->exited, 1) != nrw - 1) return;  // the last releaser finishes the CTA
    __threadfence_block();
    fence_acq_rel_sys();  // every store this CTA made is visible system-wide
    if (tr) p.trace[(size_t)blockIdx.x * kTraceWords + kTrStoreReadWait] = ring->fence_ns;
    if (p.handshake) {
      // end of call (every simple-protocol call on real peers): the last CTA of this rank tells
      // every peer "done with your buffers" and waits until every peer is done
      // with ours, so the call completes only when no peer still reads our
      // sendbuf or writes our recvbuf.
      uint32_t* cnt = x.me->flags + p.ctl + kCtlCounter;
      uint32_t old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
      if ((int)old + 1 == per_rank) {
        atomicExch(cnt, 0u);
        fence_acq_rel_sys();
        for (int q = 0; q < p.P; ++q)
          if (q != x.rank) st_relaxed_sys(p.rk[q].flags + p.ctl + kCtlDone + x.rank, cur_epoch());
        for (int q = 0; q < p.P; ++q)
          if (q != x.rank && !wait_one(p, x.me->flags + p.ctl + kCtlDone + q)) break;
        if (tr) p.trace[(size_t)blockIdx.x * kTraceWords + kTrEndAbs] = globaltimer_ns();
      }
    }
    return;
  }

  if (tid < 32) {
    // ================================================= producer (one thread)
    // Out-of-order issue: among the next job of every phase, take the first
    // (in phase order A..E) whose flags are already set, subject to
    //   - per chunk, phase order: job (ph, c) only after every job of the
    //     previous active phase for chunk c has been issued (local stores of
    //     an earlier phase must precede the release of a later one);
    //   - a window: phase A runs at most p_window chunks ahead of the last
    //     active phase.
    // Every wait is still on peers' earlier phases of the same chunk, so the
    // in-order schedule is one possible execution and progress is guaranteed.
    if (tid != 0) return;
    const bool tr = p.trace != nullptr;
    uint64_t tr_flag = 0, tr_empty = 0;
    const uint64_t t_start = tr ? globaltimer_ns() : 0;
    int last = -1;
    int64_t* const cur = ps->cur;
    int* const nj = ps->nj;
    int* const prev = ps->prev;
    int* const sub = ps->sub;
    int* const wpos = ps->wpos;  // flags of jobs[ph] already seen set
    int* const have = ps->have;  // jobs[ph] (shared memory): next job of every phase, built once per job
    int first = -1;  // first active phase: the one that takes a new chunk
    for (int ph = 0, pa = -1; ph < 5; ++ph) {
      nj[ph] = njobs(x, ph);
      cur[ph] = nj[ph] > 0 ? 0 : m;  // inactive phases are "done"
      sub[ph] = 0;
      prev[ph] = pa;
      wpos[ph] = 0;
      have[ph] = 0;
      if (nj[ph] > 0) {
        pa = last = ph;
        if (first < 0) first = ph;
      }
    }
    const int64_t window = 6;
    // Chunks of this CTA. Static: j, j+C, ... (m of them). Dynamic (p.dyn):
    // claimed one at a time from the rank's per-slice counter when the first
    // active phase needs a new chunk (within the window), the next claim's
    // atomic already in flight; a CTA on a fast SM ends up with more chunks.
    // Deadlock-free as the static schedule: every rank claims in increasing
    // chunk order, a claimed chunk's first phase never waits (A) or waits only
    // on peers' earlier phases of the same chunk, and the lowest unfinished
    // chunk is claimed on every rank.
    const bool dyn = p.dyn != 0;
    unsigned* const ctr = dyn ? p.claims + claim_index(x.rank, (int)(cur_epoch() & 1u), l) : nullptr;
    unsigned pending = dyn ? atomicAdd(ctr, 1u) : 0u;
    bool claim_done = !dyn;
    ps->nclaimed = 0;
    auto limit = [&]() -> int64_t { return dyn ? ps->nclaimed : m; };
    auto chunk_of = [&](int64_t ord) -> int64_t { return dyn ? ps->chunk[ord % kClaimRing] : j + ord * p.C; };
    int64_t k = 0;  // global tile counter
    bool ok = true;
    // Start-of-call handshake (every simple-protocol call on real peers): a
    // peer's sendbuf is final and its recvbuf free once its kernel has started
    // (stream order). The first CTA of each rank publishes the call signature
    // (host call_signature: job set, buffer offsets in the registrations,
    // count, dtype, chunking) and then its enter flag; every CTA compares
    // every peer's signature with its own before its first job that writes a
    // recvbuf or reads a peer's sendbuf (Job::entry), so ranks that disagree
    // (one zero-copy, one staged; other offsets or counts) stop with
    // LANE_ERR_MISMATCH before touching a user buffer, instead of exchanging
    // wrong data or waiting for flags that never come. Scratch-only jobs (A,
    // B into S1/S2) run meanwhile, so the handshake's round trip overlaps
    // data movement. The sig slots are rewritten only in the next call,
    // after the end barrier.
    const uint32_t my_sig = p.sig ^ (x.rank == p.sig_skew ? 1u : 0u);
    bool entered = !p.handshake;
    int enter_seen = 0;  // peers (in rank order, skipping this one) whose enter flag was seen
    if (p.handshake && blockIdx.x % per_rank == 0) {
      for (int q = 0; q < p.P; ++q)
        if (q != x.rank) st_relaxed_sys(p.rk[q].flags + p.ctl + kCtlSig + x.rank, my_sig);
      fence_acq_rel_sys();
      for (int q = 0; q < p.P; ++q)
        if (q != x.rank) st_relaxed_sys(p.rk[q].flags + p.ctl + kCtlEnter + x.rank, cur_epoch());
    }
    // Non-blocking: true once every peer's enter flag is set and the
    // signatures agree (ok = false on a mismatch).
    auto try_enter = [&]() -> bool {
      while (enter_seen < p.P) {
        if (enter_seen == x.rank) {
          ++enter_seen;
          continue;
        }
        if (!flag_ready(p, x.me->flags + p.ctl + kCtlEnter + enter_seen)) return false;
        ++enter_seen;
      }
      for (int q = 0; q < p.P; ++q) {
        if (q == x.rank) continue;
        uint32_t v;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(x.me->flags + p.ctl + kCtlSig + q) : "memory");
        if (v != my_sig) {
          atomicExch(p.abort_flag, 1u);
          *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_MISMATCH);
          __threadfence_system();
          ok = false;
          return false;
        }
      }
      fence_async_global();
      if (tr) p.trace[(size_t)blockIdx.x * kTraceWords + kTrEnterWait] = globaltimer_ns() - t_start;
      entered = true;
      return true;
    };
    if (tr) p.trace[(size_t)blockIdx.x * kTraceWords + kTrStartAbs] = t_start;
    uint64_t t_idle = 0;
    while (ok) {
      int pick = -1;
      bool any_left = false;
      for (int ph = 0; ph < 5 && pick < 0; ++ph) {
        if (nj[ph] == 0) continue;
        if (cur[ph] >= limit()) {
          if (claim_done || ph != first) {
            if (!claim_done) any_left = true;  // later phases wait for the next claim
            continue;
          }
          if (last != first && cur[first] - cur[last] >= window) {
            any_left = true;
            continue;
          }
          const unsigned c = pending;  // take the claim in flight, start the next
          if ((int64_t)c >= nc) {
            claim_done = true;
            continue;
          }
          pending = atomicAdd(ctr, 1u);
          ps->chunk[ps->nclaimed % kClaimRing] = (int64_t)c;
          ++ps->nclaimed;
        }
        any_left = true;
        if (prev[ph] >= 0 && cur[ph] >= cur[prev[ph]]) continue;  // previous phase not issued yet
        // the window: phase A (static; as before) or the first active phase (dynamic, which also
        // bounds the claim ring) runs at most `window` chunks ahead of the last phase
        if (ph == first && (first == 0 || dyn) && last != first && cur[first] - cur[last] >= window) continue;
        if (!have[ph]) {
          make_job(x, ph, chunk_geo(p, cb, sl, chunk_of(cur[ph])), sub[ph], jobs[ph]);
          have[ph] = 1;
          wpos[ph] = 0;
        }
        const Job& Jc = jobs[ph];
        if (Jc.entry && !entered && !try_enter()) {
          if (!ok) break;
          continue;
        }
        while (wpos[ph] < Jc.nwait && flag_ready(p, Jc.wait[wpos[ph]])) ++wpos[ph];
        if (wpos[ph] == Jc.nwait) pick = ph;
      }
      if (!any_left) break;
      if (pick < 0) {  // nothing ready: watchdog + abort checks
        const uint64_t now = globaltimer_ns();
        if (t_idle == 0) t_idle = now;
        if (*reinterpret_cast<volatile uint32_t*>(p.abort_flag)) ok = false;
        if (now - t_idle > p.timeout_ns) {
          atomicExch(p.abort_flag, 1u);
          *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_TIMEOUT);
          __threadfence_system();
          ok = false;
        }
        continue;
      }
      if (t_idle) {
        if (tr) tr_flag += globaltimer_ns() - t_idle;
        t_idle = 0;
      }
      const Job& J = jobs[pick];
      if (J.nwait) fence_async_global();  // acquired flags ordered before the async-proxy (TMA) reads
      have[pick] = 0;  // J stays valid until the next make_job of this phase
      // advance the phase cursor
      if (++sub[pick] == nj[pick]) {
        sub[pick] = 0;
        ++cur[pick];
      }
      const int64_t T = tile_granules(J.nsrc);
      const int64_t nt = J.len > 0 ? (J.len + T - 1) / T : 1;  // empty jobs keep one empty tile
      for (int64_t t = 0; t < nt && ok; ++t, ++k) {
        const int s = (int)(k % kStages);
        if (k >= kStages) {
          const uint32_t par = (uint32_t)(((k / kStages) - 1) & 1);
          uint32_t spins = 0;
          const uint64_t te = tr ? globaltimer_ns() : 0;
          while (!mbar_try_wait(&empty[s], par)) {
            if ((++spins & 1023u) == 0 && *reinterpret_cast<volatile uint32_t*>(p.abort_flag)) {
              ok = false;
              break;
            }
          }
          if (tr) tr_empty += globaltimer_ns() - te;
          if (!ok) break;
        }
        const int64_t g0 = t * T;
        const int64_t tl = J.len - g0 < T ? J.len - g0 : T;  // may be 0 (empty job)
        const bool inpart = x.msg.partial_g >= J.m0 + g0 && x.msg.partial_g < J.m0 + g0 + tl;
        const bool xpart = J.x_mask != 0 && inpart;
        const bool rpart = J.recv_mask != 0 && inpart;
        const int64_t poff = (xpart || rpart) ? x.msg.partial_g - (J.m0 + g0) : -1;
        uint4* stage = reinterpret_cast<uint4*>(smem + (size_t)s * kStageBytes);
        TileDesc& d = desc[s];
        d.nsrc = J.nsrc;
        d.ndst = J.ndst;
        d.recv_mask = rpart ? J.recv_mask : 0u;
        d.ph = J.ph;
        d.T = T;
        d.tl = tl;
        d.poff = poff;
        for (int dd = 0; dd < J.ndst; ++dd) d.dst[dd] = J.dst[dd] + g0;
        d.nrel = (t == nt - 1) ? J.nrel : 0;
        for (int r = 0; r < d.nrel; ++r) d.rel[r] = J.rel[r];
        uint32_t tx = 0;
        for (int i = 0; i < J.nsrc; ++i) {
          int64_t cnt = tl;
          if (xpart && ((J.x_mask >> i) & 1u)) {  // partial last granule of a sendbuf: generic load
            stage[i * T + poff] = load_partial(J.src[i] + g0 + poff, x.msg.partial_bytes);
            cnt = poff;
          }
          if (cnt > 0) tx += (uint32_t)(cnt * 16);
        }
        fence_async_smem();
        mbar_arrive_tx(&full[s], tx);
        for (int i = 0; i < J.nsrc; ++i) {
          const int64_t cnt = (xpart && ((J.x_mask >> i) & 1u)) ? poff : tl;
          if (cnt > 0) bulk_load(stage + i * T, J.src[i] + g0, (uint32_t)(cnt * 16), &full[s]);
        }
      }
    }
    // end marker (also sent after an abort so consumers exit)
    {
      const int s = (int)(k % kStages);
      if (ok && k >= kStages) {
        const uint32_t par = (uint32_t)(((k / kStages) - 1) & 1);
        uint32_t spins = 0;
        while (!mbar_try_wait(&empty[s], par))
          if ((++spins & 1023u) == 0 && *reinterpret_cast<volatile uint32_t*>(p.abort_flag)) break;
      }
      desc[s].nsrc = 0;
      if (!ok) *abort_s = 1;
      mbar_arrive_tx(&full[s], 0);
    }
    if (tr) {
      uint64_t* Tr = p.trace + (size_t)blockIdx.x * kTraceWords;
      Tr[kTrProdTotal] = globaltimer_ns() - t_start;
      Tr[kTrProdFlagWait] = tr_flag;
      Tr[kTrProdEmptyWait] = tr_empty;
      Tr[kTrProdTiles] = (uint64_t)k;
      Tr[kTrSmid] = smid();
      Tr[kTrEntryAbs] = t_entry;
    }
    return;
  }

  // ================================================ consumers (+ storer)
  const int ct = tid - kConsumerTid0;
  const bool storer = ct == 0;
  const bool tr = storer && p.trace != nullptr;
  uint64_t tr_full = 0, tr_sync = 0, tr_read = 0, tr_flush = 0, tr_bytes = 0;
  // per-phase tile time (trace): five scalars, not an array indexed by the run-time phase (stack)
  uint64_t tr_pA = 0, tr_pB = 0, tr_pC = 0, tr_pD = 0, tr_pE = 0;
  uint64_t tr_jobs = 0;
  const uint64_t t_start = tr ? globaltimer_ns() : 0;
  int64_t freed = -1;  // bulk mode: highest tile whose stage was returned to the producer
  // bulk mode: the last completed job whose release waits for its bulk stores.
  // It is released once a newer tile's stores are in flight (wait_group with
  // one newer group pending), or as soon as the storer would otherwise idle:
  // a held release may be what a peer waits for before it can feed us.
  int64_t committed = 0;  // bulk groups committed by the storer
  bool pending = false;   // a held job's release is reserved at the ring's tail (reserve_release)
  int64_t pend_g = 0;     // its last group's sequence number
  auto flush_pending = [&](int64_t newer) {
    if (!pending) return;
    bulk_wait_upto(newer);
    fence_async_global();  // the async-proxy (bulk) writes before the generic handoff
    commit_release(ring);
    pending = false;
  };
  for (int64_t k = 0;; ++k) {
    const int s = (int)(k % kStages);
    const uint32_t par = (uint32_t)((k / kStages) & 1);
    uint32_t spins = 0;
    const uint64_t tf = tr ? globaltimer_ns() : 0;
    bool aborted = false;
    while (!mbar_try_wait(&full[s], par)) {
      if (!kLsuStore && storer && pending) flush_pending(0);  // do not hold a release while idle
      if ((++spins & 1023u) == 0 && *reinterpret_cast<volatile uint32_t*>(p.abort_flag)) {
        aborted = true;
        break;
      }
    }
    if (aborted) break;
    const uint64_t t_tile = tr ? globaltimer_ns() : 0;
    if (tr) tr_full += t_tile - tf;
    const TileDesc& d = desc[s];
    const int nsrc = d.nsrc;
    if (nsrc == 0) break;
    const int64_t T = d.T, tl = d.tl, poff = d.poff;
    const int ndst = d.ndst, nrel = d.nrel, ph = d.ph;
    const uint32_t rmask = d.recv_mask;
    uint4* dst0 = d.dst[0];
    uint4* dst1 = d.dst[1];
    uint4* stage = reinterpret_cast<uint4*>(smem + (size_t)s * kStageBytes);
    if constexpr (kLsuStore) {
      for (int64_t i = ct; i < tl; i += kConsumers) {
        uint4 v;
        if (nsrc > 1) {  // canonical-order reduction in registers
          typename O::Acc acc;
          O::init(acc, stage[i]);
          for (int q = 1; q < nsrc; ++q) O::add(acc, stage[q * T + i]);
          v = O::narrow(acc);
        } else {
          v = stage[i];
        }
        for (int dd = 0; dd < ndst; ++dd) {
          uint4* dp = dd == 0 ? dst0 : (dd == 1 ? dst1 : d.dst[dd]);
          if (i == poff && ((rmask >> dd) & 1u))
            store_partial(dp + i, v, x.msg.partial_bytes);
          else
            st_cg(dp + i, v);
        }
      }
      const uint64_t ts = tr ? globaltimer_ns() : 0;
      consumers_sync();  // every consumer has read the stage and issued its stores
      if (tr) tr_sync += globaltimer_ns() - ts;
      if (storer) {
        if (nrel > 0) {  // job complete: hand its releases to the releaser warps
          const uint64_t tw = tr ? globaltimer_ns() : 0;
          publish_release(ring, rel_rec, d.rel, nrel);
          if (tr) tr_flush += globaltimer_ns() - tw;
        }
        mbar_arrive(&empty[s]);
      }
    } else {
      if (nsrc > 1) {  // canonical-order reduction, in place into slot 0
        for (int64_t i = ct; i < tl; i += kConsumers) {
          typename O::Acc acc;
          O::init(acc, stage[i]);
          for (int q = 1; q < nsrc; ++q) O::add(acc, stage[q * T + i]);
          stage[i] = O::narrow(acc);
        }
        fence_async_smem();
      }
      const uint64_t ts = tr ? globaltimer_ns() : 0;
      consumers_sync();
      if (tr) tr_sync += globaltimer_ns() - ts;
      if (storer) {
        for (int dd = 0; dd < ndst; ++dd) {
          uint4* dp = d.dst[dd];
          int64_t cnt = tl;
          if (poff >= 0 && ((rmask >> dd) & 1u)) {
            store_partial(dp + poff, stage[poff], x.msg.partial_bytes);
            cnt = poff;
          }
          if (cnt > 0) bulk_store(dp, stage, (uint32_t)(cnt * 16));
        }
        bulk_commit();
        ++committed;
        const uint64_t tq = tr ? globaltimer_ns() : 0;
        bulk_wait_read1();  // every store group but this tile's has read its smem
        if (tr) tr_read += globaltimer_ns() - tq;
        if (k >= 1 && k - 1 > freed) {  // the previous stage (and its descriptor) back to the producer
          mbar_arrive(&empty[(k - 1) % kStages]);
          freed = k - 1;
        }
        const uint64_t tw = tr ? globaltimer_ns() : 0;
        flush_pending(committed - pend_g);  // the held job's groups are older than this tile's
        if (nrel > 0) {  // job complete: hold its release until its bulk stores are done
          reserve_release(ring, rel_rec, d.rel, nrel);  // this stage's descriptor: freed only at tile k+1
          pending = true;
          pend_g = committed;
        }
        if (tr) tr_flush += globaltimer_ns() - tw;
      }
    }
    if (tr) {
      const uint64_t dt = globaltimer_ns() - t_tile;
      switch (ph) {
        case 0: tr_pA += dt; break;
        case 1: tr_pB += dt; break;
        case 2: tr_pC += dt; break;
        case 3: tr_pD += dt; break;
        default: tr_pE += dt; break;
      }
      tr_bytes += (uint64_t)tl * 16 * ndst;
      if (nrel) ++tr_jobs;
    }
  }
  if (!kLsuStore && storer) {
    flush_pending(0);
    bulk_wait_all();
  }
  if (storer) {
    __threadfence_block();
    ring->done = 1;
  }
  if (tr) {
    uint64_t* Tr = p.trace + (size_t)blockIdx.x * kTraceWords;
    Tr[kTrStoreTotal] = globaltimer_ns() - t_start;
    Tr[kTrStoreFullWait] = tr_full;
    Tr[kTrStoreSync] = tr_sync;
    Tr[kTrStoreFlush] = tr_flush;
    Tr[kTrStoreJobs] = tr_jobs;
    Tr[kTrPhaseA] = tr_pA;
    Tr[kTrPhaseB] = tr_pB;
    Tr[kTrPhaseC] = tr_pC;
    Tr[kTrPhaseD] = tr_pD;
    Tr[kTrPhaseE] = tr_pE;
    Tr[kTrBytes] = tr_bytes;
  }
}

}  // namespace tma
}  // namespace lane
