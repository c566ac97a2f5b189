// lane_ll.cuh — low-latency (LL) protocol kernel of the multi-lane allreduce
// for small and mid-size messages (sm_100a).
//
// Same method, partition and canonical reduction order as lane_tma.cuh /
// lane_kernels.cuh (Alg. 2: reduce-scatter on comm_group
// P L243, allreduce on comm_lane P L246, allgather on comm_group P L248; k
// slices, P L330-349 / L364-373). What differs is the signalling: the TMA
// engine publishes a flag per job after a system-scope fence, and that fence
// waits for every store the SM still has in flight — at small sizes every
// hop of every chunk pays it. Here every 16-byte granule travels as one
// 256-bit LL packet of four 64-bit words {data_i | epoch << 32}: each 64-bit
// word is a single-copy-atomic access, so a reader that sees the call's
// epoch in all four words holds the granule's data. No fences, no flags,
// no per-job round trip; the price is 2x the bytes on NVLink, which is why
// this protocol serves only messages up to LANE_LL_MAX_BYTES.
//
// Inboxes (per rank, per parity set, indexed chunk * stride + granule):
//   L1[s]  s < G-1 : part g of a chunk from node peer h (slot s = h<g ? h : h-1)  phase 1
//   L2[b]  b < N   : sub-part a of part g, node sum of (b,g)                    phase 2 RS
//   L3[b]  b < N   : sub-part b of part g, lane result of (b,g)                 phase 2 AG
//   L4[s]  s < G-1 : part h from node peer h (slot as L1)                       phase 3 AG
// Parity set = epoch & 1. A sender writes set e&1 in call e; the receiver
// read that set in call e-2 and finished it before it began call e-1, which
// every rank's call e-1 result depends on (allreduce), so the sender only
// reaches call e after the receiver is done with it — no credits needed.
//
// Phases per CTA (chunks j, j+C, ... of slice l; phase-major):
//   A  x[part gd]                         -> L1 of (a,gd)           (push)
//   B  sum_h (h==g ? x : L1[h]) sub-part b -> L2[a] of (b,g)        (push; own last)
//   C  sum_b L2[b] = F (sub-part a)        -> recvbuf, L3[a] of (b,g) b!=a, L4 of (a,h) h!=g
//   D  L3[b] (b != a)                      -> recvbuf, L4 of (a,h) h!=g  (phase 3 forward)
//   E  L4[h] (h != g)                      -> recvbuf
// A thread waits only on peers' earlier phases of the same chunk (handled by
// the same CTA index on every rank), so with every CTA resident no wait is
// cyclic; no intra-CTA barrier is needed (every packet carries its own flag).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_kernels.cuh"
#include "lane_plan.h"

namespace lane {
namespace ll {

#ifndef LANE_LL_MIN_BLOCKS  // CTAs per SM the register budget is sized for
#define LANE_LL_MIN_BLOCKS 1
#endif
constexpr int kThreads = 512;
constexpr int kPacketBytes = 32;  // one granule (16 B) + four 32-bit epochs

__device__ __forceinline__ void ll_store(uint64_t* line, const uint4& v, uint32_t ep) {
  const uint64_t e = (uint64_t)ep << 32;
  asm volatile("st.volatile.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(line), "l"(e | v.x), "l"(e | v.y),
               "l"(e | v.z), "l"(e | v.w)
               : "memory");
}

__device__ __forceinline__ bool ll_try(const uint64_t* line, uint32_t ep, uint4& v) {
  uint64_t a, b, c, d;
  asm volatile("ld.volatile.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(line)
               : "memory");
  v = make_uint4((uint32_t)a, (uint32_t)b, (uint32_t)c, (uint32_t)d);
  return (uint32_t)(a >> 32) == ep && (uint32_t)(b >> 32) == ep && (uint32_t)(c >> 32) == ep &&
         (uint32_t)(d >> 32) == ep;
}

// Result of a slow-path wait, returned BY VALUE: an out-parameter reference
// into a non-inlined function forces the caller's value (and its neighbours
// in arrays) through the stack (STL/LDL on the hot path).
struct Got {
  uint4 v;
  int ok;
};

// Spin until the packet carries this call's epoch; ok = 0 on timeout/abort.
__device__ __noinline__ Got ll_wait_slow(const LaneParams& p, const uint64_t* line) {
  const uint64_t t0 = globaltimer_ns();
  Got r;
  r.ok = 0;
  for (uint32_t it = 1;; ++it) {
    if (ll_try(line, cur_epoch(), r.v)) {
      r.ok = 1;
      return r;
    }
    if ((it & 255u) == 0) {
      if (*reinterpret_cast<volatile uint32_t*>(p.abort_flag)) return r;
      if (globaltimer_ns() - t0 > p.timeout_ns) {
        atomicExch(p.abort_flag, 1u);
        *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_TIMEOUT);
        __threadfence_system();
        return r;
      }
    }
  }
}

__device__ __forceinline__ bool ll_wait(const LaneParams& p, const uint64_t* line, uint4& v) {
  if (ll_try(line, cur_epoch(), v)) return true;
  const Got r = ll_wait_slow(p, line);
  v = r.v;
  return r.ok != 0;
}

// acc = sum over sources s = 0..n-1 in ascending order (the canonical order,
// R#7) of source s's granule: s == own is the local value own_v, every other
// source an LL packet at line(s). All packet loads of a batch are issued
// before any of them is waited on, so a granule pays one load latency, not n.
template <class O, class LineF>
__device__ __forceinline__ bool ll_sum(const LaneParams& p, int n, int own, const uint4& own_v, LineF line,
                                       typename O::Acc& acc) {
  constexpr int B = 2;
  for (int s0 = 0; s0 < n; s0 += B) {
    uint4 v[B];
    bool hit[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int s = s0 + u;
      hit[u] = true;
      if (s < n && s != own) hit[u] = ll_try(line(s), cur_epoch(), v[u]);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int s = s0 + u;
      if (s < n) {
        if (s == own) {
          v[u] = own_v;
        } else if (!hit[u]) {
          const Got t = ll_wait_slow(p, line(s));
          if (!t.ok) return false;
          v[u] = t.v;
        }
        if (s == 0)
          O::init(acc, v[u]);
        else
          O::add(acc, v[u]);
      }
    }
  }
  return true;
}

// Packet address of granule i of chunk c in an inbox slot.
struct Inbox {
  uint64_t* base;  // rank's LL region, current parity set
  int64_t sg, su;  // chunk strides (granules) of group-part / sub-part slots
  int64_t slot_g, slot_u;
  int G, N, cap;
  __device__ __forceinline__ uint64_t* at(int64_t slot_off, int64_t chunk_stride, int64_t c, int64_t i) const {
    return base + (slot_off + c * chunk_stride + i) * 4;
  }
  __device__ __forceinline__ uint64_t* l1(int s, int64_t c, int64_t i) const {
    return at((int64_t)s * slot_g, sg, c, i);
  }
  __device__ __forceinline__ uint64_t* l2(int b, int64_t c, int64_t i) const {
    return at((int64_t)(G - 1) * slot_g + (int64_t)b * slot_u, su, c, i);
  }
  __device__ __forceinline__ uint64_t* l3(int b, int64_t c, int64_t i) const {
    return at((int64_t)(G - 1) * slot_g + (int64_t)(N + b) * slot_u, su, c, i);
  }
  __device__ __forceinline__ uint64_t* l4(int s, int64_t c, int64_t i) const {
    return at((int64_t)(G - 1) * slot_g + (int64_t)(2 * N) * slot_u + (int64_t)s * slot_g, sg, c, i);
  }
};

// Granules per parity set (host and device agree on this layout).
LANE_HD int64_t set_granules(int G, int N, int64_t slot_g, int64_t slot_u) {
  return 2 * (int64_t)(G - 1) * slot_g + 2 * (int64_t)N * slot_u;
}

__device__ __forceinline__ uint64_t* set_base(const LaneParams& p, const RankMem& m) {
  return reinterpret_cast<uint64_t*>(m.ll) + (int64_t)(cur_epoch() & 1u) * p.ll_set * 4;
}

__device__ __forceinline__ Inbox inbox_of(const LaneParams& p, const RankMem& m) {
  Inbox b;
  b.base = set_base(p, m);
  b.sg = p.sg;
  b.su = p.su;
  b.slot_g = p.ll_slot_g;
  b.slot_u = p.ll_slot_u;
  b.G = p.G;
  b.N = p.N;
  return b;
}

// LANE_TRACE=1: per CTA, the kernel-start time and the time the LAST thread
// of the CTA finished each phase (A..E), in trace words 0..5 (ns, globaltimer).
// Per-CTA phase end times (LANE_TRACE=1) in a __shared__ array; holds only
// the kernel parameters' address and the array's, both re-derivable, so no
// register stays live across the phases for it (p.trace is re-read at use).
struct PhaseClock {
  const LaneParams* p;
  uint64_t* t;  // shared: [0] start, [1..5] phase ends
  __device__ __forceinline__ void end(int ph) const {
    if (p->trace != nullptr)
      atomicMax(reinterpret_cast<unsigned long long*>(&t[ph]), (unsigned long long)globaltimer_ns());
  }
};

__device__ __forceinline__ PhaseClock phase_clock_begin(const LaneParams& p, uint64_t* sh, uint64_t t_entry) {
  PhaseClock pc{&p, sh};
  if (p.trace != nullptr) {
    if (threadIdx.x < 8) sh[threadIdx.x] = threadIdx.x == 0 ? globaltimer_ns() : (threadIdx.x == 6 ? t_entry : 0);
    __syncthreads();
  }
  return pc;
}

__device__ __forceinline__ void phase_clock_flush(const LaneParams& p, const PhaseClock& pc) {
  if (p.trace == nullptr) return;
  __syncthreads();
  if (threadIdx.x < 8) p.trace[(size_t)blockIdx.x * kTraceWords + threadIdx.x] = pc.t[threadIdx.x];
  if (threadIdx.x == 0) p.trace[(size_t)blockIdx.x * kTraceWords + kTrSmid] = smid();
  if (threadIdx.x == 0) p.trace[(size_t)blockIdx.x * kTraceWords + kTrEntryAbs] = pc.t[6];
}

// RING2: the inter-node stage is Alg. 1 (LANE_PHASE2=ring; p.ring2), a
// separate instantiation so the default kernel keeps its register budget.
template <int DT, bool RING2 = false>
__global__ void __launch_bounds__(kThreads, LANE_LL_MIN_BLOCKS) lane_ll_kernel(const __grid_constant__ LaneParams p) {
  const uint64_t t_entry = launch_prologue(p);
  __shared__ uint64_t clk[8];
  const PhaseClock pc = phase_clock_begin(p, clk, t_entry);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int rank = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int64_t j = blockIdx.x % p.C;
  const int G = p.G, N = p.N;
  const int a = rank / G, g = rank % G;
  const uint32_t ep = cur_epoch();
  const int tid = threadIdx.x;
  constexpr int nthr = kThreads;

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(p.rk[rank].send);
  msg.recv = reinterpret_cast<uint4*>(p.rk[rank].recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sl = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  auto geo = [&](int64_t c) {
    ChunkGeo ch;
    ch.id = cb + c;
    ch.g0 = p.round_g0 + sl.start + c * p.cg;
    const int64_t rest = sl.len - c * p.cg;
    ch.len = rest < p.cg ? rest : p.cg;
    return ch;
  };
  const Inbox me = inbox_of(p, p.rk[rank]);
  auto slot_of = [&](int h, int dst_g) { return h < dst_g ? h : h - 1; };  // sender h in dst's L1/L4

  // ---------------- A: phase-1 push of the node peers' parts
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    for (int t = 1; t < G; ++t) {
      const int gd = (g + t) % G;
      const Span pd = rf_split(ch.len, G, gd);
      const Inbox dst = inbox_of(p, p.rk[a * G + gd]);
      const int s = slot_of(g, gd);
      for (int64_t i = tid; i < pd.len; i += nthr) ll_store(dst.l1(s, ch.id, i), load_x(msg, ch.g0 + pd.start + i), ep);
    }
  }

  pc.end(1);
  if constexpr (RING2) {
    // ---------------- B'/C'/D' (LANE_PHASE2=ring): the inter-node stage is
    // Alg. 1 among the lane members (P L401, L457: "the ring algorithm is
    // used in the inter-node stage"). Ring chunk t = sub-part t of part g;
    // lane member a sends to a+1. RS step s uses slot L2[s], AG step s L3[s].
    // T1 (the node sum, ascending h, one rounding) is formed on demand at the
    // ring chunk the step needs; every completed granule goes to recvbuf and
    // is forwarded to the node peers (phase 3).
    const Inbox nxt = inbox_of(p, p.rk[((a + 1) % N) * G + g]);
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      const Span gp = rf_split(ch.len, G, g);
      const int64_t width = ceil_div(gp.len, N);
      for (int64_t i = tid; i < width; i += nthr) {
        bool ok = true;
        auto t1 = [&](int t, uint4& out) {  // node sum at granule i of ring chunk t
          const int64_t gi = rf_split(gp.len, N, t).start + i;
          typename O::Acc acc;
          const uint4 xv = load_x(msg, ch.g0 + gp.start + gi);
          if (!ll_sum<O>(p, G, g, xv, [&](int h) { return me.l1(slot_of(h, g), ch.id, gi); }, acc)) return false;
          out = O::narrow(acc);
          return true;
        };
        auto deliver = [&](int t, const uint4& v) {  // final value of ring chunk t: recvbuf + phase 3
          const int64_t gi = rf_split(gp.len, N, t).start + i;
          store_out(msg, ch.g0 + gp.start + gi, v);
          for (int t2 = 1; t2 < G; ++t2) {
            const int h = (g + t2) % G;
            ll_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, gi), v, ep);
          }
        };
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < rf_split(gp.len, N, a).len) ok = t1(a, v);
        for (int s = 0; s < N - 1 && ok; ++s) {  // reduce-scatter loop (P L175-188)
          const int sp = ((a - s) % N + N) % N, rp = ((a - 1 - s) % N + N) % N;
          if (i < rf_split(gp.len, N, sp).len) ll_store(nxt.l2(s, ch.id, i), v, ep);
          if (i < rf_split(gp.len, N, rp).len) {
            uint4 w, own;
            if (!ll_wait(p, me.l2(s, ch.id, i), w) || !t1(rp, own)) {
              ok = false;
              break;
            }
            typename O::Acc acc;
            O::init(acc, w);
            O::add(acc, own);
            v = O::narrow(acc);  // one rounding per hop (R#11)
          }
        }
        if (!ok) return;
        if (i < rf_split(gp.len, N, (a + 1) % N).len) deliver((a + 1) % N, v);
        for (int s = 0; s < N - 1; ++s) {  // allgather loop (P L190-203)
          const int sp = ((a + 1 - s) % N + N) % N, rp = ((a - s) % N + N) % N;
          if (i < rf_split(gp.len, N, sp).len) ll_store(nxt.l3(s, ch.id, i), v, ep);
          if (i < rf_split(gp.len, N, rp).len) {
            if (!ll_wait(p, me.l3(s, ch.id, i), v)) return;
            deliver(rp, v);
          }
        }
      }
    }
  } else {

  // ---------------- B: phase-1 reduce (ascending h) -> phase-2 reduce-scatter push
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const Span gp = rf_split(ch.len, G, g);
    for (int t = 1; t <= N; ++t) {
      const int b = (a + t) % N;  // remote sub-parts first, own last
      const Span up = rf_split(gp.len, N, b);
      const Inbox dst = inbox_of(p, p.rk[b * G + g]);
      for (int64_t i = tid; i < up.len; i += nthr) {
        const int64_t gi = up.start + i;  // granule within part g
        typename O::Acc acc;
        const uint4 xv = load_x(msg, ch.g0 + gp.start + gi);
        if (!ll_sum<O>(p, G, g, xv, [&](int h) { return me.l1(slot_of(h, g), ch.id, gi); }, acc)) return;
        ll_store(dst.l2(a, ch.id, i), O::narrow(acc), ep);
      }
    }
  }

  pc.end(2);
  // ---------------- C: phase-2 reduce (ascending b) -> recvbuf + lane AG + phase-3 forward
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const Span gp = rf_split(ch.len, G, g);
    const Span up = rf_split(gp.len, N, a);
    for (int64_t i = tid; i < up.len; i += nthr) {
      typename O::Acc acc;
      if (!ll_sum<O>(p, N, -1, make_uint4(0, 0, 0, 0), [&](int b) { return me.l2(b, ch.id, i); }, acc)) return;
      const uint4 f = O::narrow(acc);
      store_out(msg, ch.g0 + gp.start + up.start + i, f);
      for (int t = 1; t < N; ++t) {
        const int b = (a + t) % N;
        ll_store(inbox_of(p, p.rk[b * G + g]).l3(a, ch.id, i), f, ep);
      }
      for (int t = 1; t < G; ++t) {
        const int h = (g + t) % G;
        ll_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, up.start + i), f, ep);
      }
    }
  }

  pc.end(3);
  // ---------------- D: phase-2 allgather receive -> recvbuf + phase-3 forward
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const Span gp = rf_split(ch.len, G, g);
    for (int t = 1; t < N; ++t) {
      const int b = (a + t) % N;
      const Span up = rf_split(gp.len, N, b);
      for (int64_t i = tid; i < up.len; i += nthr) {
        uint4 v;
        if (!ll_wait(p, me.l3(b, ch.id, i), v)) return;
        store_out(msg, ch.g0 + gp.start + up.start + i, v);
        for (int t2 = 1; t2 < G; ++t2) {
          const int h = (g + t2) % G;
          ll_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, up.start + i), v, ep);
        }
      }
    }
  }

  pc.end(4);
  }  // !RING2

  // ---------------- E: phase-3 allgather receive
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    for (int t = 1; t < G; ++t) {
      const int h = (g + t) % G;
      const Span ph = rf_split(ch.len, G, h);
      for (int64_t i = tid; i < ph.len; i += nthr) {
        uint4 v;
        if (!ll_wait(p, me.l4(slot_of(h, g), ch.id, i), v)) return;
        store_out(msg, ch.g0 + ph.start + i, v);
      }
    }
  }
  pc.end(5);
  phase_clock_flush(p, pc);
}

// ========================================================================
// Ring allreduce (Alg. 1 "ring_allreduce", P L150-206) on the LL
// protocol: the paper's "standard" algorithm (fig:std_vs_lane, P L393-401),
// and with k slices its "standard approach" with multiple processes per GPU
// (§3.1.1, P L335-349). Flat ring over all P ranks, rank r -> r+1.
//
// Chunk c of slice l is split into P ring parts D[0..P-1] (remainder-first,
// R#2). Reduce-scatter step s (s = 0..P-2): rank r sends part sp = r-s (its
// sendbuf part at s = 0, its running partial after) to r+1's RS slot s, and
// receives part rp = r-1-s from r-1, reducing it with its own sendbuf part in
// ONE hop in the buffer type (MPI_Reduce, P L177-181; bf16 rounds every hop,
// R#11). After P-1 steps rank r holds part r+1 complete. Allgather step s:
// send part r+1-s to r+1's AG slot s, receive part r-s. Each thread carries
// one granule index i through all 2(P-1) steps (its running value stays in
// registers); the LL packet of every hop is its own flag.
//
// Ring inbox of a rank (per parity set): RS slots s = 0..P-2, then AG slots,
// each ring_slot granules (p.ll_slot_g), chunk stride p.sg = ceil(cg/P).
LANE_HD int64_t ring_set_granules(int P, int64_t ring_slot) { return 2 * (int64_t)(P - 1) * ring_slot; }

template <int DT>
__global__ void __launch_bounds__(kThreads, LANE_LL_MIN_BLOCKS) lane_ring_ll_kernel(const __grid_constant__ LaneParams p) {
  launch_prologue(p);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int r = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int64_t j = blockIdx.x % p.C;
  const int P = p.P;
  const uint32_t ep = cur_epoch();
  const int tid = threadIdx.x;
  constexpr int nthr = kThreads;

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(p.rk[r].send);
  msg.recv = reinterpret_cast<uint4*>(p.rk[r].recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sl = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  uint64_t* const mine = set_base(p, p.rk[r]);
  uint64_t* const next = set_base(p, p.rk[(r + 1) % P]);
  const int64_t slot = p.ll_slot_g, cs = p.sg;
  auto rs = [&](uint64_t* b, int s, int64_t c, int64_t i) { return b + ((int64_t)s * slot + c * cs + i) * 4; };
  auto ag = [&](uint64_t* b, int s, int64_t c, int64_t i) {
    return b + ((int64_t)(P - 1 + s) * slot + c * cs + i) * 4;
  };

  for (int64_t c = j; c < nc; c += p.C) {
    const int64_t id = cb + c;
    const int64_t g0 = p.round_g0 + sl.start + c * p.cg;
    const int64_t clen = (sl.len - c * p.cg) < p.cg ? (sl.len - c * p.cg) : p.cg;
    const int64_t width = ceil_div(clen, P);  // longest part
    for (int64_t i = tid; i < width; i += nthr) {
      Span d = rf_split(clen, P, r);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (i < d.len) v = load_x(msg, g0 + d.start + i);
      // reduce-scatter loop (P L175-188)
      for (int s = 0; s < P - 1; ++s) {
        const int sp = ((r - s) % P + P) % P, rp = ((r - 1 - s) % P + P) % P;
        if (i < rf_split(clen, P, sp).len) ll_store(rs(next, s, id, i), v, ep);
        d = rf_split(clen, P, rp);
        if (i < d.len) {
          uint4 w;
          if (!ll_wait(p, rs(mine, s, id, i), w)) return;
          typename O::Acc acc;
          O::init(acc, w);
          O::add(acc, load_x(msg, g0 + d.start + i));
          v = O::narrow(acc);
        }
      }
      // rank r completed part r+1 (the last rp)
      d = rf_split(clen, P, (r + 1) % P);
      if (i < d.len) store_out(msg, g0 + d.start + i, v);
      // allgather loop (P L190-203)
      for (int s = 0; s < P - 1; ++s) {
        const int sp = ((r + 1 - s) % P + P) % P, rp = ((r - s) % P + P) % P;
        if (i < rf_split(clen, P, sp).len) ll_store(ag(next, s, id, i), v, ep);
        d = rf_split(clen, P, rp);
        if (i < d.len) {
          if (!ll_wait(p, ag(mine, s, id, i), v)) return;
          store_out(msg, g0 + d.start + i, v);
        }
      }
    }
  }
}

// ========================================================================
// "Approach 2" (commented-out draft of §3: "allreduce on
// node + allreduce off node") on the LL protocol: a direct node allreduce
// (reduce-scatter of part g, then every member gets every part of the node
// sum T) followed by a direct lane allreduce of the WHOLE chunk (lane part
// V_a reduced by (a,g) over b ascending, then gathered). Same association and
// rounding points as the lane method, so the same bits; 2(G-1)/G on node and
// 2(N-1)/N off node of the buffer per rank (the lane stage is not divided by G).
//
// Inboxes (per parity set): L1[G-1] (node RS, as the lane kernel), T[G] (node
// sum part h, from every node member incl. self: one thread's B result is
// another thread's C input, the packet is the hand-off), V2[N] (lane RS) and
// V3[N] (lane AG), chunk strides sg = ceil(cg/G) and sv = ceil(cg/N).
LANE_HD int64_t a2_set_granules(int G, int N, int64_t slot_g, int64_t slot_v) {
  return (int64_t)(2 * G - 1) * slot_g + 2 * (int64_t)N * slot_v;
}

template <int DT>
__global__ void __launch_bounds__(kThreads, LANE_LL_MIN_BLOCKS) lane_a2_ll_kernel(const __grid_constant__ LaneParams p) {
  launch_prologue(p);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int rank = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int64_t j = blockIdx.x % p.C;
  const int G = p.G, N = p.N;
  const int a = rank / G, g = rank % G;
  const uint32_t ep = cur_epoch();
  const int tid = threadIdx.x;
  constexpr int nthr = kThreads;

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(p.rk[rank].send);
  msg.recv = reinterpret_cast<uint4*>(p.rk[rank].recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sl = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  auto geo = [&](int64_t c) {
    ChunkGeo ch;
    ch.id = cb + c;
    ch.g0 = p.round_g0 + sl.start + c * p.cg;
    const int64_t rest = sl.len - c * p.cg;
    ch.len = rest < p.cg ? rest : p.cg;
    return ch;
  };
  const int64_t slot_g = p.ll_slot_g, slot_v = p.ll_slot_u, sg = p.sg, sv = p.su;
  auto L1 = [&](int r, int s, int64_t c, int64_t i) {
    return set_base(p, p.rk[r]) + ((int64_t)s * slot_g + c * sg + i) * 4;
  };
  auto T = [&](int r, int h, int64_t c, int64_t i) {
    return set_base(p, p.rk[r]) + ((int64_t)(G - 1 + h) * slot_g + c * sg + i) * 4;
  };
  auto V2 = [&](int r, int b, int64_t c, int64_t i) {
    return set_base(p, p.rk[r]) + ((int64_t)(2 * G - 1) * slot_g + (int64_t)b * slot_v + c * sv + i) * 4;
  };
  auto V3 = [&](int r, int b, int64_t c, int64_t i) {
    return set_base(p, p.rk[r]) + ((int64_t)(2 * G - 1) * slot_g + (int64_t)(N + b) * slot_v + c * sv + i) * 4;
  };
  auto slot_of = [&](int h, int dst_g) { return h < dst_g ? h : h - 1; };

  // ---------------- S1 push: node part gd of x -> (a,gd)
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    for (int t = 1; t < G; ++t) {
      const int gd = (g + t) % G;
      const Span pd = rf_split(ch.len, G, gd);
      for (int64_t i = tid; i < pd.len; i += nthr)
        ll_store(L1(a * G + gd, slot_of(g, gd), ch.id, i), load_x(msg, ch.g0 + pd.start + i), ep);
    }
  }
  // ---------------- S1 reduce (ascending h) + S2: node sum part g -> every node member's T[g]
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const Span gp = rf_split(ch.len, G, g);
    for (int64_t i = tid; i < gp.len; i += nthr) {
      typename O::Acc acc;
      const uint4 xv = load_x(msg, ch.g0 + gp.start + i);
      if (!ll_sum<O>(p, G, g, xv, [&](int h) { return L1(rank, slot_of(h, g), ch.id, i); }, acc)) return;
      const uint4 tv = O::narrow(acc);
      for (int t = 0; t < G; ++t) ll_store(T(a * G + (g + t) % G, g, ch.id, i), tv, ep);
    }
  }
  // ---------------- S3 push: lane part V_b of the node sum -> (b,g)'s V2[a]
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const int64_t base = ch.len / G, rem = ch.len % G, big = rem * (base + 1);
    for (int t = 1; t <= N; ++t) {
      const int b = (a + t) % N;  // own part last
      const Span vb = rf_split(ch.len, N, b);
      for (int64_t i = tid; i < vb.len; i += nthr) {
        const int64_t pos = vb.start + i;  // granule of the chunk -> its node part h
        const int h = pos < big ? (int)(pos / (base + 1)) : (int)(rem + (pos - big) / base);
        const int64_t hs = h < rem ? h * (base + 1) : big + (h - rem) * base;
        uint4 v;
        if (!ll_wait(p, T(rank, h, ch.id, pos - hs), v)) return;
        ll_store(V2(b * G + g, a, ch.id, i), v, ep);
      }
    }
  }
  // ---------------- S3 reduce (ascending b) -> recvbuf + S4 push to the lane
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    const Span va = rf_split(ch.len, N, a);
    for (int64_t i = tid; i < va.len; i += nthr) {
      typename O::Acc acc;
      if (!ll_sum<O>(p, N, -1, make_uint4(0, 0, 0, 0), [&](int b) { return V2(rank, b, ch.id, i); }, acc)) return;
      const uint4 f = O::narrow(acc);
      store_out(msg, ch.g0 + va.start + i, f);
      for (int t = 1; t < N; ++t) ll_store(V3(((a + t) % N) * G + g, a, ch.id, i), f, ep);
    }
  }
  // ---------------- S4 receive
  for (int64_t c = j; c < nc; c += p.C) {
    const ChunkGeo ch = geo(c);
    for (int t = 1; t < N; ++t) {
      const int b = (a + t) % N;
      const Span vb = rf_split(ch.len, N, b);
      for (int64_t i = tid; i < vb.len; i += nthr) {
        uint4 v;
        if (!ll_wait(p, V3(rank, b, ch.id, i), v)) return;
        store_out(msg, ch.g0 + vb.start + i, v);
      }
    }
  }
}

}  // namespace ll
}  // namespace lane
