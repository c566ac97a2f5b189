// lane_ll128.cuh — 128-byte-line low-latency protocol (LL128) kernel of the
// multi-lane allreduce for mid-size messages (sm_100a).
//
// Same method, partition and canonical reduction order as lane_ll.cuh and
// lane_tma.cuh (Alg. 2: reduce-scatter on comm_group
// P L243, allreduce on comm_lane P L246, allgather on comm_group P L248; k
// slices, P L330-349 / L364-373). What differs is the packet: the LL
// protocol pairs every 32-bit data word with a 32-bit epoch (2x the bytes on
// NVLink), which caps it near half the link rate; the simple protocol pays a
// system-scope fence per hop (5-30 us behind streaming remote stores,
// profiles/r01_fence_micro_p2.txt). Here a packet is one 128-byte line written
// by 8 consecutive lanes of a warp in ONE 16-byte-per-lane store instruction:
// lanes 0..6 carry 7 data granules, lane 7 the call's epoch in all four words
// (7/8 of the bytes are data). The reader loads the line with the same
// 8-lane pattern, lane 7 compares the epoch, and the 8 lanes agree through a
// warp shuffle. Correctness rests on the line being written and read as a
// unit (no tearing inside an aligned 128-byte line across NVLink); the PTX
// memory model does not state this, so it is an empirical property of the
// hardware (R#25), checked by the bit-exact stress tests.
//
// Inbox layout (per rank, per parity set; units = 128-byte lines):
// every chunk slot is line-aligned at SUB-PART granularity (lu = ceil(su/7)
// lines per sub-part), so that every phase — which all iterate over lane
// sub-parts — reads and writes the same line for the same granule.
//   L1[s] s < G-1 : part g of a chunk from node peer h, N sub-parts x lu lines
//   L2[b] b < N   : sub-part a of part g, node sum of (b,g), lu lines
//   L3[b] b < N   : sub-part b of part g, lane result of (b,g), lu lines
//   L4[s] s < G-1 : part h from node peer h, N sub-parts x lu lines
// Phases (A..E) and the parity-set argument are those of lane_ll.cuh. The
// lines live in their own region (RankMem::ll128), never shared with the LL
// packets: in it the last 16 bytes of a line only ever hold epochs.
// Also here: the ring allreduce (Alg. 1) on LL128 lines (lane_ring_ll128_kernel)
// and the lane kernel with Alg. 1 as its inter-node stage (RING2).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_kernels.cuh"
#include "lane_ll.cuh"
#include "lane_plan.h"

namespace lane {
namespace ll128 {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kPairGranules = 15;  // data granules per PAIR of 128-byte lines (15/16 of the bytes)
constexpr int kLineBytes = 128;
constexpr unsigned kFull = 0xffffffffu;

// Line pairs. Two consecutive 128-byte lines (an even line and the next) carry
// 15 granules: in line h (0 or 1) of pair pp, lanes 0-6 hold granules
// 15 pp + 7 h + 0..6 and lane 7 holds HALF of granule 15 pp + 14 (bytes 0-7
// in line 0, bytes 8-15 in line 1) followed by the 8-byte flag (the epoch
// twice). Every line still carries its own flag, so the line-atomicity
// reading R#25 is unchanged; the flag shrinks from 16 to 8 bytes. The two
// lines of a pair are always handled by adjacent 8-lane groups of one warp
// (flat positions 4u + grp with an even number of lines per sub-part, so the
// line's parity is grp & 1), and the two lane-7s swap halves with one shuffle.
LANE_HD int64_t lines_of(int64_t su) { return 2 * ceil_div(su, kPairGranules); }

// Granule of a sub-part (or ring part) carried by lane sl of line ln; lane 7
// of both lines of a pair carries the pair's shared granule 14.
LANE_HD int32_t line_granule(int32_t ln, int sl) {
  return kPairGranules * (ln >> 1) + (sl < 7 ? 7 * (ln & 1) + sl : 14);
}
// Whether lane sl of line ln stores its granule to the recvbuf (the shared
// granule once, from the pair's even line).
LANE_HD bool line_owner(int32_t ln, int sl) { return sl < 7 || (ln & 1) == 0; }

// Lines per parity set for a call: (G-1) L1 + (G-1) L4 slots of N*lu lines
// per chunk, N L2 + N L3 slots of lu lines per chunk.
LANE_HD int64_t set_lines(int G, int N, int64_t cap, int64_t lu) { return 2 * (int64_t)G * N * cap * lu; }

// Store this lane's 16 bytes of a line; v = the lane's granule (lane 7: the
// pair's shared granule, whole: the line's half of it goes with the flag).
__device__ __forceinline__ void line_store(uint4* line, int sl, const uint4& v, uint32_t ep) {
  const bool odd = (threadIdx.x >> 3) & 1;  // line parity within its pair (grp & 1)
  const uint4 w = sl == 7 ? (odd ? make_uint4(v.z, v.w, ep, ep) : make_uint4(v.x, v.y, ep, ep)) : v;
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(line + sl), "r"(w.x), "r"(w.y),
               "r"(w.z), "r"(w.w)
               : "memory");
}

__device__ __forceinline__ uint4 line_load(const uint4* line, int sl) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(line + sl)
               : "memory");
  return v;
}

// Warp-collective (every lane must call it, unconditionally): does the 8-lane
// group's line carry this call's epoch? Lane 7 of the group holds the flag
// words; every lane of the group gets the answer.
__device__ __forceinline__ bool group_ready(const uint4& v, int sl, uint32_t ep) {
  const bool f = sl == 7 && v.z == ep && v.w == ep;
  return __shfl_sync(kFull, f, (int)(threadIdx.x & 31) | 7);
}

// Warp-collective wait: groups with `need` reload their line until it carries
// the epoch; v = this lane's 16 bytes of the line as loaded so far. Returns the
// line (ok = 0 on timeout/abort, warp-uniform) BY VALUE (ll::Got): a reference
// out-parameter of a non-inlined function put the caller's loaded lines on
// the stack (STL.128 after every load, profiles/r01_sass_ll128.txt).
__device__ __noinline__ ll::Got wait_line(const LaneParams& p, const uint4* line, int sl, bool need, uint4 v) {
  const uint64_t t0 = globaltimer_ns();
  bool got = !need;
  ll::Got res;
  res.ok = 0;
  for (uint32_t it = 1;; ++it) {
    if (!got) v = line_load(line, sl);
    const bool r = group_ready(v, sl, cur_epoch());
    got = got || r;
    if (__all_sync(kFull, got)) {
      res.v = v;
      res.ok = 1;
      return res;
    }
    if ((it & 255u) == 0) {
      bool quit = *reinterpret_cast<volatile uint32_t*>(p.abort_flag) != 0;
      if (!quit && globaltimer_ns() - t0 > p.timeout_ns) {
        atomicExch(p.abort_flag, 1u);
        *reinterpret_cast<volatile uint32_t*>(p.err) = (uint32_t)(-LANE_ERR_TIMEOUT);
        __threadfence_system();
        quit = true;
      }
      if (__any_sync(kFull, quit)) {
        res.v = v;
        return res;
      }
    }
  }
}

// U: lines per 8-lane group per warp step (loads in flight per lane); a
// template parameter of the kernels: the host takes U = 1 for small messages
// (one warp step covers fewer lines, so more warps get work) and U = 2 above.
#ifndef LANE_LL128_U
#define LANE_LL128_U 2
#endif

// A warp step's U lines per 8-lane group: flat position, the line's
// pointer(s), whether the line exists (act: its pair holds data of the span)
// and whether this lane holds a data granule of the span (dv).
template <int U>
struct BatchT {
  bool act[U], dv[U], own[U];  // own: dv and this lane stores the granule to the recvbuf (line_owner)
  int t[U], b[U];
  int32_t ln[U], i[U];  // line in the sub-part, chunk-relative granule (< 2^31: 32-bit, fewer registers)
};

// Issue the loads of U lines (inactive lines read as zero, never loaded).
template <int U>
__device__ __forceinline__ void fetch_lines(const uint4* const (&ptr)[U], const bool (&act)[U], int sl, uint4 (&v)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = act[u] ? line_load(ptr[u], sl) : make_uint4(0, 0, 0, 0);
}

// Warp-collective: lane 7 of each line rebuilds the pair's shared granule
// from its own half and its partner line's (lane ^ 8).
template <int U>
__device__ __forceinline__ void unpack_lines(int sl, uint4 (&v)[U]) {
  const bool odd = (threadIdx.x >> 3) & 1;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t ox = __shfl_xor_sync(kFull, v[u].x, 8), oy = __shfl_xor_sync(kFull, v[u].y, 8);
    if (sl == 7) v[u] = odd ? make_uint4(ox, oy, v[u].x, v[u].y) : make_uint4(v[u].x, v[u].y, ox, oy);
  }
}

// Warp-collective: wait until every active fetched line carries the epoch
// (reloading the ones that did not yet), then unpack the shared granules.
template <int U>
__device__ __forceinline__ bool check_lines(const LaneParams& p, const uint4* const (&ptr)[U], const bool (&act)[U],
                                            int sl, uint4 (&v)[U]) {
  bool got[U], all = true;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool r = group_ready(v[u], sl, cur_epoch());
    got[u] = !act[u] || r;
    all = all && got[u];
  }
  if (!__all_sync(kFull, all)) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (!__all_sync(kFull, got[u])) {
        const ll::Got w = wait_line(p, ptr[u], sl, !got[u], v[u]);
        if (!w.ok) return false;
        v[u] = w.v;
      }
  }
  unpack_lines(sl, v);
  return true;
}

// Warp-collective: fetch U lines and wait until every active line carries the epoch.
template <int U>
__device__ __forceinline__ bool get_lines(const LaneParams& p, const uint4* const (&ptr)[U], const bool (&act)[U], int sl,
                                          uint4 (&v)[U]) {
  fetch_lines(ptr, act, sl, v);
  return check_lines(p, ptr, act, sl, v);
}

// Line index within a parity set of the lane kernel's inboxes for a call
// with cap chunks and lu lines per sub-part: (G-1) L1 slots, N L2 slots, N L3
// slots, (G-1) L4 slots; an L1/L4 slot is cap chunks x N sub-parts x lu
// lines, an L2/L3 slot cap chunks x lu lines. Host and device (the CPU tests
// check through lane_ll128_line_query that it tiles [0, set_lines) exactly).
struct Layout128 {
  int64_t slot_g, slot_u;  // lines per L1/L4 slot and per L2/L3 slot
  int64_t lu;              // lines per sub-part
  int G, N;
  LANE_HD int64_t l1(int s, int64_t c, int b, int64_t ln) const { return (int64_t)s * slot_g + (c * N + b) * lu + ln; }
  LANE_HD int64_t l2(int b, int64_t c, int64_t ln) const {
    return (int64_t)(G - 1) * slot_g + (int64_t)b * slot_u + c * lu + ln;
  }
  LANE_HD int64_t l3(int b, int64_t c, int64_t ln) const {
    return (int64_t)(G - 1) * slot_g + (int64_t)(N + b) * slot_u + c * lu + ln;
  }
  LANE_HD int64_t l4(int s, int64_t c, int b, int64_t ln) const {
    return (int64_t)(G - 1) * slot_g + (int64_t)(2 * N) * slot_u + (int64_t)s * slot_g + (c * N + b) * lu + ln;
  }
};

LANE_HD Layout128 layout128(int G, int N, int64_t cap, int64_t lu) {
  Layout128 y;
  y.slot_g = cap * N * lu;
  y.slot_u = cap * lu;
  y.lu = lu;
  y.G = G;
  y.N = N;
  return y;
}

// Line addresses of one rank's inbox (current parity set).
struct Inbox128 {
  uint4* base;  // set base (16-byte units)
  Layout128 y;
  __device__ __forceinline__ uint4* at(int64_t line) const { return base + line * 8; }
  __device__ __forceinline__ uint4* l1(int s, int64_t c, int b, int64_t ln) const { return at(y.l1(s, c, b, ln)); }
  __device__ __forceinline__ uint4* l2(int b, int64_t c, int64_t ln) const { return at(y.l2(b, c, ln)); }
  __device__ __forceinline__ uint4* l3(int b, int64_t c, int64_t ln) const { return at(y.l3(b, c, ln)); }
  __device__ __forceinline__ uint4* l4(int s, int64_t c, int b, int64_t ln) const { return at(y.l4(s, c, b, ln)); }
};

// p.ll_set = lines per parity set (stride); p.cap chunks, lu from p.su.
__device__ __forceinline__ Inbox128 inbox_of(const LaneParams& p, const RankMem& m) {
  Inbox128 b;
  b.base = reinterpret_cast<uint4*>(m.ll128) + (int64_t)(cur_epoch() & 1u) * p.ll_set * 8;
  b.y = layout128(p.G, p.N, p.cap, lines_of(p.su));
  return b;
}

// ------------------------------------------------------------------ host planner
// One-round LL128 call of ng granules, k CTA groups of at most C CTAs, inbox
// capacity M granules of message, minimum chunk cg_min: CTAs per group,
// chunk size (one chunk per CTA, k*CG <= M/4 — the sizing bound below), chunk
// count, lines per sub-part, and lines per parity set the call uses.
struct Plan128 {
  int C;
  int64_t cg, cap, lu, need;
};

inline Plan128 plan128(int G, int N, int k, int64_t ng, int C, int64_t M, int64_t cg_min) {
  Plan128 o;
  if (C < 1) C = 1;
  const int64_t slice0 = (ng + k - 1) / k;
  int64_t cg = (slice0 + C - 1) / C;
  // k*CG <= M/4 keeps the inbox sizing bound (set_capacity128): with fewer
  // than 4 CTAs per slice, CTAs take several chunks (phase-major)
  const int64_t cg_cap = M / (4 * k);
  if (cg > cg_cap) cg = cg_cap;
  if (cg < cg_min) cg = cg_min;
  const int64_t nch = n_chunks(slice0, cg);
  if (nch < C) C = (int)(nch > 0 ? nch : 1);
  o.C = C;
  o.cg = cg;
  o.cap = round_chunks(ng, k, cg);
  o.lu = lines_of(ceil_div(ceil_div(cg, G), N));
  o.need = set_lines(G, N, o.cap, o.lu);
  return o;
}

// Lines per parity set allocated at init. A call needs 2*G*N*cap*lu lines,
// lu = 2*ceil(su/15) <= 2*su/15 + 2; with G*N*su <= CG + G*N and
// cap*CG <= M + k*CG this is at most 4*(M + k*CG + cap*G*N)/15 + 4*cap*G*N
// lines; sized for k*CG <= M/4 (which plan128 keeps unless CG is the minimum
// chunk, covered by the k*cg_min term).
inline int64_t set_capacity128(int G, int N, int k, int64_t M, int64_t cg_min) {
  const int64_t chunks = M / cg_min + k + 1;
  return 2 * (2 * ceil_div(M + M / 4 + k * cg_min + chunks * G * N, kPairGranules) + 2 * (int64_t)G * N * chunks) + 64;
}

// RING2: the inter-node stage is Alg. 1 (LANE_PHASE2=ring; p.ring2), a separate
// instantiation so the default kernel keeps its register budget.
template <int DT, bool RING2 = false, int U = LANE_LL128_U>
__global__ void __launch_bounds__(kThreads, 1) lane_ll128_kernel(const __grid_constant__ LaneParams p) {
  const uint64_t t_entry = launch_prologue(p);
  using Batch = BatchT<U>;
  __shared__ uint64_t clk[8];
  const ll::PhaseClock pc = ll::phase_clock_begin(p, clk, t_entry);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int rank = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int64_t j = blockIdx.x % p.C;
  const int G = p.G, N = p.N;
  const int a = rank / G, g = rank % G;
  const uint32_t ep = cur_epoch();
  const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) >> 3, sl = threadIdx.x & 7;
  const int64_t lu = lines_of(p.su);
  const uint4 z = make_uint4(0, 0, 0, 0);

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(p.rk[rank].send);
  msg.recv = reinterpret_cast<uint4*>(p.rk[rank].recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sl_span = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sl_span.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  auto geo = [&](int64_t c) {
    ChunkGeo ch;
    ch.id = cb + c;
    ch.g0 = p.round_g0 + sl_span.start + c * p.cg;
    const int64_t rest = sl_span.len - c * p.cg;
    ch.len = rest < p.cg ? rest : p.cg;
    return ch;
  };
  const Inbox128 me = inbox_of(p, p.rk[rank]);
  auto slot_of = [&](int h, int dst_g) { return h < dst_g ? h : h - 1; };

  // Every phase walks a flat space of lines (t, b, ln) — t the peer step,
  // b the sub-part, ln the line in it (lu lines per sub-part, the unused
  // tail lines of shorter sub-parts inactive) — so all warps share the
  // phase's work; a warp step takes 4*U consecutive positions (U lines per
  // 8-lane group, positions V0 + 4u + grp). span(t, b) gives the sub-part's
  // granule span; the loop trip count is warp-uniform.
  auto walk = [&](int T, int NB, auto span, auto f) -> bool {
    const int64_t total = (int64_t)T * NB * lu;
    for (int64_t V0 = (int64_t)warp * 4 * U; V0 < total; V0 += kWarps * 4 * U) {
      Batch q;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = V0 + 4 * u + grp;
        q.act[u] = v < total;
        // positions stay far below 2^31 (total <= M/7 + G*N lines): 32-bit division
        const uint32_t v32 = q.act[u] ? (uint32_t)v : 0u, lu32 = (uint32_t)lu;
        const uint32_t r = v32 / lu32;
        q.ln[u] = (int32_t)(v32 - r * lu32);
        q.b[u] = (int)(r % (uint32_t)NB);
        q.t[u] = (int)(r / (uint32_t)NB);
        const Span up = span(q.t[u], q.b[u]);
        q.act[u] = q.act[u] && q.ln[u] < lines_of(up.len);
        q.i[u] = line_granule(q.ln[u], sl);
        q.dv[u] = q.act[u] && q.i[u] < up.len;
        q.own[u] = q.dv[u] && line_owner(q.ln[u], sl);
        q.i[u] += (int32_t)up.start;  // granule of the span's chunk-relative part
      }
      if (!f(q)) return false;
    }
    return true;
  };

  // The default path (not RING2) runs every phase through `phase`: warp step
  // s of chunk ch covers positions 4*U*s .. 4*U*s + 4*U - 1 of the chunk's
  // flat space; CTA j takes its chunks j, j+C, ..., warp w the steps w,
  // w + 16, ... (a static share). A pooled variant — the last half of every
  // chunk's steps claimed by any warp of the rank through per-phase atomic
  // counters, so fast SMs take the slow ones' tail (per-SM push rates differ
  // up to 2x, profiles/r02_trace_smid_p4.txt) — balanced the phase ends but
  // was slower at every size: the phases are link-bound, not
  // imbalance-bound.
  auto step = [&](const ChunkGeo& ch, int64_t s, int T, int NB, auto span, auto f) -> bool {
    const int64_t total = (int64_t)T * NB * lu;
    const int64_t V0 = s * 4 * U;
    Batch q;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = V0 + 4 * u + grp;
      q.act[u] = v < total;
      const uint32_t v32 = q.act[u] ? (uint32_t)v : 0u, lu32 = (uint32_t)lu;
      const uint32_t r = v32 / lu32;
      q.ln[u] = (int32_t)(v32 - r * lu32);
      q.b[u] = (int)(r % (uint32_t)NB);
      q.t[u] = (int)(r / (uint32_t)NB);
      const Span up = span(ch, q.t[u], q.b[u]);
      q.act[u] = q.act[u] && q.ln[u] < lines_of(up.len);
      q.i[u] = line_granule(q.ln[u], sl);
      q.dv[u] = q.act[u] && q.i[u] < up.len;
      q.own[u] = q.dv[u] && line_owner(q.ln[u], sl);
      q.i[u] += (int32_t)up.start;
    }
    return f(ch, q);
  };
  auto phase = [&](int T, int NB, auto span, auto f) -> bool {
    const int64_t ns = ceil_div((int64_t)T * NB * lu, 4 * U);  // warp steps per chunk
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      for (int64_t s = warp; s < ns; s += kWarps)
        if (!step(ch, s, T, NB, span, f)) return false;
    }
    return true;
  };

  // ---------------- A: phase-1 push of the node peers' parts. Flat order
  // (t, b, ln): t = sub-part order (sub-part (a+1+t) % N, the order phase B
  // consumes them in), b = destination (node peer gd = g+1+b), so the lines
  // every receiver needs first are pushed first by all its node peers.
  {
    auto span = [&](const ChunkGeo& ch, int t, int b) {
      const Span pd = rf_split(ch.len, G, (g + 1 + b) % G);
      Span up = rf_split(pd.len, N, (a + 1 + t) % N);
      up.start += pd.start;  // granule offset within the chunk
      return up;
    };
    phase(N, G - 1, span, [&](const ChunkGeo& ch, const Batch& q) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = q.dv[u] ? load_x(msg, ch.g0 + q.i[u]) : z;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q.act[u]) {
          const int gd = (g + 1 + q.b[u]) % G;
          line_store(inbox_of(p, p.rk[a * G + gd]).l1(slot_of(g, gd), ch.id, (a + 1 + q.t[u]) % N, q.ln[u]), sl,
                     x[u], ep);
        }
      return true;
    });
  }
  pc.end(1);

  if constexpr (RING2) {
    // ---------------- B'/C'/D' (LANE_PHASE2=ring): the inter-node stage is
    // Alg. 1 among the lane members (P L401, L457; R#22), as in lane_ll.cuh:
    // ring chunk t = sub-part t of part g, lane member a sends to a+1, RS
    // step s uses slot L2[s], AG step s L3[s]; the node sum T1 (ascending h,
    // one rounding) is formed on demand from the L1 lines; every completed
    // line goes to recvbuf and to the node peers' L4 (phase 3). An 8-lane
    // group carries line ln of every sub-part through all 2(N-1) steps.
    const Inbox128 nxt = inbox_of(p, p.rk[((a + 1) % N) * G + g]);
    for (int64_t c = j; c < nc; c += p.C) {
      const ChunkGeo ch = geo(c);
      const Span gp = rf_split(ch.len, G, g);
      auto widest = [&](int, int) { return Span{0, rf_split(gp.len, N, 0).len}; };  // remainder-first: sub-part 0
      const bool ok = walk(1, 1, widest, [&](const Batch& q) {
        auto up = [&](int x) { return rf_split(gp.len, N, x); };
        auto act = [&](int u, int x) { return q.act[u] && q.ln[u] < lines_of(up(x).len); };
        auto dv = [&](int u, int x) { return act(u, x) && line_granule(q.ln[u], sl) < up(x).len; };
        auto gidx = [&](int u, int x) { return ch.g0 + gp.start + up(x).start + line_granule(q.ln[u], sl); };
        // node sum of ring chunk x at this group's lines (warp-collective)
        auto t1 = [&](int x, uint4 (&out)[U]) -> bool {
          typename O::Acc acc[U];
          bool a_[U];
#pragma unroll
          for (int u = 0; u < U; ++u) a_[u] = act(u, x);
          for (int h = 0; h < G; ++h) {  // warp-uniform, ascending (R#7)
            uint4 v[U];
            if (h == g) {
#pragma unroll
              for (int u = 0; u < U; ++u) v[u] = dv(u, x) ? load_x(msg, gidx(u, x)) : z;
            } else {
              const uint4* ptr[U];
#pragma unroll
              for (int u = 0; u < U; ++u) ptr[u] = me.l1(slot_of(h, g), ch.id, x, q.ln[u]);
              if (!get_lines(p, ptr, a_, sl, v)) return false;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (h == 0)
                O::init(acc[u], v[u]);
              else
                O::add(acc[u], v[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) out[u] = O::narrow(acc[u]);
          return true;
        };
        auto deliver = [&](int x, const uint4 (&v)[U]) {  // final lines of ring chunk x: recvbuf + phase 3
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (dv(u, x) && line_owner(q.ln[u], sl)) store_out(msg, gidx(u, x), v[u]);
            if (act(u, x))
              for (int t2 = 1; t2 < G; ++t2) {
                const int h = (g + t2) % G;
                line_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, x, q.ln[u]), sl, v[u], ep);
              }
          }
        };
        uint4 v[U];
        if (!t1(a, v)) return false;
        for (int s = 0; s < N - 1; ++s) {  // reduce-scatter loop (P L175-188)
          const int sp = ((a - s) % N + N) % N, rp = ((a - 1 - s) % N + N) % N;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (act(u, sp)) line_store(nxt.l2(s, ch.id, q.ln[u]), sl, v[u], ep);
          const uint4* ptr[U];
          bool a_[U];
          uint4 w[U], own[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            ptr[u] = me.l2(s, ch.id, q.ln[u]);
            a_[u] = act(u, rp);
          }
          if (!get_lines(p, ptr, a_, sl, w)) return false;
          if (!t1(rp, own)) return false;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (a_[u]) {
              typename O::Acc acc;
              O::init(acc, w[u]);
              O::add(acc, own[u]);
              v[u] = O::narrow(acc);  // one rounding per hop (R#11)
            }
        }
        deliver((a + 1) % N, v);
        for (int s = 0; s < N - 1; ++s) {  // allgather loop (P L190-203)
          const int sp = ((a + 1 - s) % N + N) % N, rp = ((a - s) % N + N) % N;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (act(u, sp)) line_store(nxt.l3(s, ch.id, q.ln[u]), sl, v[u], ep);
          const uint4* ptr[U];
          bool a_[U];
          uint4 w[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            ptr[u] = me.l3(s, ch.id, q.ln[u]);
            a_[u] = act(u, rp);
          }
          if (!get_lines(p, ptr, a_, sl, w)) return false;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (a_[u]) v[u] = w[u];
          deliver(rp, v);
        }
        return true;
      });
      if (!ok) return;
    }
  } else {

  // ---------------- B: phase-1 reduce (ascending h) -> phase-2 reduce-scatter push
  // (t = 0..N-1 -> sub-part b = a+1+t: remote sub-parts first, own last)
  {
    auto span = [&](const ChunkGeo& ch, int t, int) {
      const Span gp = rf_split(ch.len, G, g);
      Span up = rf_split(gp.len, N, (a + 1 + t) % N);
      up.start += gp.start;
      return up;
    };
    const bool ok = phase(N, 1, span, [&](const ChunkGeo& ch, const Batch& q) {
      typename O::Acc acc[U];
      // the node's G terms two at a time: both terms' loads (own sendbuf or a
      // peer's lines) are in flight before the first epoch check — one round
      // trip per pair instead of one per term; summed ascending (R#7)
      auto fetch_term = [&](int h, const uint4* (&ptr)[U], uint4 (&v)[U]) {
        if (h == g) {
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = q.dv[u] ? load_x(msg, ch.g0 + q.i[u]) : z;
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) ptr[u] = me.l1(slot_of(h, g), ch.id, (a + 1 + q.t[u]) % N, q.ln[u]);
          fetch_lines(ptr, q.act, sl, v);
        }
      };
      for (int h0 = 0; h0 < G; h0 += 2) {  // warp-uniform
        const int h1 = h0 + 1;
        const uint4* p0[U];
        const uint4* p1[U];
        uint4 v0[U], v1[U];
        fetch_term(h0, p0, v0);
        if (h1 < G) fetch_term(h1, p1, v1);
        if (h0 != g && !check_lines(p, p0, q.act, sl, v0)) return false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (h0 == 0)
            O::init(acc[u], v0[u]);
          else
            O::add(acc[u], v0[u]);
        }
        if (h1 < G) {
          if (h1 != g && !check_lines(p, p1, q.act, sl, v1)) return false;
#pragma unroll
          for (int u = 0; u < U; ++u) O::add(acc[u], v1[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q.act[u]) {
          const int b = (a + 1 + q.t[u]) % N;
          line_store(inbox_of(p, p.rk[b * G + g]).l2(a, ch.id, q.ln[u]), sl, O::narrow(acc[u]), ep);
        }
      return true;
    });
    if (!ok) return;
  }
  pc.end(2);

  // ---------------- C: phase-2 reduce (ascending b) -> recvbuf + lane AG + phase-3 forward
  {
    auto span = [&](const ChunkGeo& ch, int, int) {
      const Span gp = rf_split(ch.len, G, g);
      Span up = rf_split(gp.len, N, a);
      up.start += gp.start;
      return up;
    };
    const bool ok = phase(1, 1, span, [&](const ChunkGeo& ch, const Batch& q) {
      typename O::Acc acc[U];
      for (int b0 = 0; b0 < N; b0 += 2) {  // warp-uniform; two lane terms in flight, ascending (R#7)
        const int b1 = b0 + 1;
        uint4 v0[U], v1[U];
        const uint4* p0[U];
        const uint4* p1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) p0[u] = me.l2(b0, ch.id, q.ln[u]);
        fetch_lines(p0, q.act, sl, v0);
        if (b1 < N) {
#pragma unroll
          for (int u = 0; u < U; ++u) p1[u] = me.l2(b1, ch.id, q.ln[u]);
          fetch_lines(p1, q.act, sl, v1);
        }
        if (!check_lines(p, p0, q.act, sl, v0)) return false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (b0 == 0)
            O::init(acc[u], v0[u]);
          else
            O::add(acc[u], v0[u]);
        }
        if (b1 < N) {
          if (!check_lines(p, p1, q.act, sl, v1)) return false;
#pragma unroll
          for (int u = 0; u < U; ++u) O::add(acc[u], v1[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint4 f = O::narrow(acc[u]);
        if (q.own[u]) store_out(msg, ch.g0 + q.i[u], f);
        if (q.act[u]) {
          for (int t = 1; t < N; ++t) {
            const int b = (a + t) % N;
            line_store(inbox_of(p, p.rk[b * G + g]).l3(a, ch.id, q.ln[u]), sl, f, ep);
          }
          for (int t = 1; t < G; ++t) {
            const int h = (g + t) % G;
            line_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, a, q.ln[u]), sl, f, ep);
          }
        }
      }
      return true;
    });
    if (!ok) return;
  }
  pc.end(3);

  // ---------------- D: phase-2 allgather receive -> recvbuf + phase-3 forward
  // (t = 0..N-2 -> lane peer b = a+1+t)
  if (N > 1) {
      auto span = [&](const ChunkGeo& ch, int t, int) {
        const Span gp = rf_split(ch.len, G, g);
        Span up = rf_split(gp.len, N, (a + 1 + t) % N);
        up.start += gp.start;
        return up;
      };
      const bool ok = phase(N - 1, 1, span, [&](const ChunkGeo& ch, const Batch& q) {
        uint4 v[U];
        const uint4* ptr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ptr[u] = me.l3((a + 1 + q.t[u]) % N, ch.id, q.ln[u]);
        if (!get_lines(p, ptr, q.act, sl, v)) return false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (q.own[u]) store_out(msg, ch.g0 + q.i[u], v[u]);
          if (q.act[u]) {
            const int b = (a + 1 + q.t[u]) % N;
            for (int t2 = 1; t2 < G; ++t2) {
              const int h = (g + t2) % G;
              line_store(inbox_of(p, p.rk[a * G + h]).l4(slot_of(g, h), ch.id, b, q.ln[u]), sl, v[u], ep);
            }
          }
        }
        return true;
      });
      if (!ok) return;
    }
  pc.end(4);
  }  // !RING2

  // ---------------- E: phase-3 allgather receive (t = 0..G-2 -> node peer h = g+1+t)
  {
    auto span = [&](const ChunkGeo& ch, int t, int b) {
      const Span ph = rf_split(ch.len, G, (g + 1 + t) % G);
      Span up = rf_split(ph.len, N, b);
      up.start += ph.start;
      return up;
    };
    const bool ok = phase(G - 1, N, span, [&](const ChunkGeo& ch, const Batch& q) {
      uint4 v[U];
      const uint4* ptr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) ptr[u] = me.l4(slot_of((g + 1 + q.t[u]) % G, g), ch.id, q.b[u], q.ln[u]);
      if (!get_lines(p, ptr, q.act, sl, v)) return false;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q.own[u]) store_out(msg, ch.g0 + q.i[u], v[u]);
      return true;
    });
    if (!ok) return;
  }
  pc.end(5);
  ll::phase_clock_flush(p, pc);
}


// ========================================================================
// Ring allreduce (Alg. 1 "ring_allreduce", P L150-206) on the LL128
// protocol: same algorithm, chunking (fixed ring chunks, R#21), rounds (the
// LL capacity, so both protocols give the same bits) and per-hop rounding
// (R#11) as lane_ring_ll_kernel; the packet is a 128-byte line. Chunk c of
// slice l is split into P ring parts (remainder-first); an 8-lane group
// carries one line of every part (granules 7 ln .. 7 ln + 6 of the part)
// through all 2(P-1) steps. Reduce-scatter step s: rank r sends its running
// partial of part r-s to r+1's RS slot s and reduces part r-1-s received from
// r-1 with its own sendbuf part; allgather step s: send part r+1-s to r+1's
// AG slot s, receive part r-s.
//
// Inbox (per parity set): RS slots s = 0..P-2 then AG slots, each
// cap * lp lines (lp = ceil(ceil(cg/P)/7) lines per ring part).
LANE_HD int64_t ring_set_lines(int P, int64_t cap, int64_t lp) { return 2 * (int64_t)(P - 1) * cap * lp; }

// Line index within a parity set of RS slot s / AG slot s, chunk c, line ln
// (host and device; tiled exactly, checked on CPU via lane_ll128_line_query).
struct RingLayout128 {
  int64_t slot, lp;  // lines per slot (cap * lp), lines per ring part
  int P;
  LANE_HD int64_t rs(int s, int64_t c, int64_t ln) const { return (int64_t)s * slot + c * lp + ln; }
  LANE_HD int64_t ag(int s, int64_t c, int64_t ln) const { return (int64_t)(P - 1 + s) * slot + c * lp + ln; }
};

LANE_HD RingLayout128 ring_layout128(int P, int64_t cap, int64_t lp) {
  RingLayout128 y;
  y.slot = cap * lp;
  y.lp = lp;
  y.P = P;
  return y;
}

template <int DT, int U = LANE_LL128_U>
__global__ void __launch_bounds__(kThreads, 1) lane_ring_ll128_kernel(const __grid_constant__ LaneParams p) {
  launch_prologue(p);
  using O = Ops<DT>;
  const int per_rank = p.k * p.C;
  const int r = p.rank0 + (int)(blockIdx.x / per_rank);
  const int l = (int)(blockIdx.x % per_rank) / p.C;
  const int j = (int)(blockIdx.x % p.C);
  const int P = p.P;
  const uint32_t ep = cur_epoch();
  const int warp = threadIdx.x >> 5, grp = (threadIdx.x & 31) >> 3, sl = threadIdx.x & 7;
  const int64_t lp = lines_of(p.sg);  // p.sg = ceil(cg / P): longest ring part
  const uint4 z = make_uint4(0, 0, 0, 0);

  Msg msg;
  msg.send = reinterpret_cast<const uint4*>(p.rk[r].send);
  msg.recv = reinterpret_cast<uint4*>(p.rk[r].recv);
  msg.partial_g = p.tail_elems < p.q ? p.ng - 1 : -1;
  msg.partial_bytes = p.tail_elems * (16 / p.q);

  const Span sls = rf_split(p.round_len, p.k, l);
  const int64_t nc = n_chunks(sls.len, p.cg);
  const int64_t cb = chunk_base(p.round_len, p.k, l, p.cg);
  const int64_t ncj = nc > j ? (nc - j + p.C - 1) / p.C : 0;  // chunks j, j+C, ... of this CTA
  uint4* const mine = reinterpret_cast<uint4*>(p.rk[r].ll128) + (int64_t)(ep & 1u) * p.ll_set * 8;
  uint4* const next = reinterpret_cast<uint4*>(p.rk[(r + 1) % P].ll128) + (int64_t)(ep & 1u) * p.ll_set * 8;
  const RingLayout128 ry = ring_layout128(P, p.cap, lp);
  auto rs = [&](uint4* b, int s, int64_t id, int64_t ln) { return b + ry.rs(s, id, ln) * 8; };
  auto ag = [&](uint4* b, int s, int64_t id, int64_t ln) { return b + ry.ag(s, id, ln) * 8; };
  auto md = [&](int x) { return ((x % P) + P) % P; };

  // flat space: (chunk of this CTA, line of a ring part); U lines per group per warp step
  const int64_t total = ncj * lp;
  for (int64_t V0 = (int64_t)warp * 4 * U; V0 < total; V0 += kWarps * 4 * U) {
    bool on[U];
    int64_t id[U], g0[U], ln[U], pb[U], pr[U];  // chunk, first granule, line, part base / remainder
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = V0 + 4 * u + grp;
      on[u] = v < total;
      const int64_t cc = on[u] ? v / lp : 0;
      ln[u] = on[u] ? v - cc * lp : 0;
      const int64_t c = j + cc * p.C;
      id[u] = cb + c;
      g0[u] = p.round_g0 + sls.start + c * p.cg;
      const int64_t rest = sls.len - c * p.cg;
      const int64_t clen = rest < p.cg ? rest : p.cg;
      pb[u] = clen / P;
      pr[u] = clen % P;
    }
    // part x of the chunk: start x*pb + min(x, pr), length pb + (x < pr)
    auto pstart = [&](int u, int x) { return (int64_t)x * pb[u] + (x < pr[u] ? x : pr[u]); };
    auto plen = [&](int u, int x) { return pb[u] + (x < pr[u] ? 1 : 0); };
    auto act = [&](int u, int x) { return on[u] && ln[u] < lines_of(plen(u, x)); };
    auto dv = [&](int u, int x) { return act(u, x) && line_granule((int32_t)ln[u], sl) < plen(u, x); };
    auto own = [&](int u, int x) { return dv(u, x) && line_owner((int32_t)ln[u], sl); };
    auto gidx = [&](int u, int x) { return g0[u] + pstart(u, x) + line_granule((int32_t)ln[u], sl); };

    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = dv(u, r) ? load_x(msg, gidx(u, r)) : z;
    // reduce-scatter loop (P L175-188)
    for (int s = 0; s < P - 1; ++s) {
      const int sp = md(r - s), rp = md(r - 1 - s);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act(u, sp)) line_store(rs(next, s, id[u], ln[u]), sl, v[u], ep);
      const uint4* ptr[U];
      bool a[U];
      uint4 w[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ptr[u] = rs(mine, s, id[u], ln[u]);
        a[u] = act(u, rp);
        x[u] = dv(u, rp) ? load_x(msg, gidx(u, rp)) : z;
      }
      if (!get_lines(p, ptr, a, sl, w)) return;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (a[u]) {
          typename O::Acc acc;
          O::init(acc, w[u]);
          O::add(acc, x[u]);
          v[u] = O::narrow(acc);  // one rounding per hop (R#11)
        }
    }
    // rank r completed part r+1 (the last rp)
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (own(u, md(r + 1))) store_out(msg, gidx(u, md(r + 1)), v[u]);
    // allgather loop (P L190-203)
    for (int s = 0; s < P - 1; ++s) {
      const int sp = md(r + 1 - s), rp = md(r - s);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act(u, sp)) line_store(ag(next, s, id[u], ln[u]), sl, v[u], ep);
      const uint4* ptr[U];
      bool a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ptr[u] = ag(mine, s, id[u], ln[u]);
        a[u] = act(u, rp);
      }
      uint4 w[U];
      if (!get_lines(p, ptr, a, sl, w)) return;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (a[u]) {
          v[u] = w[u];
          if (own(u, rp)) store_out(msg, gidx(u, rp), v[u]);
        }
    }
  }
}

}  // namespace ll128
}  // namespace lane
