// lane_plan.h — partition geometry and launch parameters, shared by the host
// planner (lane_host.cu) and the kernels (lane_kernels.cuh) so that the
// host-side ownership table tested on CPU is exactly what the device runs.
//
// Partition (Alg. 2 c_group/D P L228-240,
// listing s/PPG at s*l_r P L346-348; remainder-first rule lifted to 16-byte
// granules, readings R#2-R#4):
//   message granules -> rounds (fixed size, last smaller)
//     -> k slices (remainder-first)           : the paper's processes per GPU
//       -> chunks (fixed CG granules, last smaller) : pipeline unit
//         -> G group parts (remainder-first)  : phase-1 owner = GPU g
//           -> N lane sub-parts (remainder-first) : phase-2 owner = node a
#pragma once
#include <stdint.h>

#include "../../include/lane_allreduce.h"

#if defined(__CUDACC__)
#define LANE_HD __host__ __device__ __forceinline__
#else
#define LANE_HD inline
#endif

namespace lane {

constexpr int kGranuleBytes = 16;

struct Span {
  int64_t start;
  int64_t len;
};

// Piece i of `total` split into `parts`, the first total % parts pieces one
// longer (S L276-278 examples (10,4) -> 3,3,2,2).
LANE_HD Span rf_split(int64_t total, int64_t parts, int64_t i) {
  int64_t base = total / parts, rem = total % parts;
  Span s;
  s.start = i * base + (i < rem ? i : rem);
  s.len = base + (i < rem ? 1 : 0);
  return s;
}

LANE_HD int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of chunks of a slice of `len` granules.
LANE_HD int64_t n_chunks(int64_t len, int64_t cg) { return len > 0 ? ceil_div(len, cg) : 0; }

// Index of the first chunk of slice l among all chunks of the round
// (slice-major numbering), O(1).
LANE_HD int64_t chunk_base(int64_t round_len, int k, int l, int64_t cg) {
  int64_t base = round_len / k, rem = round_len % k;
  int64_t big = l < rem ? l : rem;
  int64_t small = l - big;
  return big * n_chunks(base + 1, cg) + small * n_chunks(base, cg);
}

// Total chunks of a round.
LANE_HD int64_t round_chunks(int64_t round_len, int k, int64_t cg) {
  return chunk_base(round_len, k, k, cg);
}

// Per-rank memory as seen from the launching process (peer entries are
// IPC-mapped UVA addresses; in emulated mode every entry is local).
struct RankMem {
  char* s1;          // phase-1 inbox: (G-1) slots x cap chunks x SG granules
  char* s2;          // phase-2 inbox: N slots x cap chunks x SU granules
  char* r;           // lane result R: cap chunks x SG granules
  uint32_t* flags;   // F1[G][cap] F2[N][cap] F3[N][cap] F4[G][cap]
  char* ll;          // low-latency (LL) inboxes: 2 parity sets, see lane_ll.cuh
  char* ll128;       // LL128 inboxes: 2 parity sets of 128-byte lines, see lane_ll128.cuh
  const char* send;  // user buffers (only for ranks this launch executes)
  char* recv;
};

struct LaneParams {
  RankMem rk[LANE_MAX_RANKS];
  int N, G, P, k, C;    // C = CTAs per CTA group (per k-slice)
  int rank0, nlocal;    // this launch executes ranks rank0 .. rank0+nlocal-1
  int q;                // elements per granule (16 / itemsize)
  int tail_elems;       // elements in the message's last granule (q if full)
  int64_t ng;           // granules of the whole message
  int64_t round_g0;     // first granule of this round
  int64_t round_len;    // granules in this round
  int64_t cg;           // chunk granules
  int64_t sg, su;       // slot strides (granules): max group part / sub-part
  int64_t cap;          // chunks of this round (slot stride in chunks)
  int64_t fcap;         // flag stride in chunks: the comm's fixed chunk_cap (never per call)
  uint32_t epoch;       // monotonically increasing per round, never reset
  int direct;           // 1: every rank's send/recv addressable: zero-copy jobs
  int handshake;        // 1: start/end handshake (every simple-protocol call on real peers)
  uint32_t sig;         // call signature checked in the start handshake (host: call_signature)
  int sig_skew;         // test hook (LANE_EMU_SIG_SKEW_RANK): this rank publishes sig ^ 1, else -1
  int64_t ctl;          // flag index of the control words: enter[P], done[P], CTA counter, sig[P]
  uint64_t timeout_ns;
  uint32_t* err;        // host-mapped error word (LANE_ERR_TIMEOUT on watchdog)
  uint32_t* abort_flag; // device word: set when any wait of this comm timed out
  uint64_t* trace;      // optional per-CTA stall accounting (LANE_TRACE=1), else null
  int releasers;        // TMA engine: active releaser warps (LANE_RELEASERS, default all)
  int64_t ll_slot_g;    // LL protocol: granules per group-part slot (L1, L4), per set
  int64_t ll_slot_u;    // LL protocol: granules per sub-part slot (L2, L3), per set
  int64_t ll_set;       // LL protocol: granules per parity set (both kernels agree)
  int ring2;            // LL lane kernel: 1 = ring inter-node stage (LANE_PHASE2=ring)
  int dyn;              // TMA engine: 1 = CTAs claim chunks from a per-(rank, slice) counter (LANE_DYN_CHUNKS)
  uint32_t* claims;     // those counters (claim_index), zeroed one launch ahead by every kernel
  uint32_t* epoch_dev;  // per local rank r: [r * 16] = the next launch's epoch, [r * 16 + 1] = arrivals
  int dev_epoch;        // 1: this launch takes its epoch from epoch_dev (CUDA graph mode), else from `epoch`
};

// Chunk-claim counters: one per (rank, parity set = epoch & 1, slice), 32 bytes
// apart. Every launch of a comm (any kernel) zeroes the NEXT launch's parity
// (launch_prologue); the next launch starts only after this one completed
// (stream order), so it finds them zero whatever protocol ran in between.
LANE_HD int64_t claim_index(int rank, int par, int l) {
  return (((int64_t)rank * 2 + par) * LANE_MAX_PROCS_PER_GPU + l) * 8;
}
constexpr int64_t kClaimWords = (int64_t)LANE_MAX_RANKS * 2 * LANE_MAX_PROCS_PER_GPU * 8;

// Trace record layout (kTraceWords uint64 per CTA, nanoseconds unless noted).
enum TraceField {
  kTrProdTotal = 0, kTrProdFlagWait, kTrProdEmptyWait, kTrProdTiles,
  kTrStoreTotal, kTrStoreFullWait, kTrStoreSync, kTrStoreReadWait, kTrStoreFlush, kTrStoreJobs,
  kTrPhaseA, kTrPhaseB, kTrPhaseC, kTrPhaseD, kTrPhaseE, kTrBytes,
  kTrStartAbs,   // producer start (absolute globaltimer)
  kTrEnterWait,  // producer time in the start-of-call handshake
  kTrEndAbs,     // releaser past the end-of-call barrier (absolute; rank's last CTA only)
  kTrSmid,       // SM the CTA ran on (%smid)
  kTrEntryAbs,   // CTA entry before the PDL wait (absolute)
  kTraceWords
};

// Flag indices inside RankMem::flags: F1[G] F2[N] F3[N] F4[G], each fcap
// chunks long, fcap = the comm's chunk_cap fixed at init, so one index has
// ONE meaning (flag type, peer, chunk id) in every call whatever its size.
//
// Reuse argument (flags hold epochs that only grow and are never reset): a
// waiter of call e accepts flag >= e. The flag at index (F, x, c) is written
// in call e+1 only by the same peer, for the same (F, x, c), and only after
// that peer finished call e, which needed this rank's contribution to chunk c
// of call e, which this rank produces only after its own wait on (F, x, c)
// of call e (per chunk, phases run in order). So a value >= e+1 can only be
// seen by a waiter of call e that has already passed. With a per-call stride
// the same index could mean (F2, b, c') in call e+1 while a slow rank still
// waits on it as (F1, h, c) in call e, and the early e+1 would pass for it.
// Control words follow at ctl: enter[MAX_RANKS], done[MAX_RANKS], the CTA
// counter, then sig[MAX_RANKS] (lane_tma.cuh start/end handshake).
LANE_HD int64_t f1_idx(const LaneParams& p, int h, int64_t c) { return (int64_t)h * p.fcap + c; }
LANE_HD int64_t f2_idx(const LaneParams& p, int b, int64_t c) {
  return ((int64_t)p.G + b) * p.fcap + c;
}
LANE_HD int64_t f3_idx(const LaneParams& p, int b, int64_t c) {
  return ((int64_t)p.G + p.N + b) * p.fcap + c;
}
LANE_HD int64_t f4_idx(const LaneParams& p, int h, int64_t c) {
  return ((int64_t)p.G + 2 * p.N + h) * p.fcap + c;
}
constexpr int kCtlEnter = 0;
constexpr int kCtlDone = LANE_MAX_RANKS;
constexpr int kCtlCounter = 2 * LANE_MAX_RANKS;
constexpr int kCtlSig = 2 * LANE_MAX_RANKS + 1;
constexpr int kCtlWords = 3 * LANE_MAX_RANKS + 1;

}  // namespace lane
