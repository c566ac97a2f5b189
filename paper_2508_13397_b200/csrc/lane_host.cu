// lane_host.cu — host runtime and C ABI of the multi-lane allreduce.
//
// Components: topology / lane map (N1), granule partition +
// chunk plan (N2), IPC buffer registry for the symmetric scratch and signal
// memory (N3), the multi-CTA-group scheduler / launcher (N8) and the C ABI
// (N9) declared in include/lane_allreduce.h.
//
// The paper's multi-PPG setup (P L330: the leader allocates, publishes an IPC
// handle, the others open it) becomes: every rank allocates ONE symmetric
// scratch allocation, publishes its cudaIpcMemHandle through the caller's
// all-gather, and opens every peer's. There is one process per GPU; the
// paper's k processes per GPU become k CTA groups inside the kernel.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <string>
#include <vector>

#include "../../include/lane_allreduce.h"
#include "lane_kernels.cuh"
#include "lane_ll.cuh"
#include "lane_ll128.cuh"
#include "lane_tma.cuh"
#include "lane_plan.h"

using lane::LaneParams;
using lane::RankMem;
using lane::Span;

namespace {

constexpr uint32_t kMagic = 0x4C414E45u;  // "LANE"
constexpr int kVersion = 2;

// Every setting that shapes a call's plan, read once at init (lane_comm_s::set)
// and carried in the blob: open_peers rejects ranks whose values differ.
enum SettingId {
  kSetEngine, kSetStoreMode, kSetThreads, kSetCtasPerGroup, kSetCgMax, kSetCgMin, kSetChunksPerCta,
  kSetProto, kSetLL128Max, kSetLL128Lo, kSetLL128Hi, kSetLL128CgMin, kSetLL128U1Max, kSetLLMax,
  kSetLLThresh, kSetLLCgMin, kSetLLCtas, kSetBulkMin, kSetRingCg, kSetPhase2Ring, kSetDirect,
  kSetCtasTotal, kSetReleasers, kNumSettings
};
const char* const kSettingNames[kNumSettings] = {
    "LANE_ENGINE", "LANE_STORE", "LANE_THREADS", "LANE_CTAS_PER_GROUP", "LANE_CHUNK_BYTES",
    "LANE_MIN_CHUNK_BYTES", "LANE_CHUNKS_PER_CTA", "LANE_PROTO", "LANE_LL128_MAX_BYTES",
    "LANE_LL128_MIN_BYTES", "LANE_LL128_THRESHOLD_BYTES", "LANE_LL128_MIN_CHUNK_BYTES",
    "LANE_LL128_U1_MAX_BYTES", "LANE_LL_MAX_BYTES", "LANE_LL_THRESHOLD_BYTES", "LANE_LL_MIN_CHUNK_BYTES",
    "LANE_LL_CTAS", "LANE_BULK_MIN_BYTES", "LANE_RING_CHUNK_BYTES", "LANE_PHASE2", "LANE_DIRECT",
    "LANE_CTAS_TOTAL", "LANE_RELEASERS"};

struct Blob {
  uint32_t magic;
  int32_t version;
  int32_t N, G, k, rank, device, pid;
  uint64_t s1_bytes, s2_bytes, r_bytes, flag_bytes, total_bytes;
  int64_t round_cap, chunk_cap;
  cudaIpcMemHandle_t handle;
  int32_t settings[kNumSettings];
};
static_assert(sizeof(Blob) <= LANE_HANDLE_BYTES, "blob too large");

// FNV-1a over the bytes of 64-bit values: the per-call signature the start handshake
// compares across ranks (lane_tma.cuh).
uint32_t fnv_mix(uint32_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (uint32_t)((v >> (8 * i)) & 0xFF);
    h *= 16777619u;
  }
  return h;
}

int64_t env_i64(const char* name, int64_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  char* end = nullptr;
  long long x = strtoll(v, &end, 10);
  if (end == v) return dflt;
  return (int64_t)x;
}

}  // namespace

struct lane_comm_s {
  int N = 0, G = 0, P = 0, k = 0, rank = 0, device = 0;
  bool emulated = false;
  bool connected = false;
  int threads = 512;
  int engine = 1;           // 0 = LSU (ld/st.global), 1 = TMA bulk pipeline
  int store_mode = 0;       // TMA engine stores: 0 auto (bulk from bulk_min), 1 st.global, 2 bulk
  int64_t bulk_min = 0;     // granules: auto mode uses bulk (TMA) stores from this message size
  int ctas_per_group = 0;  // 0 = choose per call
  int max_coresident = 0;  // CTAs of the kernel that fit on the device at once
  int sm_count = 0;
  int64_t round_cap = 0;   // granules of message per round (kernel launch)
  int64_t cg_max = 0, cg_min = 0;
  int chunks_per_cta = 4;
  int direct_mode = 2;     // LANE_DIRECT: registered multi-GPU job set (2 push, 3 pull-all, 4 pull-push, 0 staged)
  int direct_emu = 1;      // LANE_DIRECT in emulated mode (1 direct-pull default)
  int pdl = 0;             // LANE_PDL=1: multi-GPU launches with programmatic stream serialization
  bool emu_handshake = false;  // LANE_EMU_HANDSHAKE=1 (tests): start/end handshake in emulated mode
  int sig_skew = -1;       // LANE_EMU_SIG_SKEW_RANK (tests): that emulated rank publishes a wrong signature
  int ctas_total = 0;      // LANE_CTAS_TOTAL: simple-protocol CTAs per GPU (multi-GPU)
  int releasers = 4;       // LANE_RELEASERS (1..4)
  int64_t chunk_cap = 0;   // max chunks per round (flag capacity per flag type)
  uint64_t s1_bytes = 0, s2_bytes = 0, r_bytes = 0, flag_bytes = 0, total_bytes = 0;
  // LL protocol (lane_ll.cuh): message capacity, minimum chunk, inbox geometry
  int proto = 0;             // 0 = auto, 1 = always LL (when it fits), 2 = never LL (simple), 3 = always LL128
  int64_t ll_max = 0;        // granules: largest message the LL inboxes hold
  int64_t ll_thresh = 0;     // granules: auto mode uses LL up to this size
  int64_t ll_cg_min = 0;     // granules
  int ll_ctas = 0;           // CTAs per rank for LL launches (0 = SM count)
  int ll_coresident = 0;     // co-resident CTAs of the LL kernel on the device
  int64_t ll_slot_g = 0, ll_slot_u = 0;
  int64_t ring_slot = 0;     // granules per ring RS/AG slot (Alg. 1 on the LL protocol)
  int64_t ring_cg = 0;       // granules per pipeline chunk of the ring algorithms (fixed, R#21)
  int64_t a2_slot_v = 0;     // granules per lane slot of "approach 2" (whole-chunk lane parts)
  bool phase2_ring = false;  // LANE_PHASE2=ring: lane method with a ring inter-node stage
  int64_t ll_set = 0;        // granules per LL parity set (max of the lane and ring layouts)
  // LL128 protocol (lane_ll128.cuh): shares the LL region (one protocol per call)
  int64_t ll128_max = 0;     // granules: largest message the LL128 inboxes hold
  int64_t ll128_lo = 0;      // granules: auto mode uses LL128 above this size ...
  int64_t ll128_hi = 0;      // ... up to this size
  int64_t ll128_cg_min = 0;  // granules
  int64_t ll128_set = 0;     // lines (128 B) per LL128 parity set
  int64_t ll128_u1_max = 0;  // granules: LL128 lane kernel with U = 1 up to this size, U = 2 above
  uint64_t ll_bytes = 0;
  uint64_t ll128_bytes = 0;  // LL128 region: its own (never shared with the LL packets, see carve)
  std::vector<char*> own;    // own scratch allocations (1, or P when emulated)
  std::vector<void*> opened; // IPC-opened peer allocations
  RankMem rk[LANE_MAX_RANKS];
  cudaIpcMemHandle_t handle;
  uint32_t epoch = 0;
  uint32_t* err_host = nullptr;  // mapped pinned word
  uint32_t* err_dev = nullptr;
  uint32_t* abort_dev = nullptr;
  uint32_t* claims = nullptr;  // chunk-claim counters (lane_plan.h claim_index)
  uint32_t* epoch_dev = nullptr;  // per local rank: next epoch + arrival count (lane_kernels.cuh launch_prologue)
  int dev_epoch = 0;              // 1 once a call was captured into a CUDA graph (sticky)
  int dyn = -1;                // LANE_DYN_CHUNKS: TMA engine CTAs claim chunks dynamically (1), statically (0), auto (-1)
  uint64_t timeout_ns = 0;
  uint64_t* trace = nullptr;  // LANE_TRACE=1: kTraceWords per CTA of the last launch
  int trace_ctas = 0;
  struct Reg {             // a registered user buffer and its peers' mappings
    char* base;
    uint64_t bytes;
    char* peer[LANE_MAX_RANKS];
    bool live;
  };
  std::vector<Reg> regs;
  char* pending_reg = nullptr;  // set by register_handle, consumed by register_open
  uint64_t pending_bytes = 0;
  std::vector<std::pair<std::string, void*>> ipc_cache;  // opened peer allocations by handle
  int64_t ctl = 0;             // flag index of the control words
  std::vector<char*> stage;  // device staging for the host-buffer API
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host API
  cudaEvent_t ev_start = nullptr, ev_h[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr},
              ev_d[2] = {nullptr, nullptr};
  uint64_t stage_bytes = 0;
  std::string last_error;
  int32_t settings[kNumSettings];  // plan-shaping settings (Blob::settings)
};

namespace {

int fail(lane_comm_t c, int code, const std::string& msg) {
  if (c) c->last_error = msg;
  return code;
}

int cuda_fail(lane_comm_t c, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return fail(c, LANE_ERR_CUDA, m);
}

#define LANE_CUDA(c, call)                                   \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail((c), e_, #call); \
  } while (0)

int validate_topology(int N, int G, int k, std::string* why) {
  if (N < 1) return *why = "nodes must be >= 1", LANE_ERR_INVALID_ARG;
  if (G < 1) return *why = "gpus_per_node must be >= 1", LANE_ERR_INVALID_ARG;
  if (k < 1) return *why = "procs_per_gpu must be >= 1", LANE_ERR_INVALID_ARG;
  if ((int64_t)N * G > LANE_MAX_RANKS)
    return *why = "nodes*gpus_per_node exceeds LANE_MAX_RANKS", LANE_ERR_INVALID_ARG;
  if (k > LANE_MAX_PROCS_PER_GPU)
    return *why = "procs_per_gpu exceeds LANE_MAX_PROCS_PER_GPU", LANE_ERR_INVALID_ARG;
  return LANE_OK;
}

int itemsize_of(int dtype) { return dtype == LANE_BFLOAT16 ? 2 : 4; }

// Geometry of one rank's scratch for a comm (sizes in bytes). Every call's
// plan fits by construction: with round_len <= round_cap, CG in
// [cg_min, cg_max] and at most round_cap/CG + k chunks, a slot region needs
// chunks * ceil(CG/G) <= round_cap/G + round_cap/cg_min + k*(cg_max/G + 1).
void size_scratch(lane_comm_t c) {
  const int64_t RC = c->round_cap, G = c->G, N = c->N, k = c->k;
  c->chunk_cap = RC / c->cg_min + k + 1;
  const int64_t slot_g = RC / G + RC / c->cg_min + k * (c->cg_max / G + 1) + 16;
  const int64_t slot_u = RC / (G * N) + RC / c->cg_min + k * (c->cg_max / (G * N) + 1) + 16;
  c->s1_bytes = (uint64_t)((G - 1) * slot_g) * 16;
  c->s2_bytes = (uint64_t)(N * slot_u) * 16;
  c->r_bytes = (uint64_t)slot_g * 16;
  c->ctl = (2 * G + 2 * N) * c->chunk_cap;  // control words (lane_plan.h kCtl*) follow the chunk flags
  c->flag_bytes = (uint64_t)(c->ctl + lane::kCtlWords) * 4;
  auto al = [](uint64_t x) { return (x + 4095) & ~(uint64_t)4095; };
  c->s1_bytes = al(c->s1_bytes);
  c->s2_bytes = al(c->s2_bytes);
  c->r_bytes = al(c->r_bytes);
  c->flag_bytes = al(c->flag_bytes);
  // LL inboxes: a slot holds cap chunks of ceil(CG/G) (ceil(CG/(GN)),
  // ceil(CG/P) for the flat ring) granules. With CG >= ll_cg_min a round of
  // M granules has at most M/CG + k chunks, so cap * ceil(CG/G) <= M/G +
  // M/CG + k*CG/G + k; CG <= ceil(M/k) bounds the k*CG/G term by (M+k)/G.
  const int64_t M = c->ll_max;
  if (M > 0) {
    // (checked by brute force over M, G, N, k, CG in the design notes)
    const int64_t chunks = M / c->ll_cg_min + k + 1;
    int64_t cgmax = lane::ceil_div(M, k);
    if (cgmax < c->ring_cg) cgmax = c->ring_cg;
    if (cgmax < c->ll_cg_min) cgmax = c->ll_cg_min;
    c->ll_slot_g = lane::ceil_div(M, G) + chunks + k * (lane::ceil_div(cgmax, G) + 1) + 16;
    c->ll_slot_u = lane::ceil_div(M, G * N) + 2 * chunks + k * (lane::ceil_div(cgmax, G * N) + 2) + 16;
    c->ring_slot = lane::ceil_div(M, G * N) + chunks + k * (lane::ceil_div(cgmax, G * N) + 1) + 16;
    c->a2_slot_v = lane::ceil_div(M, N) + chunks + k * (lane::ceil_div(cgmax, N) + 1) + 16;
    const int64_t lane_set = lane::ll::set_granules((int)G, (int)N, c->ll_slot_g, c->ll_slot_u);
    const int64_t ring_set = lane::ll::ring_set_granules((int)(G * N), c->ring_slot);
    const int64_t a2_set = lane::ll::a2_set_granules((int)G, (int)N, c->ll_slot_g, c->a2_slot_v);
    c->ll_set = lane_set > ring_set ? lane_set : ring_set;
    if (a2_set > c->ll_set) c->ll_set = a2_set;
    c->ll_bytes = al((uint64_t)(2 * c->ll_set) * lane::ll::kPacketBytes);
  } else {
    c->ll_slot_g = c->ll_slot_u = c->ring_slot = c->a2_slot_v = c->ll_set = 0;
    c->ll_bytes = 0;
  }
  // LL128 set: a call needs 2*G*N*cap*lu lines (lane_ll128.cuh set_lines).
  // With G*N*su <= CG + G*N and cap*CG <= M + k*CG this is at most
  // 2*(M + k*CG + cap*G*N)/7 + 2*cap*G*N lines; sized here for k*CG <= M/4
  // (true whenever a slice spans >= 4 CTAs or CG is the minimum chunk of a
  // message >= 4*k*CG_min); the plan checks the exact need and otherwise
  // falls back to another protocol.
  const int64_t M8 = c->ll128_max;
  if (M8 > 0) {
    c->ll128_set = lane::ll128::set_capacity128((int)G, (int)N, (int)k, M8, c->ll128_cg_min);
    c->ll128_bytes = al((uint64_t)(2 * c->ll128_set) * lane::ll128::kLineBytes);
  } else {
    c->ll128_set = 0;
    c->ll128_bytes = 0;
  }
  c->total_bytes = c->s1_bytes + c->s2_bytes + c->r_bytes + c->flag_bytes + c->ll_bytes + c->ll128_bytes;
}

void carve(lane_comm_t c, char* base, RankMem* m) {
  m->s1 = base;
  m->s2 = base + c->s1_bytes;
  m->r = base + c->s1_bytes + c->s2_bytes;
  m->flags = reinterpret_cast<uint32_t*>(base + c->s1_bytes + c->s2_bytes + c->r_bytes);
  m->ll = c->ll_bytes ? base + c->s1_bytes + c->s2_bytes + c->r_bytes + c->flag_bytes : nullptr;
  // The LL128 lines get their own region: in it the last 16 bytes of every
  // 128-byte line only ever hold epochs (every LL128 layout is line-aligned),
  // and the LL region's packets only ever hold epochs in their high words. A
  // shared region would let one protocol's user data sit where the other
  // reads its epoch, so data equal to the current epoch could pass for a
  // fresh packet.
  m->ll128 = c->ll128_bytes ? base + c->s1_bytes + c->s2_bytes + c->r_bytes + c->flag_bytes + c->ll_bytes : nullptr;
  m->send = nullptr;
  m->recv = nullptr;
}

template <int DT>
int occupancy_of(int engine, int threads) {
  int nb = 0;
  if (engine == 1) {
    cudaFuncSetAttribute(lane::tma::lane_tma_kernel<DT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         lane::tma::kSmemBytes);
    cudaFuncSetAttribute(lane::tma::lane_tma_kernel<DT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         lane::tma::kSmemBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lane::tma::lane_tma_kernel<DT, true>, lane::tma::kThreads,
                                                  lane::tma::kSmemBytes);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lane::lane_allreduce_kernel<DT>, threads, 0);
  }
  return nb;
}

template <int DT>
int ll_occupancy_of() {
  int nb = 0, nr = 0, na = 0;
  int nb2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lane::ll::lane_ll_kernel<DT>, lane::ll::kThreads, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, lane::ll::lane_ll_kernel<DT, true>, lane::ll::kThreads, 0);
  nb = nb < nb2 ? nb : nb2;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nr, lane::ll::lane_ring_ll_kernel<DT>, lane::ll::kThreads, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&na, lane::ll::lane_a2_ll_kernel<DT>, lane::ll::kThreads, 0);
  nb = nb < nr ? nb : nr;
  return nb < na ? nb : na;
}

thread_local std::string g_init_error;  // errors of init calls that return no comm

int common_init_impl(lane_comm_t c, int N, int G, int k, int rank, int device, bool emulated) {
  c->N = N;
  c->G = G;
  c->P = N * G;
  c->k = k;
  c->rank = rank;
  c->device = device;
  c->emulated = emulated;
  c->threads = (int)env_i64("LANE_THREADS", 512);
  {
    const char* e = getenv("LANE_ENGINE");
    c->engine = (e && strcmp(e, "lsu") == 0) ? 0 : 1;
    const char* st = getenv("LANE_STORE");
    c->store_mode = !st ? 0 : (strcmp(st, "lsu") == 0 ? 1 : (strcmp(st, "bulk") == 0 ? 2 : 0));
  }
  if (c->threads < 64 || c->threads > 512 || c->threads % 32)
    return fail(c, LANE_ERR_INVALID_ARG, "LANE_THREADS must be a multiple of 32 in [64, 512]");
  c->ctas_per_group = (int)env_i64("LANE_CTAS_PER_GROUP", 0);
  c->round_cap = env_i64("LANE_ROUND_BYTES", (int64_t)1 << 30) / 16;
  // Largest pipeline chunk. Multi-GPU: 1 MiB chunks cost the all-to-all layouts up to 10% at 1 GiB
  // (1x4 615 vs 690 GB/s with 256 KiB; 4x1 652 vs 683 with 512 KiB; 2x2 neutral:
  // profiles/r02_chunk_budget_p4.txt). Emulated (HBM-bound, every rank in one launch): 1 MiB
  // (512 KiB chunks cost the N = 1 bench 8%: 4.30 -> 4.66 ms).
  c->cg_max = env_i64("LANE_CHUNK_BYTES", emulated ? (1 << 20) : (N == 1 ? (256 << 10) : (512 << 10))) / 16;
  c->cg_min = env_i64("LANE_MIN_CHUNK_BYTES", 128 << 10) / 16;
  c->chunks_per_cta = (int)env_i64("LANE_CHUNKS_PER_CTA", 4);
  if (c->chunks_per_cta < 1) c->chunks_per_cta = 1;
  if (c->round_cap < 1024) return fail(c, LANE_ERR_INVALID_ARG, "LANE_ROUND_BYTES must be >= 16 KiB");
  if (c->cg_min < 16) c->cg_min = 16;
  if (c->cg_max < c->cg_min) c->cg_max = c->cg_min;
  c->timeout_ns = (uint64_t)env_i64("LANE_TIMEOUT_MS", 20000) * 1000000ull;
  {
    const char* pr = getenv("LANE_PROTO");
    c->proto = !pr ? 0
                   : (strcmp(pr, "ll") == 0       ? 1
                      : strcmp(pr, "simple") == 0 ? 2
                      : strcmp(pr, "ll128") == 0  ? 3
                                                  : 0);
  }
  // auto range from the P = 2 / P = 4 protocol sweeps (profiles/r01_sizes_protocols_ll128.txt):
  // LL128 capacity (one round of at most this much message uses the LL128 inboxes)
  c->ll128_max = env_i64("LANE_LL128_MAX_BYTES", 32 << 20) / 16;
  if (c->ll128_max < 0) c->ll128_max = 0;
  // Default protocol ranges, from the measured crossovers (profiles/r02_protocol_crossovers.txt,
  // P = 2 and 4, every layout): LL128 beats LL from 1 MiB at P = 4 (above 512 KiB) and from
  // 4 MiB at P = 2; the simple protocol beats LL128 above 32 MiB when both phases span GPUs
  // (N > 1, G > 1: four dependent hops per chunk), above 24 MiB for one-GPU nodes (G = 1),
  // above 16 MiB for one node (N = 1).
  c->ll128_lo = env_i64("LANE_LL128_MIN_BYTES", N * G == 2 ? (2 << 20) : (512 << 10)) / 16;
  c->ll128_hi = env_i64("LANE_LL128_THRESHOLD_BYTES", (N > 1 && G > 1) ? (32 << 20) : (G == 1 ? (24 << 20) : (16 << 20))) / 16;
  c->ll128_cg_min = env_i64("LANE_LL128_MIN_CHUNK_BYTES", 16 << 10) / 16;
  c->ll128_u1_max = env_i64("LANE_LL128_U1_MAX_BYTES", 4 << 20) / 16;
  if (c->ll128_cg_min < 64) c->ll128_cg_min = 64;
  c->ll_max = env_i64("LANE_LL_MAX_BYTES", 16 << 20) / 16;
  if (c->ll_max < 0) c->ll_max = 0;
  c->ll_thresh = env_i64("LANE_LL_THRESHOLD_BYTES", 8 << 20) / 16;
  c->ll_cg_min = env_i64("LANE_LL_MIN_CHUNK_BYTES", 4 << 10) / 16;
  if (c->ll_cg_min < 16) c->ll_cg_min = 16;
  c->ll_ctas = (int)env_i64("LANE_LL_CTAS", 0);
  c->bulk_min = env_i64("LANE_BULK_MIN_BYTES", 16 << 20) / 16;
  c->ring_cg = env_i64("LANE_RING_CHUNK_BYTES", 64 << 10) / 16;
  if (c->ring_cg < c->ll_cg_min) c->ring_cg = c->ll_cg_min;
  {
    const char* p2 = getenv("LANE_PHASE2");
    c->phase2_ring = p2 && strcmp(p2, "ring") == 0;
  }
  // PDL is opt-in: it hides the launch gap in a microbenchmark (tools/launch_micro.cu) but measured
  // no gain in the allreduce and cost ~2% at 1 GiB on 1x4 / 4x1 (profiles/r02_pdl_ab_p4.txt)
  c->pdl = env_i64("LANE_PDL", 0) != 0;
  c->dyn = (int)env_i64("LANE_DYN_CHUNKS", -1);
  c->direct_mode = (int)env_i64("LANE_DIRECT", 2);
  if (c->direct_mode != 0 && c->direct_mode != 3 && c->direct_mode != 4) c->direct_mode = 2;  // 1 (pull): emulated only
  c->direct_emu = (int)env_i64("LANE_DIRECT", 1);
  if (c->direct_emu < 0 || c->direct_emu > 4) c->direct_emu = 1;
  c->emu_handshake = env_i64("LANE_EMU_HANDSHAKE", 0) != 0;
  c->sig_skew = emulated ? (int)env_i64("LANE_EMU_SIG_SKEW_RANK", -1) : -1;
  c->ctas_total = (int)env_i64("LANE_CTAS_TOTAL", 0);
  c->releasers = (int)env_i64("LANE_RELEASERS", lane::tma::kReleasers);
  if (c->releasers < 1) c->releasers = 1;
  if (c->releasers > lane::tma::kReleasers) c->releasers = lane::tma::kReleasers;
  {
    int32_t* v = c->settings;
    v[kSetEngine] = c->engine;
    v[kSetStoreMode] = c->store_mode;
    v[kSetThreads] = c->threads;
    v[kSetCtasPerGroup] = c->ctas_per_group;
    v[kSetCgMax] = (int32_t)c->cg_max;
    v[kSetCgMin] = (int32_t)c->cg_min;
    v[kSetChunksPerCta] = c->chunks_per_cta;
    v[kSetProto] = c->proto;
    v[kSetLL128Max] = (int32_t)c->ll128_max;
    v[kSetLL128Lo] = (int32_t)c->ll128_lo;
    v[kSetLL128Hi] = (int32_t)c->ll128_hi;
    v[kSetLL128CgMin] = (int32_t)c->ll128_cg_min;
    v[kSetLL128U1Max] = (int32_t)c->ll128_u1_max;
    v[kSetLLMax] = (int32_t)c->ll_max;
    v[kSetLLThresh] = (int32_t)c->ll_thresh;
    v[kSetLLCgMin] = (int32_t)c->ll_cg_min;
    v[kSetLLCtas] = c->ll_ctas;
    v[kSetBulkMin] = (int32_t)c->bulk_min;
    v[kSetRingCg] = (int32_t)c->ring_cg;
    v[kSetPhase2Ring] = c->phase2_ring ? 1 : 0;
    v[kSetDirect] = c->direct_mode;
    v[kSetCtasTotal] = c->ctas_total;
    v[kSetReleasers] = c->releasers;
  }
  size_scratch(c);

  LANE_CUDA(c, cudaSetDevice(device));
  LANE_CUDA(c, cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  int occ = occupancy_of<0>(c->engine, c->threads);
  int o1 = occupancy_of<1>(c->engine, c->threads), o2 = occupancy_of<2>(c->engine, c->threads);
  occ = occ < o1 ? occ : o1;
  occ = occ < o2 ? occ : o2;
  if (occ < 1) occ = 1;
  c->max_coresident = occ * c->sm_count;
  {
    int l0 = ll_occupancy_of<0>(), l1 = ll_occupancy_of<1>(), l2 = ll_occupancy_of<2>();
    int lo = l0 < l1 ? l0 : l1;
    lo = lo < l2 ? lo : l2;
    int m0 = 0, m1 = 0, m2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m0, lane::ll128::lane_ll128_kernel<0>, lane::ll128::kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m1, lane::ll128::lane_ll128_kernel<1>, lane::ll128::kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m2, lane::ll128::lane_ll128_kernel<2>, lane::ll128::kThreads, 0);
    lo = lo < m0 ? lo : m0;
    lo = lo < m1 ? lo : m1;
    lo = lo < m2 ? lo : m2;
    for (const void* f : {(const void*)lane::ll128::lane_ll128_kernel<0, false, 1>,
                          (const void*)lane::ll128::lane_ll128_kernel<1, false, 1>,
                          (const void*)lane::ll128::lane_ll128_kernel<2, false, 1>,
                          (const void*)lane::ll128::lane_ll128_kernel<0, true, 1>,
                          (const void*)lane::ll128::lane_ll128_kernel<1, true, 1>,
                          (const void*)lane::ll128::lane_ll128_kernel<2, true, 1>}) {
      int mr = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mr, f, lane::ll128::kThreads, 0);
      lo = lo < mr ? lo : mr;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m0, lane::ll128::lane_ring_ll128_kernel<0>, lane::ll128::kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m1, lane::ll128::lane_ring_ll128_kernel<1>, lane::ll128::kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m2, lane::ll128::lane_ring_ll128_kernel<2>, lane::ll128::kThreads, 0);
    lo = lo < m0 ? lo : m0;
    lo = lo < m1 ? lo : m1;
    lo = lo < m2 ? lo : m2;
    c->ll_coresident = (lo < 1 ? 1 : lo) * c->sm_count;
  }

  const int nalloc = emulated ? c->P : 1;
  for (int i = 0; i < nalloc; ++i) {
    char* p = nullptr;
    LANE_CUDA(c, cudaMalloc(&p, c->total_bytes));
    c->own.push_back(p);
    // flags must read 0 before any peer can write an epoch >= 1
    LANE_CUDA(c, cudaMemset(p + c->s1_bytes + c->s2_bytes + c->r_bytes, 0,
                            c->flag_bytes + c->ll_bytes + c->ll128_bytes));
  }
  LANE_CUDA(c, cudaHostAlloc(&c->err_host, 64, cudaHostAllocMapped));
  memset(c->err_host, 0, 64);
  LANE_CUDA(c, cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0));
  LANE_CUDA(c, cudaMalloc(&c->abort_dev, 64));
  LANE_CUDA(c, cudaMemset(c->abort_dev, 0, 64));
  LANE_CUDA(c, cudaMalloc(&c->claims, lane::kClaimWords * 4));
  LANE_CUDA(c, cudaMemset(c->claims, 0, lane::kClaimWords * 4));
  {
    uint32_t init[LANE_MAX_RANKS * 16];
    memset(init, 0, sizeof(init));
    for (int r = 0; r < LANE_MAX_RANKS; ++r) init[r * 16] = 1u;  // the first launch's epoch (c->epoch + 1)
    LANE_CUDA(c, cudaMalloc(&c->epoch_dev, sizeof(init)));
    LANE_CUDA(c, cudaMemcpy(c->epoch_dev, init, sizeof(init), cudaMemcpyHostToDevice));
  }
  if (env_i64("LANE_TRACE", 0)) {
    const size_t nt = (size_t)(c->max_coresident > c->ll_coresident ? c->max_coresident : c->ll_coresident);
    LANE_CUDA(c, cudaMalloc(&c->trace, nt * lane::kTraceWords * 8));
    LANE_CUDA(c, cudaMemset(c->trace, 0, nt * lane::kTraceWords * 8));
  }
  LANE_CUDA(c, cudaDeviceSynchronize());
  if (emulated) {
    for (int p = 0; p < c->P; ++p) carve(c, c->own[p], &c->rk[p]);
    c->connected = true;
  } else {
    carve(c, c->own[0], &c->rk[c->rank]);
    LANE_CUDA(c, cudaIpcGetMemHandle(&c->handle, c->own[0]));
  }
  return LANE_OK;
}

void release(lane_comm_t c);

int common_init(int N, int G, int k, int rank, int device, bool emulated, lane_comm_t* out) {
  *out = nullptr;
  std::string why;
  int st = validate_topology(N, G, k, &why);
  if (st != LANE_OK) {
    g_init_error = why;
    return st;
  }
  lane_comm_t c = new lane_comm_s();
  st = common_init_impl(c, N, G, k, rank, device, emulated);
  if (st != LANE_OK) {
    g_init_error = c->last_error;
    release(c);
    return st;
  }
  *out = c;
  return LANE_OK;
}

bool overlaps_partially(const void* s, const void* r, uint64_t bytes) {
  uintptr_t a = (uintptr_t)s, b = (uintptr_t)r;
  if (a == b) return false;
  return a < b + bytes && b < a + bytes;
}

// Which kernel a plan launches (Plan::ll).
enum PlanKind : int {
  kSimple = 0,      // TMA (or LSU) engine, simple protocol, rounds of LANE_ROUND_BYTES
  kLL = 1,          // LL lane kernel, one launch (ll_plan)
  kLaneRingLL = 2,  // LL lane kernel with the ring inter-node stage (rounds, ring_plan)
  kRingLL = 3,      // flat ring, Alg. 1, on LL packets (rounds, ring_plan)
  kLL128 = 4,       // LL128 lane kernel, one launch (ll128_plan)
  kA2LL = 5,        // "approach 2" on LL packets (rounds, a2_plan)
  kRingLL128 = 6,   // flat ring on LL128 lines (rounds, ring_plan)
  kLaneRingLL128 = 7  // LL128 lane kernel with the ring inter-node stage (rounds, ring_plan)
};

struct Plan {
  int64_t ng, cg, round_len0;
  int rounds, C, tail_elems, q;
  int ll;  // PlanKind
};

// Plans whose rounds are LL-capacity sized (ll_ring_rounds launches them).
bool ll_rounds(const Plan& pl) {
  return pl.ll == kLaneRingLL || pl.ll == kRingLL || pl.ll == kA2LL || pl.ll == kRingLL128 || pl.ll == kLaneRingLL128;
}

bool ring_plan(lane_comm_t c, int64_t ng, bool lane_ring, Plan* pl);
bool a2_plan(lane_comm_t c, int64_t ng, Plan* pl);

// LL plan for a one-round message of ng granules: C CTAs per CTA group and
// chunk size; false if the LL protocol does not apply or does not fit.
bool ll128_plan(lane_comm_t c, int64_t ng, Plan* pl);

bool ll_plan(lane_comm_t c, int64_t ng, Plan* pl) {
  if (c->P > 1 && c->proto == 3) return ll128_plan(c, ng, pl);
  if (c->P > 1 && c->proto == 0 && ng > c->ll128_lo && ng <= c->ll128_hi && ll128_plan(c, ng, pl)) return true;
  if (c->P == 1 || c->ll_bytes == 0 || c->proto == 2 || ng > c->ll_max) return false;
  if (c->proto == 0 && ng > c->ll_thresh) return false;
  const int ranks_here = c->emulated ? c->P : 1;
  int budget = c->ll_ctas > 0 ? c->ll_ctas : (c->emulated ? c->ll_coresident : c->sm_count);
  if (budget > c->ll_coresident) budget = c->ll_coresident;
  int C = budget / (ranks_here * c->k);
  if (C < 1) C = 1;
  if ((int64_t)C * c->k * ranks_here > c->ll_coresident) return false;  // every CTA must be resident
  const int64_t slice0 = (ng + c->k - 1) / c->k;
  int64_t cg = (slice0 + C - 1) / C;
  if (cg < c->ll_cg_min) cg = c->ll_cg_min;
  const int64_t nch = lane::n_chunks(slice0, cg);
  if (nch < C) C = (int)(nch > 0 ? nch : 1);
  const int64_t cap = lane::round_chunks(ng, c->k, cg);
  const int64_t sg = lane::ceil_div(cg, c->G), su = lane::ceil_div(sg, c->N);
  if (cap * sg > c->ll_slot_g || cap * su > c->ll_slot_u) return false;
  pl->C = C;
  pl->cg = cg;
  pl->ll = kLL;
  return true;
}

// LL128 plan: as ll_plan, with the LL128 inbox geometry (lines).
bool ll128_plan(lane_comm_t c, int64_t ng, Plan* pl) {
  if (c->P == 1 || c->ll128_set == 0 || ng > c->ll128_max) return false;
  const int ranks_here = c->emulated ? c->P : 1;
  int budget = c->ll_ctas > 0 ? c->ll_ctas : (c->emulated ? c->ll_coresident : c->sm_count);
  if (budget > c->ll_coresident) budget = c->ll_coresident;
  int C = budget / (ranks_here * c->k);
  if (C < 1) C = 1;
  if ((int64_t)C * c->k * ranks_here > c->ll_coresident) return false;  // every CTA must be resident
  const lane::ll128::Plan128 g = lane::ll128::plan128(c->G, c->N, c->k, ng, C, c->ll128_max, c->ll128_cg_min);
  if (g.need > c->ll128_set) return false;
  pl->C = g.C;
  pl->cg = g.cg;
  pl->ll = kLL128;
  return true;
}

int make_plan(lane_comm_t c, uint64_t count, int dtype, Plan* pl) {
  const int isz = itemsize_of(dtype);
  pl->q = 16 / isz;
  pl->ng = (int64_t)((count + pl->q - 1) / pl->q);
  pl->tail_elems = (int)(count - (uint64_t)(pl->ng - 1) * pl->q);
  pl->round_len0 = pl->ng < c->round_cap ? pl->ng : c->round_cap;
  pl->rounds = (int)((pl->ng + c->round_cap - 1) / c->round_cap);
  pl->ll = kSimple;
  if (c->phase2_ring && c->P > 1) {  // the lane method with a ring inter-node stage: LL rounds only
    if (!ring_plan(c, pl->ng, true, pl))
      return fail(c, LANE_ERR_INVALID_ARG, "LANE_PHASE2=ring: CTA capacity or LL inboxes exceeded");
    return LANE_OK;
  }
  if (pl->rounds == 1 && ll_plan(c, pl->ng, pl)) return LANE_OK;
  // CTAs per CTA group: fill the device with all ranks' groups (emulated) or
  // default to 64 CTAs per GPU across the k groups (multi-GPU); env override.
  int ranks_here = c->emulated ? c->P : 1;
  int C = c->ctas_per_group;
  if (C <= 0) {
    int budget = c->emulated ? c->max_coresident : (c->ctas_total > 0 ? c->ctas_total : c->sm_count);
    if (budget > c->max_coresident) budget = c->max_coresident;
    C = budget / (ranks_here * c->k);
  }
  if (C < 1) C = 1;
  if ((int64_t)C * c->k * ranks_here > c->max_coresident)
    return fail(c, LANE_ERR_INVALID_ARG,
                "ctas_per_group*procs_per_gpu exceeds the device's co-resident CTA capacity");
  pl->C = C;
  // chunk size: give every CTA of a group about chunks_per_cta chunks (so the
  // phases of successive chunks overlap), within [cg_min, cg_max]
  int64_t slice0 = (pl->round_len0 + c->k - 1) / c->k;
  int64_t cg = (slice0 + (int64_t)C * c->chunks_per_cta - 1) / ((int64_t)C * c->chunks_per_cta);
  if (cg > c->cg_max) cg = c->cg_max;
  if (cg < c->cg_min) cg = c->cg_min;
  pl->cg = cg;
  return LANE_OK;
}

// Per-call signature compared by the start handshake (lane_tma.cuh): every
// rank of a consistent call computes the same value.
uint32_t call_signature(lane_comm_t c, const Plan& pl, int direct, int reg_s, int reg_r, uint64_t so, uint64_t ro,
                        int dtype) {
  uint32_t h = 2166136261u;
  h = fnv_mix(h, (uint64_t)direct);
  h = fnv_mix(h, (uint64_t)(int64_t)reg_s);
  h = fnv_mix(h, (uint64_t)(int64_t)reg_r);
  h = fnv_mix(h, so);
  h = fnv_mix(h, ro);
  h = fnv_mix(h, (uint64_t)pl.ng);
  h = fnv_mix(h, (uint64_t)pl.tail_elems);
  h = fnv_mix(h, (uint64_t)dtype);
  h = fnv_mix(h, (uint64_t)pl.cg);
  h = fnv_mix(h, (uint64_t)pl.C);
  h = fnv_mix(h, (uint64_t)c->k);
  return h;
}

LaneParams base_params(lane_comm_t c, const Plan& pl) {
  LaneParams p;
  memset(&p, 0, sizeof(p));
  for (int r = 0; r < c->P; ++r) p.rk[r] = c->rk[r];
  p.N = c->N;
  p.G = c->G;
  p.P = c->P;
  p.k = c->k;
  p.C = pl.C;
  p.q = pl.q;
  p.tail_elems = pl.tail_elems;
  p.ng = pl.ng;
  p.cg = pl.cg;
  p.sg = lane::ceil_div(pl.cg, c->G);
  p.su = lane::ceil_div(p.sg, c->N);
  p.timeout_ns = c->timeout_ns;
  p.err = c->err_dev;
  p.abort_flag = c->abort_dev;
  p.trace = c->trace;
  p.ctl = c->ctl;
  p.fcap = c->chunk_cap;
  p.sig_skew = c->sig_skew;
  p.releasers = c->releasers;
  p.claims = c->claims;
  p.dyn = c->dyn > 0 ? 1 : 0;
  p.epoch_dev = c->epoch_dev;
  p.dev_epoch = c->dev_epoch;
  return p;
}

// Plan of the ring algorithms on the LL protocol (flat ring, Alg. 1; lane
// method with a ring inter-node stage): rounds of at most ll_max granules
// (one launch each), each split into the comm's k slices and pipeline chunks
// of a FIXED ring_cg granules — the ring order of an element depends on its
// chunk (R#21), so the chunking must not depend on the launch configuration.
// C = CTAs per CTA group (every CTA resident). false: does not fit.
bool ring_plan(lane_comm_t c, int64_t ng, bool lane_ring, Plan* pl) {
  if (c->ll_bytes == 0) return false;
  const int ranks_here = c->emulated ? c->P : 1;
  int budget = c->ll_ctas > 0 ? c->ll_ctas : (c->emulated ? c->ll_coresident : c->sm_count);
  if (budget > c->ll_coresident) budget = c->ll_coresident;
  int C = budget / (ranks_here * c->k);
  if (C < 1) C = 1;
  if ((int64_t)C * c->k * ranks_here > c->ll_coresident) return false;
  const int64_t RC = c->ll_max, cg = c->ring_cg;
  const int64_t r0 = ng < RC ? ng : RC;
  const int64_t nch = lane::n_chunks(lane::ceil_div(r0, c->k), cg);
  if (nch < C) C = (int)(nch > 0 ? nch : 1);
  const int64_t cap = lane::round_chunks(r0, c->k, cg);  // the first round is the largest
  pl->C = C;
  pl->cg = cg;
  pl->rounds = (int)lane::ceil_div(ng, RC);
  pl->round_len0 = r0;
  // ring algorithms on LL128 lines (same rounds and chunks, hence the same
  // bits): LANE_PROTO=ll128; auto above LANE_LL128_MIN_BYTES for the flat
  // ring only (the lane kernel's ring stage measured no faster on LL128:
  // profiles/r01_sizes_lane_ring2_ll128.txt)
  if (c->ll128_set > 0 && c->proto != 1 && (c->proto == 3 || (!lane_ring && ng > c->ll128_lo))) {
    const int64_t need =
        lane_ring ? lane::ll128::set_lines(c->G, c->N, cap,
                                           lane::ll128::lines_of(lane::ceil_div(lane::ceil_div(cg, c->G), c->N)))
                  : lane::ll128::ring_set_lines(c->P, cap, lane::ll128::lines_of(lane::ceil_div(cg, c->P)));
    if (need <= c->ll128_set) {
      pl->ll = lane_ring ? kLaneRingLL128 : kRingLL128;
      return true;
    }
  }
  if (lane_ring) {
    const int64_t sg = lane::ceil_div(cg, c->G), su = lane::ceil_div(sg, c->N);
    if (cap * sg > c->ll_slot_g || cap * su > c->ll_slot_u) return false;
  } else if (cap * lane::ceil_div(cg, c->P) > c->ring_slot) {
    return false;
  }
  pl->ll = lane_ring ? kLaneRingLL : kRingLL;
  return true;
}

// Plan of "approach 2" (lane_a2_ll_kernel): rounds of at most ll_max
// granules; the chunk size follows the CTA count (the result does not depend
// on it: canonical order). false: does not fit.
bool a2_plan(lane_comm_t c, int64_t ng, Plan* pl) {
  if (c->ll_bytes == 0) return false;
  const int ranks_here = c->emulated ? c->P : 1;
  int budget = c->ll_ctas > 0 ? c->ll_ctas : (c->emulated ? c->ll_coresident : c->sm_count);
  if (budget > c->ll_coresident) budget = c->ll_coresident;
  int C = budget / (ranks_here * c->k);
  if (C < 1) C = 1;
  if ((int64_t)C * c->k * ranks_here > c->ll_coresident) return false;
  const int64_t RC = c->ll_max;
  const int64_t r0 = ng < RC ? ng : RC;
  const int64_t slice0 = lane::ceil_div(r0, c->k);
  int64_t cg = lane::ceil_div(slice0, C);
  if (cg < c->ll_cg_min) cg = c->ll_cg_min;
  const int64_t nch = lane::n_chunks(slice0, cg);
  if (nch < C) C = (int)(nch > 0 ? nch : 1);
  const int64_t cap = lane::round_chunks(r0, c->k, cg);
  if (cap * lane::ceil_div(cg, c->G) > c->ll_slot_g || cap * lane::ceil_div(cg, c->N) > c->a2_slot_v) return false;
  pl->C = C;
  pl->cg = cg;
  pl->rounds = (int)lane::ceil_div(ng, RC);
  pl->round_len0 = r0;
  pl->ll = kA2LL;
  return true;
}

// One kernel launch of a call. Emulated: cooperative (every CTA of every
// rank co-resident). Multi-GPU: plain, or with programmatic stream
// serialization (LANE_PDL=1) so the grid is scheduled while the previous grid
// in the stream drains; every kernel starts with pdl_enter() (lane_kernels.cuh),
// which waits for that grid's completion before its first memory access (a
// no-op without PDL).
cudaError_t launch_kernel(lane_comm_t c, const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                          cudaStream_t s) {
  if (c->emulated) return cudaLaunchCooperativeKernel(fn, grid, block, args, smem, s);
  if (!c->pdl) return cudaLaunchKernel(fn, grid, block, args, smem, s);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Launch the rounds of a ring_plan (kRingLL, kLaneRingLL, kRingLL128,
// kLaneRingLL128) or of an a2_plan (kA2LL).
int ll_ring_rounds(lane_comm_t c, LaneParams& p, const Plan& pl, int dtype, cudaStream_t s) {
  const int ranks_here = c->emulated ? c->P : 1;
  const bool flat = pl.ll == kRingLL, a2 = pl.ll == kA2LL, ring128 = pl.ll == kRingLL128,
             lane128 = pl.ll == kLaneRingLL128;
  const int64_t RC = c->ll_max;
  p.ll_slot_g = flat ? c->ring_slot : c->ll_slot_g;
  p.ll_slot_u = flat ? 0 : (a2 ? c->a2_slot_v : c->ll_slot_u);
  p.ll_set = (ring128 || lane128) ? c->ll128_set : c->ll_set;
  p.ring2 = (pl.ll == kLaneRingLL || lane128) ? 1 : 0;
  p.handshake = 0;
  p.direct = 0;
  p.C = pl.C;
  p.cg = pl.cg;
  p.sg = lane::ceil_div(pl.cg, (flat || ring128) ? c->P : c->G);
  p.su = flat ? 0 : (a2 ? lane::ceil_div(pl.cg, c->N) : lane::ceil_div(p.sg, c->N));
  c->trace_ctas = 0;
  for (int r = 0; r < pl.rounds; ++r) {
    p.round_g0 = (int64_t)r * RC;
    const int64_t rest = pl.ng - p.round_g0;
    p.round_len = rest < RC ? rest : RC;
    p.cap = lane::round_chunks(p.round_len, c->k, p.cg);
    p.epoch = ++c->epoch;
    void* args[] = {&p};
    const void* fn;
    if (lane128)
      fn = dtype == LANE_INT32     ? (const void*)lane::ll128::lane_ll128_kernel<0, true, 1>
           : dtype == LANE_FLOAT32 ? (const void*)lane::ll128::lane_ll128_kernel<1, true, 1>
                                   : (const void*)lane::ll128::lane_ll128_kernel<2, true, 1>;
    else if (ring128)
      fn = dtype == LANE_INT32     ? (const void*)lane::ll128::lane_ring_ll128_kernel<0>
           : dtype == LANE_FLOAT32 ? (const void*)lane::ll128::lane_ring_ll128_kernel<1>
                                   : (const void*)lane::ll128::lane_ring_ll128_kernel<2>;
    else if (a2)
      fn = dtype == LANE_INT32     ? (const void*)lane::ll::lane_a2_ll_kernel<0>
           : dtype == LANE_FLOAT32 ? (const void*)lane::ll::lane_a2_ll_kernel<1>
                                   : (const void*)lane::ll::lane_a2_ll_kernel<2>;
    else if (flat)
      fn = dtype == LANE_INT32     ? (const void*)lane::ll::lane_ring_ll_kernel<0>
           : dtype == LANE_FLOAT32 ? (const void*)lane::ll::lane_ring_ll_kernel<1>
                                   : (const void*)lane::ll::lane_ring_ll_kernel<2>;
    else  // kLaneRingLL: the lane kernel with the ring inter-node stage
      fn = dtype == LANE_INT32     ? (const void*)lane::ll::lane_ll_kernel<0, true>
           : dtype == LANE_FLOAT32 ? (const void*)lane::ll::lane_ll_kernel<1, true>
                                   : (const void*)lane::ll::lane_ll_kernel<2, true>;
    const dim3 grid((unsigned)(ranks_here * c->k * pl.C));
    cudaError_t e = launch_kernel(c, fn, grid, dim3(lane::ll::kThreads), args, 0, s);
    if (e != cudaSuccess)
      return cuda_fail(c, e, lane128   ? "lane_ll128_kernel launch (ring inter-node stage)"
                             : ring128 ? "lane_ring_ll128_kernel launch"
                             : a2    ? "lane_a2_ll_kernel launch"
                                     : (flat ? "lane_ring_ll_kernel launch" : "lane_ll_kernel launch"));
  }
  return LANE_OK;
}

int launch_rounds(lane_comm_t c, LaneParams& p, const Plan& pl, int dtype, cudaStream_t s) {
  if (ll_rounds(pl)) return ll_ring_rounds(c, p, pl, dtype, s);
  const int nlocal = p.nlocal;
  for (int r = 0; r < pl.rounds; ++r) {
    p.round_g0 = (int64_t)r * c->round_cap;
    int64_t rest = pl.ng - p.round_g0;
    p.round_len = rest < c->round_cap ? rest : c->round_cap;
    p.cap = lane::round_chunks(p.round_len, c->k, p.cg);
    // the simple protocol's flag arrays hold chunk_cap chunks (the LL plan checked its inboxes itself)
    if (pl.ll == kSimple && p.cap > c->chunk_cap) return fail(c, LANE_ERR_INVALID_ARG, "internal: chunk capacity");
    // Chunk claims (LANE_DYN_CHUNKS): auto = dynamic on real peers when a CTA has at least 6 chunks
    // of the round — there per-SM push rates differ by up to 2x and the fast CTAs take more chunks
    // (1 GiB +3%, box-independent); with fewer chunks the static round-robin is 1-3% faster
    // (profiles/r02_dyn_chunks_ab_p4.txt). Emulated: static unless forced.
    if (c->dyn < 0) p.dyn = (!c->emulated && p.cap >= 6 * (int64_t)c->k * p.C) ? 1 : 0;
    p.epoch = ++c->epoch;
    const bool tma = c->engine == 1;
    dim3 grid((unsigned)(nlocal * c->k * p.C));
    if (pl.ll == kLL128) {  // LL128 protocol: one launch, no scratch flags, no handshake
      p.ll_set = c->ll128_set;  // set stride; the layout follows from p.cap, p.su (layout128)
      p.handshake = 0;
      p.direct = 0;
      c->trace_ctas = (int)grid.x;
      void* args[] = {&p};
      const bool u1 = pl.ng <= c->ll128_u1_max;  // small messages: one line per group per warp step
      const void* fn = u1 ? (dtype == LANE_INT32     ? (const void*)lane::ll128::lane_ll128_kernel<0, false, 1>
                             : dtype == LANE_FLOAT32 ? (const void*)lane::ll128::lane_ll128_kernel<1, false, 1>
                                                     : (const void*)lane::ll128::lane_ll128_kernel<2, false, 1>)
                          : (dtype == LANE_INT32     ? (const void*)lane::ll128::lane_ll128_kernel<0>
                             : dtype == LANE_FLOAT32 ? (const void*)lane::ll128::lane_ll128_kernel<1>
                                                     : (const void*)lane::ll128::lane_ll128_kernel<2>);
      cudaError_t e = launch_kernel(c, fn, grid, dim3(lane::ll128::kThreads), args, 0, s);
      if (e != cudaSuccess) return cuda_fail(c, e, "lane_ll128_kernel launch");
      continue;
    }
    if (pl.ll != kSimple) {  // kLL (every other kind returned above): LL protocol, one launch, no scratch flags, no handshake
      p.ll_slot_g = c->ll_slot_g;
      p.ll_slot_u = c->ll_slot_u;
      p.ll_set = c->ll_set;
      p.handshake = 0;
      p.direct = 0;
      c->trace_ctas = (int)grid.x;
      void* args[] = {&p};
      const void* fn = dtype == LANE_INT32     ? (const void*)lane::ll::lane_ll_kernel<0>
                       : dtype == LANE_FLOAT32 ? (const void*)lane::ll::lane_ll_kernel<1>
                                               : (const void*)lane::ll::lane_ll_kernel<2>;
      cudaError_t e = launch_kernel(c, fn, grid, dim3(lane::ll::kThreads), args, 0, s);
      if (e != cudaSuccess) return cuda_fail(c, e, "lane_ll_kernel launch");
      continue;
    }
    c->trace_ctas = (int)grid.x;
    dim3 block((unsigned)(tma ? lane::tma::kThreads : c->threads));
    const size_t smem = tma ? (size_t)lane::tma::kSmemBytes : 0;
    cudaError_t e;
    void* args[] = {&p};
    const void* fn;
    const bool lsu_store = c->store_mode == 1 || (c->store_mode == 0 && pl.ng < c->bulk_min);
    if (tma && lsu_store)
      fn = dtype == LANE_INT32     ? (const void*)lane::tma::lane_tma_kernel<0, true>
           : dtype == LANE_FLOAT32 ? (const void*)lane::tma::lane_tma_kernel<1, true>
                                   : (const void*)lane::tma::lane_tma_kernel<2, true>;
    else if (tma)
      fn = dtype == LANE_INT32     ? (const void*)lane::tma::lane_tma_kernel<0, false>
           : dtype == LANE_FLOAT32 ? (const void*)lane::tma::lane_tma_kernel<1, false>
                                   : (const void*)lane::tma::lane_tma_kernel<2, false>;
    else
      fn = dtype == LANE_INT32     ? (const void*)lane::lane_allreduce_kernel<0>
           : dtype == LANE_FLOAT32 ? (const void*)lane::lane_allreduce_kernel<1>
                                   : (const void*)lane::lane_allreduce_kernel<2>;
    e = launch_kernel(c, fn, grid, block, args, smem, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "lane_allreduce_kernel launch");
  }
  return LANE_OK;
}

// The device-side error word (watchdog timeout, start-handshake mismatch).
int device_error(lane_comm_t c, const char* when) {
  const uint32_t w = c->err_host ? *(volatile uint32_t*)c->err_host : 0u;
  if (w == 0) return LANE_OK;
  if (w == (uint32_t)(-LANE_ERR_MISMATCH))
    return fail(c, LANE_ERR_MISMATCH,
                std::string("comm: ranks disagreed on a call (zero-copy vs staged buffers, registration, offsets, "
                            "count or dtype)") + when + "; finalize the comm");
  return fail(c, LANE_ERR_TIMEOUT, std::string("comm: a device-side wait timed out") + when);
}

// CUDA graph capture. A captured launch would replay the epoch it was captured
// with, so once a comm sees a capturing stream it switches for good to
// device-side epochs (LaneParams::dev_epoch; lane_kernels.cuh launch_prologue):
// every launch, captured or not, takes the next epoch from device memory and
// advances it there. The device word follows the host counter on every eager
// launch, so the switch can happen at any call.
int note_capture(lane_comm_t c, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaError_t e = cudaStreamIsCapturing(s, &st);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamIsCapturing");
  if (st != cudaStreamCaptureStatusNone) c->dev_epoch = 1;
  return LANE_OK;
}

// The host-buffer entry points synchronise their staging streams and cannot
// be captured.
int refuse_capture(lane_comm_t c, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaError_t e = cudaStreamIsCapturing(s, &st);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamIsCapturing");
  if (st != cudaStreamCaptureStatusNone)
    return fail(c, LANE_ERR_UNSUPPORTED, "stream: the host-buffer API cannot be captured into a CUDA graph");
  return LANE_OK;
}

int check_call(lane_comm_t c, uint64_t count, int dtype, int op) {
  if (!c) return LANE_ERR_INVALID_ARG;
  if (dtype < LANE_INT32 || dtype > LANE_BFLOAT16)
    return fail(c, LANE_ERR_UNSUPPORTED, "dtype: unsupported lane_dtype_t");
  if (op != LANE_SUM) return fail(c, LANE_ERR_UNSUPPORTED, "op: only LANE_SUM (MPI_SUM, P L341)");
  if (!c->connected)
    return fail(c, LANE_ERR_NOT_CONNECTED, "comm: lane_allreduce_open_peers has not completed");
  int e = device_error(c, " in an earlier call");
  if (e != LANE_OK) return e;
  (void)count;
  return LANE_OK;
}

int check_buffers(lane_comm_t c, const void* s, const void* r, uint64_t bytes, const char* which) {
  if (!s || !r) return fail(c, LANE_ERR_INVALID_ARG, std::string(which) + ": null buffer");
  if (((uintptr_t)s | (uintptr_t)r) & 15)
    return fail(c, LANE_ERR_MISALIGNED, std::string(which) + ": buffers must be 16-byte aligned");
  if (overlaps_partially(s, r, bytes))
    return fail(c, LANE_ERR_INVALID_ARG, std::string(which) + ": sendbuf and recvbuf partially overlap");
  return LANE_OK;
}

int copy_p1(lane_comm_t c, const void* s, void* r, const Plan& pl, cudaStream_t st) {
  if (s == r) return LANE_OK;
  const int tail_bytes = pl.tail_elems < pl.q ? pl.tail_elems * (16 / pl.q) : 0;
  int64_t blocks = (pl.ng + 511) / 512;
  if (blocks > (int64_t)c->sm_count * 4) blocks = (int64_t)c->sm_count * 4;
  lane::lane_copy_kernel<<<(unsigned)blocks, 512, 0, st>>>(
      reinterpret_cast<const uint4*>(s), reinterpret_cast<uint4*>(r), pl.ng, tail_bytes);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, "lane_copy_kernel launch");
  return LANE_OK;
}

int find_reg(lane_comm_t c, const void* ptr, uint64_t bytes) {
  const char* q = static_cast<const char*>(ptr);
  for (size_t i = 0; i < c->regs.size(); ++i) {
    const auto& r = c->regs[i];
    if (r.live && q >= r.base && q + bytes <= r.base + r.bytes) return (int)i;
  }
  return -1;
}

// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda,
// so the library still loads on hosts without a driver).
typedef int (*GetRangeFn)(unsigned long long*, size_t*, unsigned long long);

int alloc_base(lane_comm_t c, const void* ptr, char** base) {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || !f) return cuda_fail(c, e, "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
    fn = reinterpret_cast<GetRangeFn>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)ptr) != 0)
    return fail(c, LANE_ERR_INVALID_ARG, "register: ptr is not device memory from cudaMalloc");
  *base = reinterpret_cast<char*>((uintptr_t)b);
  return LANE_OK;
}

struct RegBlob {
  uint32_t magic;
  int32_t rank;
  uint64_t bytes, offset;
  cudaIpcMemHandle_t handle;
};

int ensure_stage(lane_comm_t c, uint64_t bytes) {
  const int nbuf = 4 * (c->emulated ? c->P : 1);  // 2 pipeline slots x (send, recv) per rank
  if (c->stage_bytes >= bytes && (int)c->stage.size() == nbuf) return LANE_OK;
  // Growing the staging: the copy streams and events live as long as the comm
  // (release()); only the buffers are replaced. Earlier calls' copies and
  // kernels may still use the old buffers: wait for them first.
  if (!c->stage.empty()) {
    LANE_CUDA(c, cudaDeviceSynchronize());
    for (char* p : c->stage) cudaFree(p);
  }
  c->stage.clear();
  c->stage_bytes = 0;
  for (int i = 0; i < nbuf; ++i) {
    char* p = nullptr;
    LANE_CUDA(c, cudaMalloc(&p, bytes ? bytes : 16));
    c->stage.push_back(p);
  }
  c->stage_bytes = bytes;
  return LANE_OK;
}

}  // namespace

extern "C" {

const char* lane_allreduce_version(void) { return "lane_allreduce 0.1 (sm_100a)"; }

int lane_allreduce_init_rank(int nodes, int gpus_per_node, int procs_per_gpu, int rank, int device,
                             lane_comm_t* comm) {
  if (!comm) return LANE_ERR_INVALID_ARG;
  *comm = nullptr;
  if (rank < 0 || (int64_t)rank >= (int64_t)nodes * gpus_per_node) {
    int st = validate_topology(nodes, gpus_per_node, procs_per_gpu, &g_init_error);
    if (st == LANE_OK) g_init_error = "rank: must be in [0, nodes*gpus_per_node)";
    return LANE_ERR_INVALID_ARG;
  }
  return common_init(nodes, gpus_per_node, procs_per_gpu, rank, device, false, comm);
}

int lane_allreduce_init(int nodes, int gpus_per_node, int procs_per_gpu, lane_comm_t* comm) {
  if (!comm) return LANE_ERR_INVALID_ARG;
  *comm = nullptr;
  const char* r = getenv("RANK");
  const char* lr = getenv("LOCAL_RANK");
  const char* ws = getenv("WORLD_SIZE");
  if (!r || !ws) {
    g_init_error = "RANK/WORLD_SIZE: not set (use lane_allreduce_init_rank)";
    return LANE_ERR_INVALID_ARG;
  }
  int rank = atoi(r), world = atoi(ws), local = lr ? atoi(lr) : rank;
  if ((int64_t)nodes * gpus_per_node != world) {
    g_init_error = "nodes*gpus_per_node: must equal WORLD_SIZE";
    return LANE_ERR_INVALID_ARG;
  }
  return lane_allreduce_init_rank(nodes, gpus_per_node, procs_per_gpu, rank, local, comm);
}

int lane_allreduce_init_emulated(int nodes, int gpus_per_node, int procs_per_gpu, int device,
                                 lane_comm_t* comm) {
  if (!comm) return LANE_ERR_INVALID_ARG;
  *comm = nullptr;
  return common_init(nodes, gpus_per_node, procs_per_gpu, 0, device, true, comm);
}

int lane_allreduce_get_handle(lane_comm_t c, void* blob, size_t* blob_bytes) {
  if (!c || !blob || !blob_bytes) return fail(c, LANE_ERR_INVALID_ARG, "get_handle: null argument");
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "get_handle: emulated comm has no peers");
  Blob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagic;
  b.version = kVersion;
  b.N = c->N;
  b.G = c->G;
  b.k = c->k;
  b.rank = c->rank;
  b.device = c->device;
  b.pid = (int32_t)getpid();
  b.s1_bytes = c->s1_bytes;
  b.s2_bytes = c->s2_bytes;
  b.r_bytes = c->r_bytes;
  b.flag_bytes = c->flag_bytes;
  b.total_bytes = c->total_bytes;
  b.round_cap = c->round_cap;
  b.chunk_cap = c->chunk_cap;
  b.handle = c->handle;
  memcpy(b.settings, c->settings, sizeof(b.settings));
  memcpy(blob, &b, sizeof(b));
  *blob_bytes = sizeof(b);
  return LANE_OK;
}

int lane_allreduce_open_peers(lane_comm_t c, const void* all_blobs, size_t blob_bytes) {
  if (!c || !all_blobs) return fail(c, LANE_ERR_INVALID_ARG, "open_peers: null argument");
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "open_peers: emulated comm has no peers");
  if (c->connected) return fail(c, LANE_ERR_INVALID_ARG, "open_peers: already connected");
  if (blob_bytes < sizeof(Blob)) return fail(c, LANE_ERR_INVALID_ARG, "blob_bytes: too small");
  LANE_CUDA(c, cudaSetDevice(c->device));
  const char* base = static_cast<const char*>(all_blobs);
  for (int p = 0; p < c->P; ++p) {
    Blob b;
    memcpy(&b, base + (size_t)p * blob_bytes, sizeof(b));
    if (b.magic != kMagic || b.version != kVersion)
      return fail(c, LANE_ERR_INVALID_ARG, "all_blobs[" + std::to_string(p) + "]: not a lane blob");
    if (b.rank != p) return fail(c, LANE_ERR_INVALID_ARG, "all_blobs: not in rank order");
    if (b.N != c->N || b.G != c->G || b.k != c->k)
      return fail(c, LANE_ERR_INVALID_ARG, "all_blobs: ranks disagree on (nodes, gpus_per_node, procs_per_gpu)");
    for (int i = 0; i < kNumSettings; ++i)
      if (b.settings[i] != c->settings[i])
        return fail(c, LANE_ERR_INVALID_ARG,
                    std::string("all_blobs: ranks disagree on ") + kSettingNames[i] + " (rank " + std::to_string(p) +
                        ": " + std::to_string(b.settings[i]) + ", rank " + std::to_string(c->rank) + ": " +
                        std::to_string(c->settings[i]) + "; plan-shaping LANE_* settings must match)");
    if (b.total_bytes != c->total_bytes || b.round_cap != c->round_cap || b.chunk_cap != c->chunk_cap)
      return fail(c, LANE_ERR_INVALID_ARG, "all_blobs: ranks disagree on scratch geometry (LANE_ROUND_BYTES)");
    if (p == c->rank) continue;
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcOpenMemHandle");
    c->opened.push_back(ptr);
    carve(c, static_cast<char*>(ptr), &c->rk[p]);
  }
  c->connected = true;
  return LANE_OK;
}

int lane_allreduce(lane_comm_t c, const void* sendbuf, void* recvbuf, size_t count,
                   lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce: use lane_allreduce_emulated");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  st = check_buffers(c, sendbuf, recvbuf, bytes, "lane_allreduce");
  if (st != LANE_OK) return st;
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbuf, recvbuf, pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = c->rank;
  p.nlocal = 1;
  p.rk[c->rank].send = static_cast<const char*>(sendbuf);
  p.rk[c->rank].recv = static_cast<char*>(recvbuf);
  // zero-copy when both buffers are registered (P L330: the user buffer is
  // shared through IPC handles); peers use the same offsets into theirs
  const int rs = find_reg(c, sendbuf, bytes), rr = find_reg(c, recvbuf, bytes);
  uint64_t so = 0, ro = 0;
  if (c->engine == 1 && rs >= 0 && rr >= 0 && c->direct_mode != 0) {
    const auto& S = c->regs[rs];
    const auto& R = c->regs[rr];
    so = (uint64_t)(static_cast<const char*>(sendbuf) - S.base);
    ro = (uint64_t)(static_cast<char*>(recvbuf) - R.base);
    for (int q = 0; q < c->P; ++q)
      if (q != c->rank) {
        p.rk[q].send = S.peer[q] + so;
        p.rk[q].recv = R.peer[q] + ro;
      }
    p.direct = c->direct_mode;  // push flavour by default on real peers
  }
  // The TMA engine's simple protocol always runs the start/end handshake on
  // real peers: it carries the call signature, so ranks that disagree on the
  // job set (a buffer registered on one rank only), the registrations or
  // offsets, the count or the dtype stop with LANE_ERR_MISMATCH.
  p.handshake = c->engine == 1 ? 1 : 0;
  p.sig = call_signature(c, pl, p.direct, p.direct ? rs : -1, p.direct ? rr : -1, so, ro, dtype);
  return launch_rounds(c, p, pl, dtype, s);
}

int lane_allreduce_emulated(lane_comm_t c, const void* const* sendbufs, void* const* recvbufs,
                            size_t count, lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (!c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_emulated: comm is not emulated");
  if (!sendbufs || !recvbufs) return fail(c, LANE_ERR_INVALID_ARG, "sendbufs/recvbufs: null");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  for (int r = 0; r < c->P; ++r) {
    st = check_buffers(c, sendbufs[r], recvbufs[r], bytes,
                       ("rank " + std::to_string(r)).c_str());
    if (st != LANE_OK) return st;
  }
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbufs[0], recvbufs[0], pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = 0;
  p.nlocal = c->P;
  // emulated: every buffer is addressable; pull flavour by default (fewest HBM
  // bytes), LANE_DIRECT=2 runs the push flavour of the multi-GPU path
  p.direct = c->engine == 1 ? c->direct_emu : 0;
  // test switch: the registered calls' start/end handshake (and its call
  // signature) across the emulated ranks
  p.handshake = (c->engine == 1 && c->emu_handshake) ? 1 : 0;
  p.sig = call_signature(c, pl, p.direct, -1, -1, 0, 0, dtype);
  for (int r = 0; r < c->P; ++r) {
    p.rk[r].send = static_cast<const char*>(sendbufs[r]);
    p.rk[r].recv = static_cast<char*>(recvbufs[r]);
  }
  return launch_rounds(c, p, pl, dtype, s);
}

static int ring_rounds(lane_comm_t c, LaneParams& p, const Plan& lane_pl, int dtype, cudaStream_t s) {
  if (c->ll_bytes == 0) return fail(c, LANE_ERR_INVALID_ARG, "ring: LANE_LL_MAX_BYTES is 0 (no LL inboxes)");
  Plan pl = lane_pl;
  if (!ring_plan(c, lane_pl.ng, false, &pl))
    return fail(c, LANE_ERR_INVALID_ARG, "ring: procs_per_gpu exceeds the co-resident CTA capacity or inboxes");
  return ll_ring_rounds(c, p, pl, dtype, s);
}

int lane_allreduce_ring(lane_comm_t c, const void* sendbuf, void* recvbuf, size_t count, lane_dtype_t dtype,
                        lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_ring: use lane_allreduce_ring_emulated");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  st = check_buffers(c, sendbuf, recvbuf, bytes, "lane_allreduce_ring");
  if (st != LANE_OK) return st;
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbuf, recvbuf, pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = c->rank;
  p.nlocal = 1;
  p.rk[c->rank].send = static_cast<const char*>(sendbuf);
  p.rk[c->rank].recv = static_cast<char*>(recvbuf);
  return ring_rounds(c, p, pl, dtype, s);
}

int lane_allreduce_ring_emulated(lane_comm_t c, const void* const* sendbufs, void* const* recvbufs, size_t count,
                                 lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (!c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_ring_emulated: comm is not emulated");
  if (!sendbufs || !recvbufs) return fail(c, LANE_ERR_INVALID_ARG, "sendbufs/recvbufs: null");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  for (int r = 0; r < c->P; ++r) {
    st = check_buffers(c, sendbufs[r], recvbufs[r], bytes, ("rank " + std::to_string(r)).c_str());
    if (st != LANE_OK) return st;
  }
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbufs[0], recvbufs[0], pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = 0;
  p.nlocal = c->P;
  for (int r = 0; r < c->P; ++r) {
    p.rk[r].send = static_cast<const char*>(sendbufs[r]);
    p.rk[r].recv = static_cast<char*>(recvbufs[r]);
  }
  return ring_rounds(c, p, pl, dtype, s);
}

// "Approach 2" entry points (same argument rules as lane_allreduce / _emulated).
static int a2_call(lane_comm_t c, LaneParams& p, const Plan& lane_pl, int dtype, cudaStream_t s) {
  Plan pl = lane_pl;
  if (!a2_plan(c, lane_pl.ng, &pl))
    return fail(c, LANE_ERR_INVALID_ARG, "approach2: procs_per_gpu exceeds the co-resident CTA capacity or inboxes");
  return ll_ring_rounds(c, p, pl, dtype, s);
}

int lane_allreduce_approach2(lane_comm_t c, const void* sendbuf, void* recvbuf, size_t count,
                             lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (c->emulated)
    return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_approach2: use lane_allreduce_approach2_emulated");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  st = check_buffers(c, sendbuf, recvbuf, bytes, "lane_allreduce_approach2");
  if (st != LANE_OK) return st;
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbuf, recvbuf, pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = c->rank;
  p.nlocal = 1;
  p.rk[c->rank].send = static_cast<const char*>(sendbuf);
  p.rk[c->rank].recv = static_cast<char*>(recvbuf);
  return a2_call(c, p, pl, dtype, s);
}

int lane_allreduce_approach2_emulated(lane_comm_t c, const void* const* sendbufs, void* const* recvbufs,
                                      size_t count, lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (!c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_approach2_emulated: comm is not emulated");
  if (!sendbufs || !recvbufs) return fail(c, LANE_ERR_INVALID_ARG, "sendbufs/recvbufs: null");
  if (count == 0) return LANE_OK;
  const uint64_t bytes = (uint64_t)count * itemsize_of(dtype);
  for (int r = 0; r < c->P; ++r) {
    st = check_buffers(c, sendbufs[r], recvbufs[r], bytes, ("rank " + std::to_string(r)).c_str());
    if (st != LANE_OK) return st;
  }
  Plan pl;
  st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = note_capture(c, s)) != LANE_OK) return st;
  if (c->P == 1) return copy_p1(c, sendbufs[0], recvbufs[0], pl, s);
  LaneParams p = base_params(c, pl);
  p.rank0 = 0;
  p.nlocal = c->P;
  for (int r = 0; r < c->P; ++r) {
    p.rk[r].send = static_cast<const char*>(sendbufs[r]);
    p.rk[r].recv = static_cast<char*>(recvbufs[r]);
  }
  return a2_call(c, p, pl, dtype, s);
}

// Pipelined host-buffer allreduce: the message is cut into granule-aligned
// pieces (each its own collective allreduce — results do not depend on the
// partition); piece i+1's H2D copy and piece i-1's D2H copy run on library
// streams while piece i's kernel runs on the caller's stream. Staging is
// double-buffered; the caller's stream finally waits for the last D2H.
static int host_pipeline(lane_comm_t c, const void* const* hs, void* const* hr, size_t count, int dtype, int op,
                  cudaStream_t s) {
  const int nr = c->emulated ? c->P : 1;
  const int isz = itemsize_of(dtype);
  const int q = 16 / isz;
  int64_t piece = env_i64("LANE_HOST_PIECE_BYTES", 64 << 20) / isz;
  piece = piece / q * q;
  if (piece < q) piece = q;
  if ((uint64_t)piece > count) piece = (int64_t)count;
  int st = ensure_stage(c, (uint64_t)piece * isz);
  if (st != LANE_OK) return st;
  LANE_CUDA(c, cudaSetDevice(c->device));
  if (!c->h2d) {
    LANE_CUDA(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    LANE_CUDA(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    LANE_CUDA(c, cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      LANE_CUDA(c, cudaEventCreateWithFlags(&c->ev_h[i], cudaEventDisableTiming));
      LANE_CUDA(c, cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
      LANE_CUDA(c, cudaEventCreateWithFlags(&c->ev_d[i], cudaEventDisableTiming));
    }
  }
  // staging reuse across calls is ordered through the caller's stream
  LANE_CUDA(c, cudaEventRecord(c->ev_start, s));
  LANE_CUDA(c, cudaStreamWaitEvent(c->h2d, c->ev_start, 0));
  std::vector<const void*> sends(nr);
  std::vector<void*> recvs(nr);
  const int64_t np = ((int64_t)count + piece - 1) / piece;
  for (int64_t i = 0; i < np; ++i) {
    const int slot = (int)(i & 1);
    const uint64_t off = (uint64_t)i * piece;
    const uint64_t n = ((uint64_t)piece < count - off) ? (uint64_t)piece : count - off;
    if (i >= 2) LANE_CUDA(c, cudaStreamWaitEvent(c->h2d, c->ev_k[slot], 0));  // kernel i-2 read its send slot
    for (int r = 0; r < nr; ++r) {
      char* ss = c->stage[4 * r + 2 * slot];
      LANE_CUDA(c, cudaMemcpyAsync(ss, static_cast<const char*>(hs[r]) + off * isz, n * isz,
                                   cudaMemcpyHostToDevice, c->h2d));
      sends[r] = ss;
      recvs[r] = c->stage[4 * r + 2 * slot + 1];
    }
    LANE_CUDA(c, cudaEventRecord(c->ev_h[slot], c->h2d));
    LANE_CUDA(c, cudaStreamWaitEvent(s, c->ev_h[slot], 0));
    if (i >= 2) LANE_CUDA(c, cudaStreamWaitEvent(s, c->ev_d[slot], 0));  // D2H i-2 read its recv slot
    st = c->emulated ? lane_allreduce_emulated(c, sends.data(), recvs.data(), n, (lane_dtype_t)dtype,
                                               (lane_op_t)op, s)
                     : lane_allreduce(c, sends[0], recvs[0], n, (lane_dtype_t)dtype, (lane_op_t)op, s);
    if (st != LANE_OK) return st;
    LANE_CUDA(c, cudaEventRecord(c->ev_k[slot], s));
    LANE_CUDA(c, cudaStreamWaitEvent(c->d2h, c->ev_k[slot], 0));
    for (int r = 0; r < nr; ++r)
      LANE_CUDA(c, cudaMemcpyAsync(static_cast<char*>(hr[r]) + off * isz, recvs[r], n * isz,
                                   cudaMemcpyDeviceToHost, c->d2h));
    LANE_CUDA(c, cudaEventRecord(c->ev_d[slot], c->d2h));
  }
  LANE_CUDA(c, cudaStreamWaitEvent(s, c->ev_d[(np - 1) & 1], 0));
  return LANE_OK;
}

int lane_allreduce_host(lane_comm_t c, const void* host_send, void* host_recv, size_t count,
                        lane_dtype_t dtype, lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_host: use lane_allreduce_emulated_host");
  if (count == 0) return LANE_OK;
  if (!host_send || !host_recv) return fail(c, LANE_ERR_INVALID_ARG, "host buffers: null");
  if ((st = refuse_capture(c, static_cast<cudaStream_t>(stream))) != LANE_OK) return st;
  const void* hs[1] = {host_send};
  void* hr[1] = {host_recv};
  return host_pipeline(c, hs, hr, count, dtype, op, static_cast<cudaStream_t>(stream));
}

int lane_allreduce_emulated_host(lane_comm_t c, const void* const* host_sends,
                                 void* const* host_recvs, size_t count, lane_dtype_t dtype,
                                 lane_op_t op, void* stream) {
  int st = check_call(c, count, dtype, op);
  if (st != LANE_OK) return st;
  if (!c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "lane_allreduce_emulated_host: comm is not emulated");
  if (count == 0) return LANE_OK;
  if (!host_sends || !host_recvs) return fail(c, LANE_ERR_INVALID_ARG, "host buffers: null");
  for (int r = 0; r < c->P; ++r)
    if (!host_sends[r] || !host_recvs[r]) return fail(c, LANE_ERR_INVALID_ARG, "host buffers: null");
  if ((st = refuse_capture(c, static_cast<cudaStream_t>(stream))) != LANE_OK) return st;
  return host_pipeline(c, host_sends, host_recvs, count, dtype, op, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

extern "C" {

int lane_allreduce_register_handle(lane_comm_t c, void* ptr, size_t bytes, void* blob,
                                   size_t* blob_bytes) {
  if (!c || !ptr || !blob || !blob_bytes) return fail(c, LANE_ERR_INVALID_ARG, "register: null argument");
  if (c->emulated) return fail(c, LANE_ERR_INVALID_ARG, "register: emulated comms address every buffer already");
  if ((uintptr_t)ptr & 15) return fail(c, LANE_ERR_MISALIGNED, "register: ptr must be 16-byte aligned");
  LANE_CUDA(c, cudaSetDevice(c->device));
  char* base = nullptr;
  int st = alloc_base(c, ptr, &base);
  if (st != LANE_OK) return st;
  RegBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagic ^ 0x52454721u;
  b.rank = c->rank;
  b.bytes = bytes;
  b.offset = (uint64_t)(static_cast<char*>(ptr) - base);
  LANE_CUDA(c, cudaIpcGetMemHandle(&b.handle, base));
  memcpy(blob, &b, sizeof(b));
  *blob_bytes = sizeof(b);
  c->pending_reg = static_cast<char*>(ptr);
  c->pending_bytes = bytes;
  return LANE_OK;
}

int lane_allreduce_register_open(lane_comm_t c, const void* all_blobs, size_t blob_bytes, int* reg_id) {
  if (!c || !all_blobs || !reg_id) return fail(c, LANE_ERR_INVALID_ARG, "register_open: null argument");
  if (!c->pending_reg) return fail(c, LANE_ERR_INVALID_ARG, "register_open: no register_handle pending");
  if (blob_bytes < sizeof(RegBlob)) return fail(c, LANE_ERR_INVALID_ARG, "blob_bytes: too small");
  LANE_CUDA(c, cudaSetDevice(c->device));
  lane_comm_s::Reg r;
  memset(&r, 0, sizeof(r));
  r.base = c->pending_reg;
  r.bytes = c->pending_bytes;
  r.live = true;
  const char* blobs = static_cast<const char*>(all_blobs);
  for (int q = 0; q < c->P; ++q) {
    RegBlob b;
    memcpy(&b, blobs + (size_t)q * blob_bytes, sizeof(b));
    if (b.magic != (kMagic ^ 0x52454721u) || b.rank != q)
      return fail(c, LANE_ERR_INVALID_ARG, "all_blobs: not register blobs in rank order");
    if (b.bytes != r.bytes)
      return fail(c, LANE_ERR_INVALID_ARG, "register: ranks registered buffers of different sizes");
    if (q == c->rank) {
      r.peer[q] = r.base;
      continue;
    }
    std::string key(reinterpret_cast<const char*>(&b.handle), sizeof(b.handle));
    void* mapped = nullptr;
    for (auto& e : c->ipc_cache)
      if (e.first == key) mapped = e.second;
    if (!mapped) {
      cudaError_t e = cudaIpcOpenMemHandle(&mapped, b.handle, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcOpenMemHandle (register)");
      c->ipc_cache.emplace_back(key, mapped);
    }
    r.peer[q] = static_cast<char*>(mapped) + b.offset;
  }
  c->pending_reg = nullptr;
  c->regs.push_back(r);
  *reg_id = (int)c->regs.size() - 1;
  return LANE_OK;
}

int lane_allreduce_deregister(lane_comm_t c, int reg_id) {
  if (!c || reg_id < 0 || reg_id >= (int)c->regs.size()) return fail(c, LANE_ERR_INVALID_ARG, "reg_id: unknown");
  c->regs[reg_id].live = false;
  return LANE_OK;
}

int lane_allreduce_finalize(lane_comm_t c) {
  if (!c) return LANE_ERR_INVALID_ARG;
  release(c);
  return LANE_OK;
}

}  // extern "C"

namespace {
void release(lane_comm_t c) {
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (auto& e : c->ipc_cache) cudaIpcCloseMemHandle(e.second);
  for (char* p : c->own) cudaFree(p);
  for (char* p : c->stage) cudaFree(p);
  if (c->h2d) {
    cudaStreamDestroy(c->h2d);
    cudaStreamDestroy(c->d2h);
    cudaEventDestroy(c->ev_start);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(c->ev_h[i]);
      cudaEventDestroy(c->ev_k[i]);
      cudaEventDestroy(c->ev_d[i]);
    }
  }
  if (c->abort_dev) cudaFree(c->abort_dev);
  if (c->claims) cudaFree(c->claims);
  if (c->epoch_dev) cudaFree(c->epoch_dev);
  if (c->trace) cudaFree(c->trace);
  if (c->err_host) cudaFreeHost(c->err_host);
  delete c;
}
}  // namespace

extern "C" {

const char* lane_allreduce_last_error(lane_comm_t c) {
  if (!c) return g_init_error.c_str();  // init failures return no comm
  return c->last_error.c_str();
}

int lane_allreduce_trace(lane_comm_t c, uint64_t* out, size_t max_words, size_t* n_words) {
  if (!c) return LANE_ERR_INVALID_ARG;
  if (!c->trace) return fail(c, LANE_ERR_INVALID_ARG, "trace: comm was created without LANE_TRACE=1");
  const size_t n = (size_t)c->trace_ctas * lane::kTraceWords;
  if (n_words) *n_words = n;
  if (out && max_words) {
    LANE_CUDA(c, cudaSetDevice(c->device));
    LANE_CUDA(c, cudaDeviceSynchronize());
    LANE_CUDA(c, cudaMemcpy(out, c->trace, (max_words < n ? max_words : n) * 8, cudaMemcpyDeviceToHost));
  }
  return LANE_OK;
}

int lane_allreduce_check(lane_comm_t c) {
  if (!c) return LANE_ERR_INVALID_ARG;
  return device_error(c, "");
}

int lane_allreduce_plan(lane_comm_t c, size_t count, lane_dtype_t dtype, int64_t* chunk_granules,
                        int64_t* round_granules, int* ctas_per_group, int* launches) {
  if (!c) return LANE_ERR_INVALID_ARG;
  if (dtype < LANE_INT32 || dtype > LANE_BFLOAT16)
    return fail(c, LANE_ERR_UNSUPPORTED, "dtype: unsupported lane_dtype_t");
  Plan pl;
  int st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  if (chunk_granules) *chunk_granules = pl.cg;
  if (round_granules) *round_granules = ll_rounds(pl) ? c->ll_max : c->round_cap;
  if (ctas_per_group) *ctas_per_group = pl.C;
  if (launches) *launches = count == 0 ? 0 : (c->P == 1 ? 1 : pl.rounds);
  return LANE_OK;
}

int lane_allreduce_ring_plan(lane_comm_t c, size_t count, lane_dtype_t dtype, int64_t* chunk_granules,
                             int64_t* round_granules, int* ctas_per_group, int* launches) {
  if (!c) return LANE_ERR_INVALID_ARG;
  if (dtype < LANE_INT32 || dtype > LANE_BFLOAT16)
    return fail(c, LANE_ERR_UNSUPPORTED, "dtype: unsupported lane_dtype_t");
  const int q = 16 / itemsize_of(dtype);
  Plan pl;
  memset(&pl, 0, sizeof(pl));
  pl.ng = (int64_t)((count + q - 1) / q);
  if (!ring_plan(c, pl.ng, false, &pl))
    return fail(c, LANE_ERR_INVALID_ARG, "ring: procs_per_gpu exceeds the co-resident CTA capacity or inboxes");
  if (chunk_granules) *chunk_granules = pl.cg;
  if (round_granules) *round_granules = c->ll_max;
  if (ctas_per_group) *ctas_per_group = pl.C;
  if (launches) *launches = count == 0 ? 0 : (c->P == 1 ? 1 : pl.rounds);
  return LANE_OK;
}

int lane_ll128_plan_query(int nodes, int gpus_per_node, int procs_per_gpu, int64_t granules, int ctas_per_group,
                          int64_t max_bytes, int64_t min_chunk_bytes, int64_t* out) {
  std::string why;
  int st = validate_topology(nodes, gpus_per_node, procs_per_gpu, &why);
  if (st != LANE_OK) return st;
  if (!out || granules < 0 || ctas_per_group < 1 || max_bytes < 16 || min_chunk_bytes < 16)
    return LANE_ERR_INVALID_ARG;
  const int64_t M = max_bytes / 16, cgm = min_chunk_bytes / 16;
  const lane::ll128::Plan128 g =
      lane::ll128::plan128(gpus_per_node, nodes, procs_per_gpu, granules, ctas_per_group, M, cgm);
  out[0] = g.C;
  out[1] = g.cg;
  out[2] = g.cap;
  out[3] = g.lu;
  out[4] = g.need;
  out[5] = lane::ll128::set_capacity128(gpus_per_node, nodes, procs_per_gpu, M, cgm);
  return LANE_OK;
}

int lane_ll128_line_query(int nodes, int gpus_per_node, int64_t chunks, int64_t lines_per_subpart, int kind, int slot,
                          int64_t chunk, int b, int64_t line, int64_t* index) {
  const int N = nodes, G = gpus_per_node;
  if (!index || N < 1 || G < 1 || chunks < 1 || lines_per_subpart < 1) return LANE_ERR_INVALID_ARG;
  if (chunk < 0 || chunk >= chunks || line < 0 || line >= lines_per_subpart) return LANE_ERR_INVALID_ARG;
  const lane::ll128::Layout128 y = lane::ll128::layout128(G, N, chunks, lines_per_subpart);
  const lane::ll128::RingLayout128 ry = lane::ll128::ring_layout128(N * G, chunks, lines_per_subpart);
  switch (kind) {
    case 5:
    case 6:
      if (slot < 0 || slot >= N * G - 1) return LANE_ERR_INVALID_ARG;
      *index = kind == 5 ? ry.rs(slot, chunk, line) : ry.ag(slot, chunk, line);
      return LANE_OK;
    case 1:
    case 4:
      if (slot < 0 || slot >= G - 1 || b < 0 || b >= N) return LANE_ERR_INVALID_ARG;
      *index = kind == 1 ? y.l1(slot, chunk, b, line) : y.l4(slot, chunk, b, line);
      return LANE_OK;
    case 2:
    case 3:
      if (slot < 0 || slot >= N) return LANE_ERR_INVALID_ARG;
      *index = kind == 2 ? y.l2(slot, chunk, line) : y.l3(slot, chunk, line);
      return LANE_OK;
    default:
      return LANE_ERR_INVALID_ARG;
  }
}

int lane_allreduce_ring_protocol(lane_comm_t c, size_t count, lane_dtype_t dtype, int* protocol) {
  if (!c || !protocol) return fail(c, LANE_ERR_INVALID_ARG, "ring_protocol: null argument");
  if (dtype < LANE_INT32 || dtype > LANE_BFLOAT16)
    return fail(c, LANE_ERR_UNSUPPORTED, "dtype: unsupported lane_dtype_t");
  const int q = 16 / itemsize_of(dtype);
  Plan pl;
  memset(&pl, 0, sizeof(pl));
  pl.ng = (int64_t)((count + q - 1) / q);
  if (!ring_plan(c, pl.ng, false, &pl))
    return fail(c, LANE_ERR_INVALID_ARG, "ring: procs_per_gpu exceeds the co-resident CTA capacity or inboxes");
  *protocol = pl.ll == kRingLL128 ? LANE_PROTO_LL128 : LANE_PROTO_LL;
  return LANE_OK;
}

int lane_allreduce_protocol(lane_comm_t c, size_t count, lane_dtype_t dtype, int* protocol) {
  if (!c || !protocol) return fail(c, LANE_ERR_INVALID_ARG, "protocol: null argument");
  if (dtype < LANE_INT32 || dtype > LANE_BFLOAT16)
    return fail(c, LANE_ERR_UNSUPPORTED, "dtype: unsupported lane_dtype_t");
  Plan pl;
  int st = make_plan(c, count, dtype, &pl);
  if (st != LANE_OK) return st;
  *protocol = (count == 0 || c->P == 1) ? LANE_PROTO_SIMPLE : ((pl.ll == kLL128 || pl.ll == kLaneRingLL128) ? LANE_PROTO_LL128
                                                                  : (pl.ll != kSimple ? LANE_PROTO_LL : LANE_PROTO_SIMPLE));
  return LANE_OK;
}

int lane_topology_query(int nodes, int gpus_per_node, int rank, int* node, int* gpu,
                        int* group_ranks, int* lane_ranks) {
  std::string why;
  int st = validate_topology(nodes, gpus_per_node, 1, &why);
  if (st != LANE_OK) return st;
  if (rank < 0 || rank >= nodes * gpus_per_node) return LANE_ERR_INVALID_ARG;
  const int a = rank / gpus_per_node, g = rank % gpus_per_node;  // p = a*G + g (S L90)
  if (node) *node = a;
  if (gpu) *gpu = g;
  if (group_ranks)
    for (int h = 0; h < gpus_per_node; ++h) group_ranks[h] = a * gpus_per_node + h;
  if (lane_ranks)
    for (int b = 0; b < nodes; ++b) lane_ranks[b] = b * gpus_per_node + g;
  return LANE_OK;
}

int lane_partition_query(uint64_t count, int itemsize, int nodes, int gpus_per_node,
                         int procs_per_gpu, int64_t chunk_granules, int64_t round_granules,
                         int64_t* units_out, uint64_t max_units, uint64_t* n_units) {
  std::string why;
  int st = validate_topology(nodes, gpus_per_node, procs_per_gpu, &why);
  if (st != LANE_OK) return st;
  if (itemsize != 2 && itemsize != 4) return LANE_ERR_UNSUPPORTED;
  const int q = 16 / itemsize;
  const int64_t ng = (int64_t)((count + q - 1) / q);
  const int64_t RG = round_granules > 0 ? round_granules : (ng > 0 ? ng : 1);
  const int N = nodes, G = gpus_per_node, k = procs_per_gpu;
  auto el = [&](int64_t gr) { return (int64_t)((uint64_t)gr * q < count ? (uint64_t)gr * q : count); };
  uint64_t n = 0;
  const int64_t rounds = ng > 0 ? lane::ceil_div(ng, RG) : 0;
  for (int64_t r = 0; r < rounds; ++r) {
    const int64_t r0 = r * RG, rlen = (ng - r0) < RG ? (ng - r0) : RG;
    for (int l = 0; l < k; ++l) {
      const Span sl = lane::rf_split(rlen, k, l);
      const int64_t cg = chunk_granules > 0 ? chunk_granules : (sl.len > 0 ? sl.len : 1);
      const int64_t nc = lane::n_chunks(sl.len, cg);
      for (int64_t c = 0; c < nc; ++c) {
        const int64_t c0 = r0 + sl.start + c * cg;
        const int64_t clen = (sl.len - c * cg) < cg ? (sl.len - c * cg) : cg;
        for (int g = 0; g < G; ++g) {
          const Span gp = lane::rf_split(clen, G, g);
          for (int a = 0; a < N; ++a) {
            const Span up = lane::rf_split(gp.len, N, a);
            if (units_out && n < max_units) {
              int64_t* u = units_out + 9 * n;
              u[0] = r; u[1] = l; u[2] = c; u[3] = g; u[4] = a;
              u[5] = el(c0 + gp.start);
              u[6] = el(c0 + gp.start + gp.len);
              u[7] = el(c0 + gp.start + up.start);
              u[8] = el(c0 + gp.start + up.start + up.len);
            }
            ++n;
          }
        }
      }
    }
  }
  if (n_units) *n_units = n;
  return LANE_OK;
}

}  // extern "C"
