/*
 * lane_allreduce.h — C ABI of the B200-native k-split multi-lane allreduce.
 *
 * The operation (PAPER.md = arXiv 2508.13397, cited as P Lnnn):
 *   MPI_Allreduce(sendbuf, recvbuf, s, MPI_SUM, comm)            P L341-343
 * computed as the multi-lane algorithm (Alg. 2 "lane_allreduce", P L218-251):
 *   (1) reduce-scatter among the G GPUs of a node (comm_group)  P L243
 *   (2) allreduce of slice g among GPU g of every node (comm_lane) P L246
 *   (3) allgatherv among the G GPUs of the node                 P L248
 * with the buffer split into k slices ("processes per GPU", l_r, offset
 * s*l_r, count s/PPG; P L330-349, §3.1.2 P L364-373), each slice reduced by
 * its own independent group of CTAs.
 *
 * Every phase runs in the library's own sm_100a kernel, which loads/stores
 * peer GPUs' IPC-mapped memory over NVLink 5 / NVSwitch and signals with
 * .sys-scope release/acquire flags. No NCCL, no CPU fallback.
 *
 * Conventions
 *   - Ranks: p = a*G + g (node a, GPU-in-node g), node-major.
 *   - Every function returns a lane_status_t (0 = LANE_OK); it never throws
 *     and never aborts the process. lane_allreduce_last_error() names the
 *     offending field ("configuration error naming the field").
 *   - Streams are passed as void* (a cudaStream_t; NULL = legacy default).
 *   - Device pointers must be device memory of the comm's device, 16-byte
 *     aligned (LANE_ERR_MISALIGNED otherwise). Any count is accepted.
 *   - Results are deterministic and identical on every rank: each element is
 *     reduced once, in the canonical order (ascending GPU index within the
 *     node, then ascending node), accumulating in fp32 (int32: wrap-around);
 *     bf16 is rounded to nearest-even once per reducing phase
 *     (readings R#7-R#9).
 */
#ifndef LANE_ALLREDUCE_H
#define LANE_ALLREDUCE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lane_comm_s* lane_comm_t;

typedef enum { LANE_INT32 = 0, LANE_FLOAT32 = 1, LANE_BFLOAT16 = 2 } lane_dtype_t;

/* The paper reduces with MPI_SUM only (P L341, L347). */
typedef enum { LANE_SUM = 0 } lane_op_t;

typedef enum {
  LANE_OK = 0,
  LANE_ERR_INVALID_ARG = -1,   /* bad topology/argument; last_error names it   */
  LANE_ERR_UNSUPPORTED = -2,   /* dtype or op outside the enums; capture of the
                                  host-buffer API                              */
  LANE_ERR_CUDA = -3,          /* a CUDA runtime call or launch failed         */
  LANE_ERR_NOT_CONNECTED = -4, /* lane_allreduce before lane_allreduce_open_peers
                                  (resolving an unpublished handle) */
  LANE_ERR_TIMEOUT = -5,       /* a device-side wait exceeded LANE_TIMEOUT_MS in
                                  an earlier call; the comm is unusable (finalize) */
  LANE_ERR_MISALIGNED = -6,    /* a buffer pointer is not 16-byte aligned      */
  LANE_ERR_MISMATCH = -7       /* ranks disagreed on a call in an earlier call:
                                  zero-copy vs staged (registrations), buffer
                                  offsets, count or dtype; detected by the start
                                  handshake before any buffer was touched, the
                                  comm is unusable (finalize) */
} lane_status_t;

#define LANE_MAX_RANKS 16         /* N*G; one 8-GPU box uses <= 8                 */
#define LANE_MAX_PROCS_PER_GPU 16 /* k; the paper's largest PPG is 16 (P L431)    */
#define LANE_HANDLE_BYTES 256     /* size of one rank's blob from get_handle      */

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU (torchrun). Collective: every rank calls init, then
 * get_handle; the caller all-gathers the P blobs in rank order (the paper
 * broadcasts IPC handles the same way, P L330) and every rank calls
 * open_peers. Only then may lane_allreduce be called.
 *
 * Every LANE_* environment setting that shapes a call's plan (protocol
 * thresholds and capacities, engine, store mode, chunking, CTA budgets,
 * zero-copy job set, releasers) is read ONCE at init and carried in the blob;
 * open_peers rejects ranks whose settings differ (INVALID_ARG naming the
 * setting), so every rank plans every call identically.
 */

/* Create a comm for (nodes, gpus_per_node, procs_per_gpu) = (N, G, k).
 * rank and device are read from $RANK and $LOCAL_RANK (torchrun); requires
 * N*G == $WORLD_SIZE. Allocates this rank's symmetric scratch and signal
 * memory on the device (sized by $LANE_ROUND_BYTES, default 1 GiB of message
 * per round). Errors: INVALID_ARG (any factor < 1, N*G > LANE_MAX_RANKS,
 * k > LANE_MAX_PROCS_PER_GPU, N*G != WORLD_SIZE, missing env), CUDA. */
int lane_allreduce_init(int nodes, int gpus_per_node, int procs_per_gpu, lane_comm_t* comm);

/* As lane_allreduce_init with an explicit rank in [0, N*G) and CUDA device. */
int lane_allreduce_init_rank(int nodes, int gpus_per_node, int procs_per_gpu, int rank,
                             int device, lane_comm_t* comm);

/* Write this rank's IPC blob (at most LANE_HANDLE_BYTES) into blob;
 * *blob_bytes receives its size. The caller owns blob. */
int lane_allreduce_get_handle(lane_comm_t comm, void* blob, size_t* blob_bytes);

/* all_blobs: N*G blobs of blob_bytes each, in rank order (own blob included).
 * Opens every peer's scratch/signal memory (cudaIpcOpenMemHandle) and checks
 * that all blobs describe the same (N, G, k) and geometry (INVALID_ARG
 * otherwise). The mappings are owned by the comm until finalize. */
int lane_allreduce_open_peers(lane_comm_t comm, const void* all_blobs, size_t blob_bytes);

/* Enqueue the allreduce of count elements on stream; returns immediately.
 * sendbuf/recvbuf: device pointers owned by the caller, count elements each,
 * kept alive until the stream passes this point. sendbuf == recvbuf is
 * in-place; partial overlap is INVALID_ARG. count == 0 is a no-op. Every
 * rank must call with the same (count, dtype, op) in the same order (MPI
 * collective semantics, P L341). Messages larger than the round capacity are
 * processed in several rounds (kernel launches) inside one call. The call
 * may be captured into a CUDA graph (stream capture): from the first
 * captured call on, the comm takes every launch's epoch (the generation of
 * its flags and packets) from device memory, so each replay — and every
 * later eager call — gets a fresh one; every rank must replay its graphs and
 * make its eager calls in the same order (collective semantics). The same
 * holds for the ring, approach-2 and emulated entry points; the host-buffer
 * entry points (lane_allreduce_host, _emulated_host) cannot be captured
 * (UNSUPPORTED). */
int lane_allreduce(lane_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                   lane_dtype_t dtype, lane_op_t op, void* stream);

/* Zero-copy registration of a user buffer (collective, same order on every
 * rank). The paper shares the user buffer between processes through IPC
 * handles (P L330); here every rank maps every peer's registered buffer so
 * the kernel reads peers' sendbufs and writes peers' recvbufs directly
 * (no staging through scratch). register_handle writes this rank's blob
 * (<= LANE_HANDLE_BYTES) for [ptr, ptr+bytes) — ptr must lie in a cudaMalloc
 * allocation (not a VMM/expandable segment); the caller all-gathers the blobs
 * in rank order and calls register_open, which returns reg_id. Afterwards
 * lane_allreduce on sendbuf/recvbuf inside registered buffers runs zero-copy,
 * provided every rank passes the same offsets into its registered buffers
 * (MPI-style symmetric buffers). The registration is owned by the comm until
 * deregister/finalize; errors: INVALID_ARG, MISALIGNED, CUDA. */
int lane_allreduce_register_handle(lane_comm_t comm, void* ptr, size_t bytes, void* blob,
                                   size_t* blob_bytes);
int lane_allreduce_register_open(lane_comm_t comm, const void* all_blobs, size_t blob_bytes,
                                 int* reg_id);
/* Stop using a registration (mappings are released at finalize). Call it on
 * every rank in the same order, like register: a call whose buffers are
 * zero-copy on one rank and staged on another (or at different offsets, or
 * in registrations made in a different order) is caught by the start
 * handshake of the simple protocol (the per-call signature: job set,
 * registration index and offsets, count, dtype, chunking) and fails with
 * LANE_ERR_MISMATCH on every rank, never with wrong data or a timeout. */
int lane_allreduce_deregister(lane_comm_t comm, int reg_id);

/* End-to-end variant on HOST buffers: copies host_send to a library-owned
 * device staging buffer, runs lane_allreduce, copies the result to host_recv,
 * all on stream (pinned host memory gives async copies). host_send and
 * host_recv hold count elements each (the caller guarantees the sizes; the
 * Python binding checks them). The message is cut into pieces of
 * $LANE_HOST_PIECE_BYTES (default 64 MiB), each its own allreduce, pipelined
 * over two staging slots; staging grows on demand and is owned by the comm.
 * The caller synchronizes the stream before reading host_recv. */
int lane_allreduce_host(lane_comm_t comm, const void* host_send, void* host_recv, size_t count,
                        lane_dtype_t dtype, lane_op_t op, void* stream);

/* ------------------------------------------------------------- emulated mode
 * All P = N*G ranks on ONE device: every rank's scratch lives in this
 * device's HBM and one cooperative launch runs every rank's CTAs, so the same
 * kernels (and the same cross-rank flag protocol) run without NVLink. Used
 * for single-GPU parity and for the N=1 benchmark. */
int lane_allreduce_init_emulated(int nodes, int gpus_per_node, int procs_per_gpu, int device,
                                 lane_comm_t* comm);

/* sendbufs/recvbufs: host arrays of N*G device pointers (rank order). */
int lane_allreduce_emulated(lane_comm_t comm, const void* const* sendbufs, void* const* recvbufs,
                            size_t count, lane_dtype_t dtype, lane_op_t op, void* stream);

/* Emulated end-to-end variant: host arrays of N*G HOST buffer pointers. */
int lane_allreduce_emulated_host(lane_comm_t comm, const void* const* host_sends,
                                 void* const* host_recvs, size_t count, lane_dtype_t dtype,
                                 lane_op_t op, void* stream);

/* ---------------------------------------------------- ring (Alg. 1) baseline
 * The paper's "standard" allreduce, Alg. 1 ring_allreduce (PAPER.md
 * L150-206): a flat ring over all P = N*G ranks (rank r sends to r+1),
 * P-1 reduce-scatter steps then P-1 allgather steps; with the comm's k it is
 * the paper's "standard approach" with k processes per GPU (§3.1.1, P
 * L335-349: every k-slice is ring-allreduced independently). Hand-written
 * sm_100a kernel on the LL protocol (see LANE_PROTO_LL); messages above
 * $LANE_LL_MAX_BYTES run in several launches. Unlike lane_allreduce, each
 * chunk is reduced in ring order starting at rank c with one rounding per
 * hop in the buffer type (bf16: per-hop RNE, R#11), so results
 * differ in the last bits from the multi-lane method (int32: identical).
 * Same argument rules and errors as lane_allreduce / _emulated; buffers need
 * no registration. */
int lane_allreduce_ring(lane_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                        lane_dtype_t dtype, lane_op_t op, void* stream);
int lane_allreduce_ring_emulated(lane_comm_t comm, const void* const* sendbufs, void* const* recvbufs,
                                 size_t count, lane_dtype_t dtype, lane_op_t op, void* stream);

/* The ring's plan for (count, dtype), as lane_allreduce_plan: the pipeline
 * chunk ($LANE_RING_CHUNK_BYTES, default 64 KiB; every chunk of every k-slice
 * is its own Alg. 1 ring, R#21), the round size ($LANE_LL_MAX_BYTES)
 * in granules, CTAs per CTA group and launches. Any out-pointer may be NULL.
 *
 * $LANE_PHASE2=ring (read at init) switches lane_allreduce to the paper's
 * variant with the ring as the inter-node stage (fig:full_mpi_comparison,
 * P L401, L457): phase 1 and 3 unchanged, phase 2 = Alg. 1 among the N lane
 * members on every group part (its N sub-parts are the ring chunks), one
 * rounding per hop; it runs on the LL protocol with the same fixed chunking,
 * reported by lane_allreduce_plan. */
int lane_allreduce_ring_plan(lane_comm_t comm, size_t count, lane_dtype_t dtype, int64_t* chunk_granules,
                             int64_t* round_granules, int* ctas_per_group, int* launches);

/* --------------------------------------------------- "approach 2" variant
 * PAPER.md L296-297 (a bullet of the commented-out draft of §3 "Methods":
 * "Approach 2: allreduce on node + allreduce off node"): a direct allreduce
 * among the G GPUs of each node (every member ends with the node sum of the
 * whole buffer), then a direct allreduce of the WHOLE buffer among the N
 * lane members. Same association and rounding points as lane_allreduce, so
 * identical results; the traffic is 2(G-1)/G on node plus 2(N-1)/N off node
 * of the buffer per rank (the lane stage is not divided by G — the reason
 * the paper's method reduce-scatters first). LL protocol kernel; messages
 * above $LANE_LL_MAX_BYTES run in several launches. Same argument rules and
 * errors as lane_allreduce / lane_allreduce_emulated. */
int lane_allreduce_approach2(lane_comm_t comm, const void* sendbuf, void* recvbuf, size_t count,
                             lane_dtype_t dtype, lane_op_t op, void* stream);
int lane_allreduce_approach2_emulated(lane_comm_t comm, const void* const* sendbufs, void* const* recvbufs,
                                      size_t count, lane_dtype_t dtype, lane_op_t op, void* stream);

/* ----------------------------------------------------------------- common */

/* Release scratch, IPC mappings and staging. Collective in multi-GPU mode:
 * call only after every rank's last lane_allreduce has completed. */
int lane_allreduce_finalize(lane_comm_t comm);

/* Human-readable reason for the last error on comm (never NULL). */
const char* lane_allreduce_last_error(lane_comm_t comm);

/* Poll the device-side error word (set by the wait watchdog or the start
 * handshake). Returns LANE_OK, LANE_ERR_TIMEOUT or LANE_ERR_MISMATCH. Does
 * not synchronize. */
int lane_allreduce_check(lane_comm_t comm);

/* Per-CTA stall accounting of the last launch (TMA engine), enabled by
 * creating the comm with LANE_TRACE=1: 16 uint64 per CTA (field order in
 * producer total / flag wait / empty wait / tiles,
 * storer total / full wait / sync / read wait / flush / jobs, per-phase
 * A..E time, bytes stored; nanoseconds). Synchronizes the device. Writes at
 * most max_words to out (may be NULL) and the available count to *n_words.
 * INVALID_ARG if tracing is off. */
int lane_allreduce_trace(lane_comm_t comm, uint64_t* out, size_t max_words, size_t* n_words);

/* The execution plan lane_allreduce uses for (count, dtype): chunk size and
 * round size in 16-byte granules, CTAs per CTA group, kernel launches
 * (rounds) per call. Any out-pointer may be NULL. */
int lane_allreduce_plan(lane_comm_t comm, size_t count, lane_dtype_t dtype,
                        int64_t* chunk_granules, int64_t* round_granules, int* ctas_per_group,
                        int* launches);

/* Signalling protocol of a call (both compute the same method and the same
 * bits). SIMPLE: one persistent kernel moves chunk tiles through a TMA
 * pipeline and publishes per-job epoch flags after a system-scope fence
 * (large messages; §3.1.2 phases as chunked jobs). LL: every 16-byte
 * granule travels as a 32-byte packet of four {data, epoch} 64-bit words, so
 * the reader's poll on the data is the signal (no fences; 2x NVLink bytes;
 * used up to $LANE_LL_THRESHOLD_BYTES, default 8 MiB per rank, where LL128 does
 * not take the call, and at most $LANE_LL_MAX_BYTES, default 16 MiB, the LL
 * inbox capacity). LL128: every
 * 128-byte line carries 7 granules and the epoch (lane_ll128.cuh: 8 lanes of a
 * warp write and read the line in one 16-byte-per-lane instruction; 8/7 of the
 * bytes; used above $LANE_LL128_MIN_BYTES up to $LANE_LL128_THRESHOLD_BYTES
 * per rank, at most $LANE_LL128_MAX_BYTES, default 64 MiB, its capacity).
 * $LANE_PROTO = ll | ll128 | simple forces one. */
#define LANE_PROTO_SIMPLE 0
#define LANE_PROTO_LL 1
#define LANE_PROTO_LL128 2

/* *protocol receives the protocol lane_allreduce uses for (count, dtype) on
 * this comm (LANE_PROTO_SIMPLE for count 0 and P == 1). Errors: INVALID_ARG
 * (null), UNSUPPORTED (dtype). Host only. */
int lane_allreduce_protocol(lane_comm_t comm, size_t count, lane_dtype_t dtype, int* protocol);

/* *protocol receives the protocol lane_allreduce_ring (and _ring_emulated)
 * uses for (count, dtype): LANE_PROTO_LL128 above $LANE_LL128_MIN_BYTES per
 * rank (or with $LANE_PROTO=ll128), else LANE_PROTO_LL ($LANE_PROTO=ll forces
 * it). Both give the same bits (same rounds, ring chunks and hop order).
 * Errors: INVALID_ARG (null; plan does not fit), UNSUPPORTED (dtype). Host only. */
int lane_allreduce_ring_protocol(lane_comm_t comm, size_t count, lane_dtype_t dtype, int* protocol);

/* -------------------------------------------------- host-only introspection
 * No GPU needed; used by the CPU test-suite to compare the library's own
 * topology and partition with the oracle's. */

/* Topology of rank p: node, gpu, comm_group ranks (G
 * entries) and comm_lane ranks (N entries); any out-pointer may be NULL. */
int lane_topology_query(int nodes, int gpus_per_node, int rank, int* node, int* gpu,
                        int* group_ranks, int* lane_ranks);

/* Enumerate the ownership units of a message exactly as the kernels
 * partition it: for each unit, 9 int64 values
 * {round, l, c, g, a, part_start, part_end, start, end} (element indices).
 * chunk_granules / round_granules <= 0 mean "one piece". Writes at most
 * max_units units to units_out (may be NULL) and the total in *n_units. */
int lane_partition_query(uint64_t count, int itemsize, int nodes, int gpus_per_node,
                         int procs_per_gpu, int64_t chunk_granules, int64_t round_granules,
                         int64_t* units_out, uint64_t max_units, uint64_t* n_units);

/* LL128 planner of a one-round message of `granules` 16-byte granules
 * (lane_ll128.cuh plan128), for procs_per_gpu CTA groups of at most
 * ctas_per_group CTAs and the $LANE_LL128_MAX_BYTES / _MIN_CHUNK_BYTES
 * settings: out[0..5] = {CTAs per group, chunk granules, chunks, lines per
 * sub-part, lines per parity set the call needs, lines per set allocated}.
 * The call runs on LL128 only if out[4] <= out[5]. Errors: INVALID_ARG. */
int lane_ll128_plan_query(int nodes, int gpus_per_node, int procs_per_gpu, int64_t granules, int ctas_per_group,
                          int64_t max_bytes, int64_t min_chunk_bytes, int64_t* out);

/* Index, within an LL128 parity set, of the 128-byte line `line` of lane
 * sub-part b of chunk `chunk` in inbox `kind` (1 = L1 phase-1 part from node
 * peer slot, 2 = L2 lane RS slot, 3 = L3 lane AG slot, 4 = L4 phase-3 part
 * from node peer slot; b ignored for 2 / 3) for a call with `chunks` chunks
 * and lines_per_subpart lines per sub-part (lane_ll128.cuh layout128); kinds
 * 5 / 6 = the LL128 ring's RS / AG slot `slot` < nodes*gpus_per_node - 1,
 * lines_per_subpart = lines per ring part (ring_layout128).
 * Errors: INVALID_ARG (any index out of its range). */
int lane_ll128_line_query(int nodes, int gpus_per_node, int64_t chunks, int64_t lines_per_subpart, int kind, int slot,
                          int64_t chunk, int b, int64_t line, int64_t* index);

/* Library version string. */
const char* lane_allreduce_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LANE_ALLREDUCE_H */
