/* usp_attn.h — C ABI of the B200-native USP attention forward engine.
 *
 * Drop-in for the hot path of the reference `uspsim`
 * (/root/reference/proj): the SP attention forward
 *   usp::usp_attention<T>(RankCtx&, const ProcessMesh&, q, k, v,
 *                         positions, causal)      src/usp/usp_attention.hpp:41-47
 * with its ulysses_degree x ring_degree process grid (src/simcomm/mesh.hpp:14-34),
 * zigzag/contiguous sequence layout (src/usp/partition.hpp:19-53) and
 * Q/K/V/O/LSE tensor conventions (src/numerics/tensor.hpp:19-75,
 * src/numerics/attention.hpp:90-92). Conventions mirror the reference's
 * own C ABI (include/uspsim.h): same status numbering, opaque handles,
 * explicit destroy, thread-local last error, no exceptions across the ABI.
 *
 * Tensor conventions (all row-major, device memory, caller-owned):
 *   q   bf16 (batch, T, heads,    head_size)  sequence-sharded, T = L/(U*R),
 *   k,v bf16 (batch, T, kv_heads, head_size)  rows in usp_positions_for() order
 *   o   bf16 (batch, T, heads,    head_size)  same rows / order as q
 *   lse fp32 (batch, L/R, heads/U)            natural log, HEAD-sharded, rows in
 *                                             usp_head_positions() order
 *   GQA: query head h reads kv head h / (heads / kv_heads).
 */
#ifndef USP_ATTN_H
#define USP_ATTN_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define USP_API __attribute__((visibility("default")))
#else
#define USP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Same numbering as uspsim_status (include/uspsim.h:26-31). */
typedef enum usp_status {
  USP_OK = 0,
  USP_TOLERANCE_EXCEEDED = 1,
  USP_INVALID_INPUT = 2,
  USP_INTERNAL_ERROR = 3,
} usp_status;

/* The forward's static configuration. Replaces the (ProcessMesh, shapes,
 * causal) arguments of usp_attention (usp_attention.hpp:41-47) and the
 * simulate parameters (src/api/commands.cpp:189-215). */
typedef struct usp_config {
  int32_t ulysses_degree; /* U: ProcessMesh(ulysses, ring), mesh.hpp:16      */
  int32_t ring_degree;    /* R                                                */
  int32_t rank;           /* global rank, = ring_coord*U + ulysses_coord      */
  int32_t device;         /* CUDA device ordinal of this rank                 */
  int64_t batch;
  int64_t seq_len;        /* global L                                         */
  int32_t heads;          /* hc                                               */
  int32_t kv_heads;       /* kv_hc (GQA)                                      */
  int32_t head_size;      /* hs (<= 128; 64/128 run natively, others padded)  */
  int32_t causal;         /* zigzag layout iff causal (commands.cpp:88)       */
} usp_config;

typedef struct usp_comm usp_comm;     /* transport between the mesh's ranks */
typedef struct usp_engine usp_engine; /* one rank's forward engine          */

/* ---- layout & validation (host only, no device work) ------------------- */

/* ShardSpec + check_usp_inputs rules (partition.cpp:78-92,
 * usp_attention.cpp:15-38) with the reference's messages. */
USP_API usp_status usp_config_validate(const usp_config* cfg);
/* zigzag_partition (partition.cpp:12-33): out[R * (L/R)]. */
USP_API usp_status usp_zigzag_partition(int64_t seq_len, int32_t ring, int64_t* out);
/* ShardSpec::positions_for (partition.cpp:95-105): out[T]. */
USP_API usp_status usp_positions_for(const usp_config* cfg, int32_t rank, int64_t* out);
/* gather_positions result over the Ulysses group (all_to_all_4d.cpp:128-132),
 * i.e. the rows of the head-sharded O/LSE: out[L/R]. */
USP_API usp_status usp_head_positions(const usp_config* cfg, int32_t rank, int64_t* out);
/* causal_pair_counts (partition.cpp:52-72) of the ring assignment. */
USP_API usp_status usp_causal_pair_counts(const int64_t* assignment, int32_t ring, int64_t seq_len,
                                  int64_t* counts);

/* Per-ring-step schedule of one rank: the ring source block and the tile
 * plan the kernel will run (host logic behind usp_attn_fwd). */
typedef struct usp_step_info {
  int32_t step, src_ring_coord, send_to_rank, recv_from_rank;
  int64_t full_tiles, partial_tiles, work_units, visible_pairs;
  int64_t ring_bytes_sent; /* K+V bytes shifted after this step (0 on the last) */
} usp_step_info;
USP_API usp_status usp_schedule(const usp_config* cfg, int32_t step, usp_step_info* out);
/* The step's tile plan itself (CSR over 128-row query tiles): sizes[0] =
 * query tiles, sizes[1] = list entries; tile_off[sizes[0]+1] and
 * tile_list[sizes[1]] (k tile | partial << 31) are filled when non-NULL. */
USP_API usp_status usp_step_plan(const usp_config* cfg, int32_t step, int64_t sizes[2],
                                 int32_t* tile_off, int32_t* tile_list);
/* Communication ledger of one rank's forward, in the reference CommLedger's
 * terms (src/simcomm/ledger.hpp:21-30; closed forms ledger.cpp:25-37):
 * all_to_all sends payload*(n-1)/n, ring_shift sends the buffer. */
typedef struct usp_ledger_entry {
  int32_t kind;          /* simcomm::CollectiveKind: 3 all_to_all, 4 ring_shift */
  int32_t group_first;   /* group members: first + i*stride, i < size      */
  int32_t group_size;
  int32_t group_stride;
  int32_t step;          /* per-group sequence number                       */
  int32_t tensor;        /* 0 Q, 1 K, 2 V, 3 O, 4 dO, 5 dQ, 6 dK, 7 dV      */
  int64_t payload_elems; /* per-rank logical payload, elements              */
  double bytes_sent;     /* by this rank: bf16 elements, fp32 for the
                            circulating dK/dV partials                     */
} usp_ledger_entry;
/* Planned collectives of rank cfg->rank (host only). Returns the number of
 * entries (written up to cap), or -1 on invalid input. */
USP_API int32_t usp_forward_ledger(const usp_config* cfg, usp_ledger_entry* out, int32_t cap);
/* Planned collectives of one rank's forward followed by its backward
 * (usp_attention.cpp:68-89, ring_attention.cpp:79-155): the dO all-to-all,
 * per ring step the K/V shifts (steps < R-1) and the circulating dK/dV
 * partial shifts (steps >= 1), then the dQ, dK, dV all-to-alls. */
USP_API int32_t usp_backward_ledger(const usp_config* cfg, usp_ledger_entry* out, int32_t cap);
/* Collectives the engine actually issued in its last usp_attn_fwd (and the
 * usp_attn_bwd that followed it, if any). */
USP_API int32_t usp_engine_ledger(const usp_engine* engine, usp_ledger_entry* out, int32_t cap);

/* Algorithmic FLOPs of this rank's forward: 4 * batch * (heads/U) *
 * head_size * visible (q,k) pairs. */
USP_API usp_status usp_rank_flops(const usp_config* cfg, double* flops);

/* ---- transports ---------------------------------------------------------- */

/* NCCL over NVLink/NVSwitch, one process per GPU. All ranks pass the same
 * 128-byte ncclUniqueId produced by usp_nccl_unique_id on one rank. */
USP_API usp_status usp_nccl_unique_id(uint8_t out[128]);
USP_API usp_status usp_comm_create_nccl(const uint8_t unique_id[128], int32_t world_size,
                                int32_t rank, int32_t device, usp_comm** out);
/* In-process transport: one host thread per rank, CUDA peer copies between
 * the ranks' buffers (the analogue of simcomm::World::run, world.hpp:217-236).
 * One handle is shared by all ranks of the world; ranks may share a device. */
USP_API usp_status usp_comm_create_local(int32_t world_size, usp_comm** out);
/* Peer-memory transport, one process per GPU, no NCCL: receive buffers are
 * exported with CUDA IPC and written directly by the senders (copy engines
 * over NVLink / NVSwitch, so no SMs are taken from the attention kernel);
 * cross-process ordering by GPU stream memory operations on IPC-shared
 * signals. `allgather` is a host all-gather over the world (called
 * collectively at create and when a new buffer is first exchanged):
 * recv[world_size * bytes] <- every rank's send[bytes], rank order; it must
 * stay callable for the comm's lifetime. Returns 0 on success. */
typedef int (*usp_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
USP_API usp_status usp_comm_create_p2p(int32_t world_size, int32_t rank, int32_t device,
                                       usp_allgather_fn allgather, void* ctx, usp_comm** out);
USP_API void usp_comm_destroy(usp_comm* comm);
/* Failure detection (the reference World's stuck / mismatched-collective
 * diagnosis, world.cpp:89-113 and 152-165). Every transport bounds how long
 * a collective waits for its peers: the local transport's host rendezvous
 * (keyed by group and call number, with a signature check), the NCCL
 * transport's non-blocking init/split/launch polling and its watchdog over
 * enqueued collectives (ncclCommGetAsyncError + completion events; on
 * timeout or error every communicator is aborted). Default 600 s, or
 * USP_COMM_TIMEOUT_S. A failed comm reports USP_INTERNAL_ERROR from every
 * later call with the failure ("collective mismatch on group [...] call #k:
 * rank a called X but rank b called Y", "collective deadlock ...",
 * "ring_shift call #k on ring group [...] did not complete within ...").
 * usp_comm_status returns USP_OK while healthy. */
USP_API usp_status usp_comm_set_timeout(usp_comm* comm, double seconds);
USP_API usp_status usp_comm_status(usp_comm* comm);
/* Tests: one host rendezvous of `rank` on group `members` under `signature`
 * (local transport only; no GPU work). */
USP_API usp_status usp_comm_debug_rendezvous(usp_comm* comm, int32_t rank, const int32_t* members,
                                             int32_t n, const char* signature);

/* ---- engine -------------------------------------------------------------- */

/* comm may be NULL when U*R == 1. Allocates all workspace up front. */
USP_API usp_status usp_engine_create(const usp_config* cfg, usp_comm* comm, usp_engine** out);
/* Collective over the mesh: every rank calls it with matching shapes, in
 * the same order. Asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream). */
USP_API usp_status usp_attn_fwd(usp_engine* engine, const void* q, const void* k, const void* v,
                        void* o, float* lse, void* stream);
/* usp_attn_fwd with q, k, v, o, lse in HOST memory (same layouts), the
 * host<->device copies inside the call — what a host-side caller of
 * usp_attention (usp_attention.hpp:41-47, whose Tensor4 lives in host
 * memory) binds. At U = R = 1 the copies are pipelined against the
 * attention in sequence chunks (H2D of chunk c+1 and D2H of chunk c-1
 * overlap chunk c's kernel). Pinned (page-locked) buffers are required for
 * overlap; pageable ones work but serialise. Asynchronous on `stream`: the
 * outputs are valid once the stream has been synchronised. */
USP_API usp_status usp_attn_fwd_host(usp_engine* engine, const void* q, const void* k, const void* v,
                                     void* o, float* lse, void* stream);
/* Backward of the engine's last usp_attn_fwd: the reference's
 * usp_attention_backward<T> (src/usp/usp_attention.cpp:68-89) over
 * ring_attention_backward (src/usp/ring_attention.cpp:79-155).
 *   q, k, v, o : the tensors of the preceding usp_attn_fwd on this engine
 *                (the head-sharded activations it saved are reused, as
 *                UspForward carries them);
 *   lse        : that forward's head-sharded logsumexp;
 *   dout       : dO, sequence-sharded like o (bf16);
 *   dq, dk, dv : bf16 gradients, sequence-sharded like q, k, v.
 * dK/dV partials circulate the ring in fp32 and dQ accumulates in fp32; the
 * casts to bf16 happen once at the end. Asynchronous on `stream`.
 * USP_INVALID_INPUT when no forward preceded it. */
USP_API usp_status usp_attn_bwd(usp_engine* engine, const void* q, const void* k, const void* v,
                                const void* o, const float* lse, const void* dout, void* dq,
                                void* dk, void* dv, void* stream);
/* usp_attn_bwd on every rank of a local world (one host thread per rank). */
USP_API usp_status usp_local_world_bwd(usp_engine* const* engines, int32_t world_size,
                                       const void* const* q, const void* const* k,
                                       const void* const* v, const void* const* o,
                                       const float* const* lse, const void* const* dout,
                                       void* const* dq, void* const* dk, void* const* dv,
                                       void* const* streams);
/* Launches of the engine's own kernels in the last usp_attn_fwd / _bwd. */
USP_API int32_t usp_engine_last_launches(const usp_engine* engine);
USP_API void usp_engine_destroy(usp_engine* engine);
/* Optional per-launch timing of the attention kernel: CUDA events recorded
 * around every launch on its stream while enabled. kernel_times
 * synchronises, writes up to cap durations (ms) and returns how many launches
 * were recorded since the last call (-1 on error). */
USP_API usp_status usp_engine_enable_timing(usp_engine* engine, int32_t on);
USP_API int32_t usp_engine_kernel_times(usp_engine* engine, float* ms, int32_t cap);
/* Ring overlap sizing of an engine: the K+V bytes of one ring
 * shift, the shortest ring step it hides behind (estimated from the step's
 * visible pairs), the bandwidth that needs, the CTAs given to the ring
 * communicator (NCCL maxCTAs) and the SMs the attention grid leaves free for
 * them (0 on the copy-engine transports). */
typedef struct usp_engine_info {
  int32_t num_sms, reserved_sms, ring_ctas;
  double kv_shift_bytes, ring_step_ms_est, required_gbs;
} usp_engine_info;
USP_API usp_status usp_engine_get_info(const usp_engine* engine, usp_engine_info* out);
/* Ulysses all-to-all pipelining: every member's T rows are
 * exchanged in `chunks` row chunks; ring step 0 computes chunk c as soon as it
 * has landed (the exchange of chunk c+1 overlaps it) and the last step's
 * chunk c sends its O rows while chunk c+1 computes. Default 2 when U > 1,
 * bs = 1, T divides into whole query tiles and the transport is not the
 * peer-memory one (whose exchange is already fused into the kernels);
 * 1 = one exchange each way. USP_INVALID_INPUT when the rows do not divide.
 * Results are bitwise identical for every chunk count. */
USP_API usp_status usp_engine_set_a2a_chunks(usp_engine* engine, int32_t chunks);
USP_API int32_t usp_engine_a2a_chunks(const usp_engine* engine);
/* Backward algorithm. Default (off): one fused kernel per ring step computes
 * dK, dV and dQ (five GEMMs per tile pair; dQ partials are reduced into fp32
 * by TMA in arrival order, so dQ's summation order — and its last bits — may
 * differ run to run). On: two kernels per step (dK/dV, then dQ, which
 * recomputes S and dP) with every sum in a fixed order — bitwise
 * reproducible backward. Takes effect at the next usp_attn_bwd. */
USP_API usp_status usp_engine_set_deterministic(usp_engine* engine, int32_t on);
/* Overrides the SMs the attention grid leaves free for a concurrent
 * communication kernel (0 .. #SMs-1). */
USP_API usp_status usp_engine_set_reserved_sms(usp_engine* engine, int32_t n);
/* Per-stage breakdown of the forwards run while timing was on (events on
 * the caller's stream after each stage; a stage's time is the gap to the
 * previous one): pack, a2a_in (or pack_a2a_in for the direct peer-memory
 * exchange), wait<t> (exposed part of the K/V shift into ring step t),
 * attn<t>, a2a_out, unpack; shift<t> is the K/V transfer itself on the comm
 * stream. Summed per name over the forwards (count = how many). Synchronises
 * and clears; returns the number of stages (written up to cap), -1 on error. */
typedef struct usp_stage_time {
  char name[24];
  double ms_total;
  int32_t count;
} usp_stage_time;
USP_API int32_t usp_engine_stage_times(usp_engine* engine, usp_stage_time* out, int32_t cap);
/* Parity instrumentation (tests): while on, the forward kernel counts every
 * (warp, key tile) whose lazy O rescale fired, i.e. the running row max grew
 * by more than 8 in log2 units and O was multiplied by alpha = 2^(m_old -
 * m_new) (SoftmaxState::update's rescale, attention.cpp:209-226). Turning it
 * on or off resets the count; rescale_count synchronises the device. */
USP_API usp_status usp_engine_debug_counters(usp_engine* engine, int32_t on);
USP_API usp_status usp_engine_rescale_count(usp_engine* engine, int64_t* out);

/* Runs usp_attn_fwd on every rank of a local world, one host thread per
 * rank (engines[i] must belong to rank i); blocks until all are issued. */
USP_API usp_status usp_local_world_fwd(usp_engine* const* engines, int32_t world_size,
                               const void* const* q, const void* const* k,
                               const void* const* v, void* const* o, float* const* lse,
                               void* const* streams);

/* ---- diagnostics --------------------------------------------------------- */
USP_API const char* usp_last_error(void);
USP_API const char* usp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* USP_ATTN_H */
