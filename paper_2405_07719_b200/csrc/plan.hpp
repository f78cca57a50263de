// plan.hpp — host-side layout and schedule logic of the USP forward.
//
// Pure C++ (no CUDA): the process mesh, the zigzag / even sequence layout,
// the Ulysses and Ring group structure, and the per-ring-step tile plan the
// attention kernel consumes. Every rule restates the reference:
//   ProcessMesh          src/simcomm/mesh.cpp:8-57
//   zigzag/even layout   src/usp/partition.cpp:12-50
//   ShardSpec checks     src/usp/partition.cpp:74-105
//   usp input checks     src/usp/usp_attention.cpp:15-38
//   ring step order      src/usp/ring_attention.cpp:62-75
//   causal mask          src/numerics/attention.hpp:32-34
#pragma once

#include <cstdint>
#include <stdexcept>
#include <cstdlib>
#include <string>
#include <vector>

namespace uspb200 {

// Mirrors uspsim::ErrorCode (src/common/error.hpp:11-17).
enum class ErrorCode { kInvalidArgument, kConstraint, kCommMismatch, kNumeric, kInternal };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] void throw_invalid(const std::string& what);

// Development knobs (A/B experiments, traces): the environment is read only
// in builds with -DUSPB_DEV (build.py variants); the product library ignores
// it (USP_COMM_TIMEOUT_S, a documented setting, is the exception).
inline const char* dev_env(const char* name) {
#ifdef USPB_DEV
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
[[noreturn]] void throw_constraint(const std::string& what);

struct MeshShape {
  int ulysses = 1, ring = 1;
  int world() const { return ulysses * ring; }
  int ulysses_coord(int rank) const;              // rank % U       (mesh.cpp:23-26)
  int ring_coord(int rank) const;                 // rank / U       (mesh.cpp:28-31)
  int rank_of(int u, int r) const;                // r * U + u      (mesh.cpp:33-39)
  std::vector<int> ulysses_group(int rank) const; // mesh row       (mesh.cpp:41-48)
  std::vector<int> ring_group(int rank) const;    // mesh column    (mesh.cpp:50-57)
};

struct UspShape {
  MeshShape mesh;
  int64_t batch = 1, seq_len = 0;
  int heads = 0, kv_heads = 0, head_size = 0;
  bool causal = false;

  // Reference validation, same rules and message substrings.
  void validate() const;
  int64_t tokens_per_rank() const { return seq_len / mesh.world(); }       // T
  int64_t tokens_per_ring_rank() const { return seq_len / mesh.ring; }     // U*T
  int local_heads() const { return heads / mesh.ulysses; }
  int local_kv_heads() const { return kv_heads / mesh.ulysses; }
  // The head size the tcgen05 kernel runs at (zero padding is exact).
  int kernel_head_size() const { return head_size <= 64 ? 64 : 128; }
};

std::vector<int64_t> zigzag_partition(int64_t seq_len, int ring);  // flattened R x L/R
std::vector<int64_t> even_partition(int64_t seq_len, int ring);
std::vector<int64_t> causal_pair_counts(const std::vector<int64_t>& flat, int ring,
                                        int64_t seq_len);
// ShardSpec::positions_for (zigzag iff causal, as commands.cpp:88 does).
std::vector<int64_t> positions_for(const UspShape& s, int rank);
// gather_positions over the Ulysses group == the ring list of ring coord r.
std::vector<int64_t> head_positions(const UspShape& s, int rank);

// The ring source block at step t for ring coordinate r (ring_attention.cpp:63).
inline int ring_source(int r, int step, int ring) { return (r - step + ring) % ring; }

// Per-ring-step tile plan for the attention kernel.
struct StepPlan {
  int q_len = 0, k_len = 0, n_q_tiles = 0, n_k_tiles = 0;
  std::vector<int32_t> q_pos;      // effective positions, padded to 128
  std::vector<int32_t> k_pos;      // effective positions, padded to 128 (INT32_MAX)
  std::vector<int32_t> tile_off;   // CSR offsets, n_q_tiles + 1
  std::vector<int32_t> tile_list;  // k tile | partial << 31
  std::vector<uint32_t> units;     // q_tile | head_pair << 16 | batch << 24, LPT order
  int64_t full_tiles = 0, partial_tiles = 0, visible_pairs = 0;
};

// q_pos/k_pos are ORIGINAL token positions; causal == false makes every key
// visible (BlockMask::none). include_empty keeps query tiles with no visible
// key tile in the unit list (needed by first/last ring steps so every row is
// written). head_pairs = local q heads / NQ.
// pairs_per_kv = head pairs sharing one kv head (GQA group / NQ); the unit
// order keeps CTAs that run concurrently on the same kv head (L2 reuse of
// the streamed K/V tiles) — see plan.cpp.
// rows_per_unit: query rows per work unit (128, or 256 when the kernel runs
// two adjacent 128-row tiles of one head; the tile list is then the union of
// both tiles' visible key tiles, classified over all 256 rows).
StepPlan plan_step(const std::vector<int64_t>& q_pos, const std::vector<int64_t>& k_pos,
                   bool causal, int64_t batch, int head_pairs, bool include_empty,
                   int pairs_per_kv = 1, int rows_per_unit = 128);

// How the forward kernel fills its two q tiles per CTA: two q heads of one
// GQA group over the same rows when the local group is even (K/V tiles and
// masks shared), otherwise two adjacent 128-row tiles of ONE head (MHA and
// odd groups; K/V tiles shared, key-tile list = union, per-element masks).
// With a 4-head (or larger multiple) local group at head size 128, a 2-CTA
// cluster runs both head pairs of a head quad and shares each K/V tile by
// TMA multicast (unit = q tile x head quad).
struct FwdTiling {
  bool pair_rows;    // two row tiles of one head (else two heads)
  int head_units;    // head slots per unit list entry (head pairs, quads or heads)
  int units_per_kv;  // head slots sharing one kv head
  int rows_per_unit; // 128 or 256
  bool cluster;      // 2-CTA clusters over head quads
};
// q_rows / batch / sms: a short sequence keeps 128-row units when pairing
// rows would leave fewer units than SMs (measured faster below ~4K rows).
FwdTiling fwd_tiling(int local_heads, int local_kv_heads, int kernel_head_size, int64_t q_rows = 1 << 30,
                     int64_t batch = 1, int sms = 148);

// The same block transposed for the dK/dV kernel: CSR over KEY tiles
// (tile_list = q tile | partial << 31, same partial flags), units
// k_tile | kv_head << 16 | batch << 24 in kv-head-major LPT order.
// include_empty keeps key tiles no query sees (their dK/dV rows are
// written as zeros when the kernel does not accumulate).
StepPlan transpose_plan(const StepPlan& fwd, int64_t batch, int kv_heads, bool include_empty);
// The same over PAIRS of adjacent key tiles (2p, 2p+1) for the dK/dV
// kernel's 2-CTA clusters: CSR over pairs, list = union of the two tiles'
// q tiles (partial when partial for either or seen by only one), units
// pair | kv_head << 16 | b << 24; k_pos padded to a whole number of pairs.
StepPlan transpose_plan_pairs(const StepPlan& fwd, int64_t batch, int kv_heads, bool include_empty);

// One communication event of a rank's forward, in the reference ledger's
// terms (src/simcomm/ledger.hpp:21-30, closed forms ledger.cpp:25-37).
struct LedgerEvent {
  int kind;             // simcomm::CollectiveKind: 3 all_to_all, 4 ring_shift
  int group_first, group_size, group_stride;
  int step;             // per-group sequence number
  int tensor;           // 0 Q, 1 K, 2 V, 3 O
  int64_t payload_elems;  // per-rank logical payload, elements
  double bytes_sent;      // by this rank, at elem_bytes per element
};
// The collectives usp_attn_fwd issues on `rank` (Alg. 1 order): Q, K, V
// all-to-alls, 2(R-1) ring shifts (K then V per step), the O all-to-all.
// The reference's two position all_gathers are absent (static layout).
std::vector<LedgerEvent> forward_ledger(const UspShape& s, int rank, int elem_bytes);
// forward_ledger followed by the backward's collectives
// (usp_attention.cpp:68-89, ring_attention.cpp:79-155): dO all-to-all;
// per ring step t: K, V shifts (t < R-1), then the circulating dK, dV
// partial shifts (t >= 1, at grad_bytes per element); dQ, dK, dV
// all-to-alls. Tensor ids 4 dO, 5 dQ, 6 dK, 7 dV.
std::vector<LedgerEvent> backward_ledger(const UspShape& s, int rank, int elem_bytes, int grad_bytes);

// Exact unmasked (q, k) pair count of one block, summed over the block
// (causal_pair_counts semantics, partition.cpp:52-72) — for FLOP accounting.
int64_t visible_pairs(const std::vector<int64_t>& q_pos, const std::vector<int64_t>& k_pos,
                      bool causal);

}  // namespace uspb200
