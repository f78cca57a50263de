// engine.cu — one rank's USP attention forward and the C ABI (include/usp_attn.h).
//
// usp_attn_fwd is the B200 restatement of usp::usp_attention<T>
// (reference src/usp/usp_attention.cpp:43-65), i.e. the paper's Algorithm 1:
//   1. Ulysses all-to-all of Q, K, V, sequence-sharded -> head-sharded
//      (all_to_all_4d(.,2,1), usp_attention.cpp:54-56): pack transposes
//      (reshard.cu) + ONE grouped exchange for all three tensors;
//   2. ring attention over the ring group (ring_attention.cpp:45-76): R
//      launches of the tcgen05 attention kernel, step t on the K/V block of
//      ring source (r - t) mod R, while K/V for step t+1 are shifted on a
//      side stream into the other half of a double buffer; the online-softmax
//      merge across steps is fused into the kernel epilogue;
//   3. the inverse all-to-all for O (all_to_all_4d(.,1,2), :63).
// The per-rank position all_gathers of the reference (usp_attention.cpp:53,
// ring_attention.cpp:56) are not needed: the layout is static, so every
// rank computes all positions on the host (plan.cpp).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/usp_attn.h"
#include "fa_bwd.hpp"
#include "fa_fwd.hpp"
#include "plan.hpp"
#include "reshard.hpp"
#include "transport.hpp"

namespace uspb200 {

cudaError_t launch_fa_fwd(const FwdParams& p, int nq, int hs, int grid, cudaStream_t stream);

#define USPB_CHECK(x)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw Error(ErrorCode::kInternal, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw Error(ErrorCode::kInternal, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

// (hs, heads, seq, batch) bf16 tensor; box = one 128-row x 64-column block
// of one head, 128-byte swizzled to match the UMMA SW128 descriptors.
static CUtensorMap make_tmap(const void* base, int64_t hs, int64_t heads, int64_t seq,
                             int64_t batch, uint32_t box_rows = kTileM) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(hs), static_cast<cuuint64_t>(heads),
                              static_cast<cuuint64_t>(seq), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(hs * 2),
                                 static_cast<cuuint64_t>(heads * hs * 2),
                                 static_cast<cuuint64_t>(seq * heads * hs * 2)};
  const cuuint32_t box[4] = {64, 1, box_rows, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::ostringstream os;
    os << "cuTensorMapEncodeTiled failed (" << int(r) << "); base " << base
       << " must be 16-byte aligned";
    throw Error(ErrorCode::kInvalidArgument, os.str());
  }
  return m;
}

// fp32 (hs, heads, seq, batch) map for the fused backward's TMA reductions:
// box (32 columns, 1, 32 rows, 1) = 128-byte rows, 128B-swizzled in shared memory.
static CUtensorMap make_tmap_f32(void* base, int64_t hs, int64_t heads, int64_t seq, int64_t batch) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(hs), static_cast<cuuint64_t>(heads),
                              static_cast<cuuint64_t>(seq), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(hs * 4), static_cast<cuuint64_t>(heads * hs * 4),
                                 static_cast<cuuint64_t>(seq * heads * hs * 4)};
  const cuuint32_t box[4] = {32, 1, 32, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::ostringstream os;
    os << "cuTensorMapEncodeTiled (fp32) failed (" << int(r) << ")";
    throw Error(ErrorCode::kInternal, os.str());
  }
  return m;
}

// ------------------------------------------------------------ device memory
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) : bytes(n) {
    if (n) USPB_CHECK(cudaMalloc(&p, n));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <class T>
static DevBuf upload(const std::vector<T>& v) {
  DevBuf b(std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) USPB_CHECK(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return b;
}

struct DevStep {
  StepPlan host;
  DevBuf q_pos, k_pos, tile_off, tile_list, units;
  EpiMode mode = EpiMode::kSingle;
};

// ------------------------------------------------------------------ Engine
class Engine {
 public:
  Engine(const usp_config& c, Transport* tr) : cfg_(c), tr_(tr) {
    shape_ = to_shape(c);
    shape_.validate();
    const int world = shape_.mesh.world();
    if (c.rank < 0 || c.rank >= world) throw_invalid("rank outside the mesh");
    if (world > 1 && !tr_) throw_invalid("a transport (usp_comm) is required when U*R > 1");
    if (tr_ && tr_->world_size() != world) throw_invalid("transport world size does not match U*R");
    U_ = shape_.mesh.ulysses;
    R_ = shape_.mesh.ring;
    u_ = shape_.mesh.ulysses_coord(c.rank);
    r_ = shape_.mesh.ring_coord(c.rank);
    B_ = shape_.batch;
    T_ = shape_.tokens_per_rank();
    Tr_ = shape_.tokens_per_ring_rank();
    H_ = shape_.heads;
    KV_ = shape_.kv_heads;
    hl_ = shape_.local_heads();
    kvl_ = shape_.local_kv_heads();
    hs_ = shape_.head_size;
    hsk_ = shape_.kernel_head_size();
    const int group = hl_ / kvl_;
    USPB_CHECK(cudaSetDevice(c.device));
    USPB_CHECK(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, c.device));
    tiling_ = fwd_tiling(hl_, kvl_, hsk_, Tr_, B_, num_sms_);
    nq_ = (tiling_.pair_rows || group % 2 == 0) ? 2 : 1;
    cluster_ = tiling_.cluster;  // 2-CTA clusters sharing K/V tiles by TMA multicast
    static const int cluster_mode = [] {  // 2: cta_group::2 MMAs on the same clusters (experimental)
      const char* e = dev_env("USP_FA_CLUSTER");
      return e ? std::atoi(e) : 1;
    }();
    cluster_mode_ = cluster_ ? (cluster_mode == 2 ? 2 : 1) : 0;


    const size_t e = 2;  // bf16
    const bool reshape = U_ > 1 || hs_ != hsk_;
    q_part_ = size_t(B_) * T_ * hl_ * hsk_ * e;
    kv_part_ = size_t(B_) * T_ * kvl_ * hsk_ * e;
    const size_t q_heads = size_t(B_) * Tr_ * hl_ * hsk_ * e;
    const size_t kv_heads = size_t(B_) * Tr_ * kvl_ * hsk_ * e;
    kv_bytes_ = kv_heads;
    if (reshape) {
      q_h_ = DevBuf(q_heads);
      kv0_ = DevBuf(2 * kv_heads);
      o_h_ = DevBuf(q_heads);
    }
    if (U_ > 1) {
      send_ = DevBuf(U_ * (q_part_ + 2 * kv_part_));
      if (B_ > 1) recv_ = DevBuf(U_ * (q_part_ + 2 * kv_part_));
      o_recv_ = DevBuf(U_ * q_part_);
      if (B_ > 1) o_send_ = DevBuf(U_ * q_part_);
    }
    if (R_ > 1) {
      kv_ring_[0] = DevBuf(2 * kv_heads);
      if (R_ > 2) kv_ring_[1] = DevBuf(2 * kv_heads);
      o_acc_ = DevBuf(size_t(B_) * Tr_ * hl_ * hsk_ * sizeof(float));
      lse_acc_ = DevBuf(size_t(B_) * Tr_ * hl_ * sizeof(float));
      USPB_CHECK(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking));
      for (int t = 0; t < R_; ++t) {
        cudaEvent_t a, b;
        USPB_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        USPB_CHECK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        ev_pre_.push_back(a);
        ev_recv_.push_back(b);
      }
    }

    sched_ = DevBuf(64);
    USPB_CHECK(cudaMemset(sched_.p, 0, 64));

    // Static layout -> per-step tile plans (the reference all_gathers these
    // positions at run time; here they are known at create).
    const auto my_pos = head_positions(shape_, c.rank);
    for (int t = 0; t < R_; ++t) {
      const int src = ring_source(r_, t, R_);
      const auto k_pos = head_positions(shape_, shape_.mesh.rank_of(u_, src));
      DevStep st;
      st.mode = R_ == 1 ? EpiMode::kSingle
                        : (t == 0 ? EpiMode::kFirst : (t == R_ - 1 ? EpiMode::kLast : EpiMode::kMiddle));
      const bool include_empty = st.mode != EpiMode::kMiddle;
      st.host = plan_step(my_pos, k_pos, shape_.causal, B_, tiling_.head_units, include_empty,
                          tiling_.units_per_kv, tiling_.rows_per_unit);
      st.q_pos = upload(st.host.q_pos);
      st.k_pos = upload(st.host.k_pos);
      st.tile_off = upload(st.host.tile_off);
      st.tile_list = upload(st.host.tile_list);
      st.units = upload(st.host.units);
      steps_.push_back(std::move(st));
    }

    // Ring overlap sizing. The K+V block shifted after step t
    // must land before step t+1 starts, i.e. within step t's attention:
    // required bandwidth = 2 * kv_bytes / t_step(t), t_step from the
    // step's visible pairs at the measured forward rate (kFwdTflops), taken
    // with 2x margin over the shortest shifted-behind step. An NVLink
    // send/recv channel of NCCL moves >= kCtaGBs (conservative; measured on
    // the box by tools/overlap_nccl.py), so the ring communicator gets
    // ceil(2 * required / kCtaGBs) CTAs (1..16) and, because a CTA needs an
    // SM the persistent attention grid would otherwise hold, the attention
    // grid leaves that many SMs free (NCCL transport only; the copy-engine
    // transports take no SMs).
    if (R_ > 1) {
      constexpr double kFwdTflops = 1300.0, kCtaGBs = 20.0;
      double t_min = 1e30;
      for (int t = 0; t + 1 < R_; ++t) {
        const double f = 4.0 * double(B_) * hl_ * hs_ * double(steps_[t].host.visible_pairs);
        t_min = std::min(t_min, f / (kFwdTflops * 1e12));
      }
      kv_shift_bytes_ = 2.0 * double(kv_bytes_);
      step_ms_est_ = t_min * 1e3;
      required_gbs_ = t_min > 0 && t_min < 1e29 ? kv_shift_bytes_ / t_min / 1e9 : 0.0;
      ring_ctas_ = std::min(16, std::max(1, static_cast<int>(std::ceil(2.0 * required_gbs_ / kCtaGBs))));
      reserved_sms_ = (tr_ && tr_->comm_uses_sms()) ? ring_ctas_ : 0;
    }
    // Ulysses exchanges pipelined in row chunks: default two
    // chunks wherever the exchange goes through a transport collective (not
    // the peer-memory direct exchange) at bs = 1. On NCCL the chunk exchanges
    // that overlap the attention run on a second Ulysses communicator capped
    // at a2a_ctas CTAs, and the attention grid leaves that many SMs: sized
    // like the ring (2x the bandwidth an overlapped chunk of Q / O needs to
    // land within one chunk of attention, at a conservative 20 GB/s per CTA),
    // from the shape alone so every rank computes the same values.
    const int rows_unit = tiling_.rows_per_unit;
    const bool chunkable = U_ > 1 && B_ == 1 && tr_ && !tr_->peer_memory() && T_ % (2 * rows_unit) == 0;
    if (chunkable) {
      constexpr double kFwdTflops = 1300.0, kCtaGBs = 20.0;
      const double L = double(shape_.seq_len);
      const double pairs = shape_.causal ? L * (L + 1) / 2 : L * L;
      const double f_rank = 4.0 * double(B_) * double(H_) * hs_ * pairs / double(U_ * R_);
      const int C = 2;
      const double t_chunk = f_rank / R_ / C / (kFwdTflops * 1e12);
      const double bytes = double(U_ - 1) * double(q_part_) / C;
      const double gbs = t_chunk > 0 ? bytes / t_chunk / 1e9 : 0.0;
      if (tr_->comm_uses_sms()) {
        a2a_ctas_ = std::min(16, std::max(1, static_cast<int>(std::ceil(2.0 * gbs / kCtaGBs))));
        reserved_sms_ = std::max(reserved_sms_, a2a_ctas_);
      }
      configure_chunks(C);
    }
    if (tr_) groups_ = tr_->make_groups(c.rank, shape_.mesh.ulysses_group(c.rank),
                                        shape_.mesh.ring_group(c.rank), ring_ctas_, a2a_ctas_);
  }

  // Row-chunk plans of the ring steps whose attention overlaps a Ulysses
  // exchange: step 0 (a2a in) and step R-1 (a2a out). Chunk c of every
  // member's T rows = rows [c T/C, (c+1) T/C): unit u belongs to chunk
  // ((first row of u) mod T) / (T / C).
  void configure_chunks(int C) {
    if (C < 1 || (C > 1 && (U_ < 2 || B_ != 1 || T_ % (int64_t(C) * tiling_.rows_per_unit) != 0)))
      throw_invalid("a2a chunks must divide every member's rows into whole query tiles (U > 1, bs = 1)");
    a2a_steps_.clear();
    a2a_chunks_ = C;
    if (C == 1) return;
    if (!comm_stream_) USPB_CHECK(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking));
    while (static_cast<int>(ev_in_.size()) < C) {
      cudaEvent_t a, b;
      USPB_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      USPB_CHECK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      ev_in_.push_back(a);
      ev_attn_.push_back(b);
    }
    if (!ev_chunk_misc_[0])
      for (auto& e : ev_chunk_misc_) USPB_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const int64_t rows = T_ / C, per = tiling_.rows_per_unit;
    for (int si : {0, R_ - 1}) {
      if (si == R_ - 1 && si == 0 && !a2a_steps_.empty()) break;  // R = 1: one split step
      std::vector<DevStep> cs(C);
      const StepPlan& h = steps_[si].host;
      for (int c = 0; c < C; ++c) {
        cs[c].host = h;
        cs[c].host.units.clear();
        cs[c].mode = steps_[si].mode;
      }
      for (uint32_t u : h.units) {
        const int64_t row0 = int64_t(u & 0xFFFF) * per;
        cs[static_cast<size_t>((row0 % T_) / rows)].host.units.push_back(u);
      }
      for (auto& d : cs) {
        d.q_pos = upload(d.host.q_pos);
        d.k_pos = upload(d.host.k_pos);
        d.tile_off = upload(d.host.tile_off);
        d.tile_list = upload(d.host.tile_list);
        d.units = upload(d.host.units);
      }
      a2a_steps_.push_back(std::move(cs));
    }
  }

 public:
  struct Info {
    int num_sms, reserved_sms, ring_ctas;
    double kv_shift_bytes, step_ms_est, required_gbs;
  };
  Info info() const {
    return {num_sms_, reserved_sms_, ring_ctas_, kv_shift_bytes_, step_ms_est_, required_gbs_};
  }
  // SMs the attention grid leaves free for a concurrent communication kernel
  // (default: the sizing above).
  void set_deterministic(bool on) { deterministic_ = on; }  // plans follow at the next backward
  void set_a2a_chunks(int n) { configure_chunks(n); }
  int a2a_chunks() const { return a2a_chunks_; }
  void set_reserved_sms(int n) {
    if (n < 0 || n >= num_sms_) throw_invalid("reserved SMs must be in [0, #SMs)");
    reserved_sms_ = n;
  }

 private:
  int ring_ctas_ = 1, reserved_sms_ = 0, a2a_ctas_ = 0, a2a_chunks_ = 1;
  // Direct exchange over a peer-memory transport at bs = 1:
  // the pack kernels store Q/K/V parts straight into the owning members'
  // head-sharded buffers (no staging, no copy), and the last attention step
  // stores O rows straight into the owners' receive buffers.
  bool direct_a2a() const {
    static const bool direct_ok = [] {
      const char* e = dev_env("USP_DIRECT_A2A");
      return !e || std::atoi(e) != 0;
    }();
    return direct_ok && U_ > 1 && B_ == 1 && U_ <= 16 && tr_ && tr_->peer_memory();
  }
  // usp_attn_fwd_host with chunked all-to-alls (fwd_host_a2a): the caller's
  // host buffers, read by fwd()'s chunked branches
  struct HostIo {
    const void *q, *k, *v;
    void* o;
    float* lse;
  };
  const HostIo* hio_ = nullptr;
  std::vector<cudaEvent_t> ev_hq_, ev_ho_;
  // a2a_steps_[0]: step 0 split in row chunks (a2a in overlap);
  // a2a_steps_[1] (R > 1): step R-1 (a2a out overlap)
  std::vector<std::vector<DevStep>> a2a_steps_;
  std::vector<cudaEvent_t> ev_in_, ev_attn_;
  cudaEvent_t ev_chunk_misc_[2] = {nullptr, nullptr};  // packed, last a2a out done
  double kv_shift_bytes_ = 0, step_ms_est_ = 0, required_gbs_ = 0;

 public:

  ~Engine() {
    if (tr_) {
      try {  // peer-memory mappings of this engine's buffers (advice r1)
        tr_->release_buffers({q_h_.p, kv0_.p, o_h_.p, send_.p, recv_.p, o_send_.p, o_recv_.p, kv_ring_[0].p,
                              kv_ring_[1].p, do_h_.p, grad_h_.p, grad_recv_.p, acc_dkv_[0].p, acc_dkv_[1].p,
                              own_dkv_.p, dq_acc_.p});
      } catch (...) {
      }
    }
    for (auto e : event_pool_) cudaEventDestroy(e);
    for (auto e : stage_pool_) cudaEventDestroy(e);
    for (auto e : ev_pre_) cudaEventDestroy(e);
    for (auto e : ev_recv_) cudaEventDestroy(e);
    for (auto e : ev_in_) cudaEventDestroy(e);
    for (auto e : ev_attn_) cudaEventDestroy(e);
    for (auto e : ev_hq_) cudaEventDestroy(e);
    for (auto e : ev_ho_) cudaEventDestroy(e);
    for (auto e : ev_chunk_misc_)
      if (e) cudaEventDestroy(e);
    for (auto e : ev_acc_) cudaEventDestroy(e);
    if (comm_stream_) cudaStreamDestroy(comm_stream_);
    for (auto e : ev_chunk_in_) cudaEventDestroy(e);
    for (auto e : ev_chunk_out_) cudaEventDestroy(e);
    if (ev_entry_) cudaEventDestroy(ev_entry_);
    if (ev_kv_) cudaEventDestroy(ev_kv_);
    if (ev_drained_) cudaEventDestroy(ev_drained_);
    if (h2d_stream_) cudaStreamDestroy(h2d_stream_);
    if (d2h_stream_) cudaStreamDestroy(d2h_stream_);
  }

  static UspShape to_shape(const usp_config& c) {
    UspShape s;
    s.mesh.ulysses = c.ulysses_degree;
    s.mesh.ring = c.ring_degree;
    s.batch = c.batch;
    s.seq_len = c.seq_len;
    s.heads = c.heads;
    s.kv_heads = c.kv_heads;
    s.head_size = c.head_size;
    s.causal = c.causal != 0;
    return s;
  }

  int last_launches() const { return launches_; }

  void fwd(const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
    USPB_CHECK(cudaSetDevice(cfg_.device));
    for (const void* ptr : {q, k, v, static_cast<const void*>(o), static_cast<const void*>(lse)})
      if (!ptr || reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
        throw_invalid("q, k, v, o, lse must be non-null 16-byte aligned device pointers");
    launches_ = 0;
    ledger_.clear();
    have_fwd_ = false;
    stage_begin(st);
    const size_t e = 2;
    const bool reshape = U_ > 1 || hs_ != hsk_;
    const void* qh = q;
    const void* kh = k;
    const void* vh = v;
    uint8_t* kv0 = kv0_.as<uint8_t>();
    const bool direct = direct_a2a();
    const bool chunked = !direct && a2a_chunks_ > 1;
    if (direct) {
      // -- 1. Ulysses in, fused with the pack: part m of my Q/K/V rows ->
      //    member m's rows [u*T, (u+1)*T) of its head-sharded Q / K / V
      void* pq[16];
      void* pkv[16];
      for (int m = 0; m < U_; ++m) {
        pq[m] = tr_->ulysses_peer_ptr(*groups_, q_h_.p, m, U_ * q_part_);
        pkv[m] = tr_->ulysses_peer_ptr(*groups_, kv0_.p, m, 2 * kv_bytes_);
      }
      tr_->ulysses_ready(*groups_, st);  // every member's Q/K/V buffers are free
      batch_begin();
      for (int m = 0; m < U_; ++m) {
        pack_part(q, static_cast<uint8_t*>(pq[m]) + u_ * q_part_, H_, hl_, m, st);
        pack_part(k, static_cast<uint8_t*>(pkv[m]) + u_ * kv_part_, KV_, kvl_, m, st);
        pack_part(v, static_cast<uint8_t*>(pkv[m]) + kv_bytes_ + u_ * kv_part_, KV_, kvl_, m, st);
      }
      batch_flush(st);
      tr_->ulysses_done(*groups_, st);  // every member's parts for me have landed
      stage(st, "pack_a2a_in");
      record_a2a(0, q_part_);
      record_a2a(1, kv_part_);
      record_a2a(2, kv_part_);
      qh = q_h_.p;
      kh = kv0;
      vh = kv0 + kv_bytes_;
    } else if (chunked) {
      // -- 1. Ulysses in, pipelined: pack once, then C
      //    exchanges on comm_stream_, chunk c = rows [c T/C, (c+1) T/C) of
      //    every member's part (K / V whole in chunk 0: every q row needs
      //    every key); ring step 0 runs chunk c as soon as it has landed, so
      //    the exchange of chunk c+1 overlaps the attention of chunk c.
      //    Received in place (bs = 1), no unpack.
      uint8_t* sq = send_.as<uint8_t>();
      uint8_t* sk = sq + U_ * q_part_;
      uint8_t* sv = sk + U_ * kv_part_;
      const size_t qs = q_part_ / a2a_chunks_;
      const int64_t rc = T_ / a2a_chunks_;
      if (hio_) {
        // host buffers (fwd_host_a2a): on h2d_stream_, K and V go up and are
        // packed, then Q row chunk c goes up and is packed — rows
        // [c T/C, (c+1) T/C) of the caller's shard are exactly chunk c of
        // every member's part — so exchange c starts once its rows landed.
        const size_t qrow = size_t(H_) * hs_ * 2, kvrow = size_t(KV_) * hs_ * 2;
        USPB_CHECK(cudaMemcpyAsync(const_cast<void*>(k), hio_->k, T_ * kvrow, cudaMemcpyHostToDevice, h2d_stream_));
        USPB_CHECK(cudaMemcpyAsync(const_cast<void*>(v), hio_->v, T_ * kvrow, cudaMemcpyHostToDevice, h2d_stream_));
        batch_begin();
        pack_heads(k, sk, KV_, kvl_, h2d_stream_);
        pack_heads(v, sv, KV_, kvl_, h2d_stream_);
        batch_flush(h2d_stream_);
        for (int c = 0; c < a2a_chunks_; ++c) {
          const size_t off = size_t(c) * rc * qrow;
          USPB_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(const_cast<void*>(q)) + off,
                                     static_cast<const uint8_t*>(hio_->q) + off, rc * qrow, cudaMemcpyHostToDevice,
                                     h2d_stream_));
          pack_heads(q, sq, H_, hl_, h2d_stream_, c * rc, (c + 1) * rc);
          USPB_CHECK(cudaEventRecord(ev_hq_[c], h2d_stream_));
        }
      } else {
        batch_begin();
        pack_heads(q, sq, H_, hl_, st);
        pack_heads(k, sk, KV_, kvl_, st);
        pack_heads(v, sv, KV_, kvl_, st);
        batch_flush(st);
        stage(st, "pack");
        USPB_CHECK(cudaEventRecord(ev_chunk_misc_[0], st));
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_chunk_misc_[0], 0));
      }
      for (int c = 0; c < a2a_chunks_; ++c) {
        if (hio_) USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_hq_[c], 0));
        std::vector<std::vector<A2APart>> parts(c == 0 ? 3 : 1, std::vector<A2APart>(U_));
        for (int p = 0; p < U_; ++p) {
          parts[0][p] = {sq + p * q_part_ + c * qs, q_h_.as<uint8_t>() + p * q_part_ + c * qs};
          if (c == 0) {
            parts[1][p] = {sk + p * kv_part_, kv0 + p * kv_part_};
            parts[2][p] = {sv + p * kv_part_, kv0 + kv_bytes_ + p * kv_part_};
          }
        }
        cudaEvent_t s0 = side_event(comm_stream_);
        if (c == 0)
          tr_->all_to_all(*groups_, parts, {qs, kv_part_, kv_part_}, comm_stream_);
        else
          tr_->all_to_all(*groups_, parts, {qs}, comm_stream_, /*overlapped=*/true);
        side_span("a2a_in." + std::to_string(c), s0, side_event(comm_stream_));
        USPB_CHECK(cudaEventRecord(ev_in_[c], comm_stream_));
      }
      record_a2a(0, q_part_);
      record_a2a(1, kv_part_);
      record_a2a(2, kv_part_);
      qh = q_h_.p;
      kh = kv0;
      vh = kv0 + kv_bytes_;
    } else if (U_ > 1) {
      // -- 1. Ulysses in: pack (b,T,H,hs) -> [peer][b][T][H/U][hsk], one exchange
      uint8_t* sq = send_.as<uint8_t>();
      uint8_t* sk = sq + U_ * q_part_;
      uint8_t* sv = sk + U_ * kv_part_;
      batch_begin();
      pack_heads(q, sq, H_, hl_, st);
      pack_heads(k, sk, KV_, kvl_, st);
      pack_heads(v, sv, KV_, kvl_, st);
      batch_flush(st);
      stage(st, "pack");
      uint8_t* rq = B_ > 1 ? recv_.as<uint8_t>() : nullptr;
      uint8_t* rk = rq ? rq + U_ * q_part_ : nullptr;
      uint8_t* rv = rk ? rk + U_ * kv_part_ : nullptr;
      std::vector<std::vector<A2APart>> parts(3, std::vector<A2APart>(U_));
      for (int p = 0; p < U_; ++p) {
        // bs == 1: part p is exactly rows [p*T, (p+1)*T) of the head-sharded
        // tensor, so it is received in place (no unpack kernel).
        parts[0][p] = {sq + p * q_part_, rq ? rq + p * q_part_ : q_h_.as<uint8_t>() + p * q_part_};
        parts[1][p] = {sk + p * kv_part_, rk ? rk + p * kv_part_ : kv0 + p * kv_part_};
        parts[2][p] = {sv + p * kv_part_, rv ? rv + p * kv_part_ : kv0 + kv_bytes_ + p * kv_part_};
      }
      tr_->all_to_all(*groups_, parts, {q_part_, kv_part_, kv_part_}, st);
      stage(st, "a2a_in");
      record_a2a(0, q_part_);
      record_a2a(1, kv_part_);
      record_a2a(2, kv_part_);
      if (B_ > 1) {
        batch_begin();
        gather_seq(rq, q_h_.p, hl_, st);
        gather_seq(rk, kv0, kvl_, st);
        gather_seq(rv, kv0 + kv_bytes_, kvl_, st);
        batch_flush(st);
        stage(st, "unpack_in");
      }
      qh = q_h_.p;
      kh = kv0;
      vh = kv0 + kv_bytes_;
    } else {
      // U == 1: the reference's all-to-alls are no-ops (0 bytes); keep the
      // ledger entries it would record.
      record_a2a(0, q_part_);
      record_a2a(1, kv_part_);
      record_a2a(2, kv_part_);
    }
    if (U_ == 1 && reshape) {
      pad_rows(q, q_h_.p, B_ * T_ * H_, st);
      pad_rows(k, kv0, B_ * T_ * KV_, st);
      pad_rows(v, kv0 + kv_bytes_, B_ * T_ * KV_, st);
      stage(st, "pad");
      qh = q_h_.p;
      kh = kv0;
      vh = kv0 + kv_bytes_;
    }

    // -- 2. ring: R kernel launches, K/V shifted one step ahead on comm_stream_
    void* o_heads = reshape ? o_h_.p : o;
    const CUtensorMap tm_q = make_tmap(qh, hsk_, hl_, Tr_, B_);
    auto kbuf = [&](int t) -> const void* {
      if (t == 0) return kh;
      return kv_ring_[(t - 1) & 1].p;
    };
    auto vbuf = [&](int t) -> const void* {
      if (t == 0) return vh;
      return kv_ring_[(t - 1) & 1].as<uint8_t>() + kv_bytes_;
    };
    // Direct O: over a peer-memory transport the last step's
    // epilogue stores each O row straight into the owning Ulysses member's
    // receive buffer, so the O all-to-all overlaps the attention tile by tile.
    const bool direct_o = direct;
    void* o_peer[16] = {};
    if (direct_o)
      for (int m = 0; m < U_; ++m) o_peer[m] = tr_->ulysses_peer_ptr(*groups_, o_recv_.p, m, U_ * q_part_);
    for (int t = 0; t < R_; ++t) {
      if (t + 1 < R_) {
        USPB_CHECK(cudaEventRecord(ev_pre_[t], st));  // buf(t) ready, buf(t+1) free
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_pre_[t], 0));
        record_shift(1);
        record_shift(2);
        cudaEvent_t sh0 = side_event(comm_stream_);
        tr_->ring_shift(*groups_, {kbuf(t), vbuf(t)},
                        {const_cast<void*>(kbuf(t + 1)), const_cast<void*>(vbuf(t + 1))},
                        {kv_bytes_, kv_bytes_}, comm_stream_);
        side_span("shift" + std::to_string(t + 1), sh0, side_event(comm_stream_));
        USPB_CHECK(cudaEventRecord(ev_recv_[t], comm_stream_));
      }
      if (t > 0) {
        USPB_CHECK(cudaStreamWaitEvent(st, ev_recv_[t - 1], 0));
        stage(st, "wait" + std::to_string(t));  // exposed part of the shift into step t
      }
      const bool last = t == R_ - 1;
      if (direct_o && last) tr_->ulysses_ready(*groups_, st);  // every member's o_recv_ is free
      if (chunked && (t == 0 || last)) {
        // row chunks: wait for chunk c's Q (step 0); after the last step's
        // chunk c, its O rows go out while chunk c+1 computes
        const std::vector<DevStep>& cs = a2a_steps_[t == 0 ? 0 : 1];
        const size_t qs = q_part_ / a2a_chunks_;
        for (int c = 0; c < a2a_chunks_; ++c) {
          if (t == 0) {
            USPB_CHECK(cudaStreamWaitEvent(st, ev_in_[c], 0));
            stage(st, "wait_in." + std::to_string(c));  // exposed part of chunk c's exchange
          }
          launch_plan(cs[c], tm_q, kbuf(t), vbuf(t), o_heads, lse, Tr_, Tr_, st);
          stage(st, "attn" + std::to_string(t) + "." + std::to_string(c));
          if (!last) continue;
          USPB_CHECK(cudaEventRecord(ev_attn_[c], st));
          USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_attn_[c], 0));
          std::vector<std::vector<A2APart>> parts(1, std::vector<A2APart>(U_));
          uint8_t* osend = static_cast<uint8_t*>(o_heads);
          for (int p = 0; p < U_; ++p)
            parts[0][p] = {osend + p * q_part_ + c * qs, o_recv_.as<uint8_t>() + p * q_part_ + c * qs};
          cudaEvent_t s0 = side_event(comm_stream_);
          tr_->all_to_all(*groups_, parts, {qs}, comm_stream_, /*overlapped=*/c + 1 < a2a_chunks_);
          side_span("a2a_out." + std::to_string(c), s0, side_event(comm_stream_));
          if (hio_) {
            // host buffers: chunk c's O rows are unpacked behind their
            // exchange and go down while chunk c+1 computes; LSE (written by
            // the attention in place) goes down after the last chunk
            const int64_t rc = T_ / a2a_chunks_;
            const size_t qrow = size_t(H_) * hs_ * 2;
            unpack_heads(o_recv_.p, o, comm_stream_, 0, 0, c * rc, (c + 1) * rc);
            if (c + 1 == a2a_chunks_) {
              USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_attn_[c], 0));
              USPB_CHECK(cudaMemcpyAsync(hio_->lse, lse, size_t(B_) * Tr_ * hl_ * sizeof(float),
                                         cudaMemcpyDeviceToHost, d2h_stream_));
            }
            USPB_CHECK(cudaEventRecord(ev_ho_[c], comm_stream_));
            USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_ho_[c], 0));
            USPB_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(hio_->o) + c * rc * qrow,
                                       static_cast<uint8_t*>(o) + c * rc * qrow, rc * qrow, cudaMemcpyDeviceToHost,
                                       d2h_stream_));
          }
        }
        continue;
      }
      launch_step(t, tm_q, kbuf(t), vbuf(t), o_heads, lse, st, direct_o && last ? o_peer : nullptr);
      stage(st, "attn" + std::to_string(t));
    }

    // -- 3. Ulysses out: [peer][b][T][H/U] -> (b, T, H, hs)
    if (chunked) {
      USPB_CHECK(cudaEventRecord(ev_chunk_misc_[1], comm_stream_));
      USPB_CHECK(cudaStreamWaitEvent(st, ev_chunk_misc_[1], 0));
      stage(st, "a2a_out");  // exposed part: the last chunk's exchange
      record_a2a(3, q_part_);
      if (!hio_) {  // (host buffers: unpacked per chunk above)
        unpack_heads(o_recv_.p, o, st);
        stage(st, "unpack");
      }
    } else if (direct_o) {
      tr_->ulysses_done(*groups_, st);  // every member's rows for me have landed
      stage(st, "a2a_out");
      record_a2a(3, q_part_);
      unpack_heads(o_recv_.p, o, st);
      stage(st, "unpack");
    } else if (U_ > 1) {
      uint8_t* osend = o_h_.as<uint8_t>();
      if (B_ > 1) {
        split_seq(o_h_.p, o_send_.p, st);
        osend = o_send_.as<uint8_t>();
        stage(st, "pack_out");
      }
      std::vector<std::vector<A2APart>> parts(1, std::vector<A2APart>(U_));
      for (int p = 0; p < U_; ++p)
        parts[0][p] = {osend + p * q_part_, o_recv_.as<uint8_t>() + p * q_part_};
      tr_->all_to_all(*groups_, parts, {q_part_}, st);
      stage(st, "a2a_out");
      record_a2a(3, q_part_);
      unpack_heads(o_recv_.p, o, st);
      stage(st, "unpack");
    } else {
      record_a2a(3, q_part_);
    }
    if (U_ == 1 && reshape) {
      RowPermute rp;
      rp.src = o_h_.p;
      rp.dst = o;
      rp.dims[3] = B_ * T_ * H_;
      rp.src_stride[3] = rp.dst_stride[3] = 1;
      rp.hs_src = hsk_;
      rp.hs_dst = hs_;
      permute(rp, st);
      stage(st, "unpad");
    }
    (void)e;
    have_fwd_ = true;
    fwd_ledger_size_ = ledger_.size();
  }

  // ------------------------------------------------------------ host buffers
  // usp_attn_fwd_host: the same forward with Q/K/V/O/LSE in host memory; the
  // host<->device copies are part of the call. At U = R = 1 (bs 1, native
  // head size) the sequence is cut into row chunks [r0, r1): chunk c's Q/K/V
  // rows go up on h2d_stream_, its attention launch (query rows of chunk c
  // against keys [0, r1) when causal — positions are the identity at
  // U = R = 1 — or all keys otherwise) waits only for them, and its O/LSE
  // rows go down on d2h_stream_. PCIe traffic then overlaps the attention of
  // the neighbouring chunks instead of adding to it (chunk_bounds() sizes the
  // chunks so it does). A pure ring pipelines in fwd_host_ring, chunked
  // Ulysses exchanges in fwd_host_a2a; other meshes copy the whole shard
  // around fwd().
  void fwd_host(const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
    USPB_CHECK(cudaSetDevice(cfg_.device));
    for (const void* ptr : {q, k, v, static_cast<const void*>(o), static_cast<const void*>(lse)})
      if (!ptr) throw_invalid("q, k, v, o, lse must be non-null host pointers");
    const size_t qb = size_t(B_) * T_ * H_ * hs_ * 2, kvb = size_t(B_) * T_ * KV_ * hs_ * 2;
    const size_t lb = size_t(B_) * Tr_ * hl_ * sizeof(float);
    if (!hq_.p) {
      hq_ = DevBuf(qb);
      hk_ = DevBuf(kvb);
      hv_ = DevBuf(kvb);
      ho_ = DevBuf(qb);
      hlse_ = DevBuf(lb);
      USPB_CHECK(cudaStreamCreateWithFlags(&h2d_stream_, cudaStreamNonBlocking));
      USPB_CHECK(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking));
      const unsigned fl = dev_env("USP_HOST_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
      USPB_CHECK(cudaEventCreateWithFlags(&ev_entry_, fl));
      USPB_CHECK(cudaEventCreateWithFlags(&ev_drained_, fl));
    }
    const bool reshape = U_ > 1 || hs_ != hsk_;
    if (U_ == 1 && R_ > 1 && B_ == 1 && !reshape && Tr_ >= 4 * kTileM) {
      fwd_host_ring(q, k, v, o, lse, st);
      return;
    }
    if (U_ > 1 && !direct_a2a() && a2a_chunks_ > 1) {
      fwd_host_a2a(q, k, v, o, lse, st);
      return;
    }
    const std::vector<int64_t> bounds = chunk_bounds();
    if (U_ > 1 || R_ > 1 || B_ > 1 || reshape || bounds.size() <= 2) {
      USPB_CHECK(cudaMemcpyAsync(hq_.p, q, qb, cudaMemcpyHostToDevice, st));
      USPB_CHECK(cudaMemcpyAsync(hk_.p, k, kvb, cudaMemcpyHostToDevice, st));
      USPB_CHECK(cudaMemcpyAsync(hv_.p, v, kvb, cudaMemcpyHostToDevice, st));
      fwd(hq_.p, hk_.p, hv_.p, ho_.p, hlse_.as<float>(), st);
      USPB_CHECK(cudaMemcpyAsync(o, ho_.p, qb, cudaMemcpyDeviceToHost, st));
      USPB_CHECK(cudaMemcpyAsync(lse, hlse_.p, lb, cudaMemcpyDeviceToHost, st));
      return;
    }
    ensure_chunk_plans(bounds);
    launches_ = 0;
    ledger_.clear();
    for (int tsr = 0; tsr < 4; ++tsr) record_a2a(tsr, tsr == 0 || tsr == 3 ? q_part_ : kv_part_);
    const int n = static_cast<int>(chunk_steps_.size());
    const size_t qrow = size_t(H_) * hs_ * 2, kvrow = size_t(KV_) * hs_ * 2, lrow = size_t(hl_) * 4;
    auto up = [&](DevBuf& d, const void* h, int64_t r0, int64_t r1, size_t row) {
      USPB_CHECK(cudaMemcpyAsync(d.as<uint8_t>() + r0 * row, static_cast<const uint8_t*>(h) + r0 * row,
                                 (r1 - r0) * row, cudaMemcpyHostToDevice, h2d_stream_));
    };
    // the previous call's kernels may still read the staging buffers
    USPB_CHECK(cudaEventRecord(ev_entry_, st));
    USPB_CHECK(cudaStreamWaitEvent(h2d_stream_, ev_entry_, 0));
    USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_entry_, 0));
    if (!shape_.causal) {
      up(hk_, k, 0, Tr_, kvrow);
      up(hv_, v, 0, Tr_, kvrow);
    }
    for (int c = 0; c < n; ++c) {
      const int64_t r0 = bounds[c], r1 = bounds[c + 1];
      if (shape_.causal) {
        up(hk_, k, r0, r1, kvrow);
        up(hv_, v, r0, r1, kvrow);
      }
      up(hq_, q, r0, r1, qrow);
      USPB_CHECK(cudaEventRecord(ev_chunk_in_[c], h2d_stream_));
      USPB_CHECK(cudaStreamWaitEvent(st, ev_chunk_in_[c], 0));
      const int64_t k_len = shape_.causal ? r1 : Tr_;
      const CUtensorMap tm_q = make_tmap(hq_.as<uint8_t>() + r0 * qrow, hsk_, hl_, r1 - r0, B_);
      launch_plan(chunk_steps_[c], tm_q, hk_.p, hv_.p, ho_.as<uint8_t>() + r0 * qrow,
                  hlse_.as<float>() + r0 * hl_, r1 - r0, k_len, st);
      USPB_CHECK(cudaEventRecord(ev_chunk_out_[c], st));
      USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_chunk_out_[c], 0));
      USPB_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(o) + r0 * qrow, ho_.as<uint8_t>() + r0 * qrow,
                                 (r1 - r0) * qrow, cudaMemcpyDeviceToHost, d2h_stream_));
      USPB_CHECK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(lse) + r0 * lrow, hlse_.as<uint8_t>() + r0 * lrow,
                                 (r1 - r0) * lrow, cudaMemcpyDeviceToHost, d2h_stream_));
    }
    USPB_CHECK(cudaEventRecord(ev_drained_, d2h_stream_));
    USPB_CHECK(cudaStreamWaitEvent(st, ev_drained_, 0));
    have_fwd_ = true;
    fwd_ledger_size_ = ledger_.size();
    static const bool trace = dev_env("USP_HOST_TRACE") != nullptr;  // development timeline
    if (trace) {
      USPB_CHECK(cudaStreamSynchronize(st));
      auto at = [&](cudaEvent_t e) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_entry_, e);
        return ms;
      };
      for (int c = 0; c < n; ++c)
        std::fprintf(stderr, "chunk %2d rows [%7lld,%7lld): inputs ready %8.3f ms, attention done %8.3f ms\n", c,
                     static_cast<long long>(bounds[c]), static_cast<long long>(bounds[c + 1]), at(ev_chunk_in_[c]),
                     at(ev_chunk_out_[c]));
      std::fprintf(stderr, "drained %8.3f ms\n", at(ev_drained_));
    }
  }

  // usp_attn_fwd_host with chunked Ulysses all-to-alls (U > 1, bs 1, not
  // the direct peer-memory exchange): fwd() itself, with the host copies
  // woven into its chunk pipeline (hio_): K/V up and packed, then per row
  // chunk c Q up -> pack -> exchange c -> step-0 attention of chunk c; at
  // the last step exchange c -> unpack -> O rows down, so only the first
  // chunk's upload and the last chunk's download are exposed. Same kernels
  // and plans as fwd(): bitwise the device-resident results.
  void fwd_host_a2a(const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
    const int C = a2a_chunks_;
    if (static_cast<int>(ev_hq_.size()) != C) {
      for (auto e : ev_hq_) cudaEventDestroy(e);
      for (auto e : ev_ho_) cudaEventDestroy(e);
      ev_hq_.assign(C, nullptr);
      ev_ho_.assign(C, nullptr);
      for (int c = 0; c < C; ++c) {
        USPB_CHECK(cudaEventCreateWithFlags(&ev_hq_[c], cudaEventDisableTiming));
        USPB_CHECK(cudaEventCreateWithFlags(&ev_ho_[c], cudaEventDisableTiming));
      }
    }
    // the previous call's kernels and exchanges may still use the staging
    // and send buffers (its fwd() ended with st waiting for comm_stream_)
    USPB_CHECK(cudaEventRecord(ev_entry_, st));
    USPB_CHECK(cudaStreamWaitEvent(h2d_stream_, ev_entry_, 0));
    USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_entry_, 0));
    const HostIo io{q, k, v, o, lse};
    hio_ = &io;
    try {
      fwd(hq_.p, hk_.p, hv_.p, ho_.p, hlse_.as<float>(), st);
    } catch (...) {
      hio_ = nullptr;
      throw;
    }
    hio_ = nullptr;
    USPB_CHECK(cudaEventRecord(ev_drained_, d2h_stream_));
    USPB_CHECK(cudaStreamWaitEvent(st, ev_drained_, 0));
  }

  // usp_attn_fwd_host on a pure ring (U = 1, R > 1, bs 1): K and V go up
  // first, so the ring's first K/V shift starts while Q is still uploading;
  // Q follows in row chunks, each chunk's step-0 attention (own K/V block)
  // launched as soon as it has landed; the last ring step runs per row chunk
  // too, each chunk's O/LSE rows downloaded while the next chunk computes.
  // Every launch walks the same key tiles in the same order as fwd(), so
  // the results are bitwise those of the device-resident forward.
  void fwd_host_ring(const void* q, const void* k, const void* v, void* o, float* lse, cudaStream_t st) {
    ensure_ring_chunk_plans();
    launches_ = 0;
    ledger_.clear();
    have_fwd_ = false;
    for (int tsr = 0; tsr < 3; ++tsr) record_a2a(tsr, tsr == 0 ? q_part_ : kv_part_);
    const size_t qrow = size_t(H_) * hs_ * 2, kvrow = size_t(KV_) * hs_ * 2, lrow = size_t(hl_) * 4;
    const int n = static_cast<int>(ring_bounds_.size()) - 1;
    USPB_CHECK(cudaEventRecord(ev_entry_, st));
    USPB_CHECK(cudaStreamWaitEvent(h2d_stream_, ev_entry_, 0));
    USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_entry_, 0));
    USPB_CHECK(cudaMemcpyAsync(hk_.p, k, Tr_ * kvrow, cudaMemcpyHostToDevice, h2d_stream_));
    USPB_CHECK(cudaMemcpyAsync(hv_.p, v, Tr_ * kvrow, cudaMemcpyHostToDevice, h2d_stream_));
    USPB_CHECK(cudaEventRecord(ev_kv_, h2d_stream_));
    USPB_CHECK(cudaStreamWaitEvent(st, ev_kv_, 0));
    auto kbuf = [&](int t) -> const void* { return t == 0 ? hk_.p : kv_ring_[(t - 1) & 1].p; };
    auto vbuf = [&](int t) -> const void* {
      return t == 0 ? hv_.p : static_cast<const void*>(kv_ring_[(t - 1) & 1].as<uint8_t>() + kv_bytes_);
    };
    const CUtensorMap tm_q = make_tmap(hq_.p, hsk_, hl_, Tr_, B_);
    for (int t = 0; t < R_; ++t) {
      if (t + 1 < R_) {
        USPB_CHECK(cudaEventRecord(ev_pre_[t], st));
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_pre_[t], 0));
        record_shift(1);
        record_shift(2);
        tr_->ring_shift(*groups_, {kbuf(t), vbuf(t)},
                        {const_cast<void*>(kbuf(t + 1)), const_cast<void*>(vbuf(t + 1))},
                        {kv_bytes_, kv_bytes_}, comm_stream_);
        USPB_CHECK(cudaEventRecord(ev_recv_[t], comm_stream_));
      }
      if (t > 0) USPB_CHECK(cudaStreamWaitEvent(st, ev_recv_[t - 1], 0));
      if (t != 0 && t != R_ - 1) {
        launch_step(t, tm_q, kbuf(t), vbuf(t), ho_.p, hlse_.as<float>(), st);
        continue;
      }
      for (int c = 0; c < n; ++c) {
        const int64_t r0 = ring_bounds_[c], r1 = ring_bounds_[c + 1];
        if (t == 0) {
          USPB_CHECK(cudaMemcpyAsync(hq_.as<uint8_t>() + r0 * qrow, static_cast<const uint8_t*>(q) + r0 * qrow,
                                     (r1 - r0) * qrow, cudaMemcpyHostToDevice, h2d_stream_));
          USPB_CHECK(cudaEventRecord(ev_chunk_in_[c], h2d_stream_));
          USPB_CHECK(cudaStreamWaitEvent(st, ev_chunk_in_[c], 0));
        }
        const CUtensorMap tmc = make_tmap(hq_.as<uint8_t>() + r0 * qrow, hsk_, hl_, r1 - r0, B_);
        launch_plan(t == 0 ? ring_first_[c] : ring_last_[c], tmc, kbuf(t), vbuf(t), ho_.as<uint8_t>() + r0 * qrow,
                    hlse_.as<float>() + r0 * hl_, r1 - r0, Tr_, st, nullptr, r0);
        if (t == R_ - 1) {
          USPB_CHECK(cudaEventRecord(ev_chunk_out_[c], st));
          USPB_CHECK(cudaStreamWaitEvent(d2h_stream_, ev_chunk_out_[c], 0));
          USPB_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(o) + r0 * qrow, ho_.as<uint8_t>() + r0 * qrow,
                                     (r1 - r0) * qrow, cudaMemcpyDeviceToHost, d2h_stream_));
          USPB_CHECK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(lse) + r0 * lrow, hlse_.as<uint8_t>() + r0 * lrow,
                                     (r1 - r0) * lrow, cudaMemcpyDeviceToHost, d2h_stream_));
        }
      }
    }
    record_a2a(3, q_part_);
    USPB_CHECK(cudaEventRecord(ev_drained_, d2h_stream_));
    USPB_CHECK(cudaStreamWaitEvent(st, ev_drained_, 0));
    have_fwd_ = true;
    fwd_ledger_size_ = ledger_.size();
  }

  // Row chunks of the pure-ring host path (4 chunks of whole tiles) and the
  // step-0 (kFirst) / last-step (kLast) plans restricted to each.
  void ensure_ring_chunk_plans() {
    if (!ring_first_.empty()) return;
    const int64_t c = std::max<int64_t>((Tr_ / 4 + kTileM - 1) / kTileM * kTileM, kTileM);
    ring_bounds_ = {0};
    for (int64_t r = c; r < Tr_; r += c) ring_bounds_.push_back(r);
    ring_bounds_.push_back(Tr_);
    const auto my_pos = head_positions(shape_, cfg_.rank);
    const auto k_first = head_positions(shape_, shape_.mesh.rank_of(u_, ring_source(r_, 0, R_)));
    const auto k_last = head_positions(shape_, shape_.mesh.rank_of(u_, ring_source(r_, R_ - 1, R_)));
    for (size_t i = 0; i + 1 < ring_bounds_.size(); ++i) {
      const std::vector<int64_t> qp(my_pos.begin() + ring_bounds_[i], my_pos.begin() + ring_bounds_[i + 1]);
      DevStep f, l;
      upload_plan(f, plan_step(qp, k_first, shape_.causal, B_, tiling_.head_units, true, tiling_.units_per_kv,
                               tiling_.rows_per_unit));
      f.mode = EpiMode::kFirst;
      upload_plan(l, plan_step(qp, k_last, shape_.causal, B_, tiling_.head_units, true, tiling_.units_per_kv,
                               tiling_.rows_per_unit));
      l.mode = EpiMode::kLast;
      ring_first_.push_back(std::move(f));
      ring_last_.push_back(std::move(l));
    }
    const unsigned fl = dev_env("USP_HOST_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
    USPB_CHECK(cudaEventCreateWithFlags(&ev_kv_, fl));
    while (ev_chunk_in_.size() < ring_first_.size()) {
      cudaEvent_t a, e;
      USPB_CHECK(cudaEventCreateWithFlags(&a, fl));
      USPB_CHECK(cudaEventCreateWithFlags(&e, fl));
      ev_chunk_in_.push_back(a);
      ev_chunk_out_.push_back(e);
    }
  }

  // Chunk boundaries (whole 128-row tiles). Causal: row p's attention grows
  // with p but its upload does not, so early chunks are compute-light and the
  // pipeline would wait on PCIe. The chunks therefore grow with the work that
  // hides them: each next chunk is as large as the previous chunk's attention
  // can cover at ~50 GB/s H2D and ~1.2 PFLOP/s (clamped to [1K rows, L/8]),
  // and the last 8K rows form their own chunk so the final, exposed O
  // download is short (measured timeline: tools/host_trace.py). Non-causal:
  // 8 equal chunks. USP_HOST_CHUNKS=n forces n equal chunks; sequences of
  // 8K rows or fewer are a single chunk (plain copies around fwd()).
  std::vector<int64_t> chunk_bounds() const {
    static const int forced = [] {
      const char* e = dev_env("USP_HOST_CHUNKS");
      return e ? std::max(1, std::atoi(e)) : 0;
    }();
    auto tiles = [](int64_t r) { return (r + kTileM - 1) / kTileM * kTileM; };
    std::vector<int64_t> b{0};
    if (Tr_ <= 8192) {
      b.push_back(Tr_);
      return b;
    }
    if (forced || !shape_.causal) {
      const int n = forced ? forced : 8;
      const int64_t c = std::max<int64_t>(tiles((Tr_ + n - 1) / n), 4096);
      for (int64_t r = c; r < Tr_; r += c) b.push_back(r);
      b.push_back(Tr_);
      return b;
    }
    const double up_s_per_row = double((H_ + 2 * KV_) * hs_ * 2) / 50e9;
    const double att_s_per_pair = 4.0 * hl_ * hs_ / 1.2e15;
    const int64_t big = std::max<int64_t>(tiles(Tr_ / 8), 1024);
    static const int64_t tail_rows = [] {  // development knob (default 8192 rows)
      const char* e = dev_env("USP_HOST_TAIL");
      return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(8192);
    }();
    const int64_t tail = Tr_ > 4 * 8192 ? tiles(tail_rows) : 0;
    int64_t prev = 0, r = 1024;
    while (r < Tr_ - tail) {
      b.push_back(r);
      const double covered = att_s_per_pair * 0.5 * (double(r) * r - double(prev) * prev);
      const int64_t next = std::clamp<int64_t>(tiles(int64_t(covered / up_s_per_row)) / kTileM * kTileM, 1024, big);
      prev = r;
      r += next;
    }
    if (tail && b.back() != Tr_ - tail) b.push_back(Tr_ - tail);
    b.push_back(Tr_);
    return b;
  }

  void ensure_chunk_plans(const std::vector<int64_t>& bounds) {
    if (!chunk_steps_.empty() && chunk_bounds_ == bounds) return;
    chunk_steps_.clear();
    for (auto e : ev_chunk_in_) cudaEventDestroy(e);
    for (auto e : ev_chunk_out_) cudaEventDestroy(e);
    ev_chunk_in_.clear();
    ev_chunk_out_.clear();
    chunk_bounds_ = bounds;
    const auto pos = head_positions(shape_, cfg_.rank);
    for (size_t i = 0; i < pos.size(); ++i)
      if (pos[i] != int64_t(i)) throw Error(ErrorCode::kInternal, "chunked forward needs identity positions");
    for (size_t c = 0; c + 1 < bounds.size(); ++c) {
      const int64_t r0 = bounds[c], r1 = bounds[c + 1];
      const std::vector<int64_t> qp(pos.begin() + r0, pos.begin() + r1);
      const std::vector<int64_t> kp(pos.begin(), pos.begin() + (shape_.causal ? r1 : Tr_));
      DevStep d;
      upload_plan(d, plan_step(qp, kp, shape_.causal, B_, tiling_.head_units, true, tiling_.units_per_kv,
                               tiling_.rows_per_unit));
      d.mode = EpiMode::kSingle;
      chunk_steps_.push_back(std::move(d));
      cudaEvent_t a, e;
      const unsigned fl = dev_env("USP_HOST_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
      USPB_CHECK(cudaEventCreateWithFlags(&a, fl));
      USPB_CHECK(cudaEventCreateWithFlags(&e, fl));
      ev_chunk_in_.push_back(a);
      ev_chunk_out_.push_back(e);
    }
  }

  // ---------------------------------------------------------------- backward
  // usp_attention_backward (usp_attention.cpp:68-89): dO all-to-all in,
  // ring backward over the saved head-sharded Q, K, V, O, LSE, then the dQ,
  // dK, dV all-to-alls out. The ring (ring_attention.cpp:79-155): step t runs
  // the dK/dV kernel on K/V block src=(r-t) mod R and the dQ kernel; the
  // rank's own block contribution (t=0) stays home, the partial of the block
  // being visited circulates: created at t=1, accumulated (blk + acc) at
  // t>=2, shifted after every t>=1, so after R-1 hops each rank holds the sum
  // of the other ranks' contributions to its own block; dK = acc + own.
  void bwd(const void* q, const void* k, const void* v, const void* o, const float* lse,
           const void* dout, void* dq, void* dk, void* dv, cudaStream_t st) {
    USPB_CHECK(cudaSetDevice(cfg_.device));
    for (const void* ptr : {q, k, v, o, static_cast<const void*>(lse), dout, static_cast<const void*>(dq),
                            static_cast<const void*>(dk), static_cast<const void*>(dv)})
      if (!ptr || reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
        throw_invalid("q, k, v, o, lse, dout, dq, dk, dv must be non-null 16-byte aligned device pointers");
    if (!have_fwd_) throw_invalid("logsumexp does not match the forward shard (missing forward artifacts?)");
    ensure_bwd_buffers();
    launches_ = 0;
    ledger_.resize(fwd_ledger_size_);  // drop a previous backward's events, keep the forward's
    const bool reshape = U_ > 1 || hs_ != hsk_;
    const void* qh = reshape ? q_h_.p : q;
    const void* kh = reshape ? kv0_.p : k;
    const void* vh = reshape ? static_cast<const void*>(kv0_.as<uint8_t>() + kv_bytes_) : v;
    const void* oh = reshape ? o_h_.p : o;
    const void* doh = dout;
    // -- 1. dO: sequence-sharded -> head-sharded (all_to_all_4d(.,2,1), :79)
    if (U_ > 1) {
      uint8_t* sq = send_.as<uint8_t>();
      pack_heads(dout, sq, H_, hl_, st);
      uint8_t* rq = B_ > 1 ? recv_.as<uint8_t>() : nullptr;
      std::vector<std::vector<A2APart>> parts(1, std::vector<A2APart>(U_));
      for (int p = 0; p < U_; ++p)
        parts[0][p] = {sq + p * q_part_, rq ? rq + p * q_part_ : do_h_.as<uint8_t>() + p * q_part_};
      tr_->all_to_all(*groups_, parts, {q_part_}, st);
      if (B_ > 1) gather_seq(rq, do_h_.p, hl_, st);
      doh = do_h_.p;
    } else if (reshape) {
      pad_rows(dout, do_h_.p, B_ * T_ * H_, st);
      doh = do_h_.p;
    }
    record_a2a(4, q_part_);
    // delta = rowsum(dO * O) (output_dot_rows, attention.cpp:266-280)
    const bool fused = use_fused_bwd();
    const float inv_scale = static_cast<float>(1.0 / std::sqrt(double(hs_)));
    USPB_CHECK(launch_bwd_delta(oh, doh, delta_.as<float>(), B_, Tr_, hl_, hsk_, lse,
                                (fused ? bwd_steps_[0].fused : bwd_steps_[0].dkdv).q_pos.as<int32_t>(),
                                qvec_.as<float>(), fused ? inv_scale : 1.f, st));
    ++launches_;

    // -- 2. ring backward
    const CUtensorMap tm_q = make_tmap(qh, hsk_, hl_, Tr_, B_);
    const CUtensorMap tm_do = make_tmap(doh, hsk_, hl_, Tr_, B_);
    auto kbuf = [&](int t) -> const void* { return t == 0 ? kh : kv_ring_[(t - 1) & 1].p; };
    auto vbuf = [&](int t) -> const void* {
      return t == 0 ? vh : static_cast<const void*>(kv_ring_[(t - 1) & 1].as<uint8_t>() + kv_bytes_);
    };
    const size_t gkv = size_t(B_) * Tr_ * kvl_ * hsk_;  // fp32 elements of one of dK / dV
    float* own = own_dkv_.as<float>();
    int cur = 0;  // acc_dkv_[cur] holds the circulating partial
    if (fused) {
      ring_bwd_fused(tm_q, tm_do, kbuf, vbuf, lse, gkv, cur, st);
    } else {
    for (int t = 0; t < R_; ++t) {
      if (t + 1 < R_) {
        USPB_CHECK(cudaEventRecord(ev_pre_[t], st));
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_pre_[t], 0));
        record_shift(1);
        record_shift(2);
        tr_->ring_shift(*groups_, {kbuf(t), vbuf(t)},
                        {const_cast<void*>(kbuf(t + 1)), const_cast<void*>(vbuf(t + 1))},
                        {kv_bytes_, kv_bytes_}, comm_stream_);
        USPB_CHECK(cudaEventRecord(ev_recv_[t], comm_stream_));
      }
      if (t > 0) USPB_CHECK(cudaStreamWaitEvent(st, ev_recv_[t - 1], 0));  // K/V(t) (and acc) landed
      const BwdStep& bs = bwd_steps_[t];
      float* tgt = t == 0 ? own : acc_dkv_[cur].as<float>();
      launch_bwd_kernel(0, bs.dkdv, tm_q, tm_do, kbuf(t), vbuf(t), lse, nullptr, tgt, tgt + gkv,
                        t >= 2, st);
      if (t >= 1) {
        // ship the partial to the next ring rank (overlaps the dQ kernel)
        USPB_CHECK(cudaEventRecord(ev_acc_[t], st));
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_acc_[t], 0));
        record_shift(6, 4);
        record_shift(7, 4);
        float* a = acc_dkv_[cur].as<float>();
        float* b = acc_dkv_[cur ^ 1].as<float>();
        tr_->ring_shift(*groups_, {a, a + gkv}, {b, b + gkv}, {gkv * 4, gkv * 4}, comm_stream_);
        cur ^= 1;
        // the next step's kernels wait on ev_recv_[t], recorded after this shift
        if (t + 1 < R_) {
          USPB_CHECK(cudaEventRecord(ev_recv_[t], comm_stream_));
        } else {
          USPB_CHECK(cudaEventRecord(ev_acc_[0], comm_stream_));
        }
      }
      launch_bwd_kernel(1, bs.dq, tm_q, tm_do, kbuf(t), vbuf(t), lse, dq_acc_.as<float>(), nullptr,
                        nullptr, t > 0, st);
    }
    if (R_ > 1) USPB_CHECK(cudaStreamWaitEvent(st, ev_acc_[0], 0));
    }

    // -- 3. casts (+ dK = acc + own) and the dQ, dK, dV all-to-alls out
    const float* acc = R_ > 1 ? acc_dkv_[cur].as<float>() : nullptr;
    const float* dk_a = R_ > 1 ? acc : own;
    const float* dk_b = R_ > 1 ? own : nullptr;
    const float* dv_a = R_ > 1 ? acc + gkv : own + gkv;
    const float* dv_b = R_ > 1 ? own + gkv : nullptr;
    if (U_ == 1) {
      cast(dq_acc_.as<float>(), nullptr, dq, B_ * T_ * H_, st);
      cast(dk_a, dk_b, dk, B_ * T_ * KV_, st);
      cast(dv_a, dv_b, dv, B_ * T_ * KV_, st);
      record_a2a(5, q_part_);
      record_a2a(6, kv_part_);
      record_a2a(7, kv_part_);
      return;
    }
    // head-sharded bf16 gradients -> [peer][b][T][local] -> a2a -> (b, T, heads, hs)
    uint8_t* gq = grad_h_.as<uint8_t>();
    uint8_t* gk = gq + U_ * q_part_;
    uint8_t* gv = gk + U_ * kv_part_;
    const int64_t qrows = B_ * Tr_ * hl_, kvrows = B_ * Tr_ * kvl_;
    USPB_CHECK(launch_cast_rows(dq_acc_.as<float>(), nullptr, gq, qrows, hsk_, hsk_, st));
    USPB_CHECK(launch_cast_rows(dk_a, dk_b, gk, kvrows, hsk_, hsk_, st));
    USPB_CHECK(launch_cast_rows(dv_a, dv_b, gv, kvrows, hsk_, hsk_, st));
    launches_ += 3;
    uint8_t* sq = gq;
    uint8_t* sk = gk;
    uint8_t* sv = gv;
    if (B_ > 1) {
      sq = send_.as<uint8_t>();
      sk = sq + U_ * q_part_;
      sv = sk + U_ * kv_part_;
      split_seq(gq, sq, st, hl_);
      split_seq(gk, sk, st, kvl_);
      split_seq(gv, sv, st, kvl_);
    }
    uint8_t* rq = grad_recv_.as<uint8_t>();
    uint8_t* rk = rq + U_ * q_part_;
    uint8_t* rv = rk + U_ * kv_part_;
    std::vector<std::vector<A2APart>> parts(3, std::vector<A2APart>(U_));
    for (int p = 0; p < U_; ++p) {
      parts[0][p] = {sq + p * q_part_, rq + p * q_part_};
      parts[1][p] = {sk + p * kv_part_, rk + p * kv_part_};
      parts[2][p] = {sv + p * kv_part_, rv + p * kv_part_};
    }
    tr_->all_to_all(*groups_, parts, {q_part_, kv_part_, kv_part_}, st);
    record_a2a(5, q_part_);
    record_a2a(6, kv_part_);
    record_a2a(7, kv_part_);
    batch_begin();
    unpack_heads(rq, dq, st, H_, hl_);
    unpack_heads(rk, dk, st, KV_, kvl_);
    unpack_heads(rv, dv, st, KV_, kvl_);
    batch_flush(st);
  }

  double rank_flops() const {
    double pairs = 0;
    for (const auto& s : steps_) pairs += double(s.host.visible_pairs);
    return 4.0 * double(B_) * hl_ * hs_ * pairs;
  }

 private:
  // Row permutations go through the TMA bulk-copy kernel; between
  // batch_begin() and batch_flush() they are collected and launched as ONE
  // kernel (the Q, K, V packs; every peer part of the direct exchange).
  void permute(const RowPermute& rp, cudaStream_t st) {
    if (batching_) {
      batch_.push_back(rp);
      return;
    }
    int n = 0;
    USPB_CHECK(launch_row_permute_multi(&rp, 1, num_sms_, st, &n));
    launches_ += n;
  }
  void batch_begin() {
    batching_ = true;
    batch_.clear();
  }
  void batch_flush(cudaStream_t st) {
    batching_ = false;
    if (batch_.empty()) return;
    int n = 0;
    USPB_CHECK(launch_row_permute_multi(batch_.data(), static_cast<int>(batch_.size()), num_sms_, st, &n));
    launches_ += n;
    batch_.clear();
  }
  bool batching_ = false;
  std::vector<RowPermute> batch_;
  // (b, T, heads, hs) -> [peer][b][T][heads/U][hsk]
  // (bs 1: rows [r0, r1) of every part only, r1 = 0 meaning all T rows)
  void pack_heads(const void* src, void* dst, int heads, int local, cudaStream_t st, int64_t r0 = 0,
                  int64_t r1 = 0) {
    if (r1 == 0) r1 = T_;
    RowPermute rp;
    rp.src = static_cast<const uint8_t*>(src) + size_t(r0) * heads * hs_ * 2;
    rp.dst = static_cast<uint8_t*>(dst) + size_t(r0) * local * hsk_ * 2;
    rp.dims[0] = U_;
    rp.dims[1] = B_;
    rp.dims[2] = r1 - r0;
    rp.dims[3] = local;
    rp.src_stride[0] = local;
    rp.src_stride[1] = T_ * heads;
    rp.src_stride[2] = heads;
    rp.src_stride[3] = 1;
    rp.dst_stride[0] = B_ * T_ * local;
    rp.dst_stride[1] = T_ * local;
    rp.dst_stride[2] = local;
    rp.dst_stride[3] = 1;
    rp.hs_src = hs_;
    rp.hs_dst = hsk_;
    permute(rp, st);
  }
  // bs == 1: Ulysses part m of (T, heads, hs) -> dst (T, local, hsk) rows
  void pack_part(const void* src, void* dst, int heads, int local, int m, cudaStream_t st) {
    RowPermute rp;
    rp.src = static_cast<const uint8_t*>(src) + size_t(m) * local * hs_ * 2;
    rp.dst = dst;
    rp.dims[2] = T_;
    rp.dims[3] = local;
    rp.src_stride[2] = heads;
    rp.src_stride[3] = 1;
    rp.dst_stride[2] = local;
    rp.dst_stride[3] = 1;
    rp.hs_src = hs_;
    rp.hs_dst = hsk_;
    permute(rp, st);
  }
  // [src][b][T][local] -> (b, U*T, local)   (bs > 1 receive placement)
  void gather_seq(const void* src, void* dst, int local, cudaStream_t st) {
    RowPermute rp;
    rp.src = src;
    rp.dst = dst;
    rp.dims[0] = U_;
    rp.dims[1] = B_;
    rp.dims[2] = T_;
    rp.dims[3] = local;
    rp.src_stride[0] = B_ * T_ * local;
    rp.src_stride[1] = T_ * local;
    rp.src_stride[2] = local;
    rp.src_stride[3] = 1;
    rp.dst_stride[0] = T_ * local;
    rp.dst_stride[1] = Tr_ * local;
    rp.dst_stride[2] = local;
    rp.dst_stride[3] = 1;
    rp.hs_src = rp.hs_dst = hsk_;
    permute(rp, st);
  }
  // (b, U*T, local) -> [dst][b][T][local]   (bs > 1 send staging for O)
  void split_seq(const void* src, void* dst, cudaStream_t st, int local = 0) {
    if (!local) local = hl_;
    RowPermute rp;
    rp.src = src;
    rp.dst = dst;
    rp.dims[0] = U_;
    rp.dims[1] = B_;
    rp.dims[2] = T_;
    rp.dims[3] = local;
    rp.src_stride[0] = T_ * local;
    rp.src_stride[1] = Tr_ * local;
    rp.src_stride[2] = local;
    rp.src_stride[3] = 1;
    rp.dst_stride[0] = B_ * T_ * local;
    rp.dst_stride[1] = T_ * local;
    rp.dst_stride[2] = local;
    rp.dst_stride[3] = 1;
    rp.hs_src = rp.hs_dst = hsk_;
    permute(rp, st);
  }
  // [src][b][T][local][hsk] -> (b, T, heads, hs), heads [src*local, (src+1)*local)
  void unpack_heads(const void* src, void* dst, cudaStream_t st, int heads = 0, int local = 0, int64_t r0 = 0,
                    int64_t r1 = 0) {
    if (!heads) heads = H_;
    if (!local) local = hl_;
    if (r1 == 0) r1 = T_;
    RowPermute rp;
    rp.src = static_cast<const uint8_t*>(src) + size_t(r0) * local * hsk_ * 2;
    rp.dst = static_cast<uint8_t*>(dst) + size_t(r0) * heads * hs_ * 2;
    rp.dims[0] = U_;
    rp.dims[1] = B_;
    rp.dims[2] = r1 - r0;
    rp.dims[3] = local;
    rp.src_stride[0] = B_ * T_ * local;
    rp.src_stride[1] = T_ * local;
    rp.src_stride[2] = local;
    rp.src_stride[3] = 1;
    rp.dst_stride[0] = local;
    rp.dst_stride[1] = T_ * heads;
    rp.dst_stride[2] = heads;
    rp.dst_stride[3] = 1;
    rp.hs_src = hsk_;
    rp.hs_dst = hs_;
    permute(rp, st);
  }
  void pad_rows(const void* src, void* dst, int64_t rows, cudaStream_t st) {
    RowPermute rp;
    rp.src = src;
    rp.dst = dst;
    rp.dims[3] = rows;
    rp.src_stride[3] = rp.dst_stride[3] = 1;
    rp.hs_src = hs_;
    rp.hs_dst = hsk_;
    permute(rp, st);
  }

  void cast(const float* a, const float* b, void* dst, int64_t rows, cudaStream_t st) {
    USPB_CHECK(launch_cast_rows(a, b, dst, rows, hsk_, hs_, st));
    ++launches_;
  }

  // Ring backward with the fused kernel (ring_attention.cpp:79-155): step t
  // runs ONE kernel on K/V block src = (r - t) mod R that writes this step's
  // dK/dV block and reduces its dQ contribution into dq_acc_ (zeroed first).
  // The circulating partial is formed as in the reference: t = 0 keeps the
  // own block, t = 1 starts the partial, t >= 2 adds the block into the
  // received partial (add_into, :129-134) — the kernel writes the block to a
  // scratch buffer so it does not wait for the partial's shift, only the
  // small fp32 add does. Shifts: K/V ahead of the kernel (as the forward),
  // the partial after the add; both on comm_stream_, overlapping the next
  // step's kernel.
  template <class KB, class VB>
  void ring_bwd_fused(const CUtensorMap& tm_q, const CUtensorMap& tm_do, KB kbuf, VB vbuf, const float* lse,
                      size_t gkv, int& cur, cudaStream_t st) {
    USPB_CHECK(cudaMemsetAsync(dq_acc_.p, 0, dq_acc_.bytes, st));
    float* own = own_dkv_.as<float>();
    for (int t = 0; t < R_; ++t) {
      if (t + 1 < R_) {
        USPB_CHECK(cudaEventRecord(ev_pre_[t], st));  // kernel t-1 done with buf(t+1)
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_pre_[t], 0));
        record_shift(1);
        record_shift(2);
        tr_->ring_shift(*groups_, {kbuf(t), vbuf(t)},
                        {const_cast<void*>(kbuf(t + 1)), const_cast<void*>(vbuf(t + 1))},
                        {kv_bytes_, kv_bytes_}, comm_stream_);
        USPB_CHECK(cudaEventRecord(ev_recv_[t], comm_stream_));
      }
      if (t > 0) USPB_CHECK(cudaStreamWaitEvent(st, ev_recv_[t - 1], 0));  // K/V(t) landed
      float* tgt = t == 0 ? own : (t == 1 ? acc_dkv_[cur].as<float>() : blk_dkv_.as<float>());
      launch_bwd_kernel(2, bwd_steps_[t].fused, tm_q, tm_do, kbuf(t), vbuf(t), lse, dq_acc_.as<float>(), tgt,
                        tgt + gkv, false, st);
      if (t >= 1) {
        float* a = acc_dkv_[cur].as<float>();
        if (t >= 2) {  // the partial shifted after step t-1 has landed: partial = block + partial
          USPB_CHECK(cudaStreamWaitEvent(st, ev_acc_[0], 0));
          USPB_CHECK(launch_add_f32(blk_dkv_.as<float>(), a, static_cast<int64_t>(2 * gkv), st));
          ++launches_;
        }
        USPB_CHECK(cudaEventRecord(ev_acc_[t], st));
        USPB_CHECK(cudaStreamWaitEvent(comm_stream_, ev_acc_[t], 0));
        record_shift(6, 4);
        record_shift(7, 4);
        float* b = acc_dkv_[cur ^ 1].as<float>();
        tr_->ring_shift(*groups_, {a, a + gkv}, {b, b + gkv}, {gkv * 4, gkv * 4}, comm_stream_);
        cur ^= 1;
        USPB_CHECK(cudaEventRecord(ev_acc_[0], comm_stream_));
      }
    }
    if (R_ > 1) USPB_CHECK(cudaStreamWaitEvent(st, ev_acc_[0], 0));
  }

  struct BwdStep {
    DevStep dq, dkdv;  // two-kernel (deterministic) backward
    DevStep fused;     // one-kernel backward: dK/dV units over single key tiles
  };
  // The fused backward (one kernel per ring step, dQ reduced in fp32 by
  // TMA) is the default; usp_engine_set_deterministic
  // selects the two-kernel path, whose dQ is accumulated in a fixed order and
  // is bitwise reproducible.
  bool use_fused_bwd() const { return !deterministic_; }  // kernel head sizes 64 and 128
  static void upload_plan(DevStep& d, StepPlan&& h) {
    d.host = std::move(h);
    d.q_pos = upload(d.host.q_pos);
    d.k_pos = upload(d.host.k_pos);
    d.tile_off = upload(d.host.tile_off);
    d.tile_list = upload(d.host.tile_list);
    d.units = upload(d.host.units);
  }

  void ensure_bwd_buffers() {
    const bool fused = use_fused_bwd();
    if (!bwd_steps_.empty() && bwd_fused_built_ == fused) return;
    const size_t kv_elems = size_t(B_) * Tr_ * kvl_ * hsk_;
    if (fused && R_ > 2 && !blk_dkv_.p) blk_dkv_ = DevBuf(2 * kv_elems * sizeof(float));
    if (!bwd_steps_.empty()) {  // mode switch: rebuild the plans only
      bwd_steps_.clear();
      build_bwd_plans(fused);
      return;
    }
    const bool reshape = U_ > 1 || hs_ != hsk_;
    const size_t q_heads = size_t(B_) * Tr_ * hl_ * hsk_;
    const size_t kv_heads = size_t(B_) * Tr_ * kvl_ * hsk_;
    if (reshape) do_h_ = DevBuf(q_heads * 2);
    delta_ = DevBuf(size_t(B_) * Tr_ * hl_ * sizeof(float));
    qvec_ = DevBuf(size_t(B_) * hl_ * ((Tr_ + kTileM - 1) / kTileM) * 384 * sizeof(float));
    dq_acc_ = DevBuf(q_heads * sizeof(float));
    own_dkv_ = DevBuf(2 * kv_heads * sizeof(float));
    if (R_ > 1) {
      acc_dkv_[0] = DevBuf(2 * kv_heads * sizeof(float));
      acc_dkv_[1] = DevBuf(2 * kv_heads * sizeof(float));
      for (int t = 0; t < R_; ++t) {
        cudaEvent_t a;
        USPB_CHECK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        ev_acc_.push_back(a);
      }
    }
    if (U_ > 1) {
      grad_h_ = DevBuf(U_ * (q_part_ + 2 * kv_part_));
      grad_recv_ = DevBuf(U_ * (q_part_ + 2 * kv_part_));
    }
    build_bwd_plans(fused);
  }

  void build_bwd_plans(bool fused) {
    bwd_fused_built_ = fused;
    const int group = hl_ / kvl_;
    static const bool bwd_cluster_env = [] {
      const char* e = dev_env("USP_BWD_CLUSTER");
      return !e || std::atoi(e) != 0;
    }();
    bwd_cluster_ = bwd_cluster_env && hsk_ == 128 && group % 2 == 0;
    static const bool dkdv_cluster_env = [] {
      const char* e = dev_env("USP_BWD_DKDV_CLUSTER");
      return !e || std::atoi(e) != 0;
    }();
    dkdv_cluster_ = dkdv_cluster_env && hsk_ == 128;
    const auto my_pos = head_positions(shape_, cfg_.rank);
    for (int t = 0; t < R_; ++t) {
      const int src = ring_source(r_, t, R_);
      const auto k_pos = head_positions(shape_, shape_.mesh.rank_of(u_, src));
      BwdStep bs;
      // dQ: t = 0 writes every row (empties included), later steps accumulate
      StepPlan fq = plan_step(my_pos, k_pos, shape_.causal, B_, hl_, t == 0, group);
      if (fused) {  // dK/dV units write every key row at every step (fresh block each time)
        upload_plan(bs.fused, transpose_plan(fq, B_, kvl_, true));
        bwd_steps_.push_back(std::move(bs));
        continue;
      }
      // dK/dV: t = 0 (own) and t = 1 (new partial) write every key row
      // (over key-tile pairs when 2-CTA clusters share the Q / dO tiles)
      upload_plan(bs.dkdv, dkdv_cluster_ ? transpose_plan_pairs(fq, B_, kvl_, t <= 1)
                                         : transpose_plan(fq, B_, kvl_, t <= 1));
      if (bwd_cluster_)  // dQ over head pairs (2-CTA clusters sharing K/V by multicast)
        upload_plan(bs.dq, plan_step(my_pos, k_pos, shape_.causal, B_, hl_ / 2, t == 0, group / 2));
      else
        upload_plan(bs.dq, std::move(fq));
      bwd_steps_.push_back(std::move(bs));
    }
  }

  // kind: 0 dK/dV kernel, 1 dQ kernel, 2 fused kernel
  void launch_bwd_kernel(int kind, const DevStep& s, const CUtensorMap& tm_q, const CUtensorMap& tm_do,
                         const void* kb, const void* vb, const float* lse, float* dq, float* dk, float* dv,
                         bool accumulate, cudaStream_t st) {
    if (s.host.units.empty()) return;
    BwdParams p;
    std::memset(&p, 0, sizeof(p));
    p.tm_q = tm_q;
    p.tm_do = tm_do;
    p.tm_k = make_tmap(kb, hsk_, kvl_, Tr_, B_);
    p.tm_v = make_tmap(vb, hsk_, kvl_, Tr_, B_);
    p.lse = lse;
    p.delta = delta_.as<float>();
    p.qvec = qvec_.as<float>();
    p.n_q_tiles = static_cast<int>((Tr_ + kTileM - 1) / kTileM);
    p.dq = dq;
    p.dk = dk;
    p.dv = dv;
    if (kind == 2) p.tm_dq = make_tmap_f32(dq, hsk_, hl_, Tr_, B_);
    p.units = s.units.as<uint32_t>();
    p.tile_off = s.tile_off.as<int32_t>();
    p.tile_list = s.tile_list.as<int32_t>();
    p.q_pos = s.q_pos.as<int32_t>();
    p.k_pos = s.k_pos.as<int32_t>();
    p.sched = sched_.as<int>() + 4 * (kind + 1);
    p.num_units = static_cast<int>(s.host.units.size());
    p.batch = static_cast<int>(B_);
    p.q_len = static_cast<int>(Tr_);
    p.k_len = static_cast<int>(Tr_);
    p.heads = hl_;
    p.kv_heads = kvl_;
    p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(double(hs_)));
    p.inv_scale = static_cast<float>(1.0 / std::sqrt(double(hs_)));
    p.accumulate = accumulate ? 1 : 0;
    p.cluster = kind == 2 ? 0 : ((kind == 1 ? bwd_cluster_ : dkdv_cluster_) ? 1 : 0);
    static const char* bwd_trace = dev_env("USP_BWD_TRACE");  // development timeline
    if (bwd_trace && std::string(bwd_trace) == (kind == 2 ? "fused" : kind == 1 ? "dq" : "dkdv")) {
      if (!trace_buf_.p) trace_buf_ = DevBuf(sizeof(unsigned long long) * kTraceTiles * kTraceEvents);
      USPB_CHECK(cudaMemsetAsync(trace_buf_.p, 0, trace_buf_.bytes, st));
      p.trace = trace_buf_.as<unsigned long long>();
    }
    const int reserve = reserved_sms_;
    const int slots = std::max(1, num_sms_ - reserve);
    const int grid = p.cluster ? std::max(2, std::min(2 * p.num_units, slots) & ~1) : std::min(p.num_units, slots);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing_) {
      e0 = timing_event(2 * timed_.size());
      e1 = timing_event(2 * timed_.size() + 1);
      USPB_CHECK(cudaEventRecord(e0, st));
    }
    USPB_CHECK(kind == 2   ? launch_bwd_fused(p, hsk_, grid, st)
               : kind == 1 ? launch_bwd_dq(p, hsk_, grid, st)
                           : launch_bwd_dkdv(p, hsk_, grid, st));
    ++launches_;
    if (timing_) {
      USPB_CHECK(cudaEventRecord(e1, st));
      timed_.push_back({e0, e1});
    }
  }

  void launch_step(int t, const CUtensorMap& tm_q, const void* kb, const void* vb, void* o_heads,
                   float* lse, cudaStream_t st, void* const* o_peer = nullptr) {
    launch_plan(steps_[t], tm_q, kb, vb, o_heads, lse, Tr_, Tr_, st, o_peer);
  }

  // One attention launch over plan s: q_len query rows (tm_q, o, lse start
  // at the plan's first row) against the first k_len rows of K/V.
  void launch_plan(const DevStep& s, const CUtensorMap& tm_q, const void* kb, const void* vb,
                   void* o_heads, float* lse, int64_t q_len, int64_t k_len, cudaStream_t st,
                   void* const* o_peer = nullptr, int64_t row0 = 0) {
    if (s.host.units.empty()) return;
    FwdParams p;
    std::memset(&p, 0, sizeof(p));
    p.tm_q = tm_q;
    p.tm_k = make_tmap(kb, hsk_, kvl_, k_len, B_);
    p.tm_v = make_tmap(vb, hsk_, kvl_, k_len, B_);
    p.o = o_heads;
    p.lse = lse;
    p.o_acc = o_acc_.p ? o_acc_.as<float>() + row0 * hl_ * hsk_ : nullptr;  // bs 1 when row0 > 0
    p.lse_acc = lse_acc_.p ? lse_acc_.as<float>() + row0 * hl_ : nullptr;
    p.units = s.units.as<uint32_t>();
    p.tile_off = s.tile_off.as<int32_t>();
    p.tile_list = s.tile_list.as<int32_t>();
    p.q_pos = s.q_pos.as<int32_t>();
    p.k_pos = s.k_pos.as<int32_t>();
    p.sched = sched_.as<int>();
    p.num_units = static_cast<int>(s.host.units.size());
    p.batch = static_cast<int>(B_);
    p.q_len = static_cast<int>(q_len);
    p.k_len = static_cast<int>(k_len);
    p.heads = hl_;
    p.kv_heads = kvl_;
    p.mode = static_cast<int>(s.mode);
    p.pair_rows = tiling_.pair_rows ? 1 : 0;
    p.cluster = cluster_mode_;
    if (cluster_mode_ == 2) p.tm_k64 = make_tmap(kb, hsk_, kvl_, k_len, B_, 64);
    if (o_peer) {
      for (int m = 0; m < U_; ++m) p.o_peer[m] = o_peer[m];
      p.o_part_rows = static_cast<int>(T_);
      p.o_me = u_;
    }
    p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(double(hs_)));
    static const int kv_hint = [] {
      const char* e = dev_env("USP_KV_HINT");
      return e ? std::atoi(e) : 0;
    }();
    p.kv_hint = kv_hint;
    static const int dbg = [] {
      const char* e = dev_env("USP_FA_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    p.debug_flags = dbg;
    p.rescale_count = count_rescale_ ? dbg_count_.as<unsigned long long>() : nullptr;
    static const bool trace = dev_env("USP_FA_TRACE") != nullptr;
    if (trace) {
      if (!trace_buf_.p) trace_buf_ = DevBuf(sizeof(unsigned long long) * kTraceTiles * kTraceEvents);
      USPB_CHECK(cudaMemsetAsync(trace_buf_.p, 0, trace_buf_.bytes, st));
      p.trace = trace_buf_.as<unsigned long long>();
    }
    const int reserve = reserved_sms_;
    const int slots = std::max(1, num_sms_ - reserve);
    // cluster mode: two CTAs (one per SM of a TPC) per unit, an even grid
    const int grid = cluster_ ? std::max(2, std::min(2 * p.num_units, slots) & ~1) : std::min(p.num_units, slots);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing_) {
      e0 = timing_event(2 * timed_.size());
      e1 = timing_event(2 * timed_.size() + 1);
      USPB_CHECK(cudaEventRecord(e0, st));
    }
    USPB_CHECK(launch_fa_fwd(p, nq_, hsk_, grid, st));
    ++launches_;
    if (timing_) {
      USPB_CHECK(cudaEventRecord(e1, st));
      timed_.push_back({e0, e1});
    }
  }

  // Per-launch CUDA-event timing of the attention kernel, recorded on the
  // stream it is launched on (for roofline accounting).
  cudaEvent_t timing_event(size_t i) {
    while (event_pool_.size() <= i) {
      cudaEvent_t e;
      USPB_CHECK(cudaEventCreate(&e));
      event_pool_.push_back(e);
    }
    return event_pool_[i];
  }

 public:
  // Per-stage timing of the forward (bench.py's breakdown): while timing is
  // on, fwd() records an event on the caller's stream after every stage
  // (pack, a2a_in, wait<t> = the exposed part of the K/V shift into step t,
  // attn<t>, a2a_out, unpack, ...); a stage's time is the gap to the previous
  // event. Comm-stream spans (shift<t>: the K/V transfer itself) are timed
  // between their own two events.
  struct StageTime {
    std::string name;
    double ms = 0;
    int count = 0;
  };
  std::vector<StageTime> stage_times() {
    std::vector<StageTime> out;
    auto add = [&](const std::string& n, float ms) {
      for (auto& x : out)
        if (x.name == n) {
          x.ms += ms;
          ++x.count;
          return;
        }
      out.push_back({n, ms, 1});
    };
    for (const auto& run : stage_runs_) {
      for (size_t i = 1; i < run.size(); ++i) {
        USPB_CHECK(cudaEventSynchronize(run[i].second));
        float ms = 0.f;
        USPB_CHECK(cudaEventElapsedTime(&ms, run[i - 1].second, run[i].second));
        add(run[i].first, ms);
      }
    }
    for (const auto& sp : side_spans_) {
      USPB_CHECK(cudaEventSynchronize(sp.end));
      float ms = 0.f;
      USPB_CHECK(cudaEventElapsedTime(&ms, sp.begin, sp.end));
      add(sp.name, ms);
    }
    stage_runs_.clear();
    side_spans_.clear();
    stage_used_ = 0;
    return out;
  }

  // Parity instrumentation: counts the forward kernel's lazy O rescales.
  void debug_counters(bool on) {
    USPB_CHECK(cudaSetDevice(cfg_.device));
    if (!dbg_count_.p) dbg_count_ = DevBuf(sizeof(unsigned long long));
    USPB_CHECK(cudaMemset(dbg_count_.p, 0, sizeof(unsigned long long)));
    count_rescale_ = on;
  }
  int64_t rescale_count() {
    if (!dbg_count_.p) return 0;
    USPB_CHECK(cudaSetDevice(cfg_.device));
    unsigned long long v = 0;
    USPB_CHECK(cudaDeviceSynchronize());
    USPB_CHECK(cudaMemcpy(&v, dbg_count_.p, sizeof(v), cudaMemcpyDeviceToHost));
    return static_cast<int64_t>(v);
  }
  void enable_timing(bool on) {
    timing_ = on;
    timed_.clear();
    stage_runs_.clear();
    side_spans_.clear();
    stage_used_ = 0;
  }
  int kernel_times(float* ms, int cap) {
    int n = 0;
    for (const auto& pr : timed_) {
      USPB_CHECK(cudaEventSynchronize(pr.second));
      float t = 0.f;
      USPB_CHECK(cudaEventElapsedTime(&t, pr.first, pr.second));
      if (n < cap) ms[n] = t;
      ++n;
    }
    timed_.clear();
    return n;
  }

 private:
  struct SideSpan {
    std::string name;
    cudaEvent_t begin, end;
  };
  std::vector<std::vector<std::pair<std::string, cudaEvent_t>>> stage_runs_;
  std::vector<SideSpan> side_spans_;
  std::vector<cudaEvent_t> stage_pool_;
  size_t stage_used_ = 0;
  cudaEvent_t stage_event() {
    if (stage_used_ == stage_pool_.size()) {
      cudaEvent_t e;
      USPB_CHECK(cudaEventCreate(&e));
      stage_pool_.push_back(e);
    }
    return stage_pool_[stage_used_++];
  }
  void stage_begin(cudaStream_t st) {
    if (!timing_) return;
    stage_runs_.emplace_back();
    stage(st, "begin");
  }
  void stage(cudaStream_t st, const std::string& name) {
    if (!timing_ || stage_runs_.empty()) return;
    cudaEvent_t e = stage_event();
    USPB_CHECK(cudaEventRecord(e, st));
    stage_runs_.back().emplace_back(name, e);
  }
  cudaEvent_t side_event(cudaStream_t st) {
    if (!timing_) return nullptr;
    cudaEvent_t e = stage_event();
    USPB_CHECK(cudaEventRecord(e, st));
    return e;
  }
  void side_span(const std::string& name, cudaEvent_t b, cudaEvent_t e) {
    if (b && e) side_spans_.push_back({name, b, e});
  }
  bool timing_ = false;
  bool count_rescale_ = false;
  DevBuf dbg_count_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed_;
  std::vector<cudaEvent_t> event_pool_;

  usp_config cfg_;
  Transport* tr_;
  std::shared_ptr<Groups> groups_;
  UspShape shape_;
  int U_ = 1, R_ = 1, u_ = 0, r_ = 0, H_ = 0, KV_ = 0, hl_ = 0, kvl_ = 0, hs_ = 0, hsk_ = 0, nq_ = 1;
  FwdTiling tiling_{};
  bool cluster_ = false;
  bool bwd_cluster_ = false;
  bool dkdv_cluster_ = false;
  bool deterministic_ = false;
  bool bwd_fused_built_ = false;
  DevBuf blk_dkv_;  // fused backward, R > 2: this step's dK/dV block before it joins the partial
  int cluster_mode_ = 0;
  int64_t B_ = 1, T_ = 0, Tr_ = 0;
  int num_sms_ = 148;
  size_t q_part_ = 0, kv_part_ = 0, kv_bytes_ = 0;
  DevBuf q_h_, kv0_, o_h_, send_, recv_, o_send_, o_recv_, o_acc_, lse_acc_;
  DevBuf kv_ring_[2];
  // backward (allocated by the first usp_attn_bwd)
  DevBuf do_h_, delta_, qvec_, dq_acc_, own_dkv_, grad_h_, grad_recv_;
  DevBuf acc_dkv_[2];
  std::vector<BwdStep> bwd_steps_;
  // usp_attn_fwd_host staging and its chunk pipeline
  DevBuf hq_, hk_, hv_, ho_, hlse_;
  std::vector<DevStep> chunk_steps_;
  std::vector<DevStep> ring_first_, ring_last_;  // pure-ring host path
  std::vector<int64_t> ring_bounds_;
  cudaEvent_t ev_kv_ = nullptr;
  std::vector<int64_t> chunk_bounds_;
  cudaStream_t h2d_stream_ = nullptr, d2h_stream_ = nullptr;
  cudaEvent_t ev_entry_ = nullptr, ev_drained_ = nullptr;
  std::vector<cudaEvent_t> ev_chunk_in_, ev_chunk_out_;
  std::vector<cudaEvent_t> ev_acc_;
  bool have_fwd_ = false;
  size_t fwd_ledger_size_ = 0;
  DevBuf sched_;  // unit tickets of the attention kernel (self-resetting)
  DevBuf trace_buf_;  // USP_FA_TRACE development stamps

 public:
  const void* trace_ptr() const { return trace_buf_.p; }

 private:
  std::vector<DevStep> steps_;
  cudaStream_t comm_stream_ = nullptr;
  std::vector<cudaEvent_t> ev_pre_, ev_recv_;
  int launches_ = 0;

 public:
  std::vector<LedgerEvent> ledger_;

 private:
  // Executed-collective records (bytes as moved; payload in logical elements).
  void record_a2a(int tensor, size_t part_bytes) {
    const double elems_phys = double(part_bytes) / 2.0;
    const int64_t payload = static_cast<int64_t>(elems_phys * U_ * hs_ / hsk_ + 0.5);
    ledger_.push_back({3, shape_.mesh.rank_of(0, r_), U_, 1, tensor, tensor, payload,
                       double(part_bytes) * (U_ - 1)});
  }
  void record_shift(int tensor, int elem_bytes = 2) {
    const int step = static_cast<int>(std::count_if(ledger_.begin(), ledger_.end(),
                                                    [](const LedgerEvent& e) { return e.kind == 4; }));
    ledger_.push_back({4, shape_.mesh.rank_of(u_, 0), R_, U_, step, tensor,
                       static_cast<int64_t>(double(kv_bytes_) / 2.0 * hs_ / hsk_ + 0.5),
                       double(kv_bytes_) / 2.0 * elem_bytes});
  }
};

}  // namespace uspb200

// =================================================================== C ABI
using namespace uspb200;

struct usp_comm {
  std::unique_ptr<Transport> impl;
};
struct usp_engine {
  std::unique_ptr<Engine> impl;
};

namespace {
thread_local std::string g_last_error;

template <class F>
usp_status guarded(F&& f) {
  try {
    f();
    return USP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return (e.code() == ErrorCode::kInvalidArgument || e.code() == ErrorCode::kConstraint)
               ? USP_INVALID_INPUT
               : USP_INTERNAL_ERROR;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of memory";
    return USP_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return USP_INTERNAL_ERROR;
  }
}

UspShape shape_of(const usp_config* cfg) {
  if (!cfg) throw_invalid("config is null");
  return Engine::to_shape(*cfg);
}
}  // namespace

extern "C" {

usp_status usp_config_validate(const usp_config* cfg) {
  return guarded([&] { shape_of(cfg).validate(); });
}

usp_status usp_zigzag_partition(int64_t seq_len, int32_t ring, int64_t* out) {
  return guarded([&] {
    const auto v = zigzag_partition(seq_len, ring);
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

usp_status usp_positions_for(const usp_config* cfg, int32_t rank, int64_t* out) {
  return guarded([&] {
    const UspShape s = shape_of(cfg);
    s.validate();
    const auto v = positions_for(s, rank);
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

usp_status usp_head_positions(const usp_config* cfg, int32_t rank, int64_t* out) {
  return guarded([&] {
    const UspShape s = shape_of(cfg);
    s.validate();
    const auto v = head_positions(s, rank);
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

usp_status usp_causal_pair_counts(const int64_t* assignment, int32_t ring, int64_t seq_len,
                                  int64_t* counts) {
  return guarded([&] {
    if (ring < 1 || seq_len % ring != 0) throw_invalid("assignment must cover 0..L-1 exactly once");
    std::vector<int64_t> flat(assignment, assignment + seq_len);
    const auto c = causal_pair_counts(flat, ring, seq_len);
    std::memcpy(counts, c.data(), c.size() * sizeof(int64_t));
  });
}

usp_status usp_schedule(const usp_config* cfg, int32_t step, usp_step_info* out) {
  return guarded([&] {
    const UspShape s = shape_of(cfg);
    s.validate();
    if (step < 0 || step >= s.mesh.ring) throw_invalid("step outside [0, ring_degree)");
    const int u = s.mesh.ulysses_coord(cfg->rank), r = s.mesh.ring_coord(cfg->rank);
    const int R = s.mesh.ring;
    const int src = ring_source(r, step, R);
    const int kvl = s.local_kv_heads();
    const FwdTiling tl = fwd_tiling(s.local_heads(), kvl, s.kernel_head_size(), s.tokens_per_ring_rank(), s.batch);
    const auto st = plan_step(head_positions(s, cfg->rank),
                              head_positions(s, s.mesh.rank_of(u, src)), s.causal, s.batch,
                              tl.head_units, R == 1 || step == 0 || step == R - 1, tl.units_per_kv,
                              tl.rows_per_unit);
    out->step = step;
    out->src_ring_coord = src;
    out->send_to_rank = s.mesh.rank_of(u, (r + 1) % R);
    out->recv_from_rank = s.mesh.rank_of(u, (r - 1 + R) % R);
    out->full_tiles = st.full_tiles;
    out->partial_tiles = st.partial_tiles;
    out->work_units = static_cast<int64_t>(st.units.size());
    out->visible_pairs = st.visible_pairs;
    out->ring_bytes_sent =
        step + 1 < R ? 2 * s.batch * s.tokens_per_ring_rank() * kvl * int64_t(s.head_size) * 2 : 0;
  });
}

usp_status usp_step_plan(const usp_config* cfg, int32_t step, int64_t sizes[2], int32_t* tile_off,
                         int32_t* tile_list) {
  return guarded([&] {
    const UspShape s = shape_of(cfg);
    s.validate();
    if (step < 0 || step >= s.mesh.ring) throw_invalid("step outside [0, ring_degree)");
    const int u = s.mesh.ulysses_coord(cfg->rank), r = s.mesh.ring_coord(cfg->rank);
    const int src = ring_source(r, step, s.mesh.ring);
    const auto st = plan_step(head_positions(s, cfg->rank), head_positions(s, s.mesh.rank_of(u, src)),
                              s.causal, s.batch, 1, true);
    sizes[0] = st.n_q_tiles;
    sizes[1] = static_cast<int64_t>(st.tile_list.size());
    if (tile_off) std::memcpy(tile_off, st.tile_off.data(), st.tile_off.size() * sizeof(int32_t));
    if (tile_list) std::memcpy(tile_list, st.tile_list.data(), st.tile_list.size() * sizeof(int32_t));
  });
}

static int32_t copy_ledger(const std::vector<LedgerEvent>& ev, usp_ledger_entry* out, int32_t cap) {
  for (size_t i = 0; i < ev.size() && static_cast<int32_t>(i) < cap && out; ++i)
    out[i] = {ev[i].kind, ev[i].group_first, ev[i].group_size, ev[i].group_stride, ev[i].step,
              ev[i].tensor, ev[i].payload_elems, ev[i].bytes_sent};
  return static_cast<int32_t>(ev.size());
}

int32_t usp_forward_ledger(const usp_config* cfg, usp_ledger_entry* out, int32_t cap) {
  int32_t n = -1;
  if (guarded([&] {
        const UspShape s = shape_of(cfg);
        s.validate();
        n = copy_ledger(forward_ledger(s, cfg->rank, 2), out, cap);
      }) != USP_OK)
    return -1;
  return n;
}

int32_t usp_backward_ledger(const usp_config* cfg, usp_ledger_entry* out, int32_t cap) {
  int32_t n = -1;
  if (guarded([&] {
        const UspShape s = shape_of(cfg);
        s.validate();
        n = copy_ledger(backward_ledger(s, cfg->rank, 2, 4), out, cap);
      }) != USP_OK)
    return -1;
  return n;
}

int32_t usp_engine_ledger(const usp_engine* engine, usp_ledger_entry* out, int32_t cap) {
  if (!engine) return -1;
  return copy_ledger(engine->impl->ledger_, out, cap);
}

usp_status usp_rank_flops(const usp_config* cfg, double* flops) {
  return guarded([&] {
    const UspShape s = shape_of(cfg);
    s.validate();
    const int u = s.mesh.ulysses_coord(cfg->rank), r = s.mesh.ring_coord(cfg->rank);
    const auto mine = head_positions(s, cfg->rank);
    double pairs = 0;
    for (int t = 0; t < s.mesh.ring; ++t)
      pairs += double(visible_pairs(
          mine, head_positions(s, s.mesh.rank_of(u, ring_source(r, t, s.mesh.ring))), s.causal));
    *flops = 4.0 * double(s.batch) * s.local_heads() * s.head_size * pairs;
  });
}

usp_status usp_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] { nccl_unique_id(out); });
}

usp_status usp_comm_create_nccl(const uint8_t unique_id[128], int32_t world_size, int32_t rank,
                                int32_t device, usp_comm** out) {
  if (!out) return USP_INVALID_INPUT;
  *out = nullptr;
  return guarded([&] {
    auto c = std::make_unique<usp_comm>();
    c->impl = make_nccl_transport(unique_id, world_size, rank, device);
    *out = c.release();
  });
}

usp_status usp_comm_create_local(int32_t world_size, usp_comm** out) {
  if (!out) return USP_INVALID_INPUT;
  *out = nullptr;
  return guarded([&] {
    auto c = std::make_unique<usp_comm>();
    c->impl = make_local_transport(world_size);
    *out = c.release();
  });
}

usp_status usp_comm_create_p2p(int32_t world_size, int32_t rank, int32_t device, usp_allgather_fn allgather,
                               void* ctx, usp_comm** out) {
  if (!out) return USP_INVALID_INPUT;
  *out = nullptr;
  return guarded([&] {
    auto c = std::make_unique<usp_comm>();
    c->impl = make_p2p_transport(world_size, rank, device, allgather, ctx);
    *out = c.release();
  });
}

void usp_comm_destroy(usp_comm* comm) { delete comm; }

usp_status usp_comm_set_timeout(usp_comm* comm, double seconds) {
  if (!comm || !(seconds > 0)) {
    g_last_error = "usp_comm_set_timeout: a comm and a positive timeout are required";
    return USP_INVALID_INPUT;
  }
  comm->impl->set_timeout(seconds);
  return USP_OK;
}

usp_status usp_comm_status(usp_comm* comm) {
  if (!comm) return USP_INVALID_INPUT;
  return guarded([&] {
    const std::string st = comm->impl->status();
    if (!st.empty()) throw Error(ErrorCode::kCommMismatch, st);
  });
}

usp_status usp_comm_debug_rendezvous(usp_comm* comm, int32_t rank, const int32_t* members, int32_t n,
                                     const char* signature) {
  if (!comm || !members || n < 1 || !signature) return USP_INVALID_INPUT;
  return guarded([&] {
    comm->impl->debug_rendezvous(std::vector<int>(members, members + n), rank, signature);
  });
}

usp_status usp_engine_create(const usp_config* cfg, usp_comm* comm, usp_engine** out) {
  if (!out) return USP_INVALID_INPUT;
  *out = nullptr;
  return guarded([&] {
    if (!cfg) throw_invalid("config is null");
    auto e = std::make_unique<usp_engine>();
    e->impl = std::make_unique<Engine>(*cfg, comm ? comm->impl.get() : nullptr);
    *out = e.release();
  });
}

usp_status usp_attn_fwd(usp_engine* engine, const void* q, const void* k, const void* v, void* o,
                        float* lse, void* stream) {
  return guarded([&] {
    if (!engine) throw_invalid("engine is null");
    engine->impl->fwd(q, k, v, o, lse, static_cast<cudaStream_t>(stream));
  });
}

usp_status usp_attn_fwd_host(usp_engine* engine, const void* q, const void* k, const void* v, void* o,
                             float* lse, void* stream) {
  return guarded([&] {
    if (!engine) throw_invalid("engine is null");
    engine->impl->fwd_host(q, k, v, o, lse, static_cast<cudaStream_t>(stream));
  });
}

usp_status usp_attn_bwd(usp_engine* engine, const void* q, const void* k, const void* v, const void* o,
                        const float* lse, const void* dout, void* dq, void* dk, void* dv, void* stream) {
  return guarded([&] {
    if (!engine) throw_invalid("engine is null");
    engine->impl->bwd(q, k, v, o, lse, dout, dq, dk, dv, static_cast<cudaStream_t>(stream));
  });
}

// Development: copies the USP_FA_TRACE stamps (kTraceEvents x kTraceTiles)
// to host memory; returns 0 when tracing is off.
extern "C" USP_API int usp_engine_trace_copy(const usp_engine* engine, unsigned long long* host) {
  if (!engine || !engine->impl->trace_ptr()) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, engine->impl->trace_ptr(), sizeof(unsigned long long) * kTraceTiles * kTraceEvents,
             cudaMemcpyDeviceToHost);
  return 1;
}

int32_t usp_engine_last_launches(const usp_engine* engine) {
  return engine ? engine->impl->last_launches() : 0;
}

void usp_engine_destroy(usp_engine* engine) { delete engine; }

usp_status usp_engine_enable_timing(usp_engine* engine, int32_t on) {
  return guarded([&] {
    if (!engine) throw_invalid("engine is null");
    engine->impl->enable_timing(on != 0);
  });
}

int32_t usp_engine_stage_times(usp_engine* engine, usp_stage_time* out, int32_t cap) {
  if (!engine) return -1;
  int32_t n = -1;
  if (guarded([&] {
        const auto st = engine->impl->stage_times();
        for (size_t i = 0; i < st.size() && static_cast<int32_t>(i) < cap && out; ++i) {
          std::memset(&out[i], 0, sizeof(out[i]));
          std::strncpy(out[i].name, st[i].name.c_str(), sizeof(out[i].name) - 1);
          out[i].ms_total = st[i].ms;
          out[i].count = st[i].count;
        }
        n = static_cast<int32_t>(st.size());
      }) != USP_OK)
    return -1;
  return n;
}

usp_status usp_engine_get_info(const usp_engine* engine, usp_engine_info* out) {
  if (!engine || !out) return USP_INVALID_INPUT;
  return guarded([&] {
    const auto i = engine->impl->info();
    out->num_sms = i.num_sms;
    out->reserved_sms = i.reserved_sms;
    out->ring_ctas = i.ring_ctas;
    out->kv_shift_bytes = i.kv_shift_bytes;
    out->ring_step_ms_est = i.step_ms_est;
    out->required_gbs = i.required_gbs;
  });
}

usp_status usp_engine_set_a2a_chunks(usp_engine* engine, int32_t chunks) {
  if (!engine) return USP_INVALID_INPUT;
  return guarded([&] { engine->impl->set_a2a_chunks(chunks); });
}

int32_t usp_engine_a2a_chunks(const usp_engine* engine) { return engine ? engine->impl->a2a_chunks() : -1; }

usp_status usp_engine_set_deterministic(usp_engine* engine, int32_t on) {
  if (!engine) return USP_INVALID_INPUT;
  return guarded([&] { engine->impl->set_deterministic(on != 0); });
}

usp_status usp_engine_set_reserved_sms(usp_engine* engine, int32_t n) {
  if (!engine) return USP_INVALID_INPUT;
  return guarded([&] { engine->impl->set_reserved_sms(n); });
}

usp_status usp_engine_debug_counters(usp_engine* engine, int32_t on) {
  if (!engine) return USP_INVALID_INPUT;
  return guarded([&] { engine->impl->debug_counters(on != 0); });
}

usp_status usp_engine_rescale_count(usp_engine* engine, int64_t* out) {
  if (!engine || !out) return USP_INVALID_INPUT;
  return guarded([&] { *out = engine->impl->rescale_count(); });
}

int32_t usp_engine_kernel_times(usp_engine* engine, float* ms, int32_t cap) {
  int32_t n = -1;
  if (guarded([&] { n = engine->impl->kernel_times(ms, cap); }) != USP_OK) return -1;
  return n;
}

usp_status usp_local_world_fwd(usp_engine* const* engines, int32_t world_size,
                               const void* const* q, const void* const* k, const void* const* v,
                               void* const* o, float* const* lse, void* const* streams) {
  std::vector<usp_status> rc(world_size, USP_OK);
  std::vector<std::string> err(world_size);
  std::vector<std::thread> th;
  for (int i = 0; i < world_size; ++i) {
    th.emplace_back([&, i] {
      rc[i] = usp_attn_fwd(engines[i], q[i], k[i], v[i], o[i], lse[i],
                           streams ? streams[i] : nullptr);
      if (rc[i] != USP_OK) err[i] = g_last_error;
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < world_size; ++i)
    if (rc[i] != USP_OK) {
      g_last_error = "rank " + std::to_string(i) + ": " + err[i];
      return rc[i];
    }
  return USP_OK;
}

usp_status usp_local_world_bwd(usp_engine* const* engines, int32_t world_size, const void* const* q,
                               const void* const* k, const void* const* v, const void* const* o,
                               const float* const* lse, const void* const* dout, void* const* dq,
                               void* const* dk, void* const* dv, void* const* streams) {
  std::vector<usp_status> rc(world_size, USP_OK);
  std::vector<std::string> err(world_size);
  std::vector<std::thread> th;
  for (int i = 0; i < world_size; ++i) {
    th.emplace_back([&, i] {
      rc[i] = usp_attn_bwd(engines[i], q[i], k[i], v[i], o[i], lse[i], dout[i], dq[i], dk[i], dv[i],
                           streams ? streams[i] : nullptr);
      if (rc[i] != USP_OK) err[i] = g_last_error;
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < world_size; ++i)
    if (rc[i] != USP_OK) {
      g_last_error = "rank " + std::to_string(i) + ": " + err[i];
      return rc[i];
    }
  return USP_OK;
}

const char* usp_last_error(void) { return g_last_error.c_str(); }

const char* usp_version(void) { return "0.1.0-b200"; }

}  // extern "C"
