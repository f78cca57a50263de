// ref_driver.cpp — extern "C" shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together with
// the reference's own hot-path sources where they lie under
// /root/reference/proj/src (nothing is copied into this repo) into
// oracle/_ref/libuspref.so. It exposes the reference's functions to the
// parity tests (tests/test_oracle.py pins the C restatement in
// oracle/usp_oracle.c against it bit for bit) and to bench.py's CPU baseline
// (--impl reference / cpu_baseline kind "reference").
//
// The simulate-style driver below mirrors src/api/commands.cpp:85-160
// (run_simulation) minus the backward pass: seeded globals, ShardSpec with
// zigzag iff causal, World::run of usp_attention on U*R rank threads, then
// place_rows back to original order.

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "common/error.hpp"
#include "common/random.hpp"
#include "numerics/attention.hpp"
#include "simcomm/mesh.hpp"
#include "simcomm/world.hpp"
#include "usp/partition.hpp"
#include "usp/usp_attention.hpp"

using namespace uspsim;
using numerics::Tensor4;

namespace {
thread_local std::string g_err;

template <class T>
Tensor4<T> make(const double* src, int64_t b, int64_t s, int64_t h, int64_t d) {
  Tensor4<T> t(b, s, h, d);
  for (size_t i = 0; i < t.data().size(); ++i) t.data()[i] = static_cast<T>(src[i]);
  return t;
}

template <class T>
void unload(const Tensor4<T>& t, double* dst) {
  for (size_t i = 0; i < t.data().size(); ++i) dst[i] = static_cast<double>(t.data()[i]);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code() == ErrorCode::kConstraint ? -2 : -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -3;
  }
}

std::string g_ledger_json;

// The World's communication ledger (simcomm/ledger.hpp) as JSON rows.
template <class Ledger>
std::string ledger_json(const Ledger& ledger) {
  std::string js = "[";
  bool first = true;
  for (const auto& e : ledger.entries()) {
    if (!first) js += ",";
    first = false;
    js += "{\"kind\":\"" + std::string(simcomm::collective_name(e.kind)) + "\",\"group\":\"" +
          e.group + "\",\"step\":" + std::to_string(e.step) +
          ",\"payload_elems\":" + std::to_string(e.payload_elems) + ",\"bytes_sent\":[";
    for (size_t i = 0; i < e.bytes_sent.size(); ++i) js += (i ? "," : "") + std::to_string(e.bytes_sent[i]);
    js += "]}";
  }
  return js + "]";
}

template <class T>
int usp_forward_impl(const double* q, const double* k, const double* v,
                     int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads,
                     int64_t hs, int ulysses, int ring, int causal,
                     double* out_global, double* lse, double* seconds) {
  return guarded([&] {
    const simcomm::ProcessMesh mesh(ulysses, ring);
    const usp::ShardSpec shard(mesh, seq, /*zigzag=*/causal != 0);
    const auto gq = make<T>(q, batch, seq, heads, hs);
    const auto gk = make<T>(k, batch, seq, kv_heads, hs);
    const auto gv = make<T>(v, batch, seq, kv_heads, hs);
    struct PerRank {
      Tensor4<T> out;
      std::vector<T> lse;
      std::vector<int64_t> positions;
    };
    // Sharding (extract_rows) happens before the clock starts, as inputs are
    // already resident on each rank in the GPU measurement too.
    std::vector<std::vector<int64_t>> pos(mesh.world_size());
    std::vector<Tensor4<T>> qs, ks, vs;
    for (int r = 0; r < mesh.world_size(); ++r) {
      pos[r] = shard.positions_for(r);
      qs.push_back(usp::extract_rows(gq, pos[r]));
      ks.push_back(usp::extract_rows(gk, pos[r]));
      vs.push_back(usp::extract_rows(gv, pos[r]));
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto world = simcomm::World::run<PerRank>(
        mesh.world_size(), [&](simcomm::RankCtx& ctx) {
          const int r = ctx.rank();
          auto fwd = usp::usp_attention(ctx, mesh, qs[r], ks[r], vs[r], pos[r],
                                        causal != 0);
          return PerRank{std::move(fwd.out), std::move(fwd.logsumexp), pos[r]};
        });
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    g_ledger_json = ledger_json(world.ledger);
    if (out_global) {
      Tensor4<T> out(batch, seq, heads, hs);
      for (const auto& pr : world.per_rank) usp::place_rows(out, pr.out, pr.positions);
      unload(out, out_global);
    }
    if (lse) {
      size_t off = 0;
      for (const auto& pr : world.per_rank)
        for (T x : pr.lse) lse[off++] = static_cast<double>(x);
    }
  });
}
template <class T>
int softmax_rows_impl(const double* q, const double* k, const double* v, int64_t batch, int64_t q_len,
                      int64_t k_len, int64_t heads, int64_t kv_heads, int64_t hs, int causal,
                      const int64_t* q_pos, const int64_t* k_pos, double* out, double* lse) {
  return guarded([&] {
    const auto tq = make<T>(q, batch, q_len, heads, hs);
    const auto tk = make<T>(k, batch, k_len, kv_heads, hs);
    const auto tv = make<T>(v, batch, k_len, kv_heads, hs);
    numerics::SoftmaxState<T> st(batch, q_len, heads, hs);
    const auto mask =
        causal ? numerics::BlockMask::causal(
                     std::span<const int64_t>(q_pos, static_cast<size_t>(q_len)),
                     std::span<const int64_t>(k_pos, static_cast<size_t>(k_len)))
               : numerics::BlockMask::none();
    st.update(tq, tk, tv, mask);
    const auto l = st.logsumexp();
    for (size_t i = 0; i < l.size(); ++i) lse[i] = static_cast<double>(l[i]);
    unload(st.finalize(), out);
  });
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Ledger of the last ref_usp_forward_* call (JSON array of entries).
const char* ref_last_ledger_json(void) { return g_ledger_json.c_str(); }

void ref_uniform_stream(uint64_t seed, double lo, double hi, int64_t n, double* out) {
  UniformSource src(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = src.next(lo, hi);
}

int ref_reference_attention_f64(const double* q, const double* k, const double* v,
                                int64_t batch, int64_t seq, int64_t heads,
                                int64_t kv_heads, int64_t hs, int causal,
                                const int64_t* positions, double* out) {
  return guarded([&] {
    const auto tq = make<double>(q, batch, seq, heads, hs);
    const auto tk = make<double>(k, batch, seq, kv_heads, hs);
    const auto tv = make<double>(v, batch, seq, kv_heads, hs);
    std::span<const int64_t> pos;
    if (positions) pos = std::span<const int64_t>(positions, static_cast<size_t>(seq));
    unload(numerics::reference_attention(tq, tk, tv, causal != 0, pos), out);
  });
}

// One SoftmaxState update of a query subset against a key block, then
// finalize() + logsumexp(); the sampled-row oracle of SURVEY §8(c) step 5.
// The _f32 variant is the reference's own fp32 path (commands.cpp:142-153
// casts the generator's doubles to float), used by bench.py's parity block
// for "bf16 GPU vs fp32 CPU".
int ref_softmax_rows_f64(const double* q, const double* k, const double* v,
                         int64_t batch, int64_t q_len, int64_t k_len, int64_t heads,
                         int64_t kv_heads, int64_t hs, int causal,
                         const int64_t* q_pos, const int64_t* k_pos, double* out,
                         double* lse) {
  return softmax_rows_impl<double>(q, k, v, batch, q_len, k_len, heads, kv_heads, hs, causal, q_pos,
                                   k_pos, out, lse);
}

int ref_softmax_rows_f32(const double* q, const double* k, const double* v,
                         int64_t batch, int64_t q_len, int64_t k_len, int64_t heads,
                         int64_t kv_heads, int64_t hs, int causal,
                         const int64_t* q_pos, const int64_t* k_pos, double* out,
                         double* lse) {
  return softmax_rows_impl<float>(q, k, v, batch, q_len, k_len, heads, kv_heads, hs, causal, q_pos,
                                  k_pos, out, lse);
}

int ref_zigzag_partition(int64_t seq_len, int ring, int64_t* out) {
  return guarded([&] {
    const auto parts = usp::zigzag_partition(seq_len, ring);
    size_t off = 0;
    for (const auto& p : parts)
      for (int64_t x : p) out[off++] = x;
  });
}

int ref_positions_for(int ulysses, int ring, int64_t seq_len, int zigzag, int rank,
                      int64_t* out) {
  return guarded([&] {
    const usp::ShardSpec spec(simcomm::ProcessMesh(ulysses, ring), seq_len, zigzag != 0);
    const auto p = spec.positions_for(rank);
    std::memcpy(out, p.data(), p.size() * sizeof(int64_t));
  });
}

int ref_causal_pair_counts(const int64_t* assignment, int ring, int64_t seq_len,
                           int64_t* counts) {
  return guarded([&] {
    std::vector<std::vector<int64_t>> a(ring);
    const int64_t per = seq_len / ring;
    for (int p = 0; p < ring; ++p) a[p].assign(assignment + p * per, assignment + (p + 1) * per);
    const auto c = usp::causal_pair_counts(a, seq_len);
    std::memcpy(counts, c.data(), c.size() * sizeof(int64_t));
  });
}

// usp_attention<double|float> forward over a U x R World (see file header).
int ref_usp_forward_f64(const double* q, const double* k, const double* v, int64_t batch,
                        int64_t seq, int64_t heads, int64_t kv_heads, int64_t hs,
                        int ulysses, int ring, int causal, double* out_global,
                        double* lse, double* seconds) {
  return usp_forward_impl<double>(q, k, v, batch, seq, heads, kv_heads, hs, ulysses,
                                  ring, causal, out_global, lse, seconds);
}

int ref_usp_forward_f32(const double* q, const double* k, const double* v, int64_t batch,
                        int64_t seq, int64_t heads, int64_t kv_heads, int64_t hs,
                        int ulysses, int ring, int causal, double* out_global,
                        double* lse, double* seconds) {
  return usp_forward_impl<float>(q, k, v, batch, seq, heads, kv_heads, hs, ulysses,
                                 ring, causal, out_global, lse, seconds);
}

}  // extern "C"

// Forward + backward (src/api/commands.cpp:108-121 minus the report):
// global dq, dk, dv in original token order.
extern "C" int ref_usp_fwd_bwd_f64(const double* q, const double* k, const double* v,
                                   const double* dout, int64_t batch, int64_t seq, int64_t heads,
                                   int64_t kv_heads, int64_t hs, int ulysses, int ring, int causal,
                                   double* dq_g, double* dk_g, double* dv_g) {
  return guarded([&] {
    const simcomm::ProcessMesh mesh(ulysses, ring);
    const usp::ShardSpec shard(mesh, seq, /*zigzag=*/causal != 0);
    const auto gq = make<double>(q, batch, seq, heads, hs);
    const auto gk = make<double>(k, batch, seq, kv_heads, hs);
    const auto gv = make<double>(v, batch, seq, kv_heads, hs);
    const auto gdo = make<double>(dout, batch, seq, heads, hs);
    struct PerRank {
      Tensor4<double> dq, dk, dv;
      std::vector<int64_t> positions;
    };
    auto world = simcomm::World::run<PerRank>(mesh.world_size(), [&](simcomm::RankCtx& ctx) {
      const auto positions = shard.positions_for(ctx.rank());
      const auto q_s = usp::extract_rows(gq, positions);
      const auto k_s = usp::extract_rows(gk, positions);
      const auto v_s = usp::extract_rows(gv, positions);
      const auto do_s = usp::extract_rows(gdo, positions);
      auto fwd = usp::usp_attention(ctx, mesh, q_s, k_s, v_s, positions, causal != 0);
      auto g = usp::usp_attention_backward(ctx, mesh, fwd, do_s, causal != 0);
      return PerRank{std::move(g.dq), std::move(g.dk), std::move(g.dv), positions};
    });
    g_ledger_json = ledger_json(world.ledger);
    Tensor4<double> dq(batch, seq, heads, hs), dk(batch, seq, kv_heads, hs), dv(batch, seq, kv_heads, hs);
    for (const auto& pr : world.per_rank) {
      usp::place_rows(dq, pr.dq, pr.positions);
      usp::place_rows(dk, pr.dk, pr.positions);
      usp::place_rows(dv, pr.dv, pr.positions);
    }
    unload(dq, dq_g);
    unload(dk, dk_g);
    unload(dv, dv_g);
  });
}

extern "C" int ref_reference_attention_grad_f64(const double* q, const double* k, const double* v,
                                                const double* dout, int64_t batch, int64_t seq,
                                                int64_t heads, int64_t kv_heads, int64_t hs,
                                                int causal, const int64_t* positions, double* dq,
                                                double* dk, double* dv) {
  return guarded([&] {
    const auto tq = make<double>(q, batch, seq, heads, hs);
    const auto tk = make<double>(k, batch, seq, kv_heads, hs);
    const auto tv = make<double>(v, batch, seq, kv_heads, hs);
    const auto td = make<double>(dout, batch, seq, heads, hs);
    std::span<const int64_t> pos;
    if (positions) pos = std::span<const int64_t>(positions, static_cast<size_t>(seq));
    const auto g = numerics::reference_attention_grad(tq, tk, tv, td, causal != 0, pos);
    unload(g.dq, dq);
    unload(g.dk, dk);
    unload(g.dv, dv);
  });
}
