// plan.cpp — see plan.hpp. Pure host logic; unit-tested on CPU through the
// C-ABI (tests/test_plan.py) and exercised multi-process by the gloo tests.
#include "plan.hpp"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <numeric>
#include <sstream>

#include "fa_fwd.hpp"

namespace uspb200 {

void throw_invalid(const std::string& what) { throw Error(ErrorCode::kInvalidArgument, what); }
void throw_constraint(const std::string& what) { throw Error(ErrorCode::kConstraint, what); }

static void check_rank(const MeshShape& m, int rank) {
  if (rank < 0 || rank >= m.world()) {
    std::ostringstream os;
    os << "rank " << rank << " outside mesh of size " << m.world();  // mesh.cpp:15-21
    throw_invalid(os.str());
  }
}

int MeshShape::ulysses_coord(int rank) const {
  check_rank(*this, rank);
  return rank % ulysses;
}
int MeshShape::ring_coord(int rank) const {
  check_rank(*this, rank);
  return rank / ulysses;
}
int MeshShape::rank_of(int u, int r) const {
  if (u < 0 || u >= ulysses || r < 0 || r >= ring) throw_invalid("mesh coordinates out of range");
  return r * ulysses + u;
}
std::vector<int> MeshShape::ulysses_group(int rank) const {
  const int r = ring_coord(rank);
  std::vector<int> g(ulysses);
  for (int u = 0; u < ulysses; ++u) g[u] = rank_of(u, r);
  return g;
}
std::vector<int> MeshShape::ring_group(int rank) const {
  const int u = ulysses_coord(rank);
  std::vector<int> g(ring);
  for (int r = 0; r < ring; ++r) g[r] = rank_of(u, r);
  return g;
}

void UspShape::validate() const {
  if (batch < 1 || seq_len < 1 || heads < 1 || kv_heads < 1 || head_size < 1)
    throw_invalid("Tensor4 extents must all be >= 1");  // tensor.hpp:27-29
  if (mesh.ulysses < 1 || mesh.ring < 1) throw_invalid("mesh degrees must be >= 1");
  const int ring = mesh.ring, ulysses = mesh.ulysses;
  // ShardSpec (partition.cpp:78-92); zigzag iff causal (commands.cpp:88)
  if (causal && seq_len % (2 * ring) != 0) {
    std::ostringstream os;
    os << "sequence length " << seq_len << " is not divisible by 2*ring = " << 2 * ring
       << " as the zigzag partition requires";
    throw_constraint(os.str());
  }
  if (seq_len % ring != 0) throw_constraint("sequence length is not divisible by the ring degree");
  if ((seq_len / ring) % ulysses != 0) {
    std::ostringstream os;
    os << "per-ring-rank token count " << seq_len / ring
       << " is not divisible by the ulysses degree " << ulysses;
    throw_constraint(os.str());
  }
  // check_usp_inputs (usp_attention.cpp:22-34)
  if (kv_heads % ulysses != 0 || ulysses > kv_heads) {
    std::ostringstream os;
    os << "ulysses degree " << ulysses << " exceeds or does not divide the kv head count "
       << kv_heads << "; the ulysses degree cannot exceed the number of attention heads";
    throw_constraint(os.str());
  }
  if (heads % ulysses != 0) {
    std::ostringstream os;
    os << "query head count " << heads << " is not divisible by the ulysses degree " << ulysses;
    throw_constraint(os.str());
  }
  // check_attention_shapes (attention.cpp:27-32)
  if (heads % kv_heads != 0) {
    std::ostringstream os;
    os << "query head count " << heads << " is not divisible by kv head count " << kv_heads;
    throw_invalid(os.str());
  }
  // B200 engine limits (not reference rules).
  if (head_size > 128) {
    std::ostringstream os;
    os << "head_size " << head_size << " exceeds 128, the largest the tcgen05 kernel supports";
    throw_invalid(os.str());
  }
  if (batch > 255) throw_invalid("batch above 255 is not supported by the work-unit encoding");
  // work units carry the (local) head index in 8 bits (plan.cpp units,
  // kernels decode (unit >> 16) & 0xFF)
  if (heads / ulysses > 256 || kv_heads / ulysses > 256)
    throw_invalid("more than 256 heads per Ulysses rank is not supported by the work-unit encoding");
  if (tokens_per_ring_rank() > INT32_MAX / 2 || seq_len > INT32_MAX / 2)
    throw_invalid("sequence length exceeds the int32 position range");
  if ((tokens_per_ring_rank() + kTileM - 1) / kTileM > 65535)
    throw_invalid("too many query tiles for the work-unit encoding");
}

std::vector<int64_t> zigzag_partition(int64_t seq_len, int ring) {
  if (ring < 1) throw_invalid("ring degree must be >= 1");
  if (seq_len % (2 * ring) != 0) {
    std::ostringstream os;
    os << "sequence length " << seq_len << " is not divisible by 2*ring = " << 2 * ring
       << " as the zigzag partition requires";
    throw_constraint(os.str());
  }
  const int64_t chunk = seq_len / (2 * ring);
  std::vector<int64_t> out;
  out.reserve(seq_len);
  for (int p = 0; p < ring; ++p) {  // rank p owns chunks p and 2R-1-p (partition.cpp:24-32)
    for (int64_t i = 0; i < chunk; ++i) out.push_back(chunk * p + i);
    for (int64_t i = 0; i < chunk; ++i) out.push_back(chunk * (2 * ring - 1 - p) + i);
  }
  return out;
}

std::vector<int64_t> even_partition(int64_t seq_len, int ring) {
  if (ring < 1) throw_invalid("ring degree must be >= 1");
  if (seq_len % ring != 0) throw_constraint("sequence length is not divisible by the ring degree");
  std::vector<int64_t> out(seq_len);
  std::iota(out.begin(), out.end(), 0);
  return out;
}

std::vector<int64_t> causal_pair_counts(const std::vector<int64_t>& flat, int ring,
                                        int64_t seq_len) {
  std::vector<char> seen(seq_len, 0);
  std::vector<int64_t> counts;
  const int64_t per = static_cast<int64_t>(flat.size()) / ring;
  for (int p = 0; p < ring; ++p) {
    int64_t pairs = 0;
    for (int64_t i = 0; i < per; ++i) {
      const int64_t q = flat[p * per + i];
      if (q < 0 || q >= seq_len || seen[q]) throw_invalid("assignment must cover 0..L-1 exactly once");
      seen[q] = 1;
      pairs += q + 1;
    }
    counts.push_back(pairs);
  }
  for (char s : seen)
    if (!s) throw_invalid("assignment must cover 0..L-1 exactly once");
  return counts;
}

std::vector<int64_t> head_positions(const UspShape& s, int rank) {
  const int r = s.mesh.ring_coord(rank);
  const auto lists = s.causal ? zigzag_partition(s.seq_len, s.mesh.ring)
                              : even_partition(s.seq_len, s.mesh.ring);
  const int64_t per_ring = s.tokens_per_ring_rank();
  return std::vector<int64_t>(lists.begin() + r * per_ring, lists.begin() + (r + 1) * per_ring);
}

std::vector<int64_t> positions_for(const UspShape& s, int rank) {
  const int u = s.mesh.ulysses_coord(rank);
  const auto ring_list = head_positions(s, rank);
  const int64_t per_rank = s.tokens_per_rank();
  return std::vector<int64_t>(ring_list.begin() + u * per_rank,
                              ring_list.begin() + (u + 1) * per_rank);
}

std::vector<LedgerEvent> forward_ledger(const UspShape& s, int rank, int elem_bytes) {
  std::vector<LedgerEvent> ev;
  const int U = s.mesh.ulysses, R = s.mesh.ring;
  const int u = s.mesh.ulysses_coord(rank), r = s.mesh.ring_coord(rank);
  const int64_t T = s.tokens_per_rank(), Tr = s.tokens_per_ring_rank();
  const int64_t hs = s.head_size;
  // all_to_all: payload = the rank's whole tensor; sent = payload*(n-1)/n
  // (ledger.cpp:32-33); ring_shift: sent = payload when n > 1 (:34).
  auto a2a = [&](int step, int tensor, int64_t elems) {
    ev.push_back({3, s.mesh.rank_of(0, r), U, 1, step, tensor, elems,
                  double(elems) * elem_bytes * double(U - 1) / double(U)});
  };
  // (with U == 1 the reference still records the all-to-alls, sending 0
  // bytes; the engine issues no transfer but keeps the ledger entries)
  a2a(0, 0, s.batch * T * s.heads * hs);
  a2a(1, 1, s.batch * T * s.kv_heads * hs);
  a2a(2, 2, s.batch * T * s.kv_heads * hs);
  const int64_t kv_block = s.batch * Tr * s.local_kv_heads() * hs;
  int rstep = 0;
  for (int t = 0; t + 1 < R; ++t)
    for (int tensor = 1; tensor <= 2; ++tensor)
      ev.push_back({4, s.mesh.rank_of(u, 0), R, U, rstep++, tensor, kv_block,
                    double(kv_block) * elem_bytes});
  a2a(3, 3, s.batch * Tr * s.local_heads() * hs);
  return ev;
}

std::vector<LedgerEvent> backward_ledger(const UspShape& s, int rank, int elem_bytes, int grad_bytes) {
  std::vector<LedgerEvent> ev = forward_ledger(s, rank, elem_bytes);
  const int U = s.mesh.ulysses, R = s.mesh.ring;
  const int u = s.mesh.ulysses_coord(rank), r = s.mesh.ring_coord(rank);
  const int64_t T = s.tokens_per_rank(), Tr = s.tokens_per_ring_rank();
  const int64_t hs = s.head_size;
  auto a2a = [&](int step, int tensor, int64_t elems) {
    ev.push_back({3, s.mesh.rank_of(0, r), U, 1, step, tensor, elems,
                  double(elems) * elem_bytes * double(U - 1) / double(U)});
  };
  a2a(4, 4, s.batch * T * s.heads * hs);
  const int64_t kv_block = s.batch * Tr * s.local_kv_heads() * hs;
  int rstep = static_cast<int>(std::count_if(ev.begin(), ev.end(), [](const LedgerEvent& e) { return e.kind == 4; }));
  for (int t = 0; t < R; ++t) {
    if (t + 1 < R)
      for (int tensor = 1; tensor <= 2; ++tensor)
        ev.push_back({4, s.mesh.rank_of(u, 0), R, U, rstep++, tensor, kv_block, double(kv_block) * elem_bytes});
    if (t >= 1)
      for (int tensor = 6; tensor <= 7; ++tensor)
        ev.push_back({4, s.mesh.rank_of(u, 0), R, U, rstep++, tensor, kv_block, double(kv_block) * grad_bytes});
  }
  a2a(5, 5, s.batch * Tr * s.local_heads() * hs);
  a2a(6, 6, s.batch * Tr * s.local_kv_heads() * hs);
  a2a(7, 7, s.batch * Tr * s.local_kv_heads() * hs);
  return ev;
}

int64_t visible_pairs(const std::vector<int64_t>& q_pos, const std::vector<int64_t>& k_pos,
                      bool causal) {
  if (!causal) return static_cast<int64_t>(q_pos.size()) * static_cast<int64_t>(k_pos.size());
  std::vector<int64_t> ks(k_pos);
  std::sort(ks.begin(), ks.end());
  int64_t pairs = 0;
  for (int64_t q : q_pos)
    pairs += std::upper_bound(ks.begin(), ks.end(), q) - ks.begin();  // k_pos <= q_pos
  return pairs;
}

FwdTiling fwd_tiling(int hl, int kvl, int hsk, int64_t q_rows, int64_t batch, int sms) {
  static const bool rows_ok = [] {
    const char* e = dev_env("USP_FA_PAIR_ROWS");
    return !e || std::atoi(e) != 0;
  }();
  static const bool cluster_ok = [] {
    const char* e = dev_env("USP_FA_CLUSTER");
    return !e || std::atoi(e) != 0;
  }();
  const int group = hl / kvl;
  if (group % 4 == 0 && hsk == 128 && cluster_ok) return {false, hl / 4, group / 4, kTileM, true};
  if (group % 2 == 0) return {false, hl / 2, group / 2, kTileM, false};
  const int64_t pair_units = (q_rows + 2 * kTileM - 1) / (2 * kTileM) * hl * batch;
  if (rows_ok && pair_units >= sms) return {true, hl, group, 2 * kTileM, false};
  return {false, hl, group, kTileM, false};  // one q tile per CTA (development fallback)
}

StepPlan plan_step(const std::vector<int64_t>& q_pos, const std::vector<int64_t>& k_pos,
                   bool causal, int64_t batch, int head_pairs, bool include_empty,
                   int pairs_per_kv, int rows_per_unit) {
  StepPlan p;
  const int kTileM = rows_per_unit;  // query rows per unit (shadows the 128-row tile)
  p.q_len = static_cast<int>(q_pos.size());
  p.k_len = static_cast<int>(k_pos.size());
  p.n_q_tiles = (p.q_len + kTileM - 1) / kTileM;
  p.n_k_tiles = (p.k_len + kTileN - 1) / kTileN;
  // Effective positions: masked(i, j) <=> k_eff[j] > q_eff[i]. Non-causal
  // sees every real key; padding keys are never visible.
  const int32_t kPadK = INT32_MAX, kAllQ = INT32_MAX - 1;
  p.q_pos.assign(static_cast<size_t>(p.n_q_tiles) * kTileM, kAllQ);
  p.k_pos.assign(static_cast<size_t>(p.n_k_tiles) * kTileN, kPadK);
  for (int i = 0; i < p.q_len; ++i) p.q_pos[i] = causal ? static_cast<int32_t>(q_pos[i]) : kAllQ;
  for (int j = 0; j < p.k_len; ++j) p.k_pos[j] = causal ? static_cast<int32_t>(k_pos[j]) : 0;

  std::vector<int32_t> kmin(p.n_k_tiles, INT32_MAX), kmax(p.n_k_tiles, INT32_MIN);
  std::vector<char> ragged(p.n_k_tiles, 0);
  for (int kt = 0; kt < p.n_k_tiles; ++kt) {
    for (int c = 0; c < kTileN; ++c) {
      const int j = kt * kTileN + c;
      if (j >= p.k_len) {
        ragged[kt] = 1;
        continue;
      }
      kmin[kt] = std::min(kmin[kt], p.k_pos[j]);
      kmax[kt] = std::max(kmax[kt], p.k_pos[j]);
    }
  }
  p.tile_off.assign(p.n_q_tiles + 1, 0);
  std::vector<int> cost(p.n_q_tiles, 0);
  for (int qt = 0; qt < p.n_q_tiles; ++qt) {
    int32_t qmin = INT32_MAX, qmax = INT32_MIN;
    for (int r = 0; r < kTileM; ++r) {
      const int i = qt * kTileM + r;
      if (i >= p.q_len) break;
      qmin = std::min(qmin, p.q_pos[i]);
      qmax = std::max(qmax, p.q_pos[i]);
    }
    for (int kt = 0; kt < p.n_k_tiles; ++kt) {
      if (kmin[kt] > qmax) continue;  // every key hidden from every row: skip
      const bool full = kmax[kt] <= qmin && !ragged[kt];
      p.tile_list.push_back(full ? kt : static_cast<int32_t>(static_cast<uint32_t>(kt) | 0x80000000u));
      if (full)
        ++p.full_tiles;
      else
        ++p.partial_tiles;
      ++cost[qt];
    }
    p.tile_off[qt + 1] = static_cast<int32_t>(p.tile_list.size());
  }
  // Work units in longest-processing-time-first order. Order 1 (default)
  // is kv-head-major: all CTAs resident at a time stream the SAME kv head's
  // K/V tiles, so each tile is fetched from HBM about once per wave and
  // re-read from L2 by the other CTAs; within a kv head, units go longest
  // first (LPT) so the static round-robin assignment stays balanced.
  // Order 0 is plain LPT over (q tile, batch, head pair).
  static const int order = [] {
    const char* e = dev_env("USP_UNIT_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  struct U {
    int cost, qt, b, hp, kvh;
  };
  std::vector<U> us;
  for (int qt = 0; qt < p.n_q_tiles; ++qt) {
    if (cost[qt] == 0 && !include_empty) continue;
    for (int64_t b = 0; b < batch; ++b)
      for (int hp = 0; hp < head_pairs; ++hp)
        us.push_back({cost[qt], qt, static_cast<int>(b), hp, hp / std::max(pairs_per_kv, 1)});
  }
  std::stable_sort(us.begin(), us.end(), [](const U& a, const U& b) {
    if (order == 1) {
      if (a.b != b.b) return a.b < b.b;
      if (a.kvh != b.kvh) return a.kvh < b.kvh;
    }
    if (a.cost != b.cost) return a.cost > b.cost;
    if (a.qt != b.qt) return a.qt < b.qt;
    if (a.b != b.b) return a.b < b.b;
    return a.hp < b.hp;
  });
  p.units.reserve(us.size());
  for (const U& x : us)
    p.units.push_back(static_cast<uint32_t>(x.qt) | (static_cast<uint32_t>(x.hp) << 16) |
                      (static_cast<uint32_t>(x.b) << 24));
  p.visible_pairs = visible_pairs(q_pos, k_pos, causal);
  return p;
}

StepPlan transpose_plan(const StepPlan& f, int64_t batch, int kv_heads, bool include_empty) {
  StepPlan t;
  t.q_len = f.q_len;
  t.k_len = f.k_len;
  t.n_q_tiles = f.n_q_tiles;
  t.n_k_tiles = f.n_k_tiles;
  t.q_pos = f.q_pos;
  t.k_pos = f.k_pos;
  t.full_tiles = f.full_tiles;
  t.partial_tiles = f.partial_tiles;
  t.visible_pairs = f.visible_pairs;
  std::vector<std::vector<int32_t>> by_k(f.n_k_tiles);
  for (int qt = 0; qt < f.n_q_tiles; ++qt)
    for (int e = f.tile_off[qt]; e < f.tile_off[qt + 1]; ++e) {
      const uint32_t entry = static_cast<uint32_t>(f.tile_list[e]);
      by_k[entry & 0x7FFFFFFFu].push_back(static_cast<int32_t>((entry & 0x80000000u) | uint32_t(qt)));
    }
  t.tile_off.assign(f.n_k_tiles + 1, 0);
  for (int kt = 0; kt < f.n_k_tiles; ++kt) {
    t.tile_list.insert(t.tile_list.end(), by_k[kt].begin(), by_k[kt].end());
    t.tile_off[kt + 1] = static_cast<int32_t>(t.tile_list.size());
  }
  struct U {
    int cost, kt, b, kvh;
  };
  std::vector<U> us;
  for (int kt = 0; kt < f.n_k_tiles; ++kt) {
    const int cost = static_cast<int>(by_k[kt].size());
    if (cost == 0 && !include_empty) continue;
    for (int64_t b = 0; b < batch; ++b)
      for (int h = 0; h < kv_heads; ++h) us.push_back({cost, kt, static_cast<int>(b), h});
  }
  std::stable_sort(us.begin(), us.end(), [](const U& a, const U& b) {
    if (a.b != b.b) return a.b < b.b;
    if (a.kvh != b.kvh) return a.kvh < b.kvh;
    if (a.cost != b.cost) return a.cost > b.cost;
    return a.kt < b.kt;
  });
  for (const U& x : us)
    t.units.push_back(static_cast<uint32_t>(x.kt) | (static_cast<uint32_t>(x.kvh) << 16) |
                      (static_cast<uint32_t>(x.b) << 24));
  return t;
}

StepPlan transpose_plan_pairs(const StepPlan& f, int64_t batch, int kv_heads, bool include_empty) {
  const StepPlan one = transpose_plan(f, batch, kv_heads, include_empty);
  StepPlan t = one;
  const int n_pairs = (f.n_k_tiles + 1) / 2;
  t.k_pos.resize(static_cast<size_t>(n_pairs) * 2 * kTileN, INT32_MAX);  // a missing odd tile is padding
  t.tile_off.assign(n_pairs + 1, 0);
  t.tile_list.clear();
  std::vector<int> cost(n_pairs, 0);
  for (int pr = 0; pr < n_pairs; ++pr) {
    // union of the two key tiles' q-tile lists (both ascending); partial if
    // partial for either tile or visible to only one of them
    std::vector<std::pair<int, uint32_t>> merged;  // (q tile, flags: 1 = in a, 2 = in b, 4 = partial)
    for (int side = 0; side < 2; ++side) {
      const int kt = 2 * pr + side;
      if (kt >= f.n_k_tiles) continue;
      for (int e = one.tile_off[kt]; e < one.tile_off[kt + 1]; ++e) {
        const uint32_t entry = static_cast<uint32_t>(one.tile_list[e]);
        merged.push_back({static_cast<int>(entry & 0x7FFFFFFFu), (1u << side) | ((entry >> 31) ? 4u : 0u)});
      }
    }
    std::sort(merged.begin(), merged.end());
    for (size_t i = 0; i < merged.size();) {
      uint32_t fl = 0;
      const int qt = merged[i].first;
      for (; i < merged.size() && merged[i].first == qt; ++i) fl |= merged[i].second;
      const bool partial = (fl & 4u) || (fl & 3u) != 3u;
      t.tile_list.push_back(static_cast<int32_t>(static_cast<uint32_t>(qt) | (partial ? 0x80000000u : 0u)));
    }
    t.tile_off[pr + 1] = static_cast<int32_t>(t.tile_list.size());
    cost[pr] = t.tile_off[pr + 1] - t.tile_off[pr];
  }
  struct U {
    int cost, pr, b, kvh;
  };
  std::vector<U> us;
  for (int pr = 0; pr < n_pairs; ++pr) {
    if (cost[pr] == 0 && !include_empty) continue;
    for (int64_t b = 0; b < batch; ++b)
      for (int h = 0; h < kv_heads; ++h) us.push_back({cost[pr], pr, static_cast<int>(b), h});
  }
  std::stable_sort(us.begin(), us.end(), [](const U& a, const U& b) {
    if (a.b != b.b) return a.b < b.b;
    if (a.kvh != b.kvh) return a.kvh < b.kvh;
    if (a.cost != b.cost) return a.cost > b.cost;
    return a.pr < b.pr;
  });
  t.units.clear();
  for (const U& x : us)
    t.units.push_back(static_cast<uint32_t>(x.pr) | (static_cast<uint32_t>(x.kvh) << 16) |
                      (static_cast<uint32_t>(x.b) << 24));
  return t;
}

}  // namespace uspb200
