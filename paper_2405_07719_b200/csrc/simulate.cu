// simulate.cu — the reference's public C ABI (uspsim_run, include/uspsim.h)
// served by the B200 engine; declared in include/usp_sim.h.
//
// Restates src/api/capi.cpp:33-89 (status mapping, report handle, thread-
// local last error) and src/api/commands.cpp (envelope + config digest
// :27-33, invalid_report :36-47, run_simulation :85-160, cmd_simulate
// :189-282, ledger_summary :162-187, run_command :464-491). The simulation
// itself runs on the GPU: per rank usp_attn_fwd + usp_attn_bwd through the
// in-process transport (one host thread per rank — simcomm::World::run),
// and the check is an fp64 GPU reference (check_fp64.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/usp_sim.h"
#include "json_lite.hpp"
#include "plan.hpp"

namespace uspb200 {

cudaError_t reference_attention_fp64(int64_t batch, int64_t seq, int heads, int kv_heads, int hs, bool causal,
                                     const double* q, const double* k, const double* v, const double* dout,
                                     double* out, double* dq, double* dk, double* dv, double* scratch,
                                     cudaStream_t st);

namespace sim {

using json::Value;
constexpr int kSchemaVersion = 1;  // run_report.hpp:13

struct Report {
  int exit_code = 0;
  std::string status;
  Value doc;
  std::string text, ledger_csv;
};

// run_report.cpp:8-19
std::string fnv1a_hex(const std::string& data) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char ch : data) {
    h ^= ch;
    h *= 0x100000001b3ull;
  }
  char buf[20];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

Value envelope(const std::string& command, const Value& params) {
  Value key = Value::object();
  key["command"] = command;
  key["params"] = params;
  Value e = Value::object();
  e["schema_version"] = kSchemaVersion;
  e["command"] = command;
  e["params"] = params;
  e["config_digest"] = fnv1a_hex(key.dump());
  return e;
}

Report invalid_report(const std::string& command, const Value& params, const std::string& message) {
  Report r;
  r.exit_code = 2;
  r.status = "invalid_input";
  r.doc = envelope(command, params);
  r.doc["status"] = r.status;
  r.doc["exit_code"] = r.exit_code;
  Value res = Value::object();
  res["error"] = message;
  r.doc["results"] = res;
  r.text = "error: " + message + "\n";
  return r;
}

std::string format_sci(double v) {
  char buf[48];
  std::snprintf(buf, sizeof(buf), "%.3g", v);
  return buf;
}

// ledger.cpp:83-92
std::string format_bytes(double b) {
  if (b == std::floor(b) && std::abs(b) < 9.0e15) return std::to_string(static_cast<int64_t>(b));
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", b);
  return buf;
}

const char* collective_name(int kind) {  // ledger.cpp:14-23
  switch (kind) {
    case 0: return "all_reduce";
    case 1: return "all_gather";
    case 2: return "reduce_scatter";
    case 3: return "all_to_all";
    case 4: return "ring_shift";
  }
  return "unknown";
}

// ------------------------------------------------------------------ helpers
void ok(usp_status s) {
  if (s == USP_OK) return;
  const std::string msg = usp_last_error();
  throw Error(s == USP_INVALID_INPUT ? ErrorCode::kConstraint : ErrorCode::kInternal, msg);
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ErrorCode::kInternal, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t n) { cuda_ok(cudaMalloc(&p, std::max<size_t>(n, 16)), "cudaMalloc"); }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

// double -> fp32 -> bf16, round to nearest even (what torch's
// .to(torch.bfloat16) does to an fp64 tensor); inputs are finite.
uint16_t to_bf16(double x) {
  const float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
double from_bf16(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// UniformSource (src/common/random.hpp:15-29).
struct UniformSource {
  std::mt19937_64 engine;
  explicit UniformSource(uint64_t seed) : engine(seed) {}
  double next(double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(engine() >> 11) * 0x1.0p-53);
  }
};

struct SimSpec {
  int64_t batch = 1, seq_len = 64, heads = 8, kv_heads = 8, head_size = 16;
  int ulysses = 1, ring = 1;
  bool causal = false;
  uint64_t seed = 0;
  int device = 0;
};

struct LedgerRow {
  int kind = 0;
  std::vector<int> members;
  int64_t payload = 0;
  std::vector<double> bytes;
};
using Ledger = std::map<std::pair<std::string, int64_t>, LedgerRow>;  // keyed like CommLedger

struct SimOutcome {
  Ledger ledger;
  double out_abs = 0, out_rel = 0, dq_abs = 0, dk_abs = 0, dv_abs = 0;
  double fwd_ms = 0, bwd_ms = 0;
  int64_t launches = 0;
  std::string device_name;
};

std::string group_key(const std::vector<int>& members) {
  std::string s;
  for (size_t i = 0; i < members.size(); ++i) s += (i ? "," : "") + std::to_string(members[i]);
  return s;
}

// Merges the collectives every rank's engine executed into the reference's
// (group, step) ledger. The reference numbers each group's collectives in
// call order including its position all_gathers (usp_attention.cpp:53 on the
// Ulysses group; ring_attention.cpp:56 and :95 on the ring group), which the
// B200 engine does not issue: they are counted (so steps agree) but not
// recorded.
void merge_rank_ledger(Ledger& out, const MeshShape& mesh, int rank, const std::vector<usp_ledger_entry>& ev,
                       size_t n_fwd) {
  const auto ug = mesh.ulysses_group(rank), rg = mesh.ring_group(rank);
  const std::string uk = group_key(ug), rk = group_key(rg);
  std::map<std::string, int64_t> seq;
  auto phantom = [&](const std::string& key) { seq[key]++; };
  auto real = [&](const usp_ledger_entry& e) {
    std::vector<int> members;
    for (int i = 0; i < e.group_size; ++i) members.push_back(e.group_first + i * e.group_stride);
    const std::string key = group_key(members);
    const int64_t step = seq[key]++;
    LedgerRow& row = out[{key, step}];
    row.kind = e.kind;
    row.members = members;
    row.payload = e.payload_elems;
    row.bytes.resize(members.size(), 0.0);
    const auto it = std::find(members.begin(), members.end(), rank);
    row.bytes[it - members.begin()] = e.bytes_sent;
  };
  // forward: G_u, A2A Q K V, G_r, shifts, A2A O
  phantom(uk);
  for (size_t i = 0; i < n_fwd; ++i) {
    real(ev[i]);
    if (i == 2) phantom(rk);
  }
  // backward: A2A dO, G_r, shifts, A2A dQ dK dV
  for (size_t i = n_fwd; i < ev.size(); ++i) {
    real(ev[i]);
    if (i == n_fwd) phantom(rk);
  }
}

SimOutcome run_simulation(const SimSpec& spec, bool check) {
  const int world = spec.ulysses * spec.ring;
  std::vector<usp_config> cfgs(world);
  for (int r = 0; r < world; ++r) {
    usp_config& c = cfgs[r];
    std::memset(&c, 0, sizeof(c));
    c.ulysses_degree = spec.ulysses;
    c.ring_degree = spec.ring;
    c.rank = r;
    c.device = spec.device;
    c.batch = spec.batch;
    c.seq_len = spec.seq_len;
    c.heads = static_cast<int32_t>(spec.heads);
    c.kv_heads = static_cast<int32_t>(spec.kv_heads);
    c.head_size = static_cast<int32_t>(spec.head_size);
    c.causal = spec.causal ? 1 : 0;
  }
  ok(usp_config_validate(&cfgs[0]));  // ShardSpec + check_usp_inputs, reference order and messages
  cuda_ok(cudaSetDevice(spec.device), "cudaSetDevice");

  // Q, K, V, dO from one stream, in that order, over the global tensors
  // (commands.cpp:90-102), rounded to bf16.
  const int64_t B = spec.batch, L = spec.seq_len, H = spec.heads, KV = spec.kv_heads, hs = spec.head_size;
  const size_t nq = size_t(B * L * H * hs), nkv = size_t(B * L * KV * hs);
  std::vector<uint16_t> q(nq), k(nkv), v(nkv), dout(nq);
  UniformSource src(spec.seed);
  for (auto* t : {&q, &k, &v, &dout})
    for (auto& x : *t) x = to_bf16(src.next(-1.0, 1.0));

  // per-rank shards (extract_rows by positions_for, partition.cpp:95-105)
  const int64_t T = L / world;
  std::vector<std::vector<int64_t>> pos(world, std::vector<int64_t>(T));
  for (int r = 0; r < world; ++r) ok(usp_positions_for(&cfgs[0], r, pos[r].data()));
  auto extract = [&](const std::vector<uint16_t>& g, int64_t heads, const std::vector<int64_t>& p) {
    std::vector<uint16_t> s(size_t(B * T * heads * hs));
    const size_t row = size_t(heads * hs);
    for (int64_t b = 0; b < B; ++b)
      for (int64_t t = 0; t < T; ++t)
        std::memcpy(&s[(b * T + t) * row], &g[(b * L + p[t]) * row], row * 2);
    return s;
  };

  std::unique_ptr<usp_comm, void (*)(usp_comm*)> comm(nullptr, usp_comm_destroy);
  if (world > 1) {
    usp_comm* c = nullptr;
    ok(usp_comm_create_local(world, &c));
    comm.reset(c);
  }
  std::vector<std::unique_ptr<usp_engine, void (*)(usp_engine*)>> engines;
  for (int r = 0; r < world; ++r) {
    usp_engine* e = nullptr;
    ok(usp_engine_create(&cfgs[r], comm.get(), &e));
    engines.emplace_back(e, usp_engine_destroy);
  }
  const size_t qb = size_t(B * T * H * hs) * 2, kvb = size_t(B * T * KV * hs) * 2;
  const size_t lb = size_t(B * (L / spec.ring) * (H / spec.ulysses)) * 4;
  struct RankBufs {
    std::unique_ptr<Dev> q, k, v, o, lse, dout, dq, dk, dv;
    cudaStream_t st = nullptr;
  };
  std::vector<RankBufs> rb(world);
  for (int r = 0; r < world; ++r) {
    RankBufs& x = rb[r];
    x.q = std::make_unique<Dev>(qb);
    x.k = std::make_unique<Dev>(kvb);
    x.v = std::make_unique<Dev>(kvb);
    x.o = std::make_unique<Dev>(qb);
    x.lse = std::make_unique<Dev>(lb);
    x.dout = std::make_unique<Dev>(qb);
    x.dq = std::make_unique<Dev>(qb);
    x.dk = std::make_unique<Dev>(kvb);
    x.dv = std::make_unique<Dev>(kvb);
    cuda_ok(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking), "cudaStreamCreate");
    const auto sq = extract(q, H, pos[r]), sk = extract(k, KV, pos[r]), sv = extract(v, KV, pos[r]),
               sd = extract(dout, H, pos[r]);
    cuda_ok(cudaMemcpy(x.q->p, sq.data(), qb, cudaMemcpyHostToDevice), "upload");
    cuda_ok(cudaMemcpy(x.k->p, sk.data(), kvb, cudaMemcpyHostToDevice), "upload");
    cuda_ok(cudaMemcpy(x.v->p, sv.data(), kvb, cudaMemcpyHostToDevice), "upload");
    cuda_ok(cudaMemcpy(x.dout->p, sd.data(), qb, cudaMemcpyHostToDevice), "upload");
  }
  struct StreamGuard {
    std::vector<RankBufs>& rb;
    ~StreamGuard() {
      for (auto& x : rb)
        if (x.st) cudaStreamDestroy(x.st);
    }
  } guard{rb};

  auto ptrs = [&](std::unique_ptr<Dev> RankBufs::*m) {
    std::vector<void*> p(world);
    for (int r = 0; r < world; ++r) p[r] = (rb[r].*m)->p;
    return p;
  };
  std::vector<usp_engine*> eng(world);
  std::vector<void*> streams(world);
  for (int r = 0; r < world; ++r) {
    eng[r] = engines[r].get();
    streams[r] = rb[r].st;
  }
  const auto pq = ptrs(&RankBufs::q), pk = ptrs(&RankBufs::k), pv = ptrs(&RankBufs::v), po = ptrs(&RankBufs::o),
             pl = ptrs(&RankBufs::lse), pd = ptrs(&RankBufs::dout), pdq = ptrs(&RankBufs::dq),
             pdk = ptrs(&RankBufs::dk), pdv = ptrs(&RankBufs::dv);
  std::vector<float*> pl_f(world);
  std::vector<const float*> pl_c(world);
  for (int r = 0; r < world; ++r) {
    pl_f[r] = static_cast<float*>(pl[r]);
    pl_c[r] = pl_f[r];
  }
  std::vector<const void*> cq(pq.begin(), pq.end()), ck(pk.begin(), pk.end()), cv(pv.begin(), pv.end()),
      co(po.begin(), po.end()), cd(pd.begin(), pd.end());

  SimOutcome outcome;
  using clock = std::chrono::steady_clock;
  auto t0 = clock::now();
  ok(usp_local_world_fwd(eng.data(), world, cq.data(), ck.data(), cv.data(), po.data(), pl_f.data(),
                         streams.data()));
  cuda_ok(cudaDeviceSynchronize(), "forward");
  auto t1 = clock::now();
  std::vector<size_t> n_fwd(world);
  for (int r = 0; r < world; ++r) {
    n_fwd[r] = size_t(std::max(0, usp_engine_ledger(eng[r], nullptr, 0)));
    outcome.launches += usp_engine_last_launches(eng[r]);
  }
  ok(usp_local_world_bwd(eng.data(), world, cq.data(), ck.data(), cv.data(), co.data(), pl_c.data(), cd.data(),
                         pdq.data(), pdk.data(), pdv.data(), streams.data()));
  cuda_ok(cudaDeviceSynchronize(), "backward");
  auto t2 = clock::now();
  outcome.fwd_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  outcome.bwd_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  const MeshShape mesh{spec.ulysses, spec.ring};
  for (int r = 0; r < world; ++r) {
    outcome.launches += usp_engine_last_launches(eng[r]);
    const int n = usp_engine_ledger(eng[r], nullptr, 0);
    std::vector<usp_ledger_entry> ev(std::max(n, 0));
    if (n > 0) usp_engine_ledger(eng[r], ev.data(), n);
    merge_rank_ledger(outcome.ledger, mesh, r, ev, n_fwd[r]);
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, spec.device) == cudaSuccess) outcome.device_name = prop.name;
  if (!check) return outcome;

  // gather (place_rows) in fp64
  auto gather = [&](std::unique_ptr<Dev> RankBufs::*m, int64_t heads) {
    std::vector<double> g(size_t(B * L * heads * hs));
    std::vector<uint16_t> s(size_t(B * T * heads * hs));
    const size_t row = size_t(heads * hs);
    for (int r = 0; r < world; ++r) {
      cuda_ok(cudaMemcpy(s.data(), (rb[r].*m)->p, s.size() * 2, cudaMemcpyDeviceToHost), "download");
      for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t)
          for (size_t c = 0; c < row; ++c) g[(b * L + pos[r][t]) * row + c] = from_bf16(s[(b * T + t) * row + c]);
    }
    return g;
  };
  const auto out = gather(&RankBufs::o, H), dq = gather(&RankBufs::dq, H), dk = gather(&RankBufs::dk, KV),
             dv = gather(&RankBufs::dv, KV);

  // single-device fp64 reference on the same bf16 values, on the GPU
  auto widen = [](const std::vector<uint16_t>& x) {
    std::vector<double> w(x.size());
    for (size_t i = 0; i < x.size(); ++i) w[i] = from_bf16(x[i]);
    return w;
  };
  Dev dq_in(nq * 8), dk_in(nkv * 8), dv_in(nkv * 8), ddo(nq * 8), dout_ref(nq * 8), ddq(nq * 8), ddk(nkv * 8),
      ddv(nkv * 8), scratch(size_t(B * L * H) * 3 * 8);
  const auto wq = widen(q), wk = widen(k), wv = widen(v), wd = widen(dout);
  cuda_ok(cudaMemcpy(dq_in.p, wq.data(), nq * 8, cudaMemcpyHostToDevice), "upload");
  cuda_ok(cudaMemcpy(dk_in.p, wk.data(), nkv * 8, cudaMemcpyHostToDevice), "upload");
  cuda_ok(cudaMemcpy(dv_in.p, wv.data(), nkv * 8, cudaMemcpyHostToDevice), "upload");
  cuda_ok(cudaMemcpy(ddo.p, wd.data(), nq * 8, cudaMemcpyHostToDevice), "upload");
  cuda_ok(reference_attention_fp64(B, L, int(H), int(KV), int(hs), spec.causal, static_cast<double*>(dq_in.p),
                                   static_cast<double*>(dk_in.p), static_cast<double*>(dv_in.p),
                                   static_cast<double*>(ddo.p), static_cast<double*>(dout_ref.p),
                                   static_cast<double*>(ddq.p), static_cast<double*>(ddk.p),
                                   static_cast<double*>(ddv.p), static_cast<double*>(scratch.p), nullptr),
          "reference_attention_fp64");
  cuda_ok(cudaDeviceSynchronize(), "reference_attention_fp64");
  auto fetch = [&](const Dev& d, size_t n) {
    std::vector<double> h(n);
    cuda_ok(cudaMemcpy(h.data(), d.p, n * 8, cudaMemcpyDeviceToHost), "download");
    return h;
  };
  const auto ref_o = fetch(dout_ref, nq), ref_dq = fetch(ddq, nq), ref_dk = fetch(ddk, nkv),
             ref_dv = fetch(ddv, nkv);
  // max_errors (commands.cpp:71-83)
  auto max_errors = [](const std::vector<double>& got, const std::vector<double>& want) {
    double a = 0, rel = 0;
    for (size_t i = 0; i < got.size(); ++i) {
      const double d = std::abs(got[i] - want[i]);
      a = std::max(a, d);
      rel = std::max(rel, d / std::max(std::abs(want[i]), 1e-12));
    }
    return std::make_pair(a, rel);
  };
  std::tie(outcome.out_abs, outcome.out_rel) = max_errors(out, ref_o);
  outcome.dq_abs = max_errors(dq, ref_dq).first;
  outcome.dk_abs = max_errors(dk, ref_dk).first;
  outcome.dv_abs = max_errors(dv, ref_dv).first;
  return outcome;
}

// ledger_summary (commands.cpp:162-187) over the executed collectives.
Value ledger_summary(const Ledger& ledger) {
  Value kinds = Value::object();
  for (int kind = 0; kind <= 4; ++kind) {
    int64_t events = 0;
    double bytes = 0;
    for (const auto& [key, e] : ledger) {
      if (e.kind != kind) continue;
      ++events;
      for (double b : e.bytes) bytes += b;
    }
    if (events == 0) continue;
    Value x = Value::object();
    x["events"] = events;
    x["bytes_sent"] = bytes;
    kinds[collective_name(kind)] = x;
  }
  std::map<std::string, int64_t> a2a, shifts;
  for (const auto& [key, e] : ledger) {
    if (e.kind == 3) a2a[key.first]++;
    if (e.kind == 4) shifts[key.first]++;
  }
  Value per_group = Value::object();
  if (!a2a.empty()) per_group["all_to_all"] = a2a.begin()->second;
  if (!shifts.empty()) per_group["ring_shift"] = shifts.begin()->second;
  Value s = Value::object();
  s["collectives"] = kinds;
  s["events_per_group"] = per_group;
  return s;
}

// CommLedger::to_csv (ledger.cpp:94-106)
std::string ledger_csv(const Ledger& ledger) {
  std::ostringstream os;
  os << "step,collective,group,rank,bytes\n";
  for (const auto& [key, e] : ledger)
    for (size_t i = 0; i < e.members.size(); ++i)
      os << key.second << ',' << collective_name(e.kind) << ",\"" << key.first << "\"," << e.members[i] << ','
         << format_bytes(e.bytes[i]) << '\n';
  return os.str();
}

Report cmd_simulate(const Value& params) {
  SimSpec spec;
  spec.batch = params.value("batch", int64_t(1));
  spec.seq_len = params.value("seqlen", int64_t(64));
  spec.heads = params.value("heads", int64_t(8));
  spec.kv_heads = params.value("kv_heads", spec.heads);
  spec.head_size = params.value("head_size", int64_t(16));
  spec.ulysses = params.value("ulysses", 1);
  spec.ring = params.value("ring", 1);
  spec.causal = params.value("causal", false);
  spec.seed = params.value("seed", uint64_t(0));
  spec.device = params.value("device", 0);
  const std::string precision = params.value("precision", std::string("bf16"));
  if (precision != "bf16")
    throw_invalid("precision must be \"bf16\" on the B200 engine (bf16 inputs, fp32 accumulation); \"fp32\" and "
                  "\"fp64\" are the reference CPU library's precisions");
  const bool check = params.value("check", false);
  const double tolerance = params.value("tolerance", 2e-2);
  if (spec.batch < 1 || spec.seq_len < 1 || spec.heads < 1 || spec.kv_heads < 1 || spec.head_size < 1)
    throw_invalid("simulate dimensions must all be >= 1");
  if (spec.heads % spec.kv_heads != 0) throw_invalid("heads must be divisible by kv_heads");
  if (spec.ulysses < 1 || spec.ring < 1) throw_invalid("mesh degrees must be >= 1");

  const SimOutcome outcome = run_simulation(spec, check);

  Report r;
  r.doc = envelope("simulate", params);
  Value results = Value::object();
  results["world_size"] = int64_t(spec.ulysses) * spec.ring;
  Value mesh = Value::object();
  mesh["ulysses"] = spec.ulysses;
  mesh["ring"] = spec.ring;
  results["mesh"] = mesh;
  Value shape = Value::object();
  shape["batch"] = spec.batch;
  shape["seqlen"] = spec.seq_len;
  shape["heads"] = spec.heads;
  shape["kv_heads"] = spec.kv_heads;
  shape["head_size"] = spec.head_size;
  results["shape"] = shape;
  results["causal"] = spec.causal;
  results["precision"] = "bf16";
  results["seed"] = spec.seed;
  results["ledger"] = ledger_summary(outcome.ledger);
  Value engine = Value::object();
  engine["name"] = "usp_b200";
  engine["device"] = outcome.device_name;
  engine["device_ordinal"] = spec.device;
  engine["forward_ms"] = outcome.fwd_ms;
  engine["backward_ms"] = outcome.bwd_ms;
  engine["kernel_launches"] = outcome.launches;
  engine["ledger_omits"] = "position all_gathers (static layout on the B200 engine)";
  results["engine"] = engine;

  std::ostringstream text;
  text << "simulate: mesh ulysses=" << spec.ulysses << " ring=" << spec.ring << " (world "
       << spec.ulysses * spec.ring << "), bs=" << spec.batch << " L=" << spec.seq_len << " hc=" << spec.heads
       << " kv=" << spec.kv_heads << " hs=" << spec.head_size << (spec.causal ? ", causal" : ", full")
       << ", bf16, seed " << spec.seed << "\n";
  bool passed = true;
  if (check) {
    const double worst = std::max({outcome.out_abs, outcome.dq_abs, outcome.dk_abs, outcome.dv_abs});
    passed = worst <= tolerance;
    Value c = Value::object();
    c["max_abs_out"] = outcome.out_abs;
    c["max_rel_out"] = outcome.out_rel;
    c["max_abs_dq"] = outcome.dq_abs;
    c["max_abs_dk"] = outcome.dk_abs;
    c["max_abs_dv"] = outcome.dv_abs;
    c["tolerance"] = tolerance;
    c["passed"] = passed;
    results["check"] = c;
    text << "oracle check: |out-ref| " << format_sci(outcome.out_abs) << " (rel " << format_sci(outcome.out_rel)
         << "), |dq| " << format_sci(outcome.dq_abs) << ", |dk| " << format_sci(outcome.dk_abs) << ", |dv| "
         << format_sci(outcome.dv_abs) << " vs tolerance " << format_sci(tolerance) << ": "
         << (passed ? "PASS" : "FAIL") << "\n";
  }
  const Value& lj = results.at("ledger").at("collectives");
  text << "ledger:";
  for (const auto& [name, x] : lj.items())
    text << " " << name << "=" << x.at("events").get_int() << " events/"
         << format_sci(x.at("bytes_sent").get_double()) << " bytes";
  text << "\n";

  r.exit_code = passed ? 0 : 1;
  r.status = passed ? "ok" : "tolerance_exceeded";
  r.doc["status"] = r.status;
  r.doc["exit_code"] = r.exit_code;
  r.doc["results"] = results;
  r.text = text.str();
  r.ledger_csv = ledger_csv(outcome.ledger);
  return r;
}

// cmd_balance (commands.cpp:414-462): the zigzag vs contiguous causal load of
// each ring rank — host arithmetic over the layout the engine itself uses
// (plan.cpp zigzag_partition / even_partition / causal_pair_counts).
Report cmd_balance(const Value& params) {
  const int64_t seq_len = params.value("seqlen", int64_t(16));
  const int ring = params.value("ring", 4);
  const auto zz = zigzag_partition(seq_len, ring);
  const auto ev = even_partition(seq_len, ring);
  const auto zc = causal_pair_counts(zz, ring, seq_len);
  const auto ec = causal_pair_counts(ev, ring, seq_len);
  const int64_t per = ring > 0 ? seq_len / ring : 0;
  auto arr = [](const std::vector<int64_t>& v, size_t b, size_t e) {
    Value a = Value::array();
    for (size_t i = b; i < e; ++i) a.push_back(v[i]);
    return a;
  };
  const double skew = double(ec.back()) / double(ec.front());
  Report r;
  r.doc = envelope("balance", params);
  Value results = Value::object();
  results["seqlen"] = seq_len;
  results["ring"] = ring;
  results["zigzag_counts"] = arr(zc, 0, zc.size());
  results["even_counts"] = arr(ec, 0, ec.size());
  results["even_skew"] = skew;
  std::ostringstream text;
  text << "balance: L=" << seq_len << " ring=" << ring << "\n";
  if (seq_len <= 64) {
    Value lists = Value::array();
    for (int p = 0; p < ring; ++p) {
      lists.push_back(arr(zz, size_t(p * per), size_t((p + 1) * per)));
      text << "  ring rank " << p << " tokens [";
      for (int64_t i = 0; i < per; ++i) text << (i ? "," : "") << zz[size_t(p * per + i)];
      text << "]\n";
    }
    results["zigzag_assignment"] = lists;
  }
  auto print_counts = [&](const char* name, const std::vector<int64_t>& counts) {
    text << "  " << name << " causal pair counts:";
    for (int64_t c : counts) text << " " << c;
    text << "\n";
  };
  print_counts("zigzag", zc);
  print_counts("even  ", ec);
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%g", skew);  // std::ostream's default double format
  text << "  even skew last/first = " << buf << "\n";
  r.exit_code = 0;
  r.status = "ok";
  r.doc["status"] = r.status;
  r.doc["exit_code"] = r.exit_code;
  r.doc["results"] = results;
  r.text = text.str();
  return r;
}

// run_command (commands.cpp:464-491)
Report run_command(const Value& request) {
  std::string command;
  Value params = Value::object();
  try {
    command = request.at("command").get_string();
    if (request.contains("params")) params = request.at("params");
  } catch (const json::Error& e) {
    return invalid_report("", request, std::string("bad request envelope: ") + e.what());
  }
  try {
    if (command == "simulate") return cmd_simulate(params);
    if (command == "balance") return cmd_balance(params);
    if (command == "cost" || command == "plan")
      return invalid_report(command, params,
                            "command \"" + command +
                                "\" is analytic (host-only) and not served by the B200 engine; use the "
                                "reference uspsim library for it");
    return invalid_report(command, params, "unknown command: " + command);
  } catch (const json::Error& e) {
    return invalid_report(command, params, std::string("malformed params: ") + e.what());
  } catch (const Error& e) {
    if (e.code() == ErrorCode::kInternal)
      return invalid_report(command, params, std::string("internal error: ") + e.what());
    return invalid_report(command, params, e.what());
  } catch (const std::exception& e) {
    return invalid_report(command, params, std::string("internal error: ") + e.what());
  }
}

thread_local std::string g_last_error;

}  // namespace sim
}  // namespace uspb200

// ================================================================== C ABI
using namespace uspb200;

struct uspsim_report {
  sim::Report impl;
  std::string json_dump;
};

extern "C" {

uspsim_status uspsim_run(const char* request_json, uspsim_report** out_report) {
  if (out_report == nullptr) return USPSIM_INVALID_INPUT;
  *out_report = nullptr;
  if (request_json == nullptr) {
    sim::g_last_error = "request_json is null";
    return USPSIM_INVALID_INPUT;
  }
  try {
    json::Value request;
    try {
      request = json::parse(request_json);
    } catch (const json::Error& e) {
      sim::g_last_error = std::string("request is not valid JSON: ") + e.what();
      return USPSIM_INVALID_INPUT;
    }
    auto* handle = new uspsim_report{sim::run_command(request), {}};
    handle->json_dump = handle->impl.doc.dump();
    *out_report = handle;
    switch (handle->impl.exit_code) {
      case 0: return USPSIM_OK;
      case 1: return USPSIM_TOLERANCE_EXCEEDED;
      case 2: return USPSIM_INVALID_INPUT;
      default: return USPSIM_INTERNAL_ERROR;
    }
  } catch (const std::bad_alloc&) {
    sim::g_last_error = "out of memory";
    return USPSIM_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    sim::g_last_error = e.what();
    return USPSIM_INTERNAL_ERROR;
  }
}

const char* uspsim_report_json(const uspsim_report* report) {
  return report == nullptr ? "" : report->json_dump.c_str();
}
const char* uspsim_report_text(const uspsim_report* report) {
  return report == nullptr ? "" : report->impl.text.c_str();
}
const char* uspsim_report_ledger_csv(const uspsim_report* report) {
  return report == nullptr ? "" : report->impl.ledger_csv.c_str();
}
int uspsim_report_exit_code(const uspsim_report* report) { return report == nullptr ? 2 : report->impl.exit_code; }
void uspsim_report_free(uspsim_report* report) { delete report; }
const char* uspsim_last_error(void) { return sim::g_last_error.c_str(); }
const char* uspsim_version(void) { return "0.1.0-b200"; }

}  // extern "C"
