// transport.cpp — NCCL (one process per GPU) and in-process transports.
//
// NCCL is resolved with dlopen at first use, so the library loads on hosts
// without NCCL and binds to whichever libnccl.so.2 the process already has
// (torch's, when torch is imported first). Groups are built with
// ncclCommSplit: Ulysses comm = mesh row (color = ring coord, key = u),
// Ring comm = mesh column (color = u, key = ring coord), as ProcessMesh
// defines them (reference src/simcomm/mesh.cpp:41-57).
#include "transport.hpp"

#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>

#include "plan.hpp"

namespace uspb200 {

#define USPB_CUDA(x)                                                               \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess)                                                         \
      throw Error(ErrorCode::kInternal, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

static int index_of(const std::vector<int>& g, int rank) {
  for (size_t i = 0; i < g.size(); ++i)
    if (g[i] == rank) return static_cast<int>(i);
  throw Error(ErrorCode::kInternal, "rank not in its own group");
}

// ======================================================================
// In-process transport: the B200 analogue of simcomm::World (one thread per
// rank, barrier at every collective), moving bytes with stream-ordered CUDA
// copies (copy engines; peer copies over NVLink when ranks sit on
// different GPUs).
class LocalTransport final : public Transport {
 public:
  explicit LocalTransport(int n) : n_(n), slots_(n) {}
  ~LocalTransport() override {
    for (auto& s : slots_) {
      if (s.ready) cudaEventDestroy(s.ready);
      if (s.done) cudaEventDestroy(s.done);
    }
  }
  int world_size() const override { return n_; }
  int reserved_sms() const override { return 0; }

  std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ug,
                                      const std::vector<int>& rg) override {
    auto g = std::make_shared<Groups>();
    g->rank = rank;
    g->ulysses = ug;
    g->ring = rg;
    Slot& s = slots_.at(rank);
    if (!s.ready) {
      USPB_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
      USPB_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }
    return g;
  }

  void all_to_all(const Groups& g, const std::vector<std::vector<A2APart>>& parts,
                  const std::vector<size_t>& bytes, cudaStream_t stream) override {
    Slot& me = slots_.at(g.rank);
    me.parts = parts;
    USPB_CUDA(cudaEventRecord(me.ready, stream));
    barrier();
    const int mi = index_of(g.ulysses, g.rank);
    for (size_t p = 0; p < g.ulysses.size(); ++p) {
      Slot& peer = slots_.at(g.ulysses[p]);
      if (&peer != &me) USPB_CUDA(cudaStreamWaitEvent(stream, peer.ready, 0));
      for (size_t t = 0; t < parts.size(); ++t)
        if (bytes[t])
          USPB_CUDA(cudaMemcpyAsync(me.parts[t][p].recv, peer.parts[t][mi].send, bytes[t],
                                    cudaMemcpyDefault, stream));
    }
    USPB_CUDA(cudaEventRecord(me.done, stream));
    barrier();
    for (int peer_rank : g.ulysses)
      if (peer_rank != g.rank) USPB_CUDA(cudaStreamWaitEvent(stream, slots_.at(peer_rank).done, 0));
  }

  void ring_shift(const Groups& g, const std::vector<const void*>& send,
                  const std::vector<void*>& recv, const std::vector<size_t>& bytes,
                  cudaStream_t stream) override {
    Slot& me = slots_.at(g.rank);
    me.send = send;
    USPB_CUDA(cudaEventRecord(me.ready, stream));
    barrier();
    const int n = static_cast<int>(g.ring.size());
    const int i = index_of(g.ring, g.rank);
    Slot& prev = slots_.at(g.ring[(i - 1 + n) % n]);
    Slot& next = slots_.at(g.ring[(i + 1) % n]);
    if (&prev != &me) USPB_CUDA(cudaStreamWaitEvent(stream, prev.ready, 0));
    for (size_t t = 0; t < recv.size(); ++t)
      if (bytes[t])
        USPB_CUDA(cudaMemcpyAsync(recv[t], prev.send[t], bytes[t], cudaMemcpyDefault, stream));
    USPB_CUDA(cudaEventRecord(me.done, stream));
    barrier();
    if (&next != &me) USPB_CUDA(cudaStreamWaitEvent(stream, next.done, 0));
  }

 private:
  struct Slot {
    std::vector<std::vector<A2APart>> parts;
    std::vector<const void*> send;
    cudaEvent_t ready = nullptr, done = nullptr;
  };

  void barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    const uint64_t gen = gen_;
    if (++arrived_ == n_) {
      arrived_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    // A rank that never arrives (mismatched collectives) is reported instead
    // of hanging, like the reference's stuck-collective diagnosis
    // (world.cpp:89-113).
    if (!cv_.wait_for(lk, std::chrono::seconds(600), [&] { return gen_ != gen; }))
      throw Error(ErrorCode::kCommMismatch,
                  "local transport: a rank did not reach the collective (mismatched calls?)");
  }

  int n_;
  std::vector<Slot> slots_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t gen_ = 0;
};

std::unique_ptr<Transport> make_local_transport(int world_size) {
  if (world_size < 1) throw_invalid("world size must be >= 1");
  return std::make_unique<LocalTransport>(world_size);
}

// ======================================================================
// NCCL, resolved at runtime.
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && err.empty()) err = std::string("libnccl lacks ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRankConfig =
        reinterpret_cast<decltype(api.CommInitRankConfig)>(sym("ncclCommInitRankConfig"));
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw Error(ErrorCode::kInternal, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(ErrorCode::kInternal, std::string(what) + ": " + nccl().GetErrorString(r));
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
}  // namespace

class NcclTransport final : public Transport {
 public:
  NcclTransport(const unsigned char id[128], int n, int rank, int device) : n_(n) {
    const NcclApi& api = nccl();
    USPB_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 1;
    // Only the ring communicator runs concurrently with the attention kernel
    // (whose persistent grid leaves reserved_sms() SMs for it); a K/V block
    // shift needs a few GB/s to hide behind a ring step, so a couple of CTAs
    // suffice. The Ulysses all-to-alls run between kernels and get NCCL's
    // default channel count (full NVLink bandwidth).
    max_ctas_ = std::max(1, env_int("USP_NCCL_MAX_CTAS", 2));
    nccl_check(api.CommInitRankConfig(&world_, n, uid, rank, &cfg), "ncclCommInitRankConfig");
  }
  ~NcclTransport() override {
    for (ncclComm_t c : owned_) nccl().CommDestroy(c);
    if (world_) nccl().CommDestroy(world_);
  }
  int world_size() const override { return n_; }
  int reserved_sms() const override { return env_int("USP_RESERVED_SMS", max_ctas_); }

  // Engines of the same mesh share the two sub-communicators: the splits
  // are collective over the world and every rank creates its engines in the
  // same order, so every rank hits (or misses) this cache together.
  std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ug,
                                      const std::vector<int>& rg) override {
    const auto key = std::make_pair(ug, rg);
    auto hit = groups_.find(key);
    if (hit != groups_.end()) return hit->second;
    auto g = std::make_shared<Groups>();
    g->rank = rank;
    g->ulysses = ug;
    g->ring = rg;
    ncclConfig_t ucfg = NCCL_CONFIG_INITIALIZER;
    ucfg.blocking = 1;
    ncclConfig_t rcfg = NCCL_CONFIG_INITIALIZER;
    rcfg.blocking = 1;
    rcfg.maxCTAs = max_ctas_;
    rcfg.minCTAs = 1;
    ncclComm_t uc = nullptr, rc = nullptr;
    // color = the other mesh coordinate; key = position inside the group.
    const int u = index_of(ug, rank), r = index_of(rg, rank);
    nccl_check(nccl().CommSplit(world_, /*color=*/r, /*key=*/u, &uc, &ucfg), "ncclCommSplit(ulysses)");
    nccl_check(nccl().CommSplit(world_, /*color=*/u, /*key=*/r, &rc, &rcfg), "ncclCommSplit(ring)");
    owned_.push_back(uc);
    owned_.push_back(rc);
    g->ulysses_comm = uc;
    g->ring_comm = rc;
    groups_.emplace(key, g);
    return g;
  }

  void all_to_all(const Groups& g, const std::vector<std::vector<A2APart>>& parts,
                  const std::vector<size_t>& bytes, cudaStream_t stream) override {
    const NcclApi& api = nccl();
    auto comm = static_cast<ncclComm_t>(g.ulysses_comm);
    const int me = index_of(g.ulysses, g.rank);
    // Self part: a device copy (NCCL would also copy it).
    for (size_t t = 0; t < parts.size(); ++t)
      if (bytes[t] && parts[t][me].recv != parts[t][me].send)
        USPB_CUDA(cudaMemcpyAsync(parts[t][me].recv, parts[t][me].send, bytes[t],
                                  cudaMemcpyDeviceToDevice, stream));
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (size_t t = 0; t < parts.size(); ++t) {
      for (size_t p = 0; p < g.ulysses.size(); ++p) {
        if (static_cast<int>(p) == me || !bytes[t]) continue;
        nccl_check(api.Send(parts[t][p].send, bytes[t], ncclInt8, static_cast<int>(p), comm, stream),
                   "ncclSend");
        nccl_check(api.Recv(parts[t][p].recv, bytes[t], ncclInt8, static_cast<int>(p), comm, stream),
                   "ncclRecv");
      }
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }

  void ring_shift(const Groups& g, const std::vector<const void*>& send,
                  const std::vector<void*>& recv, const std::vector<size_t>& bytes,
                  cudaStream_t stream) override {
    const NcclApi& api = nccl();
    auto comm = static_cast<ncclComm_t>(g.ring_comm);
    const int n = static_cast<int>(g.ring.size());
    const int i = index_of(g.ring, g.rank);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (size_t t = 0; t < send.size(); ++t) {
      if (!bytes[t]) continue;
      nccl_check(api.Send(send[t], bytes[t], ncclInt8, (i + 1) % n, comm, stream), "ncclSend");
      nccl_check(api.Recv(recv[t], bytes[t], ncclInt8, (i - 1 + n) % n, comm, stream), "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }

 private:
  int n_;
  int max_ctas_ = 2;
  ncclComm_t world_ = nullptr;
  std::vector<ncclComm_t> owned_;
  std::map<std::pair<std::vector<int>, std::vector<int>>, std::shared_ptr<Groups>> groups_;
};

std::unique_ptr<Transport> make_nccl_transport(const unsigned char id[128], int world_size,
                                               int rank, int device) {
  return std::make_unique<NcclTransport>(id, world_size, rank, device);
}

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &uid, sizeof(uid));
}

}  // namespace uspb200
