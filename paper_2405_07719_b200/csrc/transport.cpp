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
#include <deque>
#include <map>
#include <tuple>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>

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

double Transport::default_timeout() {
  const char* e = std::getenv("USP_COMM_TIMEOUT_S");
  const double v = e ? std::atof(e) : 0.0;
  return v > 0 ? v : 600.0;
}

static std::string group_key(const std::vector<int>& members) {
  std::ostringstream os;  // ProcessGroup::key (world.cpp:17-28)
  for (size_t i = 0; i < members.size(); ++i) os << (i ? "," : "") << members[i];
  return os.str();
}

// ======================================================================
// In-process transport: the B200 analogue of simcomm::World (one thread per
// rank, a host rendezvous per collective), moving bytes with stream-ordered
// CUDA copies (copy engines; peer copies over NVLink when ranks sit on
// different GPUs). Like World::collective (world.cpp:119-165) every
// rendezvous is keyed by (group, per-group call number) and carries a
// signature, so mismatched calls are reported ("collective mismatch on group
// [...] call #k: rank a called X but rank b called Y") and a rank that never
// arrives is reported after the timeout ("collective deadlock: ...") instead
// of hanging the world.
class LocalTransport final : public Transport {
 public:
  explicit LocalTransport(int n) : n_(n), slots_(n), status_(n, "running") {}
  ~LocalTransport() override {
    for (auto& s : slots_) {
      if (s.ready) cudaEventDestroy(s.ready);
      if (s.done) cudaEventDestroy(s.done);
    }
  }
  int world_size() const override { return n_; }
  bool comm_uses_sms() const override { return false; }
  std::string status() override {
    std::lock_guard<std::mutex> lk(mu_);
    return failure_;
  }
  void debug_rendezvous(const std::vector<int>& members, int rank, const std::string& sig) override {
    rendezvous(members, rank, sig);
  }

  std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ug, const std::vector<int>& rg, int,
                                      int) override {
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
                  const std::vector<size_t>& bytes, cudaStream_t stream, bool) override {
    std::ostringstream sig;
    sig << "all_to_all<bf16>(tensors=" << parts.size() << ",part_bytes=";
    for (size_t t = 0; t < bytes.size(); ++t) sig << (t ? "/" : "") << bytes[t];
    sig << ")";
    Slot& me = slots_.at(g.rank);
    me.parts = parts;
    USPB_CUDA(cudaEventRecord(me.ready, stream));
    rendezvous(g.ulysses, g.rank, sig.str());
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
    rendezvous(g.ulysses, g.rank, sig.str());
    for (int peer_rank : g.ulysses)
      if (peer_rank != g.rank) USPB_CUDA(cudaStreamWaitEvent(stream, slots_.at(peer_rank).done, 0));
  }

  void ring_shift(const Groups& g, const std::vector<const void*>& send,
                  const std::vector<void*>& recv, const std::vector<size_t>& bytes,
                  cudaStream_t stream) override {
    std::ostringstream sig;
    sig << "ring_shift(buffers=" << send.size() << ",bytes=" << (bytes.empty() ? 0 : bytes[0]) << ",steps=1)";
    Slot& me = slots_.at(g.rank);
    me.send = send;
    USPB_CUDA(cudaEventRecord(me.ready, stream));
    rendezvous(g.ring, g.rank, sig.str());
    const int n = static_cast<int>(g.ring.size());
    const int i = index_of(g.ring, g.rank);
    Slot& prev = slots_.at(g.ring[(i - 1 + n) % n]);
    Slot& next = slots_.at(g.ring[(i + 1) % n]);
    if (&prev != &me) USPB_CUDA(cudaStreamWaitEvent(stream, prev.ready, 0));
    for (size_t t = 0; t < recv.size(); ++t)
      if (bytes[t])
        USPB_CUDA(cudaMemcpyAsync(recv[t], prev.send[t], bytes[t], cudaMemcpyDefault, stream));
    USPB_CUDA(cudaEventRecord(me.done, stream));
    rendezvous(g.ring, g.rank, sig.str());
    if (&next != &me) USPB_CUDA(cudaStreamWaitEvent(stream, next.done, 0));
  }

 private:
  struct Slot {
    std::vector<std::vector<A2APart>> parts;
    std::vector<const void*> send;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  struct Meet {
    std::string sig;
    int first_rank = -1;
    int arrived = 0, left = 0;
    bool done = false;
  };

  void fail_locked(const std::string& msg) {
    if (failure_.empty()) failure_ = msg;
    cv_.notify_all();
  }

  void rendezvous(const std::vector<int>& members, int rank, const std::string& sig) {
    const std::string key = group_key(members);
    std::unique_lock<std::mutex> lk(mu_);
    if (!failure_.empty()) throw Error(ErrorCode::kCommMismatch, failure_);
    const int64_t seq = seq_[{rank, key}]++;
    std::ostringstream site;
    site << sig << " call #" << seq << " on group [" << key << "]";
    Meet& m = meets_[{key, seq}];
    if (m.arrived == 0) {
      m.sig = sig;
      m.first_rank = rank;
    } else if (m.sig != sig) {
      const int a = std::min(rank, m.first_rank), b = std::max(rank, m.first_rank);
      std::ostringstream os;
      os << "collective mismatch on group [" << key << "] call #" << seq << ": rank " << a << " called "
         << (a == rank ? sig : m.sig) << " but rank " << b << " called " << (b == rank ? sig : m.sig);
      fail_locked(os.str());
      throw Error(ErrorCode::kCommMismatch, failure_);
    }
    status_.at(rank) = "blocked at " + site.str();
    if (++m.arrived == static_cast<int>(members.size())) {
      m.done = true;
      cv_.notify_all();
    } else if (!cv_.wait_for(lk, std::chrono::duration<double>(timeout_s_),
                             [&] { return m.done || !failure_.empty(); })) {
      std::ostringstream os;  // world.cpp:89-113, after the timeout
      os << "collective deadlock (no progress for " << timeout_s_ << " s):";
      for (int r = 0; r < n_; ++r) os << (r ? ";" : "") << " rank " << r << ' ' << status_[r];
      fail_locked(os.str());
    }
    if (!failure_.empty() && !m.done) throw Error(ErrorCode::kCommMismatch, failure_);
    status_.at(rank) = "running";
    if (++m.left == static_cast<int>(members.size())) meets_.erase({key, seq});
  }

  int n_;
  std::vector<Slot> slots_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<std::string, int64_t>, Meet> meets_;
  std::map<std::pair<int, std::string>, int64_t> seq_;
  std::vector<std::string> status_;
  std::string failure_;
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
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
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
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
  });
  if (!err.empty()) throw Error(ErrorCode::kInternal, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(ErrorCode::kInternal, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

// Communicators are NON-BLOCKING (ncclConfig_t.blocking = 0): init, split
// and every grouped send/recv return at once and are polled with
// ncclCommGetAsyncError against the transport timeout. A watchdog thread
// follows every enqueued collective (an event recorded after it) and the
// communicators' async errors; a collective that does not complete within
// the timeout, or an NCCL error, aborts all communicators (which also frees
// the GPU from a kernel waiting for a peer that never comes) and is reported
// with the collective and its group, like the reference World's stuck /
// mismatched-collective diagnosis (world.cpp:89-113, 152-165): the next call
// on the transport, and usp_comm_status, return it.
class NcclTransport final : public Transport {
 public:
  NcclTransport(const unsigned char id[128], int n, int rank, int device) : n_(n), rank_(rank), device_(device) {
    const NcclApi& api = nccl();
    USPB_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    const ncclResult_t r = api.CommInitRankConfig(&world_, n, uid, rank, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
      if (world_) api.CommAbort(world_);
      world_ = nullptr;
      nccl_check(r, "ncclCommInitRankConfig");
    }
    std::ostringstream what;
    what << "ncclCommInitRankConfig(world of " << n << ", rank " << rank << ")";
    wait_ready(world_, what.str());
    watchdog_ = std::thread([this] { watch(); });
  }
  ~NcclTransport() override {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (watchdog_.joinable()) watchdog_.join();
    for (auto& pd : pending_) cudaEventDestroy(pd.ev);
    for (cudaEvent_t e : free_events_) cudaEventDestroy(e);
    if (!aborted_) {
      for (ncclComm_t c : owned_) nccl().CommDestroy(c);
      if (world_) nccl().CommDestroy(world_);
    }
  }
  int world_size() const override { return n_; }
  bool comm_uses_sms() const override { return true; }
  std::string status() override {
    std::lock_guard<std::mutex> lk(mu_);
    return failure_;
  }

  // Engines of the same mesh share the two sub-communicators: the splits
  // are collective over the world and every rank creates its engines in the
  // same order, so every rank hits (or misses) this cache together.
  std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ug, const std::vector<int>& rg,
                                      int ring_ctas, int a2a_ctas) override {
    check_healthy();
    const auto key = std::make_tuple(ug, rg, ring_ctas, a2a_ctas);
    auto hit = groups_.find(key);
    if (hit != groups_.end()) return hit->second;
    auto g = std::make_shared<Groups>();
    g->rank = rank;
    g->ulysses = ug;
    g->ring = rg;
    ncclConfig_t ucfg = NCCL_CONFIG_INITIALIZER;
    ucfg.blocking = 0;
    ncclConfig_t rcfg = NCCL_CONFIG_INITIALIZER;
    rcfg.blocking = 0;
    // Only the ring communicator runs concurrently with the attention kernel
    // (whose persistent grid leaves reserved_sms() SMs for it); see DESIGN §5
    // for the sizing (K/V bytes per ring step / step time, 2x margin).
    rcfg.maxCTAs = std::max(1, ring_ctas);
    rcfg.minCTAs = 1;
    ncclComm_t uc = nullptr, rc = nullptr;
    // color = the other mesh coordinate; key = position inside the group.
    const int u = index_of(ug, rank), r = index_of(rg, rank);
    split(/*color=*/r, /*key=*/u, &uc, &ucfg, "ncclCommSplit(ulysses group [" + group_key(ug) + "])");
    owned_.push_back(uc);
    split(/*color=*/u, /*key=*/r, &rc, &rcfg, "ncclCommSplit(ring group [" + group_key(rg) + "])");
    owned_.push_back(rc);
    g->ulysses_comm = uc;
    g->ring_comm = rc;
    if (a2a_ctas > 0 && ug.size() > 1) {
      // the Ulysses chunk exchanges that overlap the attention kernel
      ncclConfig_t ocfg = NCCL_CONFIG_INITIALIZER;
      ocfg.blocking = 0;
      ocfg.maxCTAs = a2a_ctas;
      ocfg.minCTAs = 1;
      ncclComm_t oc = nullptr;
      split(/*color=*/r, /*key=*/u, &oc, &ocfg, "ncclCommSplit(ulysses overlap group [" + group_key(ug) + "])");
      owned_.push_back(oc);
      g->ulysses_overlap_comm = oc;
    }
    groups_.emplace(key, g);
    return g;
  }

  void all_to_all(const Groups& g, const std::vector<std::vector<A2APart>>& parts,
                  const std::vector<size_t>& bytes, cudaStream_t stream, bool overlapped) override {
    check_healthy();
    const NcclApi& api = nccl();
    auto comm = static_cast<ncclComm_t>(overlapped && g.ulysses_overlap_comm ? g.ulysses_overlap_comm
                                                                              : g.ulysses_comm);
    const int me = index_of(g.ulysses, g.rank);
    // Self part: a device copy (NCCL would also copy it).
    for (size_t t = 0; t < parts.size(); ++t)
      if (bytes[t] && parts[t][me].recv != parts[t][me].send)
        USPB_CUDA(cudaMemcpyAsync(parts[t][me].recv, parts[t][me].send, bytes[t],
                                  cudaMemcpyDeviceToDevice, stream));
    std::ostringstream what;
    what << "all_to_all call #" << a2a_seq_++ << " on ulysses group [" << group_key(g.ulysses) << "]";
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
    group_end(comm, what.str());
    watch_collective(stream, what.str());
  }

  void ring_shift(const Groups& g, const std::vector<const void*>& send,
                  const std::vector<void*>& recv, const std::vector<size_t>& bytes,
                  cudaStream_t stream) override {
    check_healthy();
    const NcclApi& api = nccl();
    auto comm = static_cast<ncclComm_t>(g.ring_comm);
    const int n = static_cast<int>(g.ring.size());
    const int i = index_of(g.ring, g.rank);
    std::ostringstream what;
    what << "ring_shift call #" << shift_seq_++ << " on ring group [" << group_key(g.ring) << "]";
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (size_t t = 0; t < send.size(); ++t) {
      if (!bytes[t]) continue;
      nccl_check(api.Send(send[t], bytes[t], ncclInt8, (i + 1) % n, comm, stream), "ncclSend");
      nccl_check(api.Recv(recv[t], bytes[t], ncclInt8, (i - 1 + n) % n, comm, stream), "ncclRecv");
    }
    group_end(comm, what.str());
    watch_collective(stream, what.str());
  }

 private:
  struct Pending {
    cudaEvent_t ev;
    std::string what;
    std::chrono::steady_clock::time_point t0;
  };

  void check_healthy() {
    std::lock_guard<std::mutex> lk(mu_);
    if (!failure_.empty()) throw Error(ErrorCode::kCommMismatch, failure_);
  }

  // Polls a non-blocking communicator until its pending operation (init,
  // split, group launch) finished; aborts everything on error or timeout.
  void wait_ready(ncclComm_t c, const std::string& what) {
    const NcclApi& api = nccl();
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
      ncclResult_t st = ncclSuccess;
      const ncclResult_t q = api.CommGetAsyncError(c, &st);
      if (q != ncclSuccess) st = q;
      if (st == ncclSuccess) return;
      if (st != ncclInProgress) fail(what + ": " + api.GetErrorString(st));
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > timeout_s_) {
        std::ostringstream os;
        os << what << " did not complete within " << timeout_s_ << " s (rank " << rank_ << " of " << n_
           << "): a peer did not reach it (mismatched or missing calls?)";
        fail(os.str());
      }
      if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }

  void split(int color, int key, ncclComm_t* out, ncclConfig_t* cfg, const std::string& what) {
    const ncclResult_t r = nccl().CommSplit(world_, color, key, out, cfg);
    if (r != ncclSuccess && r != ncclInProgress) fail(what + ": " + nccl().GetErrorString(r));
    wait_ready(world_, what);
    if (*out) wait_ready(*out, what);
  }

  void group_end(ncclComm_t comm, const std::string& what) {
    const ncclResult_t r = nccl().GroupEnd();
    if (r == ncclInProgress) {
      wait_ready(comm, what);
    } else if (r != ncclSuccess) {
      fail(what + ": ncclGroupEnd: " + nccl().GetErrorString(r));
    }
  }

  // Aborts every communicator and records the failure; throws it.
  [[noreturn]] void fail(const std::string& msg) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      abort_locked(msg);
    }
    throw Error(ErrorCode::kCommMismatch, msg);
  }
  void abort_locked(const std::string& msg) {
    if (failure_.empty()) failure_ = "NCCL transport: " + msg;
    if (aborted_) return;
    aborted_ = true;
    for (ncclComm_t c : owned_)
      if (c) nccl().CommAbort(c);
    if (world_) nccl().CommAbort(world_);
  }

  void watch_collective(cudaStream_t stream, const std::string& what) {
    cudaEvent_t ev = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!free_events_.empty()) {
        ev = free_events_.back();
        free_events_.pop_back();
      }
    }
    if (!ev) USPB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    USPB_CUDA(cudaEventRecord(ev, stream));
    std::lock_guard<std::mutex> lk(mu_);
    pending_.push_back({ev, what, std::chrono::steady_clock::now()});
  }

  // Watchdog: completed collectives are retired in order; the oldest one's
  // age is measured from when it became the oldest (a collective queued
  // behind a long attention step is not late until the step ends).
  void watch() {
    cudaSetDevice(device_);
    const NcclApi& api = nccl();
    std::unique_lock<std::mutex> lk(mu_);
    while (!stop_) {
      cv_.wait_for(lk, std::chrono::milliseconds(50));
      if (stop_ || aborted_) continue;
      while (!pending_.empty()) {
        const cudaError_t q = cudaEventQuery(pending_.front().ev);
        if (q == cudaErrorNotReady) break;
        free_events_.push_back(pending_.front().ev);
        pending_.pop_front();
        if (!pending_.empty()) pending_.front().t0 = std::chrono::steady_clock::now();
      }
      if (!pending_.empty()) {
        const double age = std::chrono::duration<double>(std::chrono::steady_clock::now() -
                                                         pending_.front().t0).count();
        if (age > timeout_s_) {
          std::ostringstream os;
          os << pending_.front().what << " on rank " << rank_ << " did not complete within " << timeout_s_
             << " s: a peer did not reach it (mismatched or missing calls?)";
          abort_locked(os.str());
          continue;
        }
      }
      std::vector<ncclComm_t> comms(owned_.begin(), owned_.end());
      comms.push_back(world_);
      for (ncclComm_t c : comms) {
        ncclResult_t st = ncclSuccess;
        if (!c || api.CommGetAsyncError(c, &st) != ncclSuccess) continue;
        if (st != ncclSuccess && st != ncclInProgress) {
          abort_locked(std::string("asynchronous NCCL error: ") + api.GetErrorString(st));
          break;
        }
      }
    }
  }

  int n_, rank_, device_;
  ncclComm_t world_ = nullptr;
  std::vector<ncclComm_t> owned_;
  std::map<std::tuple<std::vector<int>, std::vector<int>, int, int>, std::shared_ptr<Groups>> groups_;
  int64_t a2a_seq_ = 0, shift_seq_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Pending> pending_;
  std::vector<cudaEvent_t> free_events_;
  std::string failure_;
  bool aborted_ = false, stop_ = false;
  std::thread watchdog_;
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
