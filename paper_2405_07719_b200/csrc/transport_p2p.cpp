// transport_p2p.cpp — peer-memory transport: one process per GPU, no NCCL.
//
// The two exchanges of the USP forward/backward (RankCtx::all_to_all and
// RankCtx::ring_shift, reference src/simcomm/world.hpp:134-190) as direct
// writes into the receivers' buffers over NVLink / NVSwitch:
//   * every receive buffer the engine hands to a collective is exported once
//     with cudaIpcGetMemHandle and opened by the other ranks (lazily, at the
//     first collective that uses it — all ranks issue the same collectives in
//     the same order on symmetric allocations, so the exchange is collective);
//   * data moves with stream-ordered cudaMemcpyAsync into the peer mapping:
//     copy engines, no SMs, so a ring shift runs beside an attention kernel
//     that owns every SM (comm_uses_sms() == false);
//   * ordering across processes uses GPU stream memory operations on a small
//     IPC-shared signal array: the receiver publishes "my buffer is free for
//     collective e" (cuStreamWriteValue64 into the sender's signals), the
//     sender waits for it (cuStreamWaitValue64), copies, and publishes "data
//     of collective e landed"; the receiver's stream waits for that before
//     its consumers run. Nothing blocks a host thread after setup.
// Bootstrap (handle exchange) goes through a caller-provided host all-gather
// (usp_allgather_fn: torch.distributed, MPI, a file system ...). Ranks of
// the same process share raw pointers instead of IPC handles.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <cstring>
#include <map>
#include <set>
#include <mutex>
#include <string>
#include <vector>

#include "plan.hpp"
#include "transport.hpp"

namespace uspb200 {

#define USPB_P2P_CUDA(x)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw Error(ErrorCode::kInternal, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
using PtrAttrFn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);

struct DriverApi {
  WriteValueFn write64 = nullptr;
  WaitValueFn wait64 = nullptr;
  AddrRangeFn addr_range = nullptr;
  PtrAttrFn ptr_attr = nullptr;
};

const DriverApi& driver() {
  static DriverApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    auto get = [&](const char* name) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !p) {
        if (err.empty()) err = std::string("driver entry point unavailable: ") + name;
        return nullptr;
      }
      return p;
    };
    api.write64 = reinterpret_cast<WriteValueFn>(get("cuStreamWriteValue64"));
    api.wait64 = reinterpret_cast<WaitValueFn>(get("cuStreamWaitValue64"));
    api.addr_range = reinterpret_cast<AddrRangeFn>(get("cuMemGetAddressRange"));
    api.ptr_attr = reinterpret_cast<PtrAttrFn>(get("cuPointerGetAttribute"));
  });
  if (!err.empty()) throw Error(ErrorCode::kInternal, err);
  return api;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Error(ErrorCode::kInternal, std::string(what) + " failed (" + std::to_string(r) + ")");
}

// What one rank publishes about one of its allocations.
struct Published {
  cudaIpcMemHandle_t handle;
  uint64_t base;
  uint64_t pid;
  uint64_t bytes;
};

int index_in(const std::vector<int>& g, int rank) {
  for (size_t i = 0; i < g.size(); ++i)
    if (g[i] == rank) return static_cast<int>(i);
  throw Error(ErrorCode::kInternal, "rank not in its own group");
}

}  // namespace

class P2PTransport final : public Transport {
 public:
  P2PTransport(int world, int rank, int device, AllGatherFn allgather, void* ctx)
      : n_(world), rank_(rank), device_(device), allgather_(allgather), ctx_(ctx) {
    if (world < 1 || rank < 0 || rank >= world) throw_invalid("p2p transport: rank outside the world");
    if (!allgather_) throw_invalid("p2p transport needs a host all-gather callback");
    driver();
    USPB_P2P_CUDA(cudaSetDevice(device_));
    // signals[kind][group][rank]: kind 0 = ready (receiver's buffer free),
    // 1 = done (sender's data landed); group 0 = Ulysses row, 1 = ring column
    USPB_P2P_CUDA(cudaMalloc(&signals_, kSignalBytes()));
    USPB_P2P_CUDA(cudaMemset(signals_, 0, kSignalBytes()));
    USPB_P2P_CUDA(cudaDeviceSynchronize());
    peer_signals_ = open_peers(signals_, kSignalBytes());
  }

  ~P2PTransport() override {
    cudaSetDevice(device_);
    for (auto& kv : regs_) close_peers(kv.second.peers);
    close_peers(peer_signals_);
    if (signals_) cudaFree(signals_);
  }

  int world_size() const override { return n_; }
  bool comm_uses_sms() const override { return false; }  // copy engines + stream memops only

  std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ug, const std::vector<int>& rg, int,
                                      int) override {
    if (rank != rank_) throw_invalid("p2p transport: engine rank differs from the transport's rank");
    auto g = std::make_shared<Groups>();
    g->rank = rank;
    g->ulysses = ug;
    g->ring = rg;
    return g;
  }

  void release_buffers(const std::vector<const void*>& bufs) override {
    const DriverApi& api = driver();
    for (const void* b : bufs) {
      if (!b) continue;
      CUdeviceptr base = 0;
      size_t size = 0;
      if (api.addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(b)) != CUDA_SUCCESS) continue;
      auto it = regs_.find(base);
      if (it == regs_.end()) continue;
      close_peers(it->second.peers);
      regs_.erase(it);
    }
  }

  void all_to_all(const Groups& g, const std::vector<std::vector<A2APart>>& parts,
                  const std::vector<size_t>& bytes, cudaStream_t stream, bool) override {
    const int me = index_in(g.ulysses, g.rank);
    const uint64_t e = ++epoch_[0];
    // destinations in every peer: where MY part lands in peer p's buffer is
    // where my own (self) part lands in mine — the layouts are symmetric
    std::vector<std::vector<char*>> dst(parts.size());
    for (size_t t = 0; t < parts.size(); ++t)
      for (size_t p = 0; p < g.ulysses.size(); ++p)
        dst[t].push_back(p == size_t(me) || !bytes[t] ? nullptr
                                                       : remote(parts[t][me].recv, g.ulysses[p], bytes[t]));
    for (int peer : g.ulysses)
      if (peer != rank_) signal(stream, peer, 0, 0, e);  // my receive buffers are free
    for (size_t t = 0; t < parts.size(); ++t)  // self part
      if (bytes[t] && parts[t][me].recv != parts[t][me].send)
        USPB_P2P_CUDA(cudaMemcpyAsync(parts[t][me].recv, parts[t][me].send, bytes[t], cudaMemcpyDeviceToDevice,
                                      stream));
    for (size_t p = 0; p < g.ulysses.size(); ++p) {
      const int peer = g.ulysses[p];
      if (peer == rank_) continue;
      wait(stream, 0, 0, peer, e);  // peer's buffers are free
      for (size_t t = 0; t < parts.size(); ++t)
        if (bytes[t])
          USPB_P2P_CUDA(cudaMemcpyAsync(dst[t][p], parts[t][p].send, bytes[t], cudaMemcpyDefault, stream));
      signal(stream, peer, 1, 0, e);  // my data for peer landed
    }
    for (int peer : g.ulysses)
      if (peer != rank_) wait(stream, 1, 0, peer, e);  // every peer's data for me landed
  }

  bool peer_memory() const override { return true; }
  void* ulysses_peer_ptr(const Groups& g, const void* local, int member, size_t bytes) override {
    return remote(local, g.ulysses.at(member), bytes);
  }
  void ulysses_ready(const Groups& g, cudaStream_t stream) override {
    const uint64_t e = ++epoch_[0];
    for (int peer : g.ulysses)
      if (peer != rank_) signal(stream, peer, 0, 0, e);
    for (int peer : g.ulysses)
      if (peer != rank_) wait(stream, 0, 0, peer, e);
  }
  void ulysses_done(const Groups& g, cudaStream_t stream) override {
    const uint64_t e = epoch_[0];
    for (int peer : g.ulysses)
      if (peer != rank_) signal(stream, peer, 1, 0, e);
    for (int peer : g.ulysses)
      if (peer != rank_) wait(stream, 1, 0, peer, e);
  }

  void ring_shift(const Groups& g, const std::vector<const void*>& send, const std::vector<void*>& recv,
                  const std::vector<size_t>& bytes, cudaStream_t stream) override {
    const int n = static_cast<int>(g.ring.size());
    const uint64_t e = ++epoch_[1];
    if (n == 1) return;
    const int i = index_in(g.ring, g.rank);
    const int next = g.ring[(i + 1) % n], prev = g.ring[(i - 1 + n) % n];
    std::vector<char*> dst(send.size());
    for (size_t t = 0; t < send.size(); ++t) dst[t] = bytes[t] ? remote(recv[t], next, bytes[t]) : nullptr;
    signal(stream, prev, 0, 1, e);  // prev may write into my receive buffers
    wait(stream, 0, 1, next, e);    // next's receive buffers are free
    for (size_t t = 0; t < send.size(); ++t)
      if (bytes[t]) USPB_P2P_CUDA(cudaMemcpyAsync(dst[t], send[t], bytes[t], cudaMemcpyDefault, stream));
    signal(stream, next, 1, 1, e);  // landed in next
    wait(stream, 1, 1, prev, e);    // prev's data landed in mine
  }

 private:
  size_t kSignalBytes() const { return sizeof(uint64_t) * 2 * 2 * size_t(n_); }
  size_t sig_off(int kind, int group, int from) const {
    return sizeof(uint64_t) * ((size_t(kind) * 2 + group) * n_ + from);
  }
  // rank `to` learns (kind, group, from = me) = e
  void signal(cudaStream_t st, int to, int kind, int group, uint64_t e) {
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(peer_signals_.at(to)) + sig_off(kind, group, rank_);
    cu_check(driver().write64(reinterpret_cast<CUstream>(st), a, e, 0), "cuStreamWriteValue64");
  }
  // my stream waits until (kind, group, from) >= e in my own signals
  void wait(cudaStream_t st, int kind, int group, int from, uint64_t e) {
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(signals_) + sig_off(kind, group, from);
    cu_check(driver().wait64(reinterpret_cast<CUstream>(st), a, e, CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue64");
  }

  // Peer `peer`'s address of my local receive address `local` (bytes long).
  char* remote(const void* local, int peer, size_t bytes) {
    const DriverApi& api = driver();
    CUdeviceptr base = 0;
    size_t size = 0;
    cu_check(api.addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(local)), "cuMemGetAddressRange");
    unsigned long long id = 0;
    cu_check(api.ptr_attr(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, base), "cuPointerGetAttribute");
    Reg& r = regs_[base];
    if (r.buffer_id != id) {  // new (or re-allocated) buffer: collective registration
      close_peers(r.peers);
      r.peers = open_peers(reinterpret_cast<void*>(base), size);
      r.buffer_id = id;
      r.bytes = size;
    }
    const size_t off = reinterpret_cast<uintptr_t>(local) - base;
    if (off + bytes > r.bytes) throw Error(ErrorCode::kInternal, "p2p transport: transfer exceeds its buffer");
    return static_cast<char*>(r.peers.at(peer)) + off;
  }

  // Collective: every rank publishes (handle, base, pid) of its allocation
  // and maps everybody else's.
  std::vector<void*> open_peers(void* base, size_t bytes) {
    Published mine{};
    USPB_P2P_CUDA(cudaIpcGetMemHandle(&mine.handle, base));
    mine.base = reinterpret_cast<uint64_t>(base);
    mine.pid = static_cast<uint64_t>(getpid());
    mine.bytes = bytes;
    std::vector<Published> all(n_);
    if (allgather_(&mine, all.data(), sizeof(Published), ctx_) != 0)
      throw Error(ErrorCode::kInternal, "p2p transport: host all-gather failed");
    std::vector<void*> peers(n_, nullptr);
    for (int r = 0; r < n_; ++r) {
      if (r == rank_) {
        peers[r] = base;
      } else if (all[r].pid == mine.pid) {
        peers[r] = reinterpret_cast<void*>(all[r].base);  // same process: plain pointer
      } else {
        if (all[r].bytes != bytes) throw Error(ErrorCode::kCommMismatch, "p2p transport: asymmetric buffers");
        void* p = nullptr;
        USPB_P2P_CUDA(cudaIpcOpenMemHandle(&p, all[r].handle, cudaIpcMemLazyEnablePeerAccess));
        peers[r] = p;
        opened_.insert(p);
      }
    }
    return peers;
  }
  void close_peers(std::vector<void*>& peers) {
    for (void* p : peers)
      if (p && opened_.erase(p)) cudaIpcCloseMemHandle(p);
    peers.clear();
  }

  struct Reg {
    unsigned long long buffer_id = 0;
    size_t bytes = 0;
    std::vector<void*> peers;
  };

  int n_, rank_, device_;
  AllGatherFn allgather_;
  void* ctx_;
  void* signals_ = nullptr;
  std::vector<void*> peer_signals_;
  std::map<CUdeviceptr, Reg> regs_;
  std::set<void*> opened_;
  uint64_t epoch_[2] = {0, 0};
};

std::unique_ptr<Transport> make_p2p_transport(int world_size, int rank, int device, AllGatherFn allgather,
                                              void* ctx) {
  return std::make_unique<P2PTransport>(world_size, rank, device, allgather, ctx);
}

}  // namespace uspb200
