// transport.hpp — the two exchanges of the USP forward.
//
// Semantics follow the reference's simulated collectives:
//   all_to_all  RankCtx::all_to_all  (src/simcomm/world.hpp:134-166): part p
//               of every member goes to member p, received parts land in
//               member order;
//   ring_shift  RankCtx::ring_shift  (world.hpp:169-190): send to member
//               (i+1) % n, receive from (i-1+n) % n.
// Both are stream-ordered and collective over the group: every member must
// call them in the same order (world.cpp:135-165).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace uspb200 {

struct A2APart {
  const void* send;  // my part for member p
  void* recv;        // where member p's part for me lands
};

// The two sub-groups of one rank (ProcessMesh::ulysses_group / ring_group).
struct Groups {
  int rank = 0;
  std::vector<int> ulysses, ring;
  void* ulysses_comm = nullptr;  // transport-private (ncclComm_t for NCCL)
  void* ring_comm = nullptr;
  // NCCL: a second Ulysses communicator capped at a2a_ctas CTAs, for the
  // chunk exchanges that run while the attention kernel holds the other SMs
  void* ulysses_overlap_comm = nullptr;
};

class Transport {
 public:
  virtual ~Transport() = default;
  virtual int world_size() const = 0;
  // Collective over the world: builds this rank's sub-groups. ring_ctas /
  // a2a_ctas: how many CTAs (SMs) the ring exchange / an overlapped Ulysses
  // chunk exchange may use while the attention kernel runs (NCCL maxCTAs of
  // the ring communicator and of the capped Ulysses communicator; 0 = no
  // overlapped Ulysses exchanges). Engine sizes both from the shape alone,
  // so every rank passes the same values.
  virtual std::shared_ptr<Groups> make_groups(int rank, const std::vector<int>& ulysses_group,
                                              const std::vector<int>& ring_group, int ring_ctas,
                                              int a2a_ctas = 0) = 0;
  // Several tensors exchanged in one collective over the Ulysses group:
  // parts[t][p] for tensor t and member index p, bytes[t] per part.
  // overlapped: the exchange runs concurrently with the attention kernel
  // (NCCL uses the capped communicator).
  virtual void all_to_all(const Groups& g, const std::vector<std::vector<A2APart>>& parts,
                          const std::vector<size_t>& bytes, cudaStream_t stream, bool overlapped = false) = 0;
  // Ring shift of several buffers at once (K and V) over the ring group.
  virtual void ring_shift(const Groups& g, const std::vector<const void*>& send,
                          const std::vector<void*>& recv, const std::vector<size_t>& bytes,
                          cudaStream_t stream) = 0;
  // NCCL kernels occupy SMs (the attention grid leaves ring_ctas SMs for
  // them); the local and peer-memory transports use copy engines.
  virtual bool comm_uses_sms() const = 0;

  // Peer memory (optional): the address, valid on this rank's device, of
  // Ulysses member m's copy of the symmetric buffer holding `local`
  // (collective on first use of a buffer), and a two-phase handshake that
  // brackets direct stores into peers' buffers: ulysses_ready() = every
  // member's receive buffer is free, ulysses_done() = every member's stores
  // into mine have landed. Stream-ordered.
  virtual bool peer_memory() const { return false; }
  virtual void* ulysses_peer_ptr(const Groups&, const void*, int, size_t) { return nullptr; }
  virtual void ulysses_ready(const Groups&, cudaStream_t) {}
  virtual void ulysses_done(const Groups&, cudaStream_t) {}
  // An engine is being destroyed: drop whatever the transport keeps about
  // these local buffers (peer-memory mappings). Local, not collective.
  virtual void release_buffers(const std::vector<const void*>&) {}

  // Failure detection (the reference World's stuck/mismatched-collective
  // diagnosis, src/simcomm/world.cpp:89-113, 152-165). timeout: how long a
  // collective may wait for its peers (host rendezvous, NCCL init/split, a
  // collective's completion on the GPU) before the transport reports it.
  // status(): empty while healthy, else the failure (the comm is then dead:
  // NCCL communicators aborted, every later collective throws it again).
  virtual void set_timeout(double seconds) { timeout_s_ = seconds; }
  double timeout() const { return timeout_s_; }
  virtual std::string status() { return {}; }
  // Host-side rendezvous of `rank` on group `members` under `signature`
  // (tests: the local transport's mismatch / deadlock diagnosis without a GPU).
  virtual void debug_rendezvous(const std::vector<int>&, int, const std::string&) {
    throw_invalid("debug_rendezvous: only the local transport has a host rendezvous");
  }

 protected:
  double timeout_s_ = default_timeout();
  static double default_timeout();
};

std::unique_ptr<Transport> make_local_transport(int world_size);
// Host all-gather used to bootstrap the peer-memory transport: every rank
// contributes `bytes` at `send`; `recv` receives world_size * bytes in rank
// order. Returns 0 on success.
using AllGatherFn = int (*)(const void* send, void* recv, size_t bytes, void* ctx);
std::unique_ptr<Transport> make_p2p_transport(int world_size, int rank, int device, AllGatherFn allgather,
                                              void* ctx);
std::unique_ptr<Transport> make_nccl_transport(const unsigned char unique_id[128],
                                               int world_size, int rank, int device);
void nccl_unique_id(unsigned char out[128]);

}  // namespace uspb200
