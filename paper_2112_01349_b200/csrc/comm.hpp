// comm.hpp — collectives between rank contexts (dba/comms.hpp:35-234 role).
//
// Three backends behind one interface, all in-place on device buffers and
// stream-ordered on the calling rank's stream:
//   SelfComm   K = 1: every collective is the identity.
//   GroupComm  K ranks inside one process (one host thread per rank, the
//              reference's run_on_workers model, dba/comms.hpp:214-234),
//              ranks on one or several GPUs. A host rendezvous publishes each
//              rank's device buffer, then every rank sums the K deposited
//              buffers in ascending rank order on its own stream
//              (k_sum_slots) — bit-identical to WorkerGroup::allreduce_sum
//              (dba/comms.hpp:76-81) and rank-identical by construction.
//              Cross-rank ordering uses CUDA events, so no host<->device sync
//              is needed. Also carries the reference's call-sequence / kind /
//              length validation and rendezvous timeout (dba/comms.hpp:136-193).
//   NcclComm   one process per GPU (torchrun), ncclAllReduce over NVLink /
//              NVSwitch on the rank's stream.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace dbag {

enum class DType { f32, f64 };
inline std::size_t dsize(DType t) { return t == DType::f64 ? 8 : 4; }

// One device-side all-reduce site (peer.cuh k_peer_allreduce): every rank's
// deposit slots and arrival epochs, mapped into this rank's address space.
struct PeerSite {
  static constexpr int kMaxPeers = 16;
  int k = 0, rank = 0, nslice = 0;
  std::int64_t slice = 0;               // elements per slice (one CTA each)
  std::int64_t len = 0;                 // slot capacity in elements
  void* slot[2][kMaxPeers] = {};        // rank p's deposit buffers, by epoch parity
  unsigned* flag[kMaxPeers] = {};       // rank p's per-slice arrival epochs
  unsigned* epoch = nullptr;            // this rank's per-slice epoch (local)
  // Production waits (the DPCG graph): give up on a peer after timeout_ns
  // (SolverConfig::collective_timeout) and OR bit p of an absent rank p into
  // *failed; once *failed is set, later waits return at once so the graph
  // drains and the host raises CollectiveError. 0 / null: wait indefinitely.
  unsigned long long timeout_ns = 0;
  int* failed = nullptr;
  // Slice plan, a function of (max_len, k, shared) only, so every rank
  // agrees: slices of whole 9-vectors (one camera each). One rank per device:
  // up to 148 slices (one CTA per SM folds and exchanges its cameras). Ranks
  // sharing a device: at most kSharedCap per rank — a rank's spinning CTAs wait for
  // the other ranks' passes on the same SMs, so few and small is better
  // there (and k x kSharedCap stays co-resident).
#ifndef DBAG_PEER_SHARED_CAP
#define DBAG_PEER_SHARED_CAP 48
#endif
  static constexpr int kSharedCap = DBAG_PEER_SHARED_CAP;
  static void plan(std::int64_t max_len, int k, bool shared, std::int64_t* slice, int* nslice) {
    const std::int64_t units = std::max<std::int64_t>(1, (max_len + 8) / 9);
    const std::int64_t cap = shared ? kSharedCap : std::max<std::int64_t>(1, std::min<std::int64_t>(148, 512 / std::max(k, 1)));
    const std::int64_t per = (units + cap - 1) / cap;
    *slice = per * 9;
    *nslice = static_cast<int>((units + per - 1) / per);
  }
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // data := sum over ranks (in place, device pointer, stream-ordered)
  virtual void allreduce_sum(void* data, std::int64_t count, DType t, cudaStream_t s) = 0;
  // data := max over ranks
  virtual void allreduce_max(void* data, std::int64_t count, DType t, cudaStream_t s) = 0;
  // Collective: set up a device-side all-reduce site for vectors of up to
  // max_len elements (false where the backend has none; every rank gets the
  // same answer).
  virtual bool make_peer_site(std::int64_t /*max_len*/, DType /*t*/, PeerSite* /*out*/) { return false; }
  // SolverConfig::collective_timeout (dba/solver.hpp:54): also bounds the
  // device-side peer waits of the DPCG graph (PeerSite::timeout_ns).
  virtual std::chrono::milliseconds timeout() const { return std::chrono::milliseconds(60000); }
};

class SelfComm final : public Comm {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  void allreduce_sum(void*, std::int64_t, DType, cudaStream_t) override {}
  void allreduce_max(void*, std::int64_t, DType, cudaStream_t) override {}
};

// Shard `rank` of `size` evaluated on its own: collectives are the identity
// (EdgeEvaluator / assemble_local semantics, one partition's contribution).
class LocalComm final : public Comm {
 public:
  LocalComm(int rank, int size) : rank_(rank), size_(size) {}
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void allreduce_sum(void*, std::int64_t, DType, cudaStream_t) override {}
  void allreduce_max(void*, std::int64_t, DType, cudaStream_t) override {}

 private:
  int rank_, size_;
};

// Shared state of an in-process group of K ranks.
class Group {
 public:
  // Up to kMaxRanks ranks (the slot pointers travel as one kernel argument);
  // timeout = SolverConfig::collective_timeout (dba/solver.hpp:54, 60 s).
  static constexpr int kMaxRanks = 256;
  Group(int k, std::vector<int> devices, std::chrono::milliseconds timeout = std::chrono::milliseconds(60000));
  ~Group();
  int size() const { return k_; }
  std::chrono::milliseconds timeout() const { return timeout_; }
  int device_of(int rank) const { return devices_[static_cast<std::size_t>(rank)]; }

  void allreduce(int rank, void* data, std::int64_t count, DType t, bool is_max, cudaStream_t s);
  // WorkerGroup::barrier (dba/comms.hpp:56-63): validated rendezvous.
  void barrier(int rank);
  // WorkerGroup::sequence (dba/comms.hpp:52-53): collectives entered by rank.
  std::uint64_t sequence(int rank) const;
  void abort(const std::string& why);
  bool aborted() const;
  bool make_peer_site(int rank, std::int64_t max_len, DType t, PeerSite* out);

 private:
  struct Slot {
    void* ptr = nullptr;
    std::int64_t count = 0;
    int kind = 0;  // kBarrier, or all-reduce: dtype * 2 + is_max
    std::uint64_t seq = 0;
  };
  static constexpr int kBarrier = 8;
  void rendezvous(int rank);
  void validate(int rank, std::int64_t count, int kind);
  void* scratch(int rank, std::size_t bytes);

  int k_;
  std::vector<int> devices_;
  std::chrono::milliseconds timeout_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  std::uint64_t gen_ = 0;
  std::vector<bool> here_;
  bool aborted_ = false;
  std::string why_;
  std::vector<Slot> slots_;
  std::vector<std::uint64_t> seq_;
  std::vector<cudaEvent_t> ready_, done_;
  std::vector<void*> scratch_;
  std::vector<std::size_t> scratch_bytes_;
  std::vector<std::vector<void*>> peer_mem_;  // per rank: peer-site allocations (freed with the group)
  std::vector<PeerSite> peer_dep_;            // per rank: its own buffers, published for the others
  std::vector<int> peer_ok_;                  // per rank: its site self-check
};

// Self-check of a peer site (peer.cuh k_peer_selftest); run() is collective.
class PeerCheck {
 public:
  PeerCheck(const PeerSite& s, int device);
  ~PeerCheck();
  PeerCheck(const PeerCheck&) = delete;
  PeerCheck& operator=(const PeerCheck&) = delete;
  int run(const PeerSite& s);

 private:
  int device_;
  cudaStream_t st_ = nullptr;
  double* buf_ = nullptr;
  int* bad_ = nullptr;
};

class GroupComm final : public Comm {
 public:
  GroupComm(Group* g, int rank) : g_(g), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return g_->size(); }
  void allreduce_sum(void* d, std::int64_t n, DType t, cudaStream_t s) override { g_->allreduce(rank_, d, n, t, false, s); }
  void allreduce_max(void* d, std::int64_t n, DType t, cudaStream_t s) override { g_->allreduce(rank_, d, n, t, true, s); }
  bool make_peer_site(std::int64_t max_len, DType t, PeerSite* out) override {
    return g_->make_peer_site(rank_, max_len, t, out);
  }
  std::chrono::milliseconds timeout() const override { return g_->timeout(); }

 private:
  Group* g_;
  int rank_;
};

class NcclComm final : public Comm {
 public:
  NcclComm(int rank, int nranks, const unsigned char* id128);
  ~NcclComm() override;
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void allreduce_sum(void* d, std::int64_t n, DType t, cudaStream_t s) override;
  void allreduce_max(void* d, std::int64_t n, DType t, cudaStream_t s) override;
  bool make_peer_site(std::int64_t max_len, DType t, PeerSite* out) override;
  std::chrono::milliseconds timeout() const override { return timeout_; }
  void set_timeout(std::chrono::milliseconds t) { timeout_ = t; }

 private:
  std::chrono::milliseconds timeout_{60000};
  ncclComm_t comm_ = nullptr;
  int rank_, size_;
  std::vector<void*> own_;    // local peer-site allocations
  std::vector<void*> opened_; // peers' allocations opened through CUDA IPC
};

}  // namespace dbag
