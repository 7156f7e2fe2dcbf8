// comm.cu — Group (in-process ranks) and NCCL backends of comm.hpp.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "comm.hpp"
#include "peer.cuh"

namespace dbag {
namespace {

constexpr int kMaxGroup = Group::kMaxRanks;
struct SlotPtrs {  // 2 KB: inside the 4 KB kernel-parameter limit
  const void* p[kMaxGroup];
};

// Ascending-rank fold of the K deposited buffers (dba/comms.hpp:76-81):
// acc = s0; acc += s1; ... (sum) or acc = max(acc, s_r) (max).
template <class T, bool MAX>
__global__ void k_fold_slots(std::int64_t len, int k, SlotPtrs sp, T* __restrict__ out) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(sp.p[0])[i];
    for (int r = 1; r < k; ++r) {
      const T v = static_cast<const T*>(sp.p[r])[i];
      acc = MAX ? (v > acc ? v : acc) : acc + v;
    }
    out[i] = acc;
  }
}

ncclDataType_t nccl_type(DType t) { return t == DType::f64 ? ncclDouble : ncclFloat; }

#define DBAG_NCCL(expr)                                                                           \
  do {                                                                                            \
    ncclResult_t _r = (expr);                                                                     \
    if (_r != ncclSuccess)                                                                        \
      throw ::dbag::Error(DBAG_NCCL_ERROR, std::string(#expr " failed: ") + ncclGetErrorString(_r)); \
  } while (0)

}  // namespace

Group::Group(int k, std::vector<int> devices, std::chrono::milliseconds timeout)
    : k_(k), devices_(std::move(devices)), timeout_(timeout) {
  if (k < 1) throw Error(DBAG_INVALID_ARGUMENT, "worker group needs at least one rank");
  if (k > kMaxGroup)
    throw Error(DBAG_INVALID_ARGUMENT, "in-process group supports at most " + std::to_string(kMaxGroup) + " ranks");
  if (devices_.empty()) devices_.push_back(0);
  std::vector<int> dev(static_cast<std::size_t>(k));
  for (int r = 0; r < k; ++r) dev[static_cast<std::size_t>(r)] = devices_[static_cast<std::size_t>(r) % devices_.size()];
  devices_ = dev;
  here_.assign(static_cast<std::size_t>(k), false);
  slots_.resize(static_cast<std::size_t>(k));
  seq_.assign(static_cast<std::size_t>(k), 0);
  ready_.resize(static_cast<std::size_t>(k));
  done_.resize(static_cast<std::size_t>(k));
  scratch_.assign(static_cast<std::size_t>(k), nullptr);
  scratch_bytes_.assign(static_cast<std::size_t>(k), 0);
  peer_mem_.resize(static_cast<std::size_t>(k));
  peer_dep_.resize(static_cast<std::size_t>(k));
  peer_ok_.assign(static_cast<std::size_t>(k), 0);
  int prev = 0;
  DBAG_CUDA(cudaGetDevice(&prev));
  for (int r = 0; r < k; ++r) {
    DBAG_CUDA(cudaSetDevice(device_of(r)));
    DBAG_CUDA(cudaEventCreateWithFlags(&ready_[static_cast<std::size_t>(r)], cudaEventDisableTiming));
    DBAG_CUDA(cudaEventCreateWithFlags(&done_[static_cast<std::size_t>(r)], cudaEventDisableTiming));
  }
  // Peer access between the distinct devices of the group (NVLink / NVSwitch).
  std::vector<int> uniq = devices_;
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  for (int a : uniq) {
    DBAG_CUDA(cudaSetDevice(a));
    for (int b : uniq) {
      if (a == b) continue;
      int ok = 0;
      DBAG_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok) throw Error(DBAG_CUDA_ERROR, "devices " + std::to_string(a) + " and " + std::to_string(b) + " lack peer access");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DBAG_CUDA(e);
      (void)cudaGetLastError();
    }
  }
  DBAG_CUDA(cudaSetDevice(prev));
}

Group::~Group() {
  for (int r = 0; r < k_; ++r) {
    cudaSetDevice(device_of(r));
    cudaEventDestroy(ready_[static_cast<std::size_t>(r)]);
    cudaEventDestroy(done_[static_cast<std::size_t>(r)]);
    if (scratch_[static_cast<std::size_t>(r)]) cudaFree(scratch_[static_cast<std::size_t>(r)]);
    for (void* m : peer_mem_[static_cast<std::size_t>(r)]) cudaFree(m);
  }
}

namespace {
// One allocation per rank and site: slot parity 0 | slot parity 1 | arrival
// epochs | local epochs (zeroed, complete before it is published).
struct PeerAlloc {
  void* base = nullptr;
  std::size_t slot_bytes = 0;
};
PeerAlloc peer_alloc(std::int64_t max_len, DType t, int nslice) {
  PeerAlloc a;
  a.slot_bytes = (static_cast<std::size_t>(std::max<std::int64_t>(max_len, 1)) * dsize(t) + 255) / 256 * 256;
  const std::size_t bytes = 2 * a.slot_bytes + 2 * static_cast<std::size_t>(nslice) * sizeof(unsigned);
  DBAG_CUDA(cudaMalloc(&a.base, bytes));
  DBAG_CUDA(cudaMemset(a.base, 0, bytes));
  DBAG_CUDA(cudaDeviceSynchronize());
  return a;
}
void peer_fill(const PeerAlloc& a, int nslice, int p, PeerSite* s, bool local) {
  char* b = static_cast<char*>(a.base);
  s->slot[0][p] = b;
  s->slot[1][p] = b + a.slot_bytes;
  s->flag[p] = reinterpret_cast<unsigned*>(b + 2 * a.slot_bytes);
  if (local) s->epoch = s->flag[p] + nslice;
}
}  // namespace

bool Group::make_peer_site(int rank, std::int64_t max_len, DType t, PeerSite* out) {
  if (k_ < 2 || k_ > PeerSite::kMaxPeers) return false;  // same answer on every rank
  PeerSite s;
  s.k = k_;
  s.rank = rank;
  std::vector<int> devs(devices_);
  std::sort(devs.begin(), devs.end());
  const bool shared = std::adjacent_find(devs.begin(), devs.end()) != devs.end();
  PeerSite::plan(max_len, s.k, shared, &s.slice, &s.nslice);
  s.len = std::max<std::int64_t>(max_len, 1);
  int prev = 0;
  DBAG_CUDA(cudaGetDevice(&prev));
  DBAG_CUDA(cudaSetDevice(device_of(rank)));
  const PeerAlloc a = peer_alloc(max_len, t, s.nslice);
  DBAG_CUDA(cudaSetDevice(prev));
  auto check = std::make_unique<PeerCheck>(s, device_of(rank));
  {
    std::lock_guard<std::mutex> lk(mu_);
    peer_mem_[static_cast<std::size_t>(rank)].push_back(a.base);
    PeerSite mine = s;
    peer_fill(a, s.nslice, rank, &mine, true);
    peer_dep_[static_cast<std::size_t>(rank)] = mine;
  }
  rendezvous(rank);
  {
    std::lock_guard<std::mutex> lk(mu_);
    for (int p = 0; p < k_; ++p) {
      const PeerSite& d = peer_dep_[static_cast<std::size_t>(p)];
      s.slot[0][p] = d.slot[0][p];
      s.slot[1][p] = d.slot[1][p];
      s.flag[p] = d.flag[p];
    }
    s.epoch = peer_dep_[static_cast<std::size_t>(rank)].epoch;
  }
  rendezvous(rank);  // every rank has read the table before the next site overwrites it
  // the same self-check as the IPC path (k_peer_selftest), agreed over the group
  const int ok = check->run(s);
  check.reset();  // freed before the rendezvous: no rank frees while another's check may still wait on it
  {
    std::lock_guard<std::mutex> lk(mu_);
    peer_ok_[static_cast<std::size_t>(rank)] = ok;
  }
  rendezvous(rank);
  int all = 1;
  {
    std::lock_guard<std::mutex> lk(mu_);
    for (int v : peer_ok_) all = std::min(all, v);
  }
  rendezvous(rank);  // peer_ok_ read by every rank before the next site
  if (!all) return false;
  *out = s;
  return true;
}

// Buffers of the site self-check, allocated before any rank's check kernel
// can be spinning: cudaMalloc / cudaFree may wait for the whole device, and
// with several ranks on one device that wait would starve the peer the
// spinning kernel is waiting for.
PeerCheck::PeerCheck(const PeerSite& s, int device) : device_(device) {
  int prev = 0;
  DBAG_CUDA(cudaGetDevice(&prev));
  DBAG_CUDA(cudaSetDevice(device));
  DBAG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  DBAG_CUDA(cudaMalloc(&buf_, static_cast<std::size_t>(s.slice) * std::max(s.nslice, 1) * sizeof(double)));
  DBAG_CUDA(cudaMalloc(&bad_, sizeof(int)));
  DBAG_CUDA(cudaMemset(bad_, 0, sizeof(int)));
  DBAG_CUDA(cudaDeviceSynchronize());
  DBAG_CUDA(cudaSetDevice(prev));
}
PeerCheck::~PeerCheck() {
  cudaSetDevice(device_);
  cudaFree(buf_);
  cudaFree(bad_);
  cudaStreamDestroy(st_);
}
// 1 if two all-reduces through the site give the closed-form sums on this
// rank (2 s peer timeout); DBAG_PEER_SELFTEST_FAIL=1 forces 0 (tests of the
// fallback). Collective: every rank of the site runs it; no allocation or
// device-wide synchronization between the launch and the stream sync.
int PeerCheck::run(const PeerSite& s) {
  int prev = 0;
  DBAG_CUDA(cudaGetDevice(&prev));
  DBAG_CUDA(cudaSetDevice(device_));
  dev::k_peer_selftest<double><<<s.nslice, dev::kPeerThreads, 0, st_>>>(s, buf_, 2, bad_);
  DBAG_LAUNCH_CHECK();
  int h = 1;
  DBAG_CUDA(cudaMemcpyAsync(&h, bad_, sizeof(int), cudaMemcpyDeviceToHost, st_));
  DBAG_CUDA(cudaStreamSynchronize(st_));
  DBAG_CUDA(cudaSetDevice(prev));
  const char* f = std::getenv("DBAG_PEER_SELFTEST_FAIL");
  if (f && std::string(f) == "1") return 0;
  if (h) std::fprintf(stderr, "[dbag] peer all-reduce self-check failed on rank %d of %d\n", s.rank, s.k);
  return h ? 0 : 1;
}

void Group::abort(const std::string& why) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!aborted_) {
    aborted_ = true;
    why_ = why;
  }
  cv_.notify_all();
}

bool Group::aborted() const {
  std::lock_guard<std::mutex> lk(mu_);
  return aborted_;
}

// Generation barrier with a timeout that names the absent ranks
// (dba/comms.hpp:136-165).
void Group::rendezvous(int rank) {
  std::unique_lock<std::mutex> lk(mu_);
  if (aborted_) throw Error(DBAG_COLLECTIVE, "collective aborted: " + why_);
  here_[static_cast<std::size_t>(rank)] = true;
  if (++arrived_ == k_) {
    arrived_ = 0;
    std::fill(here_.begin(), here_.end(), false);
    ++gen_;
    cv_.notify_all();
    return;
  }
  const std::uint64_t g = gen_;
  while (gen_ == g && !aborted_) {
    if (cv_.wait_for(lk, timeout_) == std::cv_status::timeout && gen_ == g && !aborted_) {
      std::string missing;
      for (int r = 0; r < k_; ++r)
        if (!here_[static_cast<std::size_t>(r)]) missing += (missing.empty() ? "" : ", ") + std::to_string(r);
      aborted_ = true;
      why_ = "collective timeout at sequence " + std::to_string(seq_[static_cast<std::size_t>(rank)]) +
             "; still waiting on ranks: " + missing;
      cv_.notify_all();
      throw Error(DBAG_COLLECTIVE, why_);
    }
  }
  if (aborted_) throw Error(DBAG_COLLECTIVE, "collective aborted: " + why_);
}

// Call-sequence / kind / length agreement (dba/comms.hpp:167-193).
void Group::validate(int rank, std::int64_t count, int kind) {
  std::lock_guard<std::mutex> lk(mu_);
  const std::uint64_t seq = seq_[static_cast<std::size_t>(rank)];
  for (int r = 0; r < k_; ++r) {
    const Slot& s = slots_[static_cast<std::size_t>(r)];
    std::string problem;
    if (s.seq != seq) problem = "is at call sequence " + std::to_string(s.seq) + ", this rank at " + std::to_string(seq);
    else if ((s.kind == kBarrier) != (kind == kBarrier) || ((s.kind ^ kind) & 1))
      problem = "entered a different collective kind";
    else if (s.kind != kind) problem = "passed a different element type";
    else if (s.count != count)
      problem = "passed length " + std::to_string(s.count) + ", this rank passed " + std::to_string(count);
    if (!problem.empty()) {
      aborted_ = true;
      why_ = "collective mismatch: rank " + std::to_string(r) + " " + problem;
      cv_.notify_all();
      throw Error(DBAG_COLLECTIVE, why_);
    }
  }
}

void Group::barrier(int rank) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (aborted_) throw Error(DBAG_COLLECTIVE, "collective aborted: " + why_);
    slots_[static_cast<std::size_t>(rank)] = Slot{nullptr, 0, kBarrier, ++seq_[static_cast<std::size_t>(rank)]};
  }
  rendezvous(rank);
  validate(rank, 0, kBarrier);
  rendezvous(rank);  // slots stay valid until every rank validated
}

std::uint64_t Group::sequence(int rank) const {
  std::lock_guard<std::mutex> lk(mu_);
  return seq_[static_cast<std::size_t>(rank)];
}

void* Group::scratch(int rank, std::size_t bytes) {
  auto& p = scratch_[static_cast<std::size_t>(rank)];
  auto& n = scratch_bytes_[static_cast<std::size_t>(rank)];
  if (n < bytes) {
    if (p) DBAG_CUDA(cudaFree(p));
    DBAG_CUDA(cudaMalloc(&p, bytes));
    n = bytes;
  }
  return p;
}

void Group::allreduce(int rank, void* data, std::int64_t count, DType t, bool is_max, cudaStream_t s) {
  if (k_ == 1) return;
  const int kind = (t == DType::f64 ? 2 : 0) + (is_max ? 1 : 0);
  const std::size_t bytes = static_cast<std::size_t>(count) * dsize(t);
  void* out = count > 0 ? scratch(rank, bytes) : nullptr;  // before publishing: no allocation inside the window
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (aborted_) throw Error(DBAG_COLLECTIVE, "collective aborted: " + why_);
    slots_[static_cast<std::size_t>(rank)] = Slot{data, count, kind, ++seq_[static_cast<std::size_t>(rank)]};
  }
  DBAG_CUDA(cudaEventRecord(ready_[static_cast<std::size_t>(rank)], s));
  rendezvous(rank);
  validate(rank, count, kind);
  SlotPtrs sp{};
  for (int r = 0; r < k_; ++r) {
    sp.p[r] = slots_[static_cast<std::size_t>(r)].ptr;
    if (r != rank) DBAG_CUDA(cudaStreamWaitEvent(s, ready_[static_cast<std::size_t>(r)], 0));
  }
  if (count > 0) {
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<std::int64_t>((count + threads - 1) / threads, 1184));
    if (t == DType::f64) {
      if (is_max) k_fold_slots<double, true><<<blocks, threads, 0, s>>>(count, k_, sp, static_cast<double*>(out));
      else k_fold_slots<double, false><<<blocks, threads, 0, s>>>(count, k_, sp, static_cast<double*>(out));
    } else {
      if (is_max) k_fold_slots<float, true><<<blocks, threads, 0, s>>>(count, k_, sp, static_cast<float*>(out));
      else k_fold_slots<float, false><<<blocks, threads, 0, s>>>(count, k_, sp, static_cast<float*>(out));
    }
    DBAG_LAUNCH_CHECK();
  }
  DBAG_CUDA(cudaEventRecord(done_[static_cast<std::size_t>(rank)], s));
  rendezvous(rank);  // every rank has enqueued its reads of the deposited sources
  for (int r = 0; r < k_; ++r)
    if (r != rank) DBAG_CUDA(cudaStreamWaitEvent(s, done_[static_cast<std::size_t>(r)], 0));
  if (count > 0) DBAG_CUDA(cudaMemcpyAsync(data, out, bytes, cudaMemcpyDeviceToDevice, s));
}

NcclComm::NcclComm(int rank, int nranks, const unsigned char* id128) : rank_(rank), size_(nranks) {
  ncclUniqueId id;
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
  std::copy(id128, id128 + 128, reinterpret_cast<unsigned char*>(id.internal));
  DBAG_NCCL(ncclCommInitRank(&comm_, nranks, id, rank));
}

NcclComm::~NcclComm() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (void* p : own_) cudaFree(p);
  if (comm_) ncclCommDestroy(comm_);
}

// Peer site across processes: each rank's allocation is exported with CUDA
// IPC, the handles are all-gathered over NCCL and opened (peer access over
// NVLink / NVSwitch). Any rank failing makes every rank return false.
bool NcclComm::make_peer_site(std::int64_t max_len, DType t, PeerSite* out) {
  // DBAG_PEER_IPC=0 keeps the host-driven NCCL loop. The mapping is
  // verified before use (k_peer_selftest: two all-reduces per slice with a
  // 2 s peer timeout, agreed over NCCL); any failure falls back to NCCL on
  // every rank. Every rank reads the same environment (torchrun).
  const char* ipc = std::getenv("DBAG_PEER_IPC");
  if (ipc && std::string(ipc) == "0") return false;
  if (size_ < 2 || size_ > PeerSite::kMaxPeers) return false;
  PeerSite s;
  s.k = size_;
  s.rank = rank_;
  PeerSite::plan(max_len, s.k, false, &s.slice, &s.nslice);  // one process per GPU
  s.len = std::max<std::int64_t>(max_len, 1);
  const PeerAlloc a = peer_alloc(max_len, t, s.nslice);
  own_.push_back(a.base);
  peer_fill(a, s.nslice, rank_, &s, true);
  int dev = 0;
  DBAG_CUDA(cudaGetDevice(&dev));
  auto check = std::make_unique<PeerCheck>(s, dev);
  constexpr int kRec = 72;  // IPC handle (64 bytes) + status
  std::vector<unsigned char> rec(static_cast<std::size_t>(kRec) * static_cast<std::size_t>(size_), 0);
  unsigned char* mine = rec.data() + static_cast<std::size_t>(rank_) * kRec;
  cudaIpcMemHandle_t h{};
  int ok = cudaIpcGetMemHandle(&h, a.base) == cudaSuccess ? 1 : 0;
  (void)cudaGetLastError();
  std::memcpy(mine, &h, sizeof(h));
  mine[64] = static_cast<unsigned char>(ok);
  unsigned char* d = nullptr;
  cudaStream_t st = nullptr;
  DBAG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DBAG_CUDA(cudaMalloc(&d, rec.size() + sizeof(int)));
  DBAG_CUDA(cudaMemcpy(d, rec.data(), rec.size(), cudaMemcpyHostToDevice));
  DBAG_NCCL(ncclAllGather(d + static_cast<std::size_t>(rank_) * kRec, d, kRec, ncclChar, comm_, st));
  DBAG_CUDA(cudaStreamSynchronize(st));
  DBAG_CUDA(cudaMemcpy(rec.data(), d, rec.size(), cudaMemcpyDeviceToHost));
  std::vector<void*> opened;
  for (int p = 0; p < size_ && ok; ++p) {
    const unsigned char* r = rec.data() + static_cast<std::size_t>(p) * kRec;
    if (!r[64]) {
      ok = 0;
      break;
    }
    if (p == rank_) continue;
    cudaIpcMemHandle_t hp;
    std::memcpy(&hp, r, sizeof(hp));
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, hp, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      (void)cudaGetLastError();
      ok = 0;
      break;
    }
    opened.push_back(ptr);
    PeerAlloc pa;
    pa.base = ptr;
    pa.slot_bytes = a.slot_bytes;
    peer_fill(pa, s.nslice, p, &s, false);
  }
  // every rank must agree: min over ranks of ok
  int* dok = reinterpret_cast<int*>(d + rec.size());
  DBAG_CUDA(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
  DBAG_NCCL(ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, comm_, st));
  DBAG_CUDA(cudaStreamSynchronize(st));
  DBAG_CUDA(cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost));
  if (ok) {  // self-check of the mapped site, then agree again
    ok = check->run(s);
    check.reset();
    DBAG_CUDA(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
    DBAG_NCCL(ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, comm_, st));
    DBAG_CUDA(cudaStreamSynchronize(st));
    DBAG_CUDA(cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost));
    if (!ok) std::fprintf(stderr, "[dbag] CUDA-IPC peer all-reduce self-check failed: NCCL loop used\n");
  }
  cudaFree(d);
  cudaStreamDestroy(st);
  if (!ok) {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    return false;
  }
  opened_.insert(opened_.end(), opened.begin(), opened.end());
  *out = s;
  return true;
}

void NcclComm::allreduce_sum(void* d, std::int64_t n, DType t, cudaStream_t s) {
  if (size_ == 1 || n == 0) return;
  DBAG_NCCL(ncclAllReduce(d, d, static_cast<size_t>(n), nccl_type(t), ncclSum, comm_, s));
}

void NcclComm::allreduce_max(void* d, std::int64_t n, DType t, cudaStream_t s) {
  if (size_ == 1 || n == 0) return;
  DBAG_NCCL(ncclAllReduce(d, d, static_cast<size_t>(n), nccl_type(t), ncclMax, comm_, s));
}

}  // namespace dbag
