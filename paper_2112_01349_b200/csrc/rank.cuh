// rank.cuh — one rank's device context: the shard, the normal equations and
// the operators of the LM inner loop, each a short sequence of sm_100a kernel
// launches on the rank's stream. The host LM loop (solver.cuh) drives it.
//
// Operator map (reference symbol -> method):
//   EdgeEvaluator::cost + detail::distributed_cost   cost()          dba/edge_eval.hpp:289, dba/solver.hpp:264
//   linearize + assemble_local + 4 all-reduces       linearize()     dba/solver.hpp:330-340
//   damp_into + FactoredBlockDiagonal::factor        damp_factor()   dba/solver.hpp:350-355
//   g = v - allreduce(E_k C^-1 w)                    rhs()           dba/solver.hpp:357-363
//   dse                                              dse()           dba/solver.hpp:149-181
//   dpcg                                             pcg()           dba/solver.hpp:202-257
//   back-substitution + trial + model terms          backsub_trial() dba/solver.hpp:371-410
//
// Point-indexed device arrays use "device point" ids (DeviceLayout: local
// points reordered for camera locality); host-facing accessors map them back
// to global point ids.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <limits>
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

#include "comm.hpp"
#include "common.hpp"
#include "dse.cuh"
#include "graph_pcg.cuh"
#include "stream.cuh"
#include "peer.cuh"
#include "lin.cuh"
#include "kernels.cuh"
#include "partition.hpp"

namespace dbag {

// One device allocation per rank, sized in advance from the shard's layout:
// the paper's predicted-size memory pool (SURVEY.md §8f
// f4). upload() reserves it once and carves every shard buffer from it, so a
// problem that does not fit fails at one cudaMalloc, before any copy, and
// nothing is allocated inside the LM loop.
class Arena {
 public:
  static constexpr std::size_t kAlign = 256;
  static std::size_t round(std::size_t b) { return (b + kAlign - 1) / kAlign * kAlign; }
  Arena() = default;
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  ~Arena() { release(); }
  void reserve(std::size_t bytes) {
    release();
    if (bytes) DBAG_CUDA(cudaMalloc(&base_, bytes));
    cap_ = bytes;
  }
  void* take(std::size_t bytes) {
    const std::size_t b = round(bytes);
    if (used_ + b > cap_)
      throw Error(DBAG_INTERNAL, "memory pool overflow: predicted " + std::to_string(cap_) + " bytes, need more");
    void* p = base_ + used_;
    used_ += b;
    return p;
  }
  std::size_t capacity() const { return cap_; }
  std::size_t used() const { return used_; }

 private:
  void release() {
    if (base_) cudaFree(base_);
    base_ = nullptr;
    cap_ = used_ = 0;
  }
  char* base_ = nullptr;
  std::size_t cap_ = 0, used_ = 0;
};

template <class T>
class DevBuf {
 public:
  using value_type = T;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(std::size_t n) {
    release();
    n_ = n;
    if (n) DBAG_CUDA(cudaMalloc(&p_, n * sizeof(T)));
    owned_ = true;
  }
  void alloc(std::size_t n, Arena& a) {  // a slice of the rank's pool
    release();
    n_ = n;
    p_ = static_cast<T*>(a.take(n * sizeof(T)));
  }
  void copy_in(const std::vector<T>& v) {
    if (v.size() > n_) throw Error(DBAG_INTERNAL, "device buffer smaller than its upload");
    if (!v.empty()) DBAG_CUDA(cudaMemcpy(p_, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void swap(DevBuf& o) {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(owned_, o.owned_);
  }

 private:
  void release() {
    if (p_ && owned_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
    owned_ = false;
  }
  T* p_ = nullptr;
  std::size_t n_ = 0;
  bool owned_ = false;
};

// Element counts of one rank's shard buffers (Rank::shard_buffers), from the
// host-side partition plan and device layout alone.
struct ShardSizes {
  std::size_t N, slots, dpt_ptr, chunk_slot, cam_part_ptr, halo_slot, part, cam_ptr, cam_glob, n_loc, n_halo_loc,
      halo, red, cm, pl, recs, n_long, ctab, xp_full, m, jb, carry, cam_list, bounce;
};

inline void check_problem(const dbag_problem& p) {
  if (p.num_cameras < 0 || p.num_points < 0 || p.num_observations < 0)
    throw Error(DBAG_SHAPE, "negative problem dimensions");
  for (std::int64_t e = 0; e < p.num_observations; ++e) {
    if (p.camera_id[e] < 0 || p.camera_id[e] >= p.num_cameras)
      throw Error(DBAG_INVALID_ARGUMENT, "edge references unknown camera " + std::to_string(p.camera_id[e]));
    if (p.point_id[e] < 0 || p.point_id[e] >= p.num_points)
      throw Error(DBAG_INVALID_ARGUMENT, "edge references unknown point " + std::to_string(p.point_id[e]));
  }
}

inline int grid_for(std::int64_t n, int threads, int cap) {
  const std::int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(b, cap)));
}

struct PcgOut {
  int iterations = 0;
  bool converged = false;
};

struct Tally {  // dba/counters.hpp:11-24
  std::uint64_t edges = 0, block_ops = 0;
};

// S: arithmetic and state type; T: storage type of the E lanes (T = S, or
// float under FP64 arithmetic: the memory-lean variant).
template <class S, class T = S>
class Rank {
 public:
  using Scalar = S;
  using Scal = dev::PcgScal<S>;
  static constexpr DType kT = sizeof(S) == 8 ? DType::f64 : DType::f32;

  Rank(int device, Comm* comm) : device_(device), comm_(comm) {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    DBAG_CUDA(cudaMallocHost(&hsc_, sizeof(Scal)));
    DBAG_CUDA(cudaMallocHost(&hbuf_, 64 * sizeof(double)));
    DBAG_CUDA(cudaEventCreate(&mark_[0]));
    DBAG_CUDA(cudaEventCreate(&mark_[1]));
    sc_.alloc(1);
    red_part_.alloc(8 * dev::kRedBlocksMax);
    red_cnt_.alloc(1);
    DBAG_CUDA(cudaMemset(red_cnt_.get(), 0, sizeof(unsigned)));
    dsc_.alloc(64);
    bad_.alloc(4);
  }
  ~Rank() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(st_);
    for (auto e : prof_ev_) cudaEventDestroy(e);
    cudaEventDestroy(mark_[0]);
    cudaEventDestroy(mark_[1]);
    cudaFreeHost(hsc_);
    cudaFreeHost(hbuf_);
    if (gsc_h_) cudaFreeHost(gsc_h_);
    destroy_graph();
    gk_destroy();
    cudaStreamDestroy(st_);
  }

  cudaStream_t stream() const { return st_; }
  int device() const { return device_; }
  const ShardPlan& plan() const { return plan_; }
  std::int64_t edges() const { return N_; }
  Tally& tally() { return tally_; }
  int last_dse_count() const { return dse_count_; }
  std::int64_t launches() const { return launches_; }

  // ------------------------------------------------------- memory pool ----
  // Jb, the per-edge [r, J, w] rows linearize hands to assembly, is live
  // only inside linearize(): it holds one batch of whole device points of at
  // most DBAG_JB_BATCH slots (default 2^23; a larger point takes a batch of
  // its own) instead of all N rows, so city-scale shards do not keep
  // 224 bytes per edge of scratch through the PCG.
  // DBAG_LIN=rows: the two-kernel assembly through per-edge Jacobian rows in
  // HBM (Jb, assembled point- then camera-major) instead of the fused
  // linearize + assemble pass (lin.cuh).
  static bool lin_rows() {
    const char* e = std::getenv("DBAG_LIN");
    return e && std::string(e) == "rows";
  }
  static std::int64_t jb_batch_cap() {
    const char* e = std::getenv("DBAG_JB_BATCH");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? v : (std::int64_t(1) << 23);
  }
  // Batch boundaries in device points (first 0, last n_loc).
  static std::vector<std::int32_t> jb_batches(const std::vector<std::int32_t>& dpt_ptr) {
    const std::int64_t cap = lin_rows() ? jb_batch_cap() : std::numeric_limits<std::int64_t>::max();
    const std::int32_t np = static_cast<std::int32_t>(dpt_ptr.size()) - 1;
    std::vector<std::int32_t> b{0};
    for (std::int32_t d = 0; d < np; ++d)
      if (d > b.back() && dpt_ptr[static_cast<std::size_t>(d) + 1] - dpt_ptr[static_cast<std::size_t>(b.back())] > cap)
        b.push_back(d);
    b.push_back(std::max(np, 0));
    return b;
  }

  static ShardSizes shard_sizes(const ShardPlan& pl, const DeviceLayout& d) {
    ShardSizes z{};
    z.N = static_cast<std::size_t>(pl.range.count);
    z.m = static_cast<std::size_t>(pl.m);
    z.slots = d.slot_dpt.size();
    z.dpt_ptr = d.dpt_ptr.size();
    z.chunk_slot = d.chunk_slot.size();
    z.cam_part_ptr = d.cam_part_ptr.size();
    z.halo_slot = d.halo_slot.size();
    z.part = static_cast<std::size_t>(d.n_part) * 9;
    z.cam_ptr = pl.cam_ptr.size();
    z.cam_glob = pl.cams.to_global.size();
    z.n_loc = static_cast<std::size_t>(pl.pts.size());
    z.n_halo_loc = 0;
    for (std::size_t lp = 0; lp < z.n_loc; ++lp) z.n_halo_loc += pl.halo_of_lpt[lp] >= 0;
    z.halo = static_cast<std::size_t>(std::max<std::int64_t>(pl.n_shared, 1)) * 12;
    z.red = std::max<std::size_t>(8 * dev::kRedBlocksMax, 2 * (z.m * 32 / 256 + 64));
    z.cm = z.m * 9;
    z.pl = z.n_loc * 3;
    z.recs = static_cast<std::size_t>(std::max<std::size_t>(d.chunk_slot.size(), 1)) * dev::Rec<T, dev::kLanesFact>::kLen;
    z.n_long = 0;
    z.ctab = 0;
    for (std::size_t t = 0; t + 1 < d.tile_chunk.size(); ++t) {
      z.n_long += d.tile_chunk[t + 1] - d.tile_chunk[t] > 1;
      z.ctab += 4 * (d.tile_chunk[t + 1] - d.tile_chunk[t] == 1);
    }
    z.xp_full = static_cast<std::size_t>(pl.n) * 3;
    const std::vector<std::int32_t> jb = jb_batches(d.dpt_ptr);
    const std::size_t nb = jb.size() - 1;
    z.jb = 0;
    if (lin_rows())
      for (std::size_t b = 0; b < nb; ++b)
        z.jb = std::max<std::size_t>(z.jb, d.dpt_ptr.empty() ? 0 : d.dpt_ptr[jb[b + 1]] - d.dpt_ptr[jb[b]]);
    z.cam_ptr = lin_rows() ? nb * pl.cam_ptr.size() : 0;  // camera-major slot lists: row assembly only
    z.carry = nb > 1 ? (pl.cam_ptr.size() - 1) * 54 : 0;
    z.cam_list = nb > 1 ? nb * (pl.cam_ptr.size() - 1) : 0;
    z.bounce = pl.ranks > 1 ? 4 * static_cast<std::size_t>(pl.ranks) : 0;  // tallies (2K) and identity probe (4K)
    return z;
  }

  // Every pool-backed buffer of the rank with its element count; the one
  // list both the prediction and the allocation walk.
  template <class F>
  static void shard_buffers(const ShardSizes& z, F&& f) {
    for (auto pm : {&Rank::slot_cam_, &Rank::slot_dpt_, &Rank::slot_edge_})
      f(pm, pm == &Rank::slot_dpt_ || pm == &Rank::slot_edge_ ? z.slots : z.N);
    f(&Rank::cslot_dslot_, lin_rows() ? z.N : 0);
    for (auto pm : {&Rank::slot_px_, &Rank::slot_py_, &Rank::slot_w_}) f(pm, z.N);
    f(&Rank::dpt_ptr_, z.dpt_ptr);
    f(&Rank::chunk_slot_, z.chunk_slot);
    f(&Rank::cam_part_ptr_, z.cam_part_ptr);
    f(&Rank::halo_slot_, z.halo_slot);
    f(&Rank::halo_pos_, z.halo_slot);
    f(&Rank::slot_chunk_, z.slots);
    f(&Rank::cam_ptr_, z.cam_ptr);
    f(&Rank::cam_glob_, z.cam_glob);
    for (auto pm : {&Rank::dpt_glob_d_, &Rank::halo_of_}) f(pm, z.n_loc);
    f(&Rank::owned_, z.n_loc);
    for (auto pm : {&Rank::halo_dpt_, &Rank::halo_idx_}) f(pm, z.n_halo_loc);
    f(&Rank::long_chunk_, z.n_long);
    f(&Rank::ctab_, z.ctab);
    f(&Rank::part_, z.part);
    f(&Rank::halo_buf_, z.halo);
    f(&Rank::halo_sum_, z.halo);
    f(&Rank::cam_ident_, z.m + 1);
    f(&Rank::red_part_, z.red);
    for (auto pm : {&Rank::xc_, &Rank::xct_, &Rank::dxc_, &Rank::v_, &Rank::g_, &Rank::r_, &Rank::z_, &Rank::p_,
                    &Rank::q_, &Rank::ctmp_, &Rank::p2_, &Rank::Rm_})
      f(pm, z.cm);
    for (auto pm : {&Rank::xp_, &Rank::xpt_, &Rank::dxp_, &Rank::w_}) f(pm, z.pl);
    for (auto pm : {&Rank::B_, &Rank::Bd_, &Rank::Binv_, &Rank::Bexp_}) f(pm, z.cm * 9);
    for (auto pm : {&Rank::C_, &Rank::Cd_}) f(pm, z.pl * 3);
    f(&Rank::Cinv_, z.pl * 3 + 16 / sizeof(S));  // slack for 16-byte-rounded reads
    f(&Rank::Jb_, z.jb * 28);
    f(&Rank::bpart_, lin_rows() ? 0 : z.part / 9 * dev::kAsmTerms);
    f(&Rank::carry_, z.carry);
    f(&Rank::cam_list_, z.cam_list);
    f(&Rank::E_, z.recs);
    f(&Rank::xp_full_, z.xp_full);
    f(&Rank::gsc_, 1);
    f(&Rank::g_pq_cam_, z.m);
    f(&Rank::g_bar_, 1);
    f(&Rank::bounce_, z.bounce);
  }

  // Device bytes upload() reserves for this shard (exact: upload checks it).
  static std::size_t predict_bytes(const ShardSizes& z) {
    std::size_t b = 0;
    shard_buffers(z, [&](auto pm, std::size_t n) {
      using Buf = std::remove_reference_t<decltype(std::declval<Rank&>().*pm)>;
      b += Arena::round(std::max<std::size_t>(n, 1) * sizeof(typename Buf::value_type));
    });
    return b;
  }
  std::size_t pool_bytes() const { return pool_.capacity(); }
  std::size_t pool_used() const { return pool_.used(); }

  // ------------------------------------------------------------ upload ----
  void upload(const dbag_problem& p, int jac_mode) {
    DBAG_CUDA(cudaSetDevice(device_));
    check_problem(p);
    jac_mode_ = jac_mode;
    destroy_graph();
    plan_ = plan_shard(p.camera_id, p.point_id, p.num_observations, p.num_cameras, p.num_points, comm_->size(),
                       comm_->rank(), dev::kTile);
    m_ = plan_.m;
    n_glob_ = plan_.n;
    n_loc_ = plan_.pts.size();
    m_loc_ = plan_.cams.size();
    N_ = plan_.range.count;
    H_ = plan_.n_shared;
    const std::int64_t base = plan_.range.start;
    lay_ = build_device_layout(plan_, p.camera_id + base, dev::kTile);
    const S* px = static_cast<const S*>(p.pixel_x);
    const S* py = static_cast<const S*>(p.pixel_y);
    const S* wt = static_cast<const S*>(p.weight);
    std::vector<std::int32_t> s_cam(N_);
    std::vector<S> s_px(N_), s_py(N_), s_w(N_);
    for (std::int64_t s = 0; s < N_; ++s) {
      const std::int64_t e = lay_.slot_edge[static_cast<std::size_t>(s)];
      s_cam[s] = p.camera_id[base + e];
      s_px[s] = px[base + e];
      s_py[s] = py[base + e];
      s_w[s] = wt ? wt[base + e] : S(1);
      if (!(s_w[s] >= S(0))) throw Error(DBAG_INVALID_ARGUMENT, "edge weight must be >= 0");
    }
    n_tiles_ = static_cast<int>(lay_.tile_pt.size()) - 1;
    n_chunks_ = static_cast<std::int32_t>(lay_.chunk_slot.size());
    n_chunk_part_ = static_cast<std::int32_t>(lay_.ucam_cam.size());
    // camera-major view (assembly of B, v)
    std::vector<std::int32_t> cptr32(plan_.cam_ptr.begin(), plan_.cam_ptr.end());
    std::vector<std::int32_t> dslot_of_edge(static_cast<std::size_t>(N_));
    for (std::int64_t s = 0; s < N_; ++s) dslot_of_edge[static_cast<std::size_t>(lay_.slot_edge[static_cast<std::size_t>(s)])] = static_cast<std::int32_t>(s);
    std::vector<std::int32_t> cslot(static_cast<std::size_t>(N_));
    for (std::int64_t c = 0; c < N_; ++c)
      cslot[static_cast<std::size_t>(c)] = dslot_of_edge[static_cast<std::size_t>(plan_.cam_blk[static_cast<std::size_t>(c)])];
    // device points
    dpt_glob_.resize(static_cast<std::size_t>(n_loc_));
    std::vector<std::int32_t> halo_of(static_cast<std::size_t>(n_loc_), -1);
    std::vector<std::uint8_t> owned(static_cast<std::size_t>(n_loc_), 1);
    std::vector<std::int32_t> hl, hi;
    for (std::int32_t d = 0; d < n_loc_; ++d) {
      const std::int32_t lp = lay_.dpt_lpt[static_cast<std::size_t>(d)];
      dpt_glob_[static_cast<std::size_t>(d)] = plan_.pts.to_global[static_cast<std::size_t>(lp)];
      halo_of[static_cast<std::size_t>(d)] = plan_.halo_of_lpt[static_cast<std::size_t>(lp)];
      owned[static_cast<std::size_t>(d)] = plan_.owned_lpt[static_cast<std::size_t>(lp)];
      if (halo_of[static_cast<std::size_t>(d)] >= 0) {
        hl.push_back(d);
        hi.push_back(halo_of[static_cast<std::size_t>(d)]);
      }
    }
    owned_h_ = owned;
    n_halo_loc_ = static_cast<std::int32_t>(hl.size());
    {  // points no edge observes: no rank holds them; they keep their x0
      std::vector<std::uint8_t> seen(static_cast<std::size_t>(p.num_points), 0);
      for (std::int64_t e = 0; e < p.num_observations; ++e) seen[static_cast<std::size_t>(p.point_id[e])] = 1;
      orphans_.clear();
      for (std::int32_t q = 0; q < p.num_points; ++q)
        if (!seen[static_cast<std::size_t>(q)]) orphans_.push_back(q);
    }
    // the whole shard in one pool allocation, sized before any copy
    const ShardSizes z = shard_sizes(plan_, lay_);
    pool_.reserve(predict_bytes(z));
    shard_buffers(z, [&](auto pm, std::size_t n) { (this->*pm).alloc(std::max<std::size_t>(n, 1), pool_); });
    if (pool_.used() != pool_.capacity()) throw Error(DBAG_INTERNAL, "memory pool prediction mismatch");
    slot_cam_.copy_in(s_cam);
    slot_dpt_.copy_in(lay_.slot_dpt);
    slot_edge_.copy_in(lay_.slot_edge);
    slot_px_.copy_in(s_px);
    slot_py_.copy_in(s_py);
    slot_w_.copy_in(s_w);
    dpt_ptr_.copy_in(lay_.dpt_ptr);
    chunk_slot_.copy_in(lay_.chunk_slot);
    {
      std::vector<std::int32_t> ident(static_cast<std::size_t>(m_) + 1);
      for (std::size_t i = 0; i < ident.size(); ++i) ident[i] = static_cast<std::int32_t>(i);
      cam_ident_.copy_in(ident);
    }
    cam_part_ptr_.copy_in(lay_.cam_part_ptr);
    halo_slot_.copy_in(lay_.halo_slot);
    slot_chunk_.copy_in(lay_.slot_chunk);
    std::vector<std::int32_t> cam_list_h;
    {  // camera-major slot lists per Jb batch, edge order inside each camera
      jb_pt_ = jb_batches(lay_.dpt_ptr);
      const std::size_t nb = jb_pt_.size() - 1, mc = cptr32.size();
      jb_ncam_.clear();
      if (nb > 1) cam_list_h.assign(nb * (mc - 1), 0);
      if (nb > 1) {
        std::vector<std::int32_t> bs(nb + 1);
        for (std::size_t b = 0; b <= nb; ++b) bs[b] = lay_.dpt_ptr[static_cast<std::size_t>(jb_pt_[b])];
        std::vector<std::int32_t> bptr(nb * mc + 1, 0), bslot(cslot.size());
        auto batch_of = [&](std::int32_t ds) {
          return static_cast<std::size_t>(std::upper_bound(bs.begin(), bs.end(), ds) - bs.begin()) - 1;
        };
        for (std::size_t lc = 0; lc + 1 < mc; ++lc)
          for (std::int32_t cs = cptr32[lc]; cs < cptr32[lc + 1]; ++cs)
            ++bptr[batch_of(cslot[static_cast<std::size_t>(cs)]) * mc + lc + 1];
        for (std::size_t i = 1; i < bptr.size(); ++i) bptr[i] += bptr[i - 1];
        std::vector<std::int32_t> fill(bptr.begin(), bptr.end() - 1);
        for (std::size_t lc = 0; lc + 1 < mc; ++lc)
          for (std::int32_t cs = cptr32[lc]; cs < cptr32[lc + 1]; ++cs) {
            const std::int32_t ds = cslot[static_cast<std::size_t>(cs)];
            bslot[static_cast<std::size_t>(fill[batch_of(ds) * mc + lc]++)] = ds;
          }
        bptr.pop_back();  // batch b's cam_ptr: bptr[b*mc .. b*mc + mc)
        jb_ncam_.assign(nb, 0);  // the cameras batch b touches, at cam_list[b*(mc-1) ..)
        for (std::size_t b = 0; b < nb; ++b)
          for (std::size_t lc = 0; lc + 1 < mc; ++lc)
            if (bptr[b * mc + lc + 1] > bptr[b * mc + lc]) cam_list_h[b * (mc - 1) + jb_ncam_[b]++] = static_cast<std::int32_t>(lc);
        cptr32.swap(bptr);
        cslot.swap(bslot);
      }
    }
    if (lin_rows()) {
      cam_ptr_.copy_in(cptr32);
      cam_list_.copy_in(cam_list_h);
      cslot_dslot_.copy_in(cslot);
    }
    cam_glob_.copy_in(plan_.cams.to_global);
    dpt_glob_d_.copy_in(dpt_glob_);
    halo_of_.copy_in(halo_of);
    owned_.copy_in(owned);
    halo_dpt_.copy_in(hl);
    halo_idx_.copy_in(hi);
    DBAG_CUDA(cudaMemset(g_bar_.get(), 0, sizeof(unsigned long long)));
    fact_ = true;
    E_.copy_in(build_records<dev::kLanesFact>(s_cam));
    // assembly partials: the halo slots' own positions are never written by
    // the fused linearize and must read as zero in the camera fold
    if (bpart_.size() > 0) DBAG_CUDA(cudaMemset(bpart_.get(), 0, bpart_.size() * sizeof(double)));
    set_state(static_cast<const S*>(p.cameras), static_cast<const S*>(p.points));
    have_system_ = false;
    setup_peer_sites();
  }

  // ---- device-side collectives of the K > 1 graph DPCG (peer.cuh) --------
  // Collective (every rank uploads): one site for the camera vector (9m) and
  // one for the halo (3H). DBAG_PEER=0 keeps the host-driven run-ahead loop.
  static bool peer_enabled() {
    const char* e = std::getenv("DBAG_PEER");
    return !(e && std::string(e) == "0");
  }
  void setup_peer_sites() {
    gk_destroy();
    if (comm_->size() < 2 || !peer_enabled()) {
      peer_ok_ = false;
      return;
    }
    const std::int64_t nc = static_cast<std::int64_t>(m_) * 9, nh = 3 * static_cast<std::int64_t>(H_);
    if (peer_ok_ && nc <= peer_cap_[0] && nh <= peer_cap_[1]) return;
    bool ok = comm_->make_peer_site(std::max<std::int64_t>(nc, 1), kT, &ps_cam_);
    ok = comm_->make_peer_site(std::max<std::int64_t>(nh, 1), kT, &ps_halo_) && ok;
    peer_ok_ = ok;
    peer_cap_[0] = nc;
    peer_cap_[1] = nh;
  }
  void gk_destroy() {
    if (gk_exec_) cudaGraphExecDestroy(gk_exec_);
    if (gk_graph_) cudaGraphDestroy(gk_graph_);
    gk_exec_ = nullptr;
    gk_graph_ = nullptr;
  }

  // Full-size host x_c (9m) and x_p (3n); this rank keeps its local points.
  // The full x_p goes to the device as is (one copy from the caller's
  // buffer, DMA-direct when it is pinned) and is permuted into device-point
  // order there.
  void set_state(const S* xc, const S* xp) {
    DBAG_CUDA(cudaSetDevice(device_));
    orphan_x_.resize(orphans_.size() * 3);
    for (std::size_t i = 0; i < orphans_.size(); ++i)
      for (int k = 0; k < 3; ++k) orphan_x_[i * 3 + k] = xp[static_cast<std::size_t>(orphans_[i]) * 3 + k];
    DBAG_CUDA(cudaMemcpyAsync(xc_.get(), xc, sizeof(S) * 9 * static_cast<std::size_t>(m_), cudaMemcpyHostToDevice, st_));
    const std::size_t full = static_cast<std::size_t>(n_glob_) * 3;
    if (xp_full_.size() < std::max<std::size_t>(full, 1)) xp_full_.alloc(std::max<std::size_t>(full, 1));
    DBAG_CUDA(cudaMemcpyAsync(xp_full_.get(), xp, sizeof(S) * full, cudaMemcpyHostToDevice, st_));
    if (n_loc_ > 0)
      launch(dev::k_point_rows<S, false>, grid_for(n_loc_, 256, 1 << 30), 256, n_loc_,
             static_cast<const std::int32_t*>(dpt_glob_d_.get()), xp_full_.get(), xp_.get());
    DBAG_CUDA(cudaStreamSynchronize(st_));
    have_system_ = false;
  }

  // Cameras and this rank's points (owned_only: points it owns) into
  // full-size host vectors; other entries are left untouched.
  void get_state(S* xc, S* xp, bool owned_only = false) {
    DBAG_CUDA(cudaSetDevice(device_));
    if (xc) DBAG_CUDA(cudaMemcpyAsync(xc, xc_.get(), sizeof(S) * 9 * static_cast<std::size_t>(m_), cudaMemcpyDeviceToHost, st_));
    if (xp && n_loc_ == n_glob_) {  // every point is local: un-permute on the device, one copy out
      const std::size_t full = static_cast<std::size_t>(n_glob_) * 3;
      if (xp_full_.size() < std::max<std::size_t>(full, 1)) xp_full_.alloc(std::max<std::size_t>(full, 1));
      if (n_loc_ > 0)
        launch(dev::k_point_rows<S, true>, grid_for(n_loc_, 256, 1 << 30), 256, n_loc_,
               static_cast<const std::int32_t*>(dpt_glob_d_.get()), xp_.get(), xp_full_.get());
      DBAG_CUDA(cudaMemcpyAsync(xp, xp_full_.get(), sizeof(S) * full, cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
      return;
    }
    std::vector<S> loc(static_cast<std::size_t>(n_loc_) * 3);
    DBAG_CUDA(cudaMemcpyAsync(loc.data(), xp_.get(), sizeof(S) * loc.size(), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    if (xp)
      for (std::int32_t d = 0; d < n_loc_; ++d) {
        if (owned_only && !owned_h_[static_cast<std::size_t>(d)]) continue;
        for (int k = 0; k < 3; ++k)
          xp[static_cast<std::size_t>(dpt_glob_[static_cast<std::size_t>(d)]) * 3 + k] = loc[static_cast<std::size_t>(d) * 3 + k];
      }
  }

  // ------------------------------------------------------------- cost ----
  // Returns the all-reduced cost (+inf if any rank saw P_z == 0); bad_edge
  // is the lowest offending global edge id over ranks, or -1.
  double cost(bool trial, std::int64_t* bad_edge) {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaMemsetAsync(bad_.get(), 0xff, sizeof(unsigned long long), st_));
    DBAG_CUDA(cudaMemsetAsync(dsc_.get(), 0, sizeof(double), st_));
    if (N_ > 0)
      launch(dev::k_cost<S>, grid_for(N_, dev::kRedThreads, dev::kRedBlocksMax), dev::kRedThreads, N_,
             slot_cam_.get(), slot_dpt_.get(), slot_edge_.get(), plan_.range.start, slot_px_.get(), slot_py_.get(),
             slot_w_.get(), trial ? xct_.get() : xc_.get(), trial ? xpt_.get() : xp_.get(), red(), dsc_.get(),
             bad_.get());
    tally_.edges += static_cast<std::uint64_t>(N_);
    comm_->allreduce_sum(dsc_.get(), 1, DType::f64, st_);
    const std::int64_t bad = agree_min_index(bad_.get());
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, dsc_.get(), sizeof(double), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    if (bad_edge) *bad_edge = bad;
    return bad >= 0 ? std::numeric_limits<double>::infinity() : hbuf_[0];
  }

  // --------------------------------------------------------- linearize ----
  void linearize() {
    if (!lin_rows()) return linearize_fused();
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaMemsetAsync(bad_.get(), 0xff, sizeof(unsigned long long), st_));
    DBAG_CUDA(cudaMemsetAsync(B_.get(), 0, B_.size() * sizeof(S), st_));
    DBAG_CUDA(cudaMemsetAsync(v_.get(), 0, v_.size() * sizeof(S), st_));
    if (jb_pt_.size() > 2) DBAG_CUDA(cudaMemsetAsync(carry_.get(), 0, carry_.size() * sizeof(double), st_));
    use_factored();
    if (m_ > 0)  // the cameras' R at the linearization point (factored records)
      launch(dev::k_cam_rotations<S>, grid_for(m_, 128, 1 << 30), 128, m_, static_cast<const S*>(xc_.get()), Rm_.get());
    auto kern = jac_mode_ == 1 ? dev::k_linearize<S, 1, T, dev::kLanesFact> : dev::k_linearize<S, 0, T, dev::kLanesFact>;
    const int nb = static_cast<int>(jb_pt_.size()) - 1;
    for (int b = 0; b < nb && N_ > 0; ++b) {  // one Jb batch of whole points at a time
      const std::int32_t d0 = jb_pt_[static_cast<std::size_t>(b)], d1 = jb_pt_[static_cast<std::size_t>(b) + 1];
      const std::int64_t s0 = lay_.dpt_ptr[static_cast<std::size_t>(d0)], s1 = lay_.dpt_ptr[static_cast<std::size_t>(d1)];
      if (s1 > s0)
        launch(kern, static_cast<int>((s1 - s0 + 127) / 128), 128, s0, s1, slot_cam_.get(), slot_dpt_.get(),
               slot_edge_.get(), plan_.range.start, slot_px_.get(), slot_py_.get(), slot_w_.get(), xc_.get(), xp_.get(),
               Jb_.get(), E_.get(), slot_chunk_.get(), chunk_slot_.get(), bad_.get());
      if (d1 > d0)
        launch(dev::k_assemble_points<S>, grid_for(d1 - d0, 128, 1 << 30), 128, d0, d1, dpt_ptr_.get(), s0, Jb_.get(),
               C_.get(), w_.get());
      const int ncam = nb > 1 ? jb_ncam_[static_cast<std::size_t>(b)] : m_loc_;
      if (ncam > 0)
        launch(dev::k_assemble_cameras<S, 256>, ncam, 256, cam_ptr_.get() + static_cast<std::size_t>(b) * (m_loc_ + 1),
               cam_glob_.get(), cslot_dslot_.get(), s0, Jb_.get(), B_.get(), v_.get(), nb > 1 ? carry_.get() : nullptr,
               nb > 1 ? cam_list_.get() + static_cast<std::size_t>(b) * m_loc_ : nullptr);
    }
    if (nb > 1 && m_loc_ > 0)
      launch(dev::k_carry_out<S>, grid_for(m_loc_, 128, 1 << 30), 128, m_loc_, cam_glob_.get(),
             static_cast<const double*>(carry_.get()), B_.get(), v_.get());
    tally_.edges += static_cast<std::uint64_t>(N_);
    const std::int64_t bad = agree_min_index(bad_.get());
    if (bad >= 0) throw degenerate_depth(bad);
    comm_->allreduce_sum(B_.get(), static_cast<std::int64_t>(m_) * 81, kT, st_);
    halo_exchange_Cw();
    comm_->allreduce_sum(v_.get(), static_cast<std::int64_t>(m_) * 9, kT, st_);
    have_system_ = true;
  }

  dev::LinArgs<S, T> lin_args() {
    dev::LinArgs<S, T> a;
    a.n_chunks = n_chunks_;
    a.rec = E_.get();
    a.chunk_slot = chunk_slot_.get();
    a.slot_cam = slot_cam_.get();
    a.slot_pt = slot_dpt_.get();
    a.slot_edge = slot_edge_.get();
    a.edge_base = plan_.range.start;
    a.px = slot_px_.get();
    a.py = slot_py_.get();
    a.w = slot_w_.get();
    a.xc = xc_.get();
    a.xp = xp_.get();
    a.C = C_.get();
    a.wv = w_.get();
    a.bpart = bpart_.get();
    a.long_chunk = long_chunk_.get();
    a.n_long = n_long_;
    a.bad_edge = bad_.get();
    return a;
  }

  // linearize + assemble_local in one pass over the chunks (lin.cuh), then
  // the camera fold of the assembly partials; all-reduces as above.
  void linearize_fused() {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaMemsetAsync(bad_.get(), 0xff, sizeof(unsigned long long), st_));
    use_factored();
    if (m_ > 0)  // the cameras' R at the linearization point (factored records)
      launch(dev::k_cam_rotations<S>, grid_for(m_, 128, 1 << 30), 128, m_, static_cast<const S*>(xc_.get()), Rm_.get());
    const dev::LinArgs<S, T> a = lin_args();
    if (n_chunks_ > 0) {
      if (jac_mode_ == 1) launch(dev::k_lin_chunk<S, 1, T, dev::kLanesFact>, n_chunks_, dev::kTile, a);
      else launch(dev::k_lin_chunk<S, 0, T, dev::kLanesFact>, n_chunks_, dev::kTile, a);
      if (n_long_ > 0) {
        if (jac_mode_ == 1) launch(dev::k_lin_long<S, 1, T, dev::kLanesFact>, n_long_, dev::kTile, a);
        else launch(dev::k_lin_long<S, 0, T, dev::kLanesFact>, n_long_, dev::kTile, a);
      }
    }
    if (m_ > 0)
      launch(dev::k_cam_assemble<S>, grid_for(static_cast<std::int64_t>(m_) * 32, 256, 1 << 30), 256, m_,
             static_cast<const std::int32_t*>(cam_part_ptr_.get()), static_cast<const double*>(bpart_.get()), B_.get(),
             v_.get());
    tally_.edges += static_cast<std::uint64_t>(N_);
    const std::int64_t bad = agree_min_index(bad_.get());
    if (bad >= 0) throw degenerate_depth(bad);
    comm_->allreduce_sum(B_.get(), static_cast<std::int64_t>(m_) * 81, kT, st_);
    halo_exchange_Cw();
    comm_->allreduce_sum(v_.get(), static_cast<std::int64_t>(m_) * 9, kT, st_);
    have_system_ = true;
  }

  // ------------------------------------------------------ damp + factor ----
  void damp_factor(double lambda, int policy) {
    DBAG_CUDA(cudaSetDevice(device_));
    lambda_ = lambda;
    policy_ = policy;
    DBAG_CUDA(cudaMemsetAsync(bad_.get(), 0xff, 2 * sizeof(unsigned long long), st_));
    const S lam = static_cast<S>(lambda);
    // C failures are reported by global point id: the reference factors the
    // full-size C in global order and names the first failing block, C
    // before B (dba/solver.hpp:354-355, dba/block_matrix.hpp:123-134).
    if (n_loc_ > 0)
      launch(dev::k_damp_factor<S, 3>, grid_for(n_loc_, 128, 1 << 30), 128, n_loc_, C_.get(), lam, policy, Cd_.get(),
             Cinv_.get(), dpt_glob_d_.get(), bad_.get());
    if (m_ > 0)
      launch(dev::k_damp_factor<S, 9>, grid_for(m_, 64, 1 << 30), 64, m_, B_.get(), lam, policy, Bd_.get(),
             Binv_.get(), static_cast<const std::int32_t*>(nullptr), bad_.get() + 1);
    if (m_ > 0)  // explicit B^-1 for the block-Jacobi preconditioner
      launch(dev::k_block_inverse<S, 9>, grid_for(m_, 64, 1 << 30), 64, m_, static_cast<const S*>(Binv_.get()),
             Bexp_.get());
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, bad_.get(), 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    unsigned long long raw[2];
    std::memcpy(raw, hbuf_, sizeof(raw));
    // Points no edge observes keep a zero C block (no rank holds them); the
    // reference factors all n blocks, so its damped zero block — lambda I or
    // lambda * 1e-6 I — fails the pivot test when it is not positive.
    if (!orphans_.empty()) {
      const S d = policy == 0 ? lam : lam * static_cast<S>(1e-6);
      if (!(d > S(0)) && !(d != d))
        raw[0] = std::min<unsigned long long>(raw[0], static_cast<unsigned long long>(orphans_.front()));
    }
    // -index (none = -inf): the max over ranks is the lowest failing index.
    const double none = -std::numeric_limits<double>::infinity();
    double agree[2] = {raw[0] == ~0ull ? none : -double(raw[0]), raw[1] == ~0ull ? none : -double(raw[1])};
    if (comm_->size() > 1) {
      double* d = dsc_.get();
      DBAG_CUDA(cudaMemcpyAsync(d + 8, agree, sizeof(agree), cudaMemcpyHostToDevice, st_));
      comm_->allreduce_max(d + 8, 2, DType::f64, st_);
      DBAG_CUDA(cudaMemcpyAsync(agree, d + 8, sizeof(agree), cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
    }
    if (std::isfinite(agree[0])) throw singular_block(static_cast<std::int64_t>(-agree[0]), 3);
    if (std::isfinite(agree[1])) throw singular_block(static_cast<std::int64_t>(-agree[1]), 9);
  }

  // ---------------------------------------------------------------- rhs ----
  void rhs() {
    DBAG_CUDA(cudaSetDevice(device_));
    fused_pass<2>(nullptr);
    tally_.block_ops += static_cast<std::uint64_t>(N_);
    if (comm_->size() == 1) {
      cam_reduce<2>(nullptr, g_.get());
    } else {
      cam_reduce<0>(nullptr, ctmp_.get());
      comm_->allreduce_sum(ctmp_.get(), static_cast<std::int64_t>(m_) * 9, kT, st_);
      const std::int64_t len = static_cast<std::int64_t>(m_) * 9;
      if (len > 0) launch(dev::k_sub<S>, grid_for(len, 256, 1 << 30), 256, len, v_.get(), ctmp_.get(), g_.get());
    }
  }

  // ---------------------------------------------------------------- DSE ----
  // q = (B_d - E C^-1 E^T) x; with PQ the epilogue also forms p.q -> alpha.
  template <bool PQ>
  void dse(const S* x, S* q) {
    const bool prof = profiling_;
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    fused_pass<0>(x);
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    if (comm_->size() == 1) {
      if (PQ) {
        cam_reduce<1>(x, q);
      } else {
        cam_reduce<0>(nullptr, ctmp_.get());
        launch(dev::k_cam_epilogue<S, false>, grid_for(m_, dev::kRedThreads, dev::kRedBlocksMax), dev::kRedThreads,
               m_, Bd_.get(), x, ctmp_.get(), q, red(), sc_.get());
      }
    } else {
      cam_reduce<0>(nullptr, ctmp_.get());
      comm_->allreduce_sum(ctmp_.get(), static_cast<std::int64_t>(m_) * 9, kT, st_);
      launch(dev::k_cam_epilogue<S, PQ>, grid_for(m_, dev::kRedThreads, dev::kRedBlocksMax), dev::kRedThreads, m_,
             Bd_.get(), x, ctmp_.get(), q, red(), sc_.get());
    }
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    tally_.block_ops += 2 * static_cast<std::uint64_t>(N_);
    ++dse_count_;
    ++dse_launches_;
  }

  // --------------------------------------------------------------- DPCG ----
  PcgOut pcg(double tol, int max_iters) {
    DBAG_CUDA(cudaSetDevice(device_));
    if (comm_->size() == 1) {
      const char* mode = std::getenv("DBAG_PCG");
      const std::string m = mode ? mode : "graph";
      if (m == "graph" && n_chunks_ > 0 && m_ > 0) return pcg_graph(tol, max_iters);
    }
    if (comm_->size() > 1 && n_chunks_ > 0 && m_ > 0) {
      const char* mode = std::getenv("DBAG_PCG");
      if (!(mode && std::string(mode) == "host")) return peer_ok_ ? pcg_graph_k(tol, max_iters) : pcg_stream(tol, max_iters);
    }
    S* x = dxc_.get();
    const std::int64_t len = static_cast<std::int64_t>(m_) * 9;
    dse_count_ = 0;
    DBAG_CUDA(cudaMemsetAsync(x, 0, sizeof(S) * std::max<std::int64_t>(len, 1), st_));
    Scal init{};
    DBAG_CUDA(cudaMemcpyAsync(sc_.get(), &init, sizeof(Scal), cudaMemcpyHostToDevice, st_));
    launch_dot(g_.get(), g_.get(), len, &sc_.get()->rhs_norm2);
    read_scal();
    const double rhs_norm = std::sqrt(hsc_->rhs_norm2);
    if (rhs_norm == 0.0) return {0, true};
    // r = g - S x0 with x0 = 0: S 0 = 0 exactly, so r = g; the reference's
    // DSE on x0 (dba/solver.hpp:217) is still counted in the tallies.
    tally_.block_ops += 2 * static_cast<std::uint64_t>(N_);
    ++dse_count_;
    DBAG_CUDA(cudaMemcpyAsync(r_.get(), g_.get(), sizeof(S) * len, cudaMemcpyDeviceToDevice, st_));
    double r_norm = rhs_norm;
    int n = 0;
    const int rb = grid_for(m_, dev::kRedThreads, dev::kRedBlocksMax);
    const int vb = grid_for(len, dev::kRedThreads, dev::kRedBlocksMax);
    while (r_norm > tol * rhs_norm && n < max_iters) {
      const std::uint64_t ops0 = tally_.block_ops;
      const int dse0 = dse_count_;
      launch(dev::k_pcg_precond_inv<S>, vb, dev::kRedThreads, m_, static_cast<const S*>(Bexp_.get()),
             static_cast<const S*>(r_.get()), z_.get(), red(), sc_.get());
      launch(dev::k_pcg_p<S>, grid_for(len, 256, 1 << 30), 256, len, z_.get(), p_.get(),
             static_cast<const Scal*>(sc_.get()));
      dse<true>(p_.get(), q_.get());
      const std::uint64_t ops1 = tally_.block_ops;
      const int dse1 = dse_count_;
      const bool refresh = (n + 1) % 50 == 0;
      if (refresh) {
        launch(dev::k_pcg_xr<S, false>, vb, dev::kRedThreads, len, p_.get(), q_.get(), x, r_.get(), red(), sc_.get());
        dse<false>(x, q_.get());
        launch(dev::k_pcg_refresh<S>, vb, dev::kRedThreads, len, g_.get(), q_.get(), r_.get(), red(), sc_.get(), 1);
      } else {
        launch(dev::k_pcg_xr<S, true>, vb, dev::kRedThreads, len, p_.get(), q_.get(), x, r_.get(), red(), sc_.get());
      }
      read_scal();
      if (hsc_->status & 1) {  // rho breakdown: thrown before this iteration's DSE
        tally_.block_ops = ops0;
        dse_count_ = dse0;
        throw Error(DBAG_PCG_BREAKDOWN, "preconditioned residual norm rho = " + std::to_string(hsc_->rho) +
                                            " at iteration " + std::to_string(n));
      }
      if (hsc_->status & 2) {  // p'q breakdown: thrown after the DSE of p
        tally_.block_ops = ops1;
        dse_count_ = dse1;
        throw Error(DBAG_PCG_BREAKDOWN, "operator lost positive definiteness (p'q = " + std::to_string(hsc_->pq) +
                                            ") at iteration " + std::to_string(n));
      }
      ++n;
      r_norm = std::sqrt(hsc_->rnorm2);
    }
    return {n, r_norm <= tol * rhs_norm};
  }

  // ---- DPCG for K > 1 ranks: the graph body's kernels, run ahead ----------
  // The same device-side state machine as the graph (k_g_init, k_g_pass,
  // k_g_fold, k_g_step; scalars, loop decision, breakdowns and refresh
  // passes all on the device), with the cross-rank steps between them: the
  // halo all-reduce + k_halo_fix after the pass, the camera fold
  // (k_cam_reduce) + its all-reduce before k_g_fold. The host enqueues
  // kRunAhead body passes at a time and reads the scalars once per batch
  // (instead of once per PCG iteration); passes after the loop decision
  // return at entry, and every rank enqueues the same collectives, so the
  // call sequence stays aligned across ranks.
  PcgOut pcg_stream(double tol, int max_iters) {
    constexpr int kRunAhead = 8;
    if (!gsc_h_) DBAG_CUDA(cudaMallocHost(&gsc_h_, sizeof(dev::GScal<S>)));
    dev::GBufs<S> B = gbufs();
    B.c_total = ctmp_.get();
    const dev::RedWs ws = red();
    dev::GScal<S>* sc = gsc_.get();
    const dev::GScal<S>* csc = sc;
    const dev::DseArgs<S, T> A = dse_args(nullptr);
    dev::GScal<S> init{};
    init.tol = tol;
    init.max_iters = max_iters;
    *gsc_h_ = init;
    DBAG_CUDA(cudaMemcpyAsync(sc, gsc_h_, sizeof(init), cudaMemcpyHostToDevice, st_));
    const int lane_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 / 3 + 255) / 256 + 1);
    const int warp_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 + 255) / 256);
    const bool prof = profiling_;
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    launch(dev::k_g_init<S>, lane_blocks, dev::kRedThreads, B, ws, sc, dev::kNoCond);
    const std::int32_t nh = static_cast<std::int32_t>(lay_.halo_slot.size());
    std::int64_t passes = 0;
    for (;;) {
      for (int u = 0; u < kRunAhead; ++u, ++passes) {
        if (H_ > 0) DBAG_CUDA(cudaMemsetAsync(halo_buf_.get(), 0, sizeof(S) * 3 * static_cast<std::size_t>(H_), st_));
        launch_pass(A, B, csc);
        if (H_ > 0) {
          comm_->allreduce_sum(halo_buf_.get(), 3 * H_, kT, st_);
          if (nh > 0) halo_fix(nh);
        }
        cam_reduce<0>(nullptr, ctmp_.get());
        comm_->allreduce_sum(ctmp_.get(), static_cast<std::int64_t>(m_) * 9, kT, st_);
        launch(dev::k_g_fold<S>, warp_blocks, dev::kRedThreads, B, csc);
        launch(dev::k_g_step<S>, lane_blocks, dev::kRedThreads, B, ws, sc, dev::kNoCond);
      }
      DBAG_CUDA(cudaMemcpyAsync(gsc_h_, sc, sizeof(dev::GScal<S>), cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
      if (gsc_h_->done) break;
    }
    if (prof) {
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    }
    collect_profile();
    const dev::GScal<S> o = *gsc_h_;
    dse_count_ = o.dse_count;
    dse_launches_ += o.dse_count;
    tally_.block_ops += 2 * static_cast<std::uint64_t>(N_) * static_cast<std::uint64_t>(o.dse_count);
    if (o.status == 1)
      throw Error(DBAG_PCG_BREAKDOWN, "preconditioned residual norm rho = " + std::to_string(o.rho) +
                                          " at iteration " + std::to_string(o.n));
    if (o.status == 2)
      throw Error(DBAG_PCG_BREAKDOWN, "operator lost positive definiteness (p'q = " + std::to_string(o.pq) +
                                          ") at iteration " + std::to_string(o.n));
    return {o.n, std::sqrt(o.rnorm2) <= tol * std::sqrt(o.rhs_norm2)};
  }

  // ---- DPCG as one CUDA graph with conditional WHILE / IF nodes (K = 1) ----
  dev::GBufs<S> gbufs() {
    dev::GBufs<S> b;
    b.m = m_;
    b.Bd = Bd_.get();
    b.Binv = Bexp_.get();
    b.g = g_.get();
    b.x = dxc_.get();
    b.r = r_.get();
    b.z = z_.get();
    b.p0 = p_.get();
    b.p1 = p2_.get();
    b.q = q_.get();
    b.cam_part_ptr = cam_part_ptr_.get();
    b.part = part_.get();
    b.pq_cam = g_pq_cam_.get();
    b.c_total = nullptr;
    return b;
  }

  static cudaGraphNode_t add_kernel(cudaGraph_t g, const cudaGraphNode_t* dep, void* func, int grid, int block,
                                    void** args, int smem = 0) {
    cudaKernelNodeParams kp{};
    kp.func = func;
    kp.gridDim = dim3(static_cast<unsigned>(std::max(grid, 1)));
    kp.blockDim = dim3(static_cast<unsigned>(block));
    kp.sharedMemBytes = static_cast<unsigned>(smem);
    kp.kernelParams = args;
    cudaGraphNode_t n;
    DBAG_CUDA(cudaGraphAddKernelNode(&n, g, dep, dep ? 1 : 0, &kp));
    return n;
  }

  // Kernel node depending on `dep` through a programmatic edge (the
  // dependent may launch once every CTA of `dep` allowed it, and waits for
  // dep's completion at its griddepcontrol.wait).
  static cudaGraphNode_t add_kernel_pdl(cudaGraph_t g, cudaGraphNode_t dep, void* func, int grid, int block,
                                        void** args, int smem = 0) {
    cudaGraphNode_t n = add_kernel(g, nullptr, func, grid, block, args, smem);
    cudaGraphEdgeData e{};
    e.from_port = cudaGraphKernelNodePortProgrammatic;
    e.type = cudaGraphDependencyTypeProgrammatic;
    DBAG_CUDA(cudaGraphAddDependencies_v2(g, &dep, &n, &e, 1));
    return n;
  }

  static cudaGraph_t add_conditional(cudaGraph_t g, const cudaGraphNode_t* dep, cudaGraphConditionalHandle h,
                                     cudaGraphConditionalNodeType type, cudaGraphNode_t* node) {
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = 1;
    DBAG_CUDA(cudaGraphAddNode(node, g, dep, dep ? 1 : 0, &np));
    return np.conditional.phGraph_out[0];
  }

  void destroy_graph() {
    if (g_exec_) cudaGraphExecDestroy(g_exec_);
    if (g_graph_) cudaGraphDestroy(g_graph_);
    g_exec_ = nullptr;
    g_graph_ = nullptr;
  }

  void build_graph() {
    destroy_graph();
    if (!gsc_h_) DBAG_CUDA(cudaMallocHost(&gsc_h_, sizeof(dev::GScal<S>)));
    dev::GBufs<S> B = gbufs();
    dev::RedWs ws = red();
    dev::GScal<S>* sc = gsc_.get();
    dev::DseArgs<S, T> A = dse_args(nullptr);
    const int cam_lane_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 / 3 + 255) / 256 + 1);
    DBAG_CUDA(cudaGraphCreate(&g_graph_, 0));
    cudaGraphConditionalHandle hw;
    DBAG_CUDA(cudaGraphConditionalHandleCreate(&hw, g_graph_, 0, 0));
    void* a_init[] = {&B, &ws, &sc, &hw};
    cudaGraphNode_t n_init = add_kernel(g_graph_, nullptr, reinterpret_cast<void*>(dev::k_g_init<S>), cam_lane_blocks,
                                        dev::kRedThreads, a_init);
    cudaGraphNode_t n_while;
    cudaGraph_t body = add_conditional(g_graph_, &n_init, hw, cudaGraphCondTypeWhile, &n_while);
    const dev::GScal<S>* csc = sc;
    void* a_pass[] = {&A, &B, &csc};
    plan_fold_step();
    cudaGraphNode_t cur = nullptr;
    g_unroll_ = DBAG_GRAPH_UNROLL;
    if (const char* ue = std::getenv("DBAG_UNROLL")) g_unroll_ = std::max(1, std::atoi(ue));
    const bool streamed = use_stream();
    const dev::ChunkTab* tab = reinterpret_cast<const dev::ChunkTab*>(ctab_.get());
    std::int32_t nn = n_norm_;
    void* a_stream[] = {&A, &B, &csc, &tab, &nn};
    for (int u = 0; u < g_unroll_; ++u) {
      void* pass = fact_ ? reinterpret_cast<void*>(dev::k_g_pass<S, T, dev::kLanesFact>)
                         : reinterpret_cast<void*>(dev::k_g_pass<S, T, dev::kLanesDense>);
      int pgrid = n_long_ + n_chunks_, pblock = dev::kTile, psmem = 0;
      void** pargs = a_pass;
      if (streamed) {
        const StreamCfg& c = stream_cfg();
        pass = c.fn;
        pgrid = c.grid;
        pblock = dev::kStreamThreads;
        psmem = c.smem;
        pargs = a_stream;
      }
      cur = u ? add_kernel_pdl(body, cur, pass, pgrid, pblock, pargs, psmem)
              : add_kernel(body, nullptr, pass, pgrid, pblock, pargs, psmem);
      cur = add_fold_step(body, cur, B, sc, hw);
    }
    DBAG_CUDA(cudaGraphInstantiate(&g_exec_, g_graph_, 0));
    g_fact_ = fact_;
  }

  // The fold + step form of a DPCG body, by m: k_g_fsc (one thread-block
  // cluster) for small m, k_g_fs (warp per camera, grid barrier) while its
  // grid is co-resident, else k_g_fold + k_g_step. DBAG_FSC=0 / DBAG_FS=0
  // force the larger-m forms.
  void plan_fold_step() {
    const int cam_warp_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 + 255) / 256);
    // fused fold + step (k_g_fs) when its warp-per-camera grid is co-resident
    int fs_per_sm = 0, sms = 0;
    DBAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fs_per_sm, dev::k_g_fs<S>, dev::kRedThreads, 0));
    DBAG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    const char* fse = std::getenv("DBAG_FS");
    g_fused_ = !(fse && std::string(fse) == "0") && cam_warp_blocks <= fs_per_sm * sms &&
               cam_warp_blocks <= dev::kRedBlocksMax;
    DBAG_CUDA(cudaMemset(g_bar_.get(), 0, sizeof(unsigned long long)));
    // small m: fold + step as one thread-block cluster (k_g_fsc)
    const char* fcl = std::getenv("DBAG_FSC");
    g_cluster_ = 0;
    g_cpw_ = m_ <= 16 * dev::kFscWarps ? 1 : 2;
    const int fsc_ctas = static_cast<int>((m_ + g_cpw_ * dev::kFscWarps - 1) / (g_cpw_ * dev::kFscWarps));
    void* fsc_fn = g_cpw_ == 1 ? reinterpret_cast<void*>(dev::k_g_fsc<S, 1>) : reinterpret_cast<void*>(dev::k_g_fsc<S, 2>);
    if (!(fcl && std::string(fcl) == "0") && m_ > 0 && fsc_ctas <= 16) {
      DBAG_CUDA(cudaFuncSetAttribute(fsc_fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(static_cast<unsigned>(fsc_ctas));
      lc.blockDim = dim3(dev::kFscThreads);
      cudaLaunchAttribute at{};
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = static_cast<unsigned>(fsc_ctas);
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      lc.attrs = &at;
      lc.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, fsc_fn, &lc) == cudaSuccess && clusters > 0) g_cluster_ = fsc_ctas;
      cudaGetLastError();
    }
  }
  // Appends the planned fold + step node(s) after `cur` (programmatic edges).
  cudaGraphNode_t add_fold_step(cudaGraph_t body, cudaGraphNode_t cur, dev::GBufs<S> B, dev::GScal<S>* sc,
                                cudaGraphConditionalHandle hw) {
    dev::RedWs ws = red();
    const dev::GScal<S>* csc = sc;
    unsigned long long* bar = g_bar_.get();
    void* a_fold[] = {&B, &csc};
    void* a_step[] = {&B, &ws, &sc, &hw};
    void* a_fs[] = {&B, &ws, &sc, &hw, &bar};
    void* a_fsc[] = {&B, &sc, &hw};
    const int cam_warp_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 + 255) / 256);
    const int cam_lane_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 / 3 + 255) / 256 + 1);
    if (g_cluster_ > 0) {
      void* fsc_fn = g_cpw_ == 1 ? reinterpret_cast<void*>(dev::k_g_fsc<S, 1>) : reinterpret_cast<void*>(dev::k_g_fsc<S, 2>);
      cur = add_kernel_pdl(body, cur, fsc_fn, g_cluster_, dev::kFscThreads, a_fsc);
      cudaLaunchAttributeValue cv{};
      cv.clusterDim.x = static_cast<unsigned>(g_cluster_);
      cv.clusterDim.y = 1;
      cv.clusterDim.z = 1;
      DBAG_CUDA(cudaGraphKernelNodeSetAttribute(cur, cudaLaunchAttributeClusterDimension, &cv));
      return cur;
    }
    if (g_fused_)
      return add_kernel_pdl(body, cur, reinterpret_cast<void*>(dev::k_g_fs<S>), cam_warp_blocks, dev::kRedThreads, a_fs);
    cur = add_kernel_pdl(body, cur, reinterpret_cast<void*>(dev::k_g_fold<S>), cam_warp_blocks, dev::kRedThreads, a_fold);
    return add_kernel_pdl(body, cur, reinterpret_cast<void*>(dev::k_g_step<S>), cam_lane_blocks, dev::kRedThreads,
                          a_step);
  }

  PcgOut pcg_graph(double tol, int max_iters) {
    if (!g_exec_ || g_fact_ != fact_) build_graph();
    dev::GScal<S> init{};
    init.tol = tol;
    init.max_iters = max_iters;
    *gsc_h_ = init;
    DBAG_CUDA(cudaMemcpyAsync(gsc_.get(), gsc_h_, sizeof(init), cudaMemcpyHostToDevice, st_));
    const bool prof = profiling_;
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    DBAG_CUDA(cudaGraphLaunch(g_exec_, st_));
    if (prof) {
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    }
    DBAG_CUDA(cudaMemcpyAsync(gsc_h_, gsc_.get(), sizeof(init), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    collect_profile();
#if DBAG_GTIMING
    {
      static unsigned long long t[dev::kTlStride * 1024];
      DBAG_CUDA(cudaMemcpyFromSymbol(t, dev::g_tl, sizeof(t)));
      const int nn = std::min(gsc_h_->n, 1023);
      double acc[8] = {0};
      int cnt = 0;
      for (int k = 1; k + 1 < nn; ++k) {
        if ((k + 1) % 50 == 0 || k % 50 == 0) continue;
        bool ok = true;
        for (int q = 0; q < 7; ++q) ok = ok && t[k * dev::kTlStride + q] != 0;
        if (!ok) continue;
        for (int q = 0; q < 6; ++q) acc[q] += double(t[k * dev::kTlStride + q + 1]) - double(t[k * dev::kTlStride + q]);
        acc[6] += double(t[(k + 1) * dev::kTlStride]) - double(t[k * dev::kTlStride + 6]);
        ++cnt;
      }
      double lr[64] = {0};
      int lc[64] = {0};
      const int u = std::max(1, std::min(g_unroll_, 64));
      for (int k = 1; k + 1 < nn; ++k) {
        if ((k + 1) % 50 == 0 || k % 50 == 0 || !t[k * dev::kTlStride + 6] || !t[(k + 1) * dev::kTlStride]) continue;
        lr[k % u] += double(t[(k + 1) * dev::kTlStride]) - double(t[k * dev::kTlStride + 6]);
        ++lc[k % u];
      }
      for (int par = 0; par < 2; ++par) {
        double a[8] = {0};
        int c2 = 0;
        for (int k = 1; k + 1 < nn; ++k) {
          if ((k + 1) % 50 == 0 || k % 50 == 0 || (k & 1) != par) continue;
          bool ok = t[(k + 1) * dev::kTlStride] != 0;
          for (int q = 0; q < 7; ++q) ok = ok && t[k * dev::kTlStride + q] != 0;
          if (!ok) continue;
          for (int q = 0; q < 6; ++q) a[q] += double(t[k * dev::kTlStride + q + 1]) - double(t[k * dev::kTlStride + q]);
          a[6] += double(t[(k + 1) * dev::kTlStride]) - double(t[k * dev::kTlStride + 6]);
          ++c2;
        }
        double st = 0.0;
        for (int k = 1; k + 1 < nn; ++k) {
          if ((k + 1) % 50 == 0 || k % 50 == 0 || (k & 1) != par || !t[(k + 1) * dev::kTlStride + 7] || !t[k * dev::kTlStride + 6]) continue;
          st += double(t[(k + 1) * dev::kTlStride + 7]) - double(t[k * dev::kTlStride + 6]);
        }
        std::fprintf(stderr, "GTIMING n%%2=%d: next-pass CTA0 start - decision %.2f; segs", par, c2 ? st / c2 / 1e3 : 0.0);
        for (int q = 0; q < 7; ++q) std::fprintf(stderr, " %.2f", c2 ? a[q] / c2 / 1e3 : 0.0);
        std::fprintf(stderr, "\n");
      }
      std::fprintf(stderr, "GTIMING loop by n mod %d (us):", u);
      for (int q = 0; q < u; ++q) std::fprintf(stderr, " %.2f", lc[q] ? lr[q] / lc[q] / 1e3 : 0.0);
      std::fprintf(stderr, "\n");
      if (cnt)
        std::fprintf(stderr, "GTIMING n=%d marks(us): pass->fs %.2f sc %.2f fold %.2f barrier %.2f pqsum %.2f step %.2f loop %.2f\n",
                     nn, acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3, acc[4] / cnt / 1e3,
                     acc[5] / cnt / 1e3, acc[6] / cnt / 1e3);
    }
#endif
    const dev::GScal<S> o = *gsc_h_;
    // k_g_init + 3 kernels per body pass (the no-op copies of the last
    // unrolled body launch too)
    const std::int64_t passes = std::max(o.dse_count - 1, 0);
    launches_ += 1 + (g_fused_ || g_cluster_ > 0 ? 2 : 3) * ((passes + g_unroll_ - 1) / g_unroll_) * g_unroll_;
    dse_count_ = o.dse_count;
    dse_launches_ += o.dse_count;
    tally_.block_ops += 2 * static_cast<std::uint64_t>(N_) * static_cast<std::uint64_t>(o.dse_count);
    if (o.status == 1)
      throw Error(DBAG_PCG_BREAKDOWN, "preconditioned residual norm rho = " + std::to_string(o.rho) +
                                          " at iteration " + std::to_string(o.n));
    if (o.status == 2)
      throw Error(DBAG_PCG_BREAKDOWN, "operator lost positive definiteness (p'q = " + std::to_string(o.pq) +
                                          ") at iteration " + std::to_string(o.n));
    return {o.n, std::sqrt(o.rnorm2) <= tol * std::sqrt(o.rhs_norm2)};
  }
  // ---- DPCG for K > 1 ranks as one CUDA graph per rank ---------------------
  // The K = 1 graph's state machine with the cross-rank steps inside the
  // WHILE body, all on the device: pass -> halo all-reduce (peer) ->
  // k_halo_fix -> camera fold of the rank's partials (k_cam_reduce) ->
  // camera all-reduce (peer) -> k_g_fold (reads the summed camera vector) ->
  // k_g_step. The ranks' graphs synchronise only through the peer
  // collectives; every loop decision is taken from rank-identical bits.
  void build_graph_k() {
    gk_destroy();
    if (!gsc_h_) DBAG_CUDA(cudaMallocHost(&gsc_h_, sizeof(dev::GScal<S>)));
    dev::GBufs<S> B = gbufs();
    dev::RedWs ws = red();
    dev::GScal<S>* sc = gsc_.get();
    // peer waits bounded by the collective timeout; absent ranks -> sc->peer_fail
    const unsigned long long tmo_ns =
        static_cast<unsigned long long>(std::max<std::int64_t>(comm_->timeout().count(), 1)) * 1000000ull;
    for (PeerSite* ps : {&ps_cam_, &ps_halo_}) {
      ps->timeout_ns = tmo_ns;
      ps->failed = &sc->peer_fail;
    }
    const dev::GScal<S>* csc = sc;
    dev::DseArgs<S, T> A = dse_args(nullptr);
    const int lane_blocks = static_cast<int>((static_cast<std::int64_t>(m_) * 32 / 3 + 255) / 256 + 1);
    DBAG_CUDA(cudaGraphCreate(&gk_graph_, 0));
    cudaGraphConditionalHandle hw;
    DBAG_CUDA(cudaGraphConditionalHandleCreate(&hw, gk_graph_, 0, 0));
    void* a_init[] = {&B, &ws, &sc, &hw};
    cudaGraphNode_t n_init = add_kernel(gk_graph_, nullptr, reinterpret_cast<void*>(dev::k_g_init<S>), lane_blocks,
                                        dev::kRedThreads, a_init);
    cudaGraphNode_t n_while;
    cudaGraph_t body = add_conditional(gk_graph_, &n_init, hw, cudaGraphCondTypeWhile, &n_while);
    void* a_pass[] = {&A, &B, &csc};
    const int* skip = &sc->done;
    // halo: all-reduce of the deposits (halo_buf: zero outside this rank's
    // points) into halo_sum, then this rank's halo slots (k_peer_halo)
    const S* hb = halo_buf_.get();
    S* hs = halo_sum_.get();
    std::int64_t nh = 3 * static_cast<std::int64_t>(H_);
    std::int32_t nhs = static_cast<std::int32_t>(lay_.halo_slot.size());
    const std::int32_t* hslot = halo_slot_.get();
    const std::int32_t* sdpt = slot_dpt_.get();
    const std::int32_t* hof = halo_of_.get();
    const S* cinv = Cinv_.get();
    const T* erec = static_cast<const T*>(fact_ ? E_.get() : Edense_.get());
    const std::int32_t* sch = slot_chunk_.get();
    const std::int32_t* chs = chunk_slot_.get();
    const std::int32_t* hpos = halo_pos_.get();
    S* part = part_.get();
    const std::int32_t* scam = slot_cam_.get();
    const S* rm = Rm_.get();
    void* a_halo[] = {&ps_halo_, &hb, &hs, &nh, &skip, &nhs, &hslot, &sdpt, &hof, &cinv, &erec, &sch, &chs, &hpos,
                      &part, &scam, &rm};
    void* halo = fact_ ? reinterpret_cast<void*>(dev::k_peer_halo<S, T, dev::kLanesFact>)
                       : reinterpret_cast<void*>(dev::k_peer_halo<S, T, dev::kLanesDense>);
    // camera side: this rank's partials folded per camera and summed over
    // ranks into ctmp (k_peer_cam); the fold + step kernels then read it as
    // one partial per camera (identity partial pointers)
    std::int32_t mm = m_;
    const std::int32_t* cpp = cam_part_ptr_.get();
    const S* cparts = part_.get();
    S* ct = ctmp_.get();
    void* a_cam[] = {&ps_cam_, &mm, &cpp, &cparts, &ct, &skip};
    dev::GBufs<S> Bk = B;
    Bk.part = ctmp_.get();
    Bk.cam_part_ptr = cam_ident_.get();
    plan_fold_step();
    cudaGraphNode_t cur = nullptr;
    gk_unroll_ = DBAG_GRAPH_UNROLL;
    if (const char* ue = std::getenv("DBAG_UNROLL")) gk_unroll_ = std::max(1, std::atoi(ue));
    void* pass = fact_ ? reinterpret_cast<void*>(dev::k_g_pass<S, T, dev::kLanesFact>)
                       : reinterpret_cast<void*>(dev::k_g_pass<S, T, dev::kLanesDense>);
    for (int u = 0; u < gk_unroll_; ++u) {
      cur = u ? add_kernel_pdl(body, cur, pass, n_long_ + n_chunks_, dev::kTile, a_pass)
              : add_kernel(body, nullptr, pass, n_long_ + n_chunks_, dev::kTile, a_pass);
      if (H_ > 0) cur = add_kernel(body, &cur, halo, 1, dev::kPeerThreads, a_halo);
      cur = add_kernel(body, &cur, reinterpret_cast<void*>(dev::k_peer_cam<S>), ps_cam_.nslice, dev::kPeerThreads,
                       a_cam);
      cur = add_fold_step(body, cur, Bk, sc, hw);
    }
    DBAG_CUDA(cudaGraphInstantiate(&gk_exec_, gk_graph_, 0));
    gk_fact_ = fact_;
  }

  PcgOut pcg_graph_k(double tol, int max_iters) {
    if (!gk_exec_ || gk_fact_ != fact_) build_graph_k();
    dev::GScal<S> init{};
    init.tol = tol;
    init.max_iters = max_iters;
    *gsc_h_ = init;
    DBAG_CUDA(cudaMemcpyAsync(gsc_.get(), gsc_h_, sizeof(init), cudaMemcpyHostToDevice, st_));
    // halo deposits: entries of other ranks' points stay zero through the solve
    if (H_ > 0) DBAG_CUDA(cudaMemsetAsync(halo_buf_.get(), 0, sizeof(S) * 3 * static_cast<std::size_t>(H_), st_));
    const bool prof = profiling_;
    if (prof) DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    DBAG_CUDA(cudaGraphLaunch(gk_exec_, st_));
    if (prof) {
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
      DBAG_CUDA(cudaEventRecord(prof_event(), st_));
    }
    DBAG_CUDA(cudaMemcpyAsync(gsc_h_, gsc_.get(), sizeof(init), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    collect_profile();
    const dev::GScal<S> o = *gsc_h_;
    if (o.peer_fail) {
      std::string who;
      for (int p = 0; p < comm_->size(); ++p)
        if (o.peer_fail & (1 << p)) who += (who.empty() ? "" : ", ") + std::to_string(p);
      throw Error(DBAG_COLLECTIVE, "collective timeout after " + std::to_string(comm_->timeout().count()) +
                                       " ms in the device all-reduce of the DPCG graph: rank(s) " + who +
                                       " did not arrive");
    }
    const std::int64_t passes = std::max(o.dse_count - 1, 0);
    const int per_body = 2 + (H_ > 0 ? 1 : 0) + (g_fused_ || g_cluster_ > 0 ? 1 : 2);
    launches_ += 1 + per_body * ((passes + gk_unroll_ - 1) / gk_unroll_) * gk_unroll_;
    dse_count_ = o.dse_count;
    dse_launches_ += o.dse_count;
    tally_.block_ops += 2 * static_cast<std::uint64_t>(N_) * static_cast<std::uint64_t>(o.dse_count);
    if (o.status == 1)
      throw Error(DBAG_PCG_BREAKDOWN, "preconditioned residual norm rho = " + std::to_string(o.rho) +
                                          " at iteration " + std::to_string(o.n));
    if (o.status == 2)
      throw Error(DBAG_PCG_BREAKDOWN, "operator lost positive definiteness (p'q = " + std::to_string(o.pq) +
                                          ") at iteration " + std::to_string(o.n));
    return {o.n, std::sqrt(o.rnorm2) <= tol * std::sqrt(o.rhs_norm2)};
  }

  // Device time of the graph body's DSE pass (k_g_pass) launched alone,
  // back to back, on the state the last graph DPCG left (bench roofline).
  double time_dse_pass(int reps) {
    DBAG_CUDA(cudaSetDevice(device_));
    if (!g_exec_) throw Error(DBAG_INVALID_ARGUMENT, "time_dse_pass needs a preceding graph DPCG");
    const dev::DseArgs<S, T> A = dse_args(nullptr);
    const dev::GBufs<S> B = gbufs();
    const dev::GScal<S>* sc = gsc_.get();
    dev::GScal<S> live = *gsc_h_;  // the finished solve's scalars, reopened
    live.done = 0;
    *gsc_h_ = live;
    DBAG_CUDA(cudaMemcpyAsync(gsc_.get(), gsc_h_, sizeof(live), cudaMemcpyHostToDevice, st_));
    cudaEvent_t e0, e1;
    DBAG_CUDA(cudaEventCreate(&e0));
    DBAG_CUDA(cudaEventCreate(&e1));
    auto one = [&] { launch_pass(A, B, sc); };
    one();  // warm-up
    DBAG_CUDA(cudaEventRecord(e0, st_));
    for (int r = 0; r < reps; ++r) one();
    DBAG_CUDA(cudaEventRecord(e1, st_));
    DBAG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    DBAG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return static_cast<double>(ms) / std::max(reps, 1);
  }


  // ------------------------------------------- back-substitution + trial ----
  void backsub_trial() {
    DBAG_CUDA(cudaSetDevice(device_));
    if (H_ > 0) DBAG_CUDA(cudaMemsetAsync(halo_buf_.get(), 0, sizeof(S) * 3 * static_cast<std::size_t>(H_), st_));
    stream_pass<1>(dxc_.get());
    if (H_ > 0) {
      comm_->allreduce_sum(halo_buf_.get(), 3 * H_, kT, st_);
      if (n_halo_loc_ > 0)
        launch(dev::k_halo_finish<S, 1>, grid_for(n_halo_loc_, 128, 1 << 30), 128, n_halo_loc_, halo_dpt_.get(),
               halo_idx_.get(), static_cast<const S*>(halo_buf_.get()), static_cast<const S*>(Cinv_.get()),
               static_cast<const S*>(w_.get()), dxp_.get());
    }
    tally_.block_ops += static_cast<std::uint64_t>(N_);
    double* d = dsc_.get();
    const int cb = grid_for(m_, dev::kRedThreads, dev::kRedBlocksMax);
    launch(dev::k_trial<S, 9>, cb, dev::kRedThreads, m_, xc_.get(), dxc_.get(), xct_.get(), B_.get(), v_.get(),
           static_cast<const std::uint8_t*>(nullptr), lambda_, policy_, red(), d + 16);
    DBAG_CUDA(cudaMemsetAsync(d + 20, 0, 4 * sizeof(double), st_));
    if (n_loc_ > 0)
      launch(dev::k_trial<S, 3>, grid_for(n_loc_, dev::kRedThreads, dev::kRedBlocksMax), dev::kRedThreads, n_loc_,
             xp_.get(), dxp_.get(), xpt_.get(), C_.get(), w_.get(), static_cast<const std::uint8_t*>(owned_.get()),
             lambda_, policy_, red(), d + 20);
    // point terms: max over ranks for d[20], sums for d[21..22]
    comm_->allreduce_max(d + 20, 1, DType::f64, st_);
    comm_->allreduce_sum(d + 21, 2, DType::f64, st_);
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, d + 16, 8 * sizeof(double), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    step_inf_ = std::max(hbuf_[0], hbuf_[4]);
    damp_term_ = policy_ == 0 ? lambda_ * (hbuf_[1] + hbuf_[5]) : hbuf_[1] + hbuf_[5];
    gv_ = hbuf_[2] + hbuf_[6];
  }

  double damping_lambda() const { return lambda_; }
  int damping_policy() const { return policy_; }

  // The full state on every rank (lm_solve returns rank 0's, and every
  // rank's is identical, dba/solver.hpp:282-285, 533): x_c is replicated;
  // x_p is zero-filled in global order, each rank scatters the points it
  // owns, and a sum-all-reduce over the communicator assembles it (every
  // entry gets exactly one nonzero contribution, so the sum is exact).
  void gather_state(S* xc, S* xp) {
    DBAG_CUDA(cudaSetDevice(device_));
    if (xc)
      DBAG_CUDA(cudaMemcpyAsync(xc, xc_.get(), sizeof(S) * 9 * static_cast<std::size_t>(m_), cudaMemcpyDeviceToHost, st_));
    const std::size_t full = static_cast<std::size_t>(n_glob_) * 3;
    DBAG_CUDA(cudaMemsetAsync(xp_full_.get(), 0, sizeof(S) * std::max<std::size_t>(full, 1), st_));
    if (n_loc_ > 0)
      launch(dev::k_owned_rows<S>, grid_for(n_loc_, 256, 1 << 30), 256, n_loc_,
             static_cast<const std::int32_t*>(dpt_glob_d_.get()), static_cast<const std::uint8_t*>(owned_.get()),
             static_cast<const S*>(xp_.get()), xp_full_.get());
    comm_->allreduce_sum(xp_full_.get(), static_cast<std::int64_t>(full), kT, st_);
    if (xp) DBAG_CUDA(cudaMemcpyAsync(xp, xp_full_.get(), sizeof(S) * full, cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    if (xp)  // unobserved points: unchanged since set_state (the reference never moves them)
      for (std::size_t i = 0; i < orphans_.size(); ++i)
        for (int k = 0; k < 3; ++k) xp[static_cast<std::size_t>(orphans_[i]) * 3 + k] = orphan_x_[i * 3 + k];
  }

  void model_terms(double* step_inf, double* damp, double* gv) const {
    *step_inf = step_inf_;
    *damp = damp_term_;
    *gv = gv_;
  }

  void accept() {
    xc_.swap(xct_);
    xp_.swap(xpt_);
    have_system_ = false;
  }

  bool have_system() const { return have_system_; }

  // ---------------------------------------------------- rank identity ----
  // |x_c|_inf and |x_p|_inf (over owned points, max over ranks).
  void state_inf(double* ic, double* ip) {
    DBAG_CUDA(cudaSetDevice(device_));
    std::vector<S> hc(static_cast<std::size_t>(m_) * 9), hp(static_cast<std::size_t>(n_loc_) * 3);
    DBAG_CUDA(cudaMemcpyAsync(hc.data(), xc_.get(), sizeof(S) * hc.size(), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaMemcpyAsync(hp.data(), xp_.get(), sizeof(S) * hp.size(), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    double a = 0, b = 0;
    for (S v : hc) a = std::max(a, double(std::abs(v)));
    for (std::int32_t d = 0; d < n_loc_; ++d)
      if (owned_h_[static_cast<std::size_t>(d)])
        for (int k = 0; k < 3; ++k) b = std::max(b, double(std::abs(hp[static_cast<std::size_t>(d) * 3 + k])));
    double* dd = dsc_.get();
    hbuf_[0] = b;
    DBAG_CUDA(cudaMemcpyAsync(dd + 30, hbuf_, sizeof(double), cudaMemcpyHostToDevice, st_));
    comm_->allreduce_max(dd + 30, 1, DType::f64, st_);
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, dd + 30, sizeof(double), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    *ic = a;
    *ip = hbuf_[0];
  }

  // Sum-all-reduce of a small host vector (at most 4K doubles: the per-rank
  // tallies and the rank-identity probe) through the pool's bounce buffer.
  void allreduce_host(double* v, int n) {
    DBAG_CUDA(cudaSetDevice(device_));
    if (comm_->size() == 1) return;
    if (bounce_.size() < static_cast<std::size_t>(n)) throw Error(DBAG_INTERNAL, "host all-reduce exceeds the bounce buffer");
    DBAG_CUDA(cudaMemcpyAsync(bounce_.get(), v, sizeof(double) * n, cudaMemcpyHostToDevice, st_));
    comm_->allreduce_sum(bounce_.get(), n, DType::f64, st_);
    DBAG_CUDA(cudaMemcpyAsync(v, bounce_.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
  }

  // ------------------------------------------------------- test hooks ----
  // Cost-path residuals of the current (or trial) state, shard edge order.
  void residuals(bool trial, S* out) {
    DBAG_CUDA(cudaSetDevice(device_));
    DevBuf<S> r;
    r.alloc(std::max<std::size_t>(static_cast<std::size_t>(N_) * 2, 1));
    if (N_ > 0)
      launch(dev::k_residuals<S>, grid_for(N_, 128, 1 << 30), 128, N_, slot_cam_.get(), slot_dpt_.get(),
             slot_edge_.get(), slot_px_.get(), slot_py_.get(), trial ? xct_.get() : xc_.get(),
             trial ? xpt_.get() : xp_.get(), r.get());
    DBAG_CUDA(cudaMemcpyAsync(out, r.get(), sizeof(S) * 2 * static_cast<std::size_t>(N_), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
  }

  void get_jacobians(S* res, S* jac) {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    std::vector<S> jb(static_cast<std::size_t>(N_) * 28);
    if (lin_rows()) {
      if (jb_pt_.size() > 2) throw Error(DBAG_INVALID_ARGUMENT, "Jacobian rows are kept for one Jb batch only");
      DBAG_CUDA(cudaMemcpy(jb.data(), Jb_.get(), sizeof(S) * jb.size(), cudaMemcpyDeviceToHost));
    } else if (N_ > 0) {
      // test hook: the fused linearize keeps no rows; recompute them at the
      // same state into a temporary (outside the pool; rewrites the same
      // records bit for bit)
      S* tmp = nullptr;
      DBAG_CUDA(cudaMalloc(&tmp, sizeof(S) * jb.size()));
      std::unique_ptr<void, void (*)(void*)> keep(tmp, [](void* q) { cudaFree(q); });
      auto kern = jac_mode_ == 1 ? dev::k_linearize<S, 1, T, dev::kLanesFact> : dev::k_linearize<S, 0, T, dev::kLanesFact>;
      DBAG_CUDA(cudaMemsetAsync(bad_.get(), 0xff, sizeof(unsigned long long), st_));
      launch(kern, static_cast<int>((N_ + 127) / 128), 128, std::int64_t(0), N_, slot_cam_.get(), slot_dpt_.get(),
             slot_edge_.get(), plan_.range.start, slot_px_.get(), slot_py_.get(), slot_w_.get(), xc_.get(), xp_.get(),
             tmp, E_.get(), slot_chunk_.get(), chunk_slot_.get(), bad_.get());
      DBAG_CUDA(cudaMemcpyAsync(jb.data(), tmp, sizeof(S) * jb.size(), cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
    }
    for (std::int64_t s = 0; s < N_; ++s) {
      const std::int64_t e = lay_.slot_edge[static_cast<std::size_t>(s)];
      const S* row = jb.data() + static_cast<std::size_t>(s) * 28;
      res[e] = row[0];
      res[N_ + e] = row[1];
      for (int j = 0; j < 12; ++j) {
        jac[static_cast<std::size_t>(j) * N_ + e] = row[2 + j];
        jac[static_cast<std::size_t>(12 + j) * N_ + e] = row[14 + j];
      }
    }
  }

  void get_system(S* B, S* C, S* E, S* v, S* w) {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    if (B) DBAG_CUDA(cudaMemcpy(B, B_.get(), sizeof(S) * 81 * static_cast<std::size_t>(m_), cudaMemcpyDeviceToHost));
    if (v) DBAG_CUDA(cudaMemcpy(v, v_.get(), sizeof(S) * 9 * static_cast<std::size_t>(m_), cudaMemcpyDeviceToHost));
    std::vector<S> c(static_cast<std::size_t>(n_loc_) * 9), ww(static_cast<std::size_t>(n_loc_) * 3);
    DBAG_CUDA(cudaMemcpy(c.data(), C_.get(), sizeof(S) * c.size(), cudaMemcpyDeviceToHost));
    DBAG_CUDA(cudaMemcpy(ww.data(), w_.get(), sizeof(S) * ww.size(), cudaMemcpyDeviceToHost));
    if (C) std::fill(C, C + static_cast<std::size_t>(n_glob_) * 9, S(0));
    if (w) std::fill(w, w + static_cast<std::size_t>(n_glob_) * 3, S(0));
    for (std::int32_t d = 0; d < n_loc_; ++d) {
      const std::size_t g = static_cast<std::size_t>(dpt_glob_[static_cast<std::size_t>(d)]);
      if (C) std::copy(c.begin() + d * 9, c.begin() + d * 9 + 9, C + g * 9);
      if (w) std::copy(ww.begin() + d * 3, ww.begin() + d * 3 + 3, w + g * 3);
    }
    if (E) {
      std::vector<std::int32_t> scam(static_cast<std::size_t>(N_));
      if (N_ > 0)
        DBAG_CUDA(cudaMemcpy(scam.data(), slot_cam_.get(), sizeof(std::int32_t) * scam.size(), cudaMemcpyDeviceToHost));
      if (fact_) {  // E = G^T Gt R (kernels.cuh kLanesFact)
        std::vector<T> e(E_.size());
        std::vector<S> R(static_cast<std::size_t>(m_) * 9);
        DBAG_CUDA(cudaMemcpy(e.data(), E_.get(), sizeof(T) * e.size(), cudaMemcpyDeviceToHost));
        DBAG_CUDA(cudaMemcpy(R.data(), Rm_.get(), sizeof(S) * R.size(), cudaMemcpyDeviceToHost));
        for (std::int64_t s = 0; s < N_; ++s) {
          const std::int64_t ed = lay_.slot_edge[static_cast<std::size_t>(s)];
          const std::size_t at = rec_offset<dev::kLanesFact>(s);
          double g[18];
          for (int k = 0; k < 18; ++k) g[k] = double(e[at + static_cast<std::size_t>(k) * dev::kTile]);
          const S* Rc = R.data() + static_cast<std::size_t>(scam[static_cast<std::size_t>(s)]) * 9;
          double jp[2][3];
          for (int r = 0; r < 2; ++r)
            for (int j = 0; j < 3; ++j)
              jp[r][j] = g[r * 9 + 3] * double(Rc[j]) + g[r * 9 + 4] * double(Rc[3 + j]) + g[r * 9 + 5] * double(Rc[6 + j]);
          for (int i = 0; i < 9; ++i)
            for (int j = 0; j < 3; ++j) E[ed * 27 + i * 3 + j] = S(g[i] * jp[0][j] + g[9 + i] * jp[1][j]);
        }
      } else {
        std::vector<T> e(Edense_.size());
        DBAG_CUDA(cudaMemcpy(e.data(), Edense_.get(), sizeof(T) * e.size(), cudaMemcpyDeviceToHost));
        for (std::int64_t s = 0; s < N_; ++s) {
          const std::int64_t ed = lay_.slot_edge[static_cast<std::size_t>(s)];
          const std::size_t at = rec_offset<dev::kLanesDense>(s);
          for (int k = 0; k < 27; ++k) E[ed * 27 + k] = S(e[at + static_cast<std::size_t>(k) * dev::kTile]);
        }
      }
    }
  }

  // Caller-fabricated system (test hook): full-size B, C, v, w and the
  // E_table of the whole problem in global edge order.
  void set_system(const S* B, const S* C, const S* E_table, const S* v, const S* w) {
    DBAG_CUDA(cudaSetDevice(device_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    if (B) DBAG_CUDA(cudaMemcpy(B_.get(), B, sizeof(S) * 81 * static_cast<std::size_t>(m_), cudaMemcpyHostToDevice));
    if (v) DBAG_CUDA(cudaMemcpy(v_.get(), v, sizeof(S) * 9 * static_cast<std::size_t>(m_), cudaMemcpyHostToDevice));
    if (C || w) {
      std::vector<S> c(static_cast<std::size_t>(n_loc_) * 9), ww(static_cast<std::size_t>(n_loc_) * 3);
      DBAG_CUDA(cudaMemcpy(c.data(), C_.get(), sizeof(S) * c.size(), cudaMemcpyDeviceToHost));
      DBAG_CUDA(cudaMemcpy(ww.data(), w_.get(), sizeof(S) * ww.size(), cudaMemcpyDeviceToHost));
      for (std::int32_t d = 0; d < n_loc_; ++d) {
        const std::size_t g = static_cast<std::size_t>(dpt_glob_[static_cast<std::size_t>(d)]);
        if (C) std::copy(C + g * 9, C + g * 9 + 9, c.begin() + d * 9);
        if (w) std::copy(w + g * 3, w + g * 3 + 3, ww.begin() + d * 3);
      }
      DBAG_CUDA(cudaMemcpy(C_.get(), c.data(), sizeof(S) * c.size(), cudaMemcpyHostToDevice));
      DBAG_CUDA(cudaMemcpy(w_.get(), ww.data(), sizeof(S) * ww.size(), cudaMemcpyHostToDevice));
    }
    if (E_table) {  // arbitrary 9x3 blocks: the dense record layout from here on
      std::vector<std::int32_t> scam(static_cast<std::size_t>(N_));
      if (N_ > 0)
        DBAG_CUDA(cudaMemcpy(scam.data(), slot_cam_.get(), sizeof(std::int32_t) * scam.size(), cudaMemcpyDeviceToHost));
      std::vector<T> e = build_records<dev::kLanesDense>(scam);
      for (std::int64_t s = 0; s < N_; ++s) {
        const std::int64_t ed = plan_.range.start + lay_.slot_edge[static_cast<std::size_t>(s)];
        const std::size_t at = rec_offset<dev::kLanesDense>(s);
        for (int k = 0; k < 27; ++k) e[at + static_cast<std::size_t>(k) * dev::kTile] = T(E_table[ed * 27 + k]);
      }
      if (Edense_.size() != e.size()) Edense_.alloc(e.size());
      Edense_.copy_in(e);
      fact_ = false;
    }
    have_system_ = true;
  }

  template <int L>
  std::size_t rec_offset(std::int64_t s) const {
    const std::int32_t c = lay_.slot_chunk[static_cast<std::size_t>(s)];
    return static_cast<std::size_t>(c) * dev::Rec<T, L>::kLen +
           static_cast<std::size_t>(s - lay_.chunk_slot[static_cast<std::size_t>(c)]);
  }

  // Fabricated blocks are already damped: factor them as-is (identity
  // damping with lambda = 0 adds exactly 0 to every diagonal entry).
  void factor_as_is() { damp_factor(0.0, 0); }

  void dse_host(const S* x, S* out) {
    DBAG_CUDA(cudaSetDevice(device_));
    const std::size_t len = static_cast<std::size_t>(m_) * 9;
    DBAG_CUDA(cudaMemcpyAsync(p_.get(), x, sizeof(S) * len, cudaMemcpyHostToDevice, st_));
    dse<false>(p_.get(), q_.get());
    DBAG_CUDA(cudaMemcpyAsync(out, q_.get(), sizeof(S) * len, cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
  }

  // One trial's intermediate results for the cross-K tests (group_operator
  // modes): 2 g (rhs), 3 dx_c after DPCG, 4 [cost_new, step_inf, damping
  // term, dx.v + dx.w], 5 v.
  void trial_probe(int mode, double tol, int max_iters, S* out) {
    DBAG_CUDA(cudaSetDevice(device_));
    const std::size_t len = static_cast<std::size_t>(m_) * 9;
    if (mode == 5) {
      DBAG_CUDA(cudaMemcpyAsync(out, v_.get(), sizeof(S) * len, cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
      return;
    }
    rhs();
    if (mode == 2) {
      DBAG_CUDA(cudaMemcpyAsync(out, g_.get(), sizeof(S) * len, cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
      return;
    }
    pcg(tol, max_iters);
    if (mode == 3) {
      DBAG_CUDA(cudaMemcpyAsync(out, dxc_.get(), sizeof(S) * len, cudaMemcpyDeviceToHost, st_));
      DBAG_CUDA(cudaStreamSynchronize(st_));
      return;
    }
    backsub_trial();
    std::int64_t bad = -1;
    const double c = cost(true, &bad);
    out[0] = S(c);
    out[1] = S(step_inf_);
    out[2] = S(damp_term_);
    out[3] = S(gv_);
  }

  PcgOut dpcg_host(const S* rhs, double tol, int max_iters, S* x_out) {
    DBAG_CUDA(cudaSetDevice(device_));
    const std::size_t len = static_cast<std::size_t>(m_) * 9;
    DBAG_CUDA(cudaMemcpyAsync(g_.get(), rhs, sizeof(S) * len, cudaMemcpyHostToDevice, st_));
    const PcgOut o = pcg(tol, max_iters);
    DBAG_CUDA(cudaMemcpyAsync(x_out, dxc_.get(), sizeof(S) * len, cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    return o;
  }

  // ---------------------------------------------------- timing hooks ----
  void mark(int which) { DBAG_CUDA(cudaEventRecord(mark_[which & 1], st_)); }
  double elapsed_ms() {
    DBAG_CUDA(cudaEventSynchronize(mark_[1]));
    float ms = 0;
    DBAG_CUDA(cudaEventElapsedTime(&ms, mark_[0], mark_[1]));
    return ms;
  }
  void set_profiling(bool on) {
    collect_profile();
    profiling_ = on;
    prof_point_ms_ = prof_cam_ms_ = 0;
    dse_launches_ = 0;
  }
  void profile(double* total, std::int64_t* launches, double* point_ms, double* cam_ms) {
    collect_profile();
    *total = prof_point_ms_ + prof_cam_ms_;
    *launches = dse_launches_;
    *point_ms = prof_point_ms_;
    *cam_ms = prof_cam_ms_;
  }
  void sync() { DBAG_CUDA(cudaStreamSynchronize(st_)); }

 private:
  template <class... KA, class... A>
  void launch(void (*k)(KA...), dim3 grid, dim3 block, A&&... args) {
    k<<<grid, block, 0, st_>>>(std::forward<A>(args)...);
    DBAG_LAUNCH_CHECK();
    ++launches_;
  }

  dev::RedWs red() { return dev::RedWs{red_part_.get(), red_cnt_.get()}; }

  void read_scal() {
    DBAG_CUDA(cudaMemcpyAsync(hsc_, sc_.get(), sizeof(Scal), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    collect_profile();
  }

  void launch_dot(const S* a, const S* b, std::int64_t len, double* out) {
    launch(dev::k_dot<S>, grid_for(len, dev::kRedThreads, dev::kRedBlocksMax), dev::kRedThreads, len, a, b, red(),
           out);
  }

  // The point-side half of the DSE (MODE 0) / rhs (MODE 2): one pass over E
  // writing the per-(chunk, camera) partials; halo points are finished after
  // their all-reduce.
  template <int MODE>
  void fused_pass(const S* x) {
    const bool halo = MODE == 0 && H_ > 0;
    if (halo) DBAG_CUDA(cudaMemsetAsync(halo_buf_.get(), 0, sizeof(S) * 3 * static_cast<std::size_t>(H_), st_));
    stream_pass<MODE>(x);
    const std::int32_t nh = static_cast<std::int32_t>(lay_.halo_slot.size());
    if (MODE == 0 && H_ > 0) {
      comm_->allreduce_sum(halo_buf_.get(), 3 * H_, kT, st_);
      if (nh > 0) halo_fix(nh);
    } else if (MODE == 2 && nh > 0) {
      // rhs: C and w are complete on every rank, so the chunk partials
      // already hold the halo slots' E_s C^-1 w; the halo slots' own
      // partials (camera-major positions halo_pos) must add nothing: zero
      // them (they still hold the last DSE's values).
      launch(dev::k_zero_rows<S, 9>, grid_for(nh, 128, 1 << 30), 128, nh, static_cast<const std::int32_t*>(halo_pos_.get()),
             part_.get());
    }
  }

  // E chunk records of L lanes (kernels.cuh kLanesFact / kLanesDense): zero
  // lanes plus each chunk's static metadata (RecMeta); the lanes are
  // (re)written by k_linearize (factored) or set_system (dense).
  template <int L>
  std::vector<T> build_records(const std::vector<std::int32_t>& s_cam) {
    const std::size_t nc = static_cast<std::size_t>(std::max(n_chunks_, 1));
    std::vector<T> recs(nc * dev::Rec<T, L>::kLen, T(0));
    std::vector<std::int32_t> long_first;
    const std::size_t nt = lay_.tile_pt.size() - 1;
    for (std::size_t t = 0; t < nt; ++t) {
      const std::int32_t p0 = lay_.tile_pt[t], p1 = lay_.tile_pt[t + 1];
      const std::int32_t s0 = lay_.dpt_ptr[static_cast<std::size_t>(p0)];
      const std::int32_t ch0 = lay_.tile_chunk[t], ch1 = lay_.tile_chunk[t + 1];
      if (ch1 - ch0 > 1) long_first.push_back(ch0);
      for (std::int32_t c = ch0; c < ch1; ++c) {
        auto* M = reinterpret_cast<dev::RecMeta*>(recs.data() + static_cast<std::size_t>(c) * dev::Rec<T, L>::kLen +
                                                  dev::Rec<T, L>::kE);
        const std::int32_t c0 = lay_.chunk_slot[static_cast<std::size_t>(c)];
        const std::int32_t c1 = (c + 1 < ch1) ? lay_.chunk_slot[static_cast<std::size_t>(c) + 1]
                                              : lay_.dpt_ptr[static_cast<std::size_t>(p1)];
        M->p0 = p0;
        M->np = p1 - p0;
        M->nslots = c1 - c0;
        M->nchunk = ch1 - ch0;
        M->ci = c - ch0;
        for (std::int32_t sl = c0; sl < c1; ++sl) {
          M->cam[sl - c0] = s_cam[static_cast<std::size_t>(sl)];
          M->pt[sl - c0] = ch1 - ch0 > 1 ? 0
                                          : static_cast<std::uint8_t>(lay_.slot_dpt[static_cast<std::size_t>(sl)] - p0);
        }
        if (ch1 - ch0 == 1)
          for (std::int32_t i = 0; i <= p1 - p0; ++i)
            M->pbeg[i] = static_cast<std::uint8_t>(lay_.dpt_ptr[static_cast<std::size_t>(p0 + i)] - s0);
        const std::int32_t u0 = lay_.chunk_ucam[static_cast<std::size_t>(c)];
        const std::int32_t u1 = lay_.chunk_ucam[static_cast<std::size_t>(c) + 1];
        M->nu = u1 - u0;
        const std::int32_t k0 = lay_.ucam_ptr[static_cast<std::size_t>(u0)];
        for (std::int32_t u = u0; u <= u1; ++u) {
          M->ubeg[u - u0] = static_cast<std::uint8_t>(lay_.ucam_ptr[static_cast<std::size_t>(u)] - k0);
          if (u < u1) M->upart[u - u0] = lay_.part_pos[static_cast<std::size_t>(u)];
          if (u < u1 && u - u0 < dev::kXsCams) M->ucam[u - u0] = lay_.ucam_cam[static_cast<std::size_t>(u)];
        }
        for (std::int32_t u = u0; u < u1; ++u)
          for (std::int32_t k = lay_.ucam_ptr[static_cast<std::size_t>(u)]; k < lay_.ucam_ptr[static_cast<std::size_t>(u) + 1];
               ++k) {
            const std::int32_t sl = lay_.ucam_slot[static_cast<std::size_t>(k)];
            M->uslot[k - k0] = static_cast<std::uint8_t>(sl);
            M->su[sl] = static_cast<std::uint8_t>(u - u0);
          }
      }
    }
    n_long_ = static_cast<std::int32_t>(long_first.size());
    long_chunk_.copy_in(long_first);
    {  // staged-chunk table of the streaming pass (stream.cuh ChunkTab)
      std::vector<std::int32_t> tab;
      for (std::size_t t = 0; t < nt; ++t) {
        if (lay_.tile_chunk[t + 1] - lay_.tile_chunk[t] != 1) continue;
        const std::int32_t p0 = lay_.tile_pt[t], np = lay_.tile_pt[t + 1] - p0;
        const std::size_t b0 = static_cast<std::size_t>(p0) * 9 * sizeof(S);
        const std::size_t nb = (b0 & 15) + static_cast<std::size_t>(std::min(np, dev::kCStage)) * 9 * sizeof(S);
        tab.push_back(lay_.tile_chunk[t]);
        tab.push_back(static_cast<std::int32_t>(b0 >> 4));
        tab.push_back(static_cast<std::int32_t>((nb + 15) / 16 * 16));
        tab.push_back(0);
      }
      n_norm_ = static_cast<std::int32_t>(tab.size() / 4);
      ctab_.copy_in(tab);
    }
    std::vector<std::int32_t> hpos(lay_.halo_slot.size());
    for (std::size_t i = 0; i < hpos.size(); ++i)
      hpos[i] = lay_.part_pos[static_cast<std::size_t>(n_chunk_part_) + i];
    halo_pos_.copy_in(hpos);
    return recs;
  }

  // Back to the factored records (linearize writes them); the graph is
  // rebuilt for the record layout on its next use.
  void use_factored() { fact_ = true; }

  void halo_fix(std::int32_t nh) {
    if (fact_)
      launch(dev::k_halo_fix<S, T, dev::kLanesFact>, grid_for(nh, 128, 1 << 30), 128, nh, halo_slot_.get(),
             slot_dpt_.get(), halo_of_.get(), static_cast<const S*>(halo_buf_.get()), static_cast<const S*>(Cinv_.get()),
             static_cast<const T*>(E_.get()), slot_chunk_.get(), chunk_slot_.get(), halo_pos_.get(), part_.get(),
             static_cast<const std::int32_t*>(slot_cam_.get()), static_cast<const S*>(Rm_.get()));
    else
      launch(dev::k_halo_fix<S, T, dev::kLanesDense>, grid_for(nh, 128, 1 << 30), 128, nh, halo_slot_.get(),
             slot_dpt_.get(), halo_of_.get(), static_cast<const S*>(halo_buf_.get()), static_cast<const S*>(Cinv_.get()),
             static_cast<const T*>(Edense_.get()), slot_chunk_.get(), chunk_slot_.get(), halo_pos_.get(), part_.get(),
             static_cast<const std::int32_t*>(slot_cam_.get()), static_cast<const S*>(Rm_.get()));
  }

  // ---- the persistent TMA-fed pass (stream.cuh) ----------------------------
  // Opt-in (DBAG_STREAM=1): measured 5 % (venice FP64) to 30 % (FP32,
  // trafalgar) slower than the one-CTA-per-chunk k_g_pass;
  // DBAG_NST sets its stage-ring depth (2, 3 or 4; 2 measured best).
  struct StreamCfg {
    void* fn = nullptr;
    int smem = 0, grid = 0;
    bool fact = false;
  };
  static bool use_stream() {
    const char* e = std::getenv("DBAG_STREAM");
    return e && std::string(e) == "1";
  }
  template <int L>
  static void* stream_fn(int nst) {
    if (nst == 2) return reinterpret_cast<void*>(dev::k_g_stream<S, T, L, 2>);
    if (nst == 4) return reinterpret_cast<void*>(dev::k_g_stream<S, T, L, 4>);
    return reinterpret_cast<void*>(dev::k_g_stream<S, T, L, 3>);
  }
  const StreamCfg& stream_cfg() {
    if (scfg_.fn && scfg_.fact == fact_) return scfg_;
    int nst = 2;
    if (const char* e = std::getenv("DBAG_NST")) nst = std::min(4, std::max(2, std::atoi(e)));
    StreamCfg c;
    c.fact = fact_;
    c.fn = fact_ ? stream_fn<dev::kLanesFact>(nst) : stream_fn<dev::kLanesDense>(nst);
    c.smem = fact_ ? dev::StreamLayout<S, T, dev::kLanesFact>::bytes(nst)
                   : dev::StreamLayout<S, T, dev::kLanesDense>::bytes(nst);
    DBAG_CUDA(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem));
    int per_sm = 0, sms = 0;
    DBAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c.fn, dev::kStreamThreads, c.smem));
    DBAG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    c.grid = std::max(1, std::min(std::max(per_sm, 1) * sms, std::max(n_norm_, n_long_)));
    scfg_ = c;
    return scfg_;
  }
  // One DSE pass of the graph body outside a graph (run-ahead loop, timing).
  void launch_pass(const dev::DseArgs<S, T>& A, const dev::GBufs<S>& B, const dev::GScal<S>* sc) {
    if (!use_stream()) {
      if (fact_) launch(dev::k_g_pass<S, T, dev::kLanesFact>, n_long_ + n_chunks_, dev::kTile, A, B, sc);
      else launch(dev::k_g_pass<S, T, dev::kLanesDense>, n_long_ + n_chunks_, dev::kTile, A, B, sc);
      return;
    }
    const StreamCfg& c = stream_cfg();
    const dev::ChunkTab* tab = reinterpret_cast<const dev::ChunkTab*>(ctab_.get());
    std::int32_t nn = n_norm_;
    void* args[] = {const_cast<dev::DseArgs<S, T>*>(&A), const_cast<dev::GBufs<S>*>(&B), &sc, &tab, &nn};
    DBAG_CUDA(cudaLaunchKernel(c.fn, dim3(static_cast<unsigned>(c.grid)), dim3(dev::kStreamThreads), args,
                               static_cast<std::size_t>(c.smem), st_));
    ++launches_;
  }

  dev::DseArgs<S, T> dse_args(const S* x) {
    dev::DseArgs<S, T> a;
    a.n_chunks = n_chunks_;
    a.rec = fact_ ? E_.get() : Edense_.get();
    a.x = x;
    a.Cinv = Cinv_.get();
    a.w = w_.get();
    a.halo_of = H_ > 0 ? halo_of_.get() : nullptr;
    a.halo_buf = halo_buf_.get();
    a.part = part_.get();
    a.out_pt = dxp_.get();
    a.long_chunk = long_chunk_.get();
    a.n_long = n_long_;
    a.pf_dist = pf_dist();
    a.Rm = Rm_.get();
    return a;
  }

  // L2 prefetch distance of the chunk pass: one wave of resident CTAs
  // (DBAG_PF overrides; 0 disables).
  std::int32_t pf_dist() {
    if (pf_dist_ < 0) {
      const char* e = std::getenv("DBAG_PF");
      if (e) {
        pf_dist_ = std::max(0, std::atoi(e));
      } else {
        int per_sm = 0, sms = 0;
        DBAG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_g_pass<S, T, dev::kLanesFact>,
                                                                 dev::kTile, 0));
        DBAG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
        pf_dist_ = per_sm * sms;
      }
    }
    return pf_dist_;
  }

  template <int MODE>
  void stream_pass(const S* x) {
    if (n_chunks_ == 0) return;
    const dev::DseArgs<S, T> a = dse_args(x);
    if (fact_) {
      launch(dev::k_dse_chunk<S, MODE, T, dev::kLanesFact>, n_chunks_, dev::kTile, a);
      if (n_long_ > 0) launch(dev::k_dse_long<S, MODE, T, dev::kLanesFact>, n_long_, dev::kTile, a);
    } else {
      launch(dev::k_dse_chunk<S, MODE, T, dev::kLanesDense>, n_chunks_, dev::kTile, a);
      if (n_long_ > 0) launch(dev::k_dse_long<S, MODE, T, dev::kLanesDense>, n_long_, dev::kTile, a);
    }
  }

  template <int EPI>
  void cam_reduce(const S* x, S* out) {
    if (m_ == 0) return;
    launch(dev::k_cam_reduce<S, EPI>, grid_for(static_cast<std::int64_t>(m_) * 32, dev::kRedThreads, 1 << 30),
           dev::kRedThreads, m_, cam_part_ptr_.get(), static_cast<const std::int32_t*>(nullptr), static_cast<const S*>(part_.get()),
           static_cast<const S*>(Bd_.get()), x, static_cast<const S*>(v_.get()), out, red(), sc_.get());
  }

  // Lowest index over ranks from a device u64 (all-ones = none); -1 if none.
  std::int64_t agree_min_index(unsigned long long* dev_bad) {
    unsigned long long raw = 0;
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, dev_bad, sizeof(raw), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    std::memcpy(&raw, hbuf_, sizeof(raw));
    if (comm_->size() == 1) return raw == ~0ull ? -1 : static_cast<std::int64_t>(raw);
    const double neg = raw == ~0ull ? -std::numeric_limits<double>::infinity() : -double(raw);
    double* d = dsc_.get();
    hbuf_[0] = neg;
    DBAG_CUDA(cudaMemcpyAsync(d + 28, hbuf_, sizeof(double), cudaMemcpyHostToDevice, st_));
    comm_->allreduce_max(d + 28, 1, DType::f64, st_);
    DBAG_CUDA(cudaMemcpyAsync(hbuf_, d + 28, sizeof(double), cudaMemcpyDeviceToHost, st_));
    DBAG_CUDA(cudaStreamSynchronize(st_));
    return std::isfinite(hbuf_[0]) ? static_cast<std::int64_t>(-hbuf_[0]) : -1;
  }

  // C (9) and w (3) of shared points summed across ranks through the halo
  // buffer (value-identical to the reference's full-size all-reduce).
  void halo_exchange_Cw() {
    if (H_ == 0) {
      comm_->allreduce_sum(halo_buf_.get(), 0, kT, st_);  // keep the collective sequence aligned
      return;
    }
    DBAG_CUDA(cudaMemsetAsync(halo_buf_.get(), 0, sizeof(S) * 12 * static_cast<std::size_t>(H_), st_));
    S* hw = halo_buf_.get() + 9 * static_cast<std::size_t>(H_);
    const int g = grid_for(std::max(n_halo_loc_, 1), 128, 1 << 30);
    if (n_halo_loc_ > 0) {
      launch(dev::k_halo_scatter<S, 9>, g, 128, n_halo_loc_, halo_dpt_.get(), halo_idx_.get(),
             static_cast<const S*>(C_.get()), halo_buf_.get());
      launch(dev::k_halo_scatter<S, 3>, g, 128, n_halo_loc_, halo_dpt_.get(), halo_idx_.get(),
             static_cast<const S*>(w_.get()), hw);
    }
    comm_->allreduce_sum(halo_buf_.get(), 12 * H_, kT, st_);
    if (n_halo_loc_ > 0) {
      launch(dev::k_halo_gather<S, 9>, g, 128, n_halo_loc_, halo_dpt_.get(), halo_idx_.get(),
             static_cast<const S*>(halo_buf_.get()), C_.get());
      launch(dev::k_halo_gather<S, 3>, g, 128, n_halo_loc_, halo_dpt_.get(), halo_idx_.get(),
             static_cast<const S*>(hw), w_.get());
    }
  }

  cudaEvent_t prof_event() {
    if (prof_next_ == prof_ev_.size()) {
      cudaEvent_t e;
      DBAG_CUDA(cudaEventCreate(&e));
      prof_ev_.push_back(e);
    }
    return prof_ev_[prof_next_++];
  }
  // Events come in groups of 3 per DSE: [start, point pass done, camera done].
  void collect_profile() {
    if (prof_next_ == 0) return;
    DBAG_CUDA(cudaStreamSynchronize(st_));
    for (std::size_t i = 0; i + 2 < prof_next_; i += 3) {
      float a = 0, b = 0;
      DBAG_CUDA(cudaEventElapsedTime(&a, prof_ev_[i], prof_ev_[i + 1]));
      DBAG_CUDA(cudaEventElapsedTime(&b, prof_ev_[i + 1], prof_ev_[i + 2]));
      prof_point_ms_ += a;
      prof_cam_ms_ += b;
    }
    prof_next_ = 0;
  }

  int device_;
  Comm* comm_;
  cudaStream_t st_ = nullptr;
  ShardPlan plan_;
  DeviceLayout lay_;
  int jac_mode_ = 0;
  std::int32_t m_ = 0, n_glob_ = 0, n_loc_ = 0, m_loc_ = 0, n_halo_loc_ = 0, n_chunk_part_ = 0;
  std::int64_t N_ = 0, H_ = 0;
  int n_tiles_ = 0;
  std::int32_t n_long_ = 0;
  std::int32_t n_norm_ = 0;  // single-chunk tiles: the streaming pass's staged chunks
  std::int32_t n_chunks_ = 0;
  bool have_system_ = false;
  double lambda_ = 0;
  int policy_ = 1;
  double step_inf_ = 0, damp_term_ = 0, gv_ = 0;
  int dse_count_ = 0;
  std::int64_t dse_launches_ = 0, launches_ = 0;
  Tally tally_;
  Scal* hsc_ = nullptr;
  double* hbuf_ = nullptr;
  cudaEvent_t mark_[2];
  bool profiling_ = false;
  std::vector<cudaEvent_t> prof_ev_;
  std::size_t prof_next_ = 0;
  double prof_point_ms_ = 0, prof_cam_ms_ = 0;
  std::vector<std::int32_t> dpt_glob_;
  std::vector<std::uint8_t> owned_h_;
  std::vector<std::int32_t> orphans_;  // global ids of points no edge observes
  std::vector<S> orphan_x_;            // their state (set_state)

  Arena pool_;  // declared first: destroyed after the buffers carved from it
  DevBuf<std::int32_t> slot_cam_, slot_dpt_, slot_edge_, dpt_ptr_, chunk_slot_, cam_part_ptr_, halo_slot_, slot_chunk_,
      long_chunk_, ctab_, cam_ident_, halo_pos_, cam_ptr_, cam_glob_, cslot_dslot_, dpt_glob_d_,
      halo_of_, halo_dpt_, halo_idx_;
  DevBuf<std::uint8_t> owned_;
  DevBuf<S> slot_px_, slot_py_, slot_w_;
  DevBuf<S> xc_, xct_, dxc_, v_, g_, r_, z_, p_, q_, ctmp_;
  DevBuf<S> xp_, xpt_, dxp_, w_;
  DevBuf<S> B_, Bd_, Binv_, Bexp_, C_, Cd_, Cinv_, p2_;
  DevBuf<dev::GScal<S>> gsc_;
  DevBuf<double> g_pq_cam_;
  DevBuf<S> xp_full_;  // x_p in global point order (state transfers)
  DevBuf<unsigned long long> g_bar_;  // k_g_fs grid barrier arrivals (monotonic)
  bool g_fused_ = false;
  int g_cluster_ = 0, g_cpw_ = 1;  // k_g_fsc cluster size (0: not used), cameras per warp
  int g_unroll_ = DBAG_GRAPH_UNROLL;
  dev::GScal<S>* gsc_h_ = nullptr;
  cudaGraph_t g_graph_ = nullptr;
  cudaGraphExec_t g_exec_ = nullptr;
  DevBuf<S> Jb_, part_, halo_buf_, halo_sum_;
  DevBuf<double> bpart_;  // camera assembly partials (lin.cuh), kAsmTerms per partial position
  DevBuf<double> carry_;               // k_assemble_cameras sums across Jb batches
  std::vector<std::int32_t> jb_pt_;    // Jb batch boundaries (device points)
  std::int32_t pf_dist_ = -1;
  StreamCfg scfg_;
  bool peer_ok_ = false;
  std::int64_t peer_cap_[2] = {0, 0};
  PeerSite ps_cam_, ps_halo_;
  cudaGraph_t gk_graph_ = nullptr;
  cudaGraphExec_t gk_exec_ = nullptr;
  int gk_unroll_ = 1;
  bool gk_fact_ = false;
  std::vector<std::int32_t> jb_ncam_;  // cameras each Jb batch touches
  DevBuf<std::int32_t> cam_list_;      // ... their local ids, m_loc per batch
  DevBuf<T> E_;       // chunk records: factored lanes G = sqrt(w) Jc (T) + RecMeta (pool)
  DevBuf<T> Edense_;  // 9x3-block records for caller-fabricated E (set_system; outside the pool)
  DevBuf<S> Rm_;      // per-camera R at the linearization point (factored records)
  bool fact_ = true, g_fact_ = true;
  DevBuf<Scal> sc_;
  DevBuf<double> red_part_, dsc_, bounce_;
  DevBuf<unsigned> red_cnt_;
  DevBuf<unsigned long long> bad_;
};

}  // namespace dbag
