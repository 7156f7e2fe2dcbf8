// partition.hpp — host-side, integer-exact edge partitioning and the device
// index layout derived from it.
//
// Bit-exact restatement of the reference's partitioning contract
// (north_star: "bit-exact edge-to-partition assignment and index ordering"):
//   partition_edges     dba/partition.hpp:76-103   contiguous chunks, the
//                                                  first N mod K ranks +1
//   LocalIndexMap       dba/partition.hpp:14-45    first-appearance order
//   build_groups        dba/block_matrix.hpp:309-320 counting sort, ascending
//                                                  edge order inside a group
// plus the B200 additions: the point-major slot permutation the kernels
// stream, the camera-major view of it, point tiles aligned to point
// boundaries, and the halo plan (points touched by more than one rank).
#pragma once

#include <algorithm>
#include <limits>
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace dbag {

struct LocalMap {
  std::vector<std::int32_t> to_local;   // global -> local, -1 if untouched
  std::vector<std::int32_t> to_global;  // local -> global, first appearance
  void build(const std::int32_t* ids, std::int64_t count, std::int32_t global_count) {
    to_local.assign(static_cast<std::size_t>(global_count), -1);
    to_global.clear();
    for (std::int64_t i = 0; i < count; ++i) {
      const std::int32_t id = ids[i];
      if (to_local[static_cast<std::size_t>(id)] < 0) {
        to_local[static_cast<std::size_t>(id)] = static_cast<std::int32_t>(to_global.size());
        to_global.push_back(id);
      }
    }
  }
  std::int32_t size() const { return static_cast<std::int32_t>(to_global.size()); }
};

// Counting sort of `key` into `groups` buckets; ids keep ascending order.
inline void group_by(const std::vector<std::int32_t>& key, std::int32_t groups, std::vector<std::int64_t>& ptr,
                     std::vector<std::int64_t>& ids) {
  ptr.assign(static_cast<std::size_t>(groups) + 1, 0);
  for (std::int32_t k : key) ++ptr[static_cast<std::size_t>(k) + 1];
  for (std::int32_t g = 0; g < groups; ++g) ptr[static_cast<std::size_t>(g) + 1] += ptr[static_cast<std::size_t>(g)];
  ids.resize(key.size());
  std::vector<std::int64_t> cursor(ptr.begin(), ptr.end() - 1);
  for (std::size_t i = 0; i < key.size(); ++i)
    ids[static_cast<std::size_t>(cursor[static_cast<std::size_t>(key[i])]++)] = static_cast<std::int64_t>(i);
}

struct EdgeRange {
  std::int64_t start = 0, count = 0;
};

inline std::vector<EdgeRange> split_edges(std::int64_t n, int k) {
  if (k < 1) throw Error(DBAG_INVALID_ARGUMENT, "worker count must be >= 1");
  if (k > n)
    throw Error(DBAG_INVALID_ARGUMENT,
                "worker count " + std::to_string(k) + " exceeds number of edges " + std::to_string(n));
  std::vector<EdgeRange> r(static_cast<std::size_t>(k));
  const std::int64_t base = n / k, extra = n % k;
  std::int64_t next = 0;
  for (int i = 0; i < k; ++i) {
    r[static_cast<std::size_t>(i)].start = next;
    r[static_cast<std::size_t>(i)].count = base + (i < extra ? 1 : 0);
    next += r[static_cast<std::size_t>(i)].count;
  }
  return r;
}

// One rank's shard of the canonical edge order with all index structures.
struct ShardPlan {
  int rank = 0, ranks = 1;
  std::int32_t m = 0, n = 0;  // global camera / point counts
  EdgeRange range;
  LocalMap cams, pts;
  std::vector<std::int32_t> cam_of, pt_of;              // per shard edge, local ids
  std::vector<std::int64_t> cam_ptr, cam_blk, pt_ptr, pt_blk;  // reference groups
  // Device layout: slot s streams edge pt_blk[s] (point-major).
  std::vector<std::int32_t> cslot_pslot;  // camera-major slot -> point-major slot
  std::vector<std::int32_t> tile_pt;      // point tiles [tile_pt[t], tile_pt[t+1])
  // Halo: shared points (touched by > 1 rank), global ascending order.
  std::int64_t n_shared = 0;
  std::vector<std::int32_t> halo_of_lpt;  // local point -> halo index or -1
  std::vector<std::uint8_t> owned_lpt;    // 1 if this rank owns the point (lowest toucher)
};

// Tiles of whole points with at most `tile` slots each; a point with more
// slots than `tile` forms a tile of its own.
inline std::vector<std::int32_t> make_point_tiles(const std::vector<std::int64_t>& pt_ptr, int tile) {
  std::vector<std::int32_t> t{0};
  const std::int32_t np = static_cast<std::int32_t>(pt_ptr.size()) - 1;
  std::int32_t p = 0;
  while (p < np) {
    const std::int64_t base = pt_ptr[static_cast<std::size_t>(p)];
    std::int32_t q = p + 1;
    while (q < np && pt_ptr[static_cast<std::size_t>(q) + 1] - base <= tile) ++q;
    t.push_back(q);
    p = q;
  }
  return t;
}

// Per-point rank coverage for the halo plan: touched by > 1 rank => shared;
// owner = lowest touching rank.
struct Coverage {
  std::vector<std::int32_t> first_rank;
  std::vector<std::int32_t> rank_count;
  std::int64_t n_shared = 0;
  std::vector<std::int64_t> shared_index;  // global point -> halo index or -1
};

inline Coverage point_coverage(const std::int32_t* pt_id, std::int32_t n, const std::vector<EdgeRange>& ranges) {
  Coverage c;
  c.first_rank.assign(static_cast<std::size_t>(n), -1);
  c.rank_count.assign(static_cast<std::size_t>(n), 0);
  std::vector<std::int32_t> last(static_cast<std::size_t>(n), -1);
  for (std::size_t r = 0; r < ranges.size(); ++r) {
    for (std::int64_t e = ranges[r].start; e < ranges[r].start + ranges[r].count; ++e) {
      const std::size_t p = static_cast<std::size_t>(pt_id[e]);
      if (last[p] != static_cast<std::int32_t>(r)) {
        last[p] = static_cast<std::int32_t>(r);
        if (c.first_rank[p] < 0) c.first_rank[p] = static_cast<std::int32_t>(r);
        ++c.rank_count[p];
      }
    }
  }
  c.shared_index.assign(static_cast<std::size_t>(n), -1);
  for (std::size_t p = 0; p < static_cast<std::size_t>(n); ++p)
    if (c.rank_count[p] > 1) c.shared_index[p] = c.n_shared++;
  return c;
}

inline ShardPlan plan_shard(const std::int32_t* cam_id, const std::int32_t* pt_id, std::int64_t num_obs,
                            std::int32_t m, std::int32_t n, int ranks, int rank, int tile = 128) {
  const auto ranges = split_edges(num_obs, ranks);
  if (rank < 0 || rank >= ranks) throw Error(DBAG_INVALID_ARGUMENT, "rank out of range");
  ShardPlan s;
  s.rank = rank;
  s.ranks = ranks;
  s.m = m;
  s.n = n;
  s.range = ranges[static_cast<std::size_t>(rank)];
  const std::int64_t cnt = s.range.count;
  s.cams.build(cam_id + s.range.start, cnt, m);
  s.pts.build(pt_id + s.range.start, cnt, n);
  s.cam_of.resize(static_cast<std::size_t>(cnt));
  s.pt_of.resize(static_cast<std::size_t>(cnt));
  for (std::int64_t i = 0; i < cnt; ++i) {
    s.cam_of[static_cast<std::size_t>(i)] = s.cams.to_local[static_cast<std::size_t>(cam_id[s.range.start + i])];
    s.pt_of[static_cast<std::size_t>(i)] = s.pts.to_local[static_cast<std::size_t>(pt_id[s.range.start + i])];
  }
  group_by(s.cam_of, s.cams.size(), s.cam_ptr, s.cam_blk);
  group_by(s.pt_of, s.pts.size(), s.pt_ptr, s.pt_blk);
  if (cnt >= (std::int64_t(1) << 31)) throw Error(DBAG_INVALID_ARGUMENT, "shard exceeds 2^31 edges; use more ranks");
  std::vector<std::int32_t> pslot_of_edge(static_cast<std::size_t>(cnt));
  for (std::int64_t sl = 0; sl < cnt; ++sl)
    pslot_of_edge[static_cast<std::size_t>(s.pt_blk[static_cast<std::size_t>(sl)])] = static_cast<std::int32_t>(sl);
  s.cslot_pslot.resize(static_cast<std::size_t>(cnt));
  for (std::int64_t c = 0; c < cnt; ++c)
    s.cslot_pslot[static_cast<std::size_t>(c)] = pslot_of_edge[static_cast<std::size_t>(s.cam_blk[static_cast<std::size_t>(c)])];
  s.tile_pt = make_point_tiles(s.pt_ptr, tile);
  s.halo_of_lpt.assign(static_cast<std::size_t>(s.pts.size()), -1);
  s.owned_lpt.assign(static_cast<std::size_t>(s.pts.size()), 1);
  if (ranks > 1) {
    const Coverage cov = point_coverage(pt_id, n, ranges);
    s.n_shared = cov.n_shared;
    for (std::int32_t lp = 0; lp < s.pts.size(); ++lp) {
      const std::size_t g = static_cast<std::size_t>(s.pts.to_global[static_cast<std::size_t>(lp)]);
      s.halo_of_lpt[static_cast<std::size_t>(lp)] = static_cast<std::int32_t>(cov.shared_index[g]);
      s.owned_lpt[static_cast<std::size_t>(lp)] = cov.first_rank[g] == rank ? 1 : 0;
    }
  }
  return s;
}

// Device layout of one shard for the DSE chunk pass (dse.cuh):
//   * device points: the shard's local points ordered by their smallest
//     camera id (ties by local id) so that a tile of consecutive points
//     touches few cameras; each point keeps its slots in edge order, so
//     per-point sums accumulate in the reference's order;
//   * tiles of whole points (<= `tile` slots, or one long point), split in
//     chunks of <= `tile` slots;
//   * per chunk, the distinct cameras it touches with their slot lists: one
//     9-wide partial per (chunk, camera), reduced per camera in chunk order
//     (deterministic, no atomics);
//   * halo slots (of points shared with other ranks) get their own partials.
struct DeviceLayout {
  std::vector<std::int32_t> dpt_lpt;      // device point -> local point
  std::vector<std::int32_t> lpt_dpt;      // local point -> device point
  std::vector<std::int32_t> slot_edge;    // device slot -> shard edge
  std::vector<std::int32_t> dpt_ptr;      // device point -> slot range
  std::vector<std::int32_t> slot_dpt;     // device slot -> device point
  std::vector<std::int32_t> tile_pt;      // tile -> device point range
  std::vector<std::int32_t> tile_chunk;   // tile -> chunk range
  std::vector<std::int32_t> chunk_slot;   // chunk -> first slot
  std::vector<std::int32_t> slot_chunk;   // slot -> chunk
  std::vector<std::int32_t> chunk_ucam;   // chunk -> range of its (camera) partials
  std::vector<std::int32_t> ucam_cam;     // partial -> global camera
  std::vector<std::int32_t> ucam_ptr;     // partial -> range in ucam_slot
  std::vector<std::int32_t> ucam_slot;    // slot offsets within the chunk
  std::vector<std::int32_t> halo_slot;    // device slots of halo points
  std::int32_t n_part = 0;                // chunk partials + halo partials
  std::vector<std::int32_t> cam_part_ptr;  // global camera -> partial ids
  std::vector<std::int32_t> cam_part;
  std::vector<std::int32_t> part_pos;      // partial id -> camera-major position
};

inline DeviceLayout build_device_layout(const ShardPlan& s, const std::int32_t* cam_id_shard, int tile) {
  DeviceLayout d;
  const std::int32_t np = s.pts.size();
  std::vector<std::int32_t> mincam(static_cast<std::size_t>(np), std::numeric_limits<std::int32_t>::max());
  for (std::size_t e = 0; e < s.pt_of.size(); ++e) {
    auto& mc = mincam[static_cast<std::size_t>(s.pt_of[e])];
    mc = std::min(mc, cam_id_shard[e]);
  }
  d.dpt_lpt.resize(static_cast<std::size_t>(np));
  for (std::int32_t i = 0; i < np; ++i) d.dpt_lpt[static_cast<std::size_t>(i)] = i;
  std::stable_sort(d.dpt_lpt.begin(), d.dpt_lpt.end(), [&](std::int32_t a, std::int32_t b) {
    return mincam[static_cast<std::size_t>(a)] < mincam[static_cast<std::size_t>(b)];
  });
  d.lpt_dpt.resize(static_cast<std::size_t>(np));
  d.dpt_ptr.assign(static_cast<std::size_t>(np) + 1, 0);
  d.slot_edge.reserve(s.pt_of.size());
  d.slot_dpt.reserve(s.pt_of.size());
  for (std::int32_t dp = 0; dp < np; ++dp) {
    const std::int32_t lp = d.dpt_lpt[static_cast<std::size_t>(dp)];
    d.lpt_dpt[static_cast<std::size_t>(lp)] = dp;
    for (std::int64_t k = s.pt_ptr[static_cast<std::size_t>(lp)]; k < s.pt_ptr[static_cast<std::size_t>(lp) + 1]; ++k) {
      d.slot_edge.push_back(static_cast<std::int32_t>(s.pt_blk[static_cast<std::size_t>(k)]));
      d.slot_dpt.push_back(dp);
    }
    d.dpt_ptr[static_cast<std::size_t>(dp) + 1] = static_cast<std::int32_t>(d.slot_edge.size());
  }
  std::vector<std::int64_t> ptr64(d.dpt_ptr.begin(), d.dpt_ptr.end());
  d.tile_pt = make_point_tiles(ptr64, tile);
  const std::size_t nt = d.tile_pt.size() - 1;
  d.tile_chunk.assign(nt + 1, 0);
  d.chunk_ucam.push_back(0);
  std::vector<std::int32_t> seen(static_cast<std::size_t>(s.m), -1), order;
  for (std::size_t t = 0; t < nt; ++t) {
    const std::int32_t s0 = d.dpt_ptr[static_cast<std::size_t>(d.tile_pt[t])];
    const std::int32_t s1 = d.dpt_ptr[static_cast<std::size_t>(d.tile_pt[t + 1])];
    for (std::int32_t c0 = s0; c0 < s1; c0 += tile) {
      const std::int32_t c1 = std::min(s1, c0 + tile);
      d.chunk_slot.push_back(c0);
      for (std::int32_t sl = c0; sl < c1; ++sl) d.slot_chunk.push_back(static_cast<std::int32_t>(d.chunk_slot.size()) - 1);
      // distinct cameras in first-appearance order, slots grouped per camera
      order.clear();
      std::vector<std::vector<std::int32_t>> lists;
      for (std::int32_t sl = c0; sl < c1; ++sl) {
        const std::int32_t cam = cam_id_shard[d.slot_edge[static_cast<std::size_t>(sl)]];
        std::int32_t& u = seen[static_cast<std::size_t>(cam)];
        if (u < 0) {
          u = static_cast<std::int32_t>(order.size());
          order.push_back(cam);
          lists.emplace_back();
        }
        lists[static_cast<std::size_t>(u)].push_back(sl - c0);
      }
      for (std::size_t u = 0; u < order.size(); ++u) {
        d.ucam_cam.push_back(order[u]);
        d.ucam_ptr.push_back(static_cast<std::int32_t>(d.ucam_slot.size()));
        d.ucam_slot.insert(d.ucam_slot.end(), lists[u].begin(), lists[u].end());
        seen[static_cast<std::size_t>(order[u])] = -1;
      }
      d.chunk_ucam.push_back(static_cast<std::int32_t>(d.ucam_cam.size()));
    }
    d.tile_chunk[t + 1] = static_cast<std::int32_t>(d.chunk_slot.size());
  }
  d.ucam_ptr.push_back(static_cast<std::int32_t>(d.ucam_slot.size()));
  // halo partials: one per slot of a shared point
  const std::int32_t n_chunk_part = static_cast<std::int32_t>(d.ucam_cam.size());
  std::vector<std::int32_t> halo_cam;
  for (std::int32_t sl = 0; sl < static_cast<std::int32_t>(d.slot_edge.size()); ++sl) {
    const std::int32_t lp = d.dpt_lpt[static_cast<std::size_t>(d.slot_dpt[static_cast<std::size_t>(sl)])];
    if (s.halo_of_lpt[static_cast<std::size_t>(lp)] >= 0) {
      d.halo_slot.push_back(sl);
      halo_cam.push_back(cam_id_shard[d.slot_edge[static_cast<std::size_t>(sl)]]);
    }
  }
  d.n_part = n_chunk_part + static_cast<std::int32_t>(d.halo_slot.size());
  // camera -> partial ids (chunk partials in chunk order, then halo partials)
  d.cam_part_ptr.assign(static_cast<std::size_t>(s.m) + 1, 0);
  for (std::int32_t c : d.ucam_cam) ++d.cam_part_ptr[static_cast<std::size_t>(c) + 1];
  for (std::int32_t c : halo_cam) ++d.cam_part_ptr[static_cast<std::size_t>(c) + 1];
  for (std::int32_t c = 0; c < s.m; ++c) d.cam_part_ptr[static_cast<std::size_t>(c) + 1] += d.cam_part_ptr[static_cast<std::size_t>(c)];
  d.cam_part.resize(static_cast<std::size_t>(d.n_part));
  std::vector<std::int32_t> cur(d.cam_part_ptr.begin(), d.cam_part_ptr.end() - 1);
  for (std::int32_t u = 0; u < n_chunk_part; ++u)
    d.cam_part[static_cast<std::size_t>(cur[static_cast<std::size_t>(d.ucam_cam[static_cast<std::size_t>(u)])]++)] = u;
  for (std::size_t h = 0; h < halo_cam.size(); ++h)
    d.cam_part[static_cast<std::size_t>(cur[static_cast<std::size_t>(halo_cam[h])]++)] = n_chunk_part + static_cast<std::int32_t>(h);
  // partials are stored camera-major: partial id -> its position
  d.part_pos.resize(static_cast<std::size_t>(d.n_part));
  for (std::int32_t k = 0; k < d.n_part; ++k) d.part_pos[static_cast<std::size_t>(d.cam_part[static_cast<std::size_t>(k)])] = k;
  return d;
}

}  // namespace dbag
