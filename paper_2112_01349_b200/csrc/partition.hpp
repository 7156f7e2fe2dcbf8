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

}  // namespace dbag
