#pragma once
#include <functional>
#include <string>
#include <vector>

#include "gd_common.cuh"

namespace gd {

// Host-side results of one census call besides the device sums.
struct CensusExtras {
  std::vector<unsigned __int128> k4tot;   // per graph: number of 4-cliques
  std::vector<unsigned __int128> c4tot2;  // per graph: 2 x number of 4-cycles (non-induced)
  std::vector<float> ms;                  // phase timings (CUDA events)
  std::vector<std::string> names;
  std::vector<int64_t> stats;
  std::vector<std::string> stats_names;
};

// Frame sharding for multi-GPU runs.  The frames of passes A-C are dealt
// round-robin (in descending-work order) to `world` shards; the slot-indexed
// partial counters are summed between passes (allreduce, in place) and the
// per-shard 128-bit totals gathered (allgather: count u64 per rank).  Every
// rank then finalizes all edges.  With no allreduce, `world` shards are
// emulated one after another on this GPU (they share the accumulators, which
// is exactly the all-reduce): the single-GPU check of the partitioning.
struct Shard {
  int rank = 0, world = 1;
  std::function<void(unsigned long long*, size_t)> allreduce;
  std::function<void(const unsigned long long*, unsigned long long*, size_t)> allgather;
  bool real() const { return (bool)allreduce; }
};

// Runs the census on device graph g.  table_dev: int64 [m][10] device buffer
// or null; sums_dev: uint64 [G][13][2]; seen_dev: uint64 [G].
void run_census(DevGraph& g, bool per_edge, long long* table_dev, unsigned long long* sums_dev,
                unsigned long long* seen_dev, CensusExtras& ex, cudaStream_t s,
                const Shard& shard = Shard());

void sums_from_table(const long long* table_dev, int64_t m, int64_t n,
                     unsigned long long* sums_dev, cudaStream_t s);

}  // namespace gd
