#pragma once
#include <algorithm>
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
  bool direct = false;  // small-graph path: sums complete, no 4-clique / 4-cycle totals
  int64_t row0 = 0;   // first canonical edge of the rows written to the table
  int64_t rows = -1;  // rows written (-1: all m)
  // in: page-locked host destination of the whole per-edge table (optional).
  // When set, a single-graph census finalizes in row chunks and copies each
  // chunk to the host on a second stream while the next one is finalized;
  // out: table_copied says the host table is complete on return.
  void* host_table = nullptr;
  bool table_copied = false;
};

// Multi-GPU census of one graph.  The frames of passes A-C are dealt
// round-robin (in descending-work order) to `world` shards; each rank owns
// the contiguous canonical edge range [r*M, (r+1)*M), M = ceil(m / world),
// and finalizes only those rows:
//   after pass A   the per-edge triangle / 4-clique counts (m x u64, packed
//                  edge-indexed) and T(x) (n x u64) are all-reduced -- pass B
//                  reads t of any edge;
//   after pass C   the per-edge partial sums of passes B and C (4 x m, u32
//                  below degree 2^16) are reduce-scattered onto the owners;
//   finalize       owned rows only; the 13 x 128-bit sums and the 4-clique /
//                  4-cycle totals of every rank are all-gathered and added.
// Volume per rank at R-MAT-20 (m = 15.7M): all-reduce 126 MB + 8 MB,
// reduce-scatter 251 MB (u32 slots) -- ~0.55 GB moved per rank at 8 ranks
// (ring: 2(W-1)/W of the all-reduced and (W-1)/W of the reduce-scattered
// bytes), against 1.26 GB for the former all-reduce of every slot array.
// With no communicator, `world` shards are emulated one after another on
// this GPU: they share the accumulators (which is exactly the all-reduce /
// reduce-scatter), and the ownership packing, unpacking and per-range
// finalize run as in a real job -- the single-GPU check of the partition.
struct Shard {
  int rank = 0, world = 1;
  std::function<void(unsigned long long*, size_t)> allreduce;
  std::function<void(const unsigned long long*, unsigned long long*, size_t)> allgather;
  // reduce_scatter(send, recv, recvcount, element bytes 4 | 8): sum
  std::function<void(const void*, void*, size_t, int)> reduce_scatter;
  bool real() const { return (bool)allreduce; }
};

// Owned canonical edge range [e0, e1) of a rank.
inline void shard_rows(int64_t m, int rank, int world, int64_t* e0, int64_t* e1) {
  const int64_t M = world > 0 ? (m + world - 1) / world : m;
  *e0 = std::min<int64_t>(m, (int64_t)rank * M);
  *e1 = std::min<int64_t>(m, *e0 + M);
}

// Runs the census on device graph g.  table_dev: int64 [m][10] device buffer
// or null; sums_dev: uint64 [G][13][2]; seen_dev: uint64 [G].
void run_census(DevGraph& g, bool per_edge, long long* table_dev, unsigned long long* sums_dev,
                unsigned long long* seen_dev, CensusExtras& ex, cudaStream_t s,
                const Shard& shard = Shard());

void sums_from_table(const long long* table_dev, int64_t m, int64_t n,
                     unsigned long long* sums_dev, cudaStream_t s);

}  // namespace gd
