// Collectives of the slab-sharded step and the slab planner.  Not part of the
// C-ABI: the C-ABI wraps these in hot_set_comm_host / hot_set_comm_nccl / hot_plan_slabs.
//
// The sharded step needs exactly three collectives, all on contiguous byte ranges of device
// buffers whose layout is identical on every rank (global row order):
//   allgather_ranges  rank r's [off[r], off[r+1]) to every rank (level-1 matrix rows after the
//                     Galerkin split, the level-0 residual and smoother output rows);
//   halo              rank r's first / last lattice planes to its two neighbours (level-0 u after
//                     each residue group of smoother waves, hot_context.cu sgs0_sharded);
//   allreduce_max     a few host ints (failure flags of sharded kernels, so every rank takes the
//                     same branch and no rank is left waiting in a collective).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/hot_c_api.h"

namespace hotb200 {

struct Comm {
  int rank = 0, size = 1;
  long long halos = 0, gathers = 0;
  virtual ~Comm() = default;
  virtual void allgather_ranges(void* dbuf, const std::vector<long long>& off, cudaStream_t s) = 0;
  virtual void halo(void* dbuf, const std::vector<long long>& edges, cudaStream_t s) = 0;
  virtual void allreduce_max(int* host_v, int n, cudaStream_t s) = 0;
};

Comm* make_host_comm(const hot_comm_host& ops);
Comm* make_nccl_comm(const unsigned char id[128], int rank, int size);
void nccl_unique_id(unsigned char id[128]);

/// hot_plan_slabs (include/hot_c_api.h); false when no admissible cut exists.
bool plan_slabs(int plane_lo, int nplanes, const long long* weight, int size, int align, int min_width, int* bounds);

}  // namespace hotb200
