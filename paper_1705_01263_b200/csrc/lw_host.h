// lw_host.h -- internal host-side interfaces shared by the translation units of liblw_b200.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "lw_qmc.cuh"

namespace lw {

// QmcDim/perm tables from the reference's DimensionTable arrays (qmc.py:274-305)
int pack_qmc_tables(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                    const int64_t* perm_offset, std::vector<QmcDim>& dims, std::vector<uint16_t>& perm);

// Vose alias table; same operation order as the oracle
int alias_build(const double* w, int64_t n, double* prob, int32_t* alias, double* pdf);

// Device BVH build (geometry.py:100-148 semantics).  d_verts [ntris*9] on the device.
// Outputs are device arrays owned by the caller after the call (cudaFree).
struct DeviceBVH {
  int64_t nnodes = 0;
  double* bounds = nullptr;      // [nnodes*6]
  long long* children = nullptr; // [nnodes*2]
  long long* order = nullptr;    // [ntris]
};
int bvh_build_device(const double* d_verts, int64_t ntris, cudaStream_t stream, DeviceBVH& out);
int64_t bvh_node_count(int64_t ntris);

}  // namespace lw
