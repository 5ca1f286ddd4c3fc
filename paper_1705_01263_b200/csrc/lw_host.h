// lw_host.h -- internal host-side interfaces shared by the translation units of liblw_b200.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/lw_b200.h"
#include "lw_envpyr.cuh"
#include "lw_lighttree.cuh"
#include "lw_qmc.cuh"

namespace lw {

void set_error(const char* fmt, ...);

// QmcDim/perm tables from the reference's DimensionTable arrays (qmc.py:274-305)
int pack_qmc_tables(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                    const int64_t* perm_offset, std::vector<QmcDim>& dims, std::vector<uint16_t>& perm);

// Vose alias table; same operation order as the oracle
int alias_build(const double* w, int64_t n, double* prob, int32_t* alias, double* pdf);

// environment pyramid (lw_envpyr.cuh; oracle ep_build): levels and per-bin top levels; `meta`
// gets sizes and offsets (its pointers are set by the caller after upload)
int env_pyramid_build(int W, int H, const double* weight, std::vector<double>& lvl, std::vector<double>& top,
                      LwEnvPyr& meta);

// light hierarchy over the emitters of positive weight (lw_lighttree.cuh; oracle lt_build):
// depth-first nodes, per-emitter branch bits and depth (-1 = not in the tree)
int light_tree_build(const double* verts, const int64_t* emit_tri, const double* weight, const int32_t* twosided,
                     int64_t nemit, std::vector<LwLightNode>& nodes, std::vector<unsigned long long>& path,
                     std::vector<int>& depth);

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

// Binned-SAH render BVH: internal nodes in breadth-first order with both
// children's boxes, leaf refs -(1 + (start<<3 | count)).
struct SahNode {
  double box[12];
  int32_t ref[2];
};
inline int32_t leaf_ref32_host(int64_t start, int64_t count) { return (int32_t)(-(1 + ((start << 3) | count))); }

// the same tree built on the GPU (lw_sah_build.cu); nodes/order are device arrays owned by the caller
struct DeviceSah {
  SahNode* nodes = nullptr;
  int* order = nullptr;
  int64_t nnodes = 0;
  int32_t root_ref = -1;
  double root_box[6];
  int levels = 0;  // binary tree depth bound (level-synchronous build iterations)
};
int sah_build_device(const double* d_verts, int64_t ntris, cudaStream_t stream, DeviceSah& out);

}  // namespace lw
