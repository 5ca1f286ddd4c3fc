// lw_bvh_build.cu -- GPU BVH build with the exact output of the reference's build_bvh
// (geometry.py:100-148): median split on the largest-extent axis (first max), triangles
// ordered by (centroid[axis], triangle id), leaves of <= 4 triangles, DFS pre-order node
// numbering, leaf children [-(start+1), count].
//
// Instead of the reference's recursive per-node lexsort, the build keeps three lists of
// triangle ids, each presorted once by (centroid_a, id) with a stable radix sort, and
// processes the tree one level at a time:
//   1. per-segment bounds: warp segmented reduction + ordered-integer atomics,
//   2. per-segment split: axis = argmax extent, half = size / 2, DFS node ids computed in
//      closed form (lw_count_nodes), leaves emit their `order` slice,
//   3. mark the left half of every segment from its split-axis list,
//   4. stable partition of all three lists inside every segment (exclusive scan + scatter),
// so every child segment is again sorted by (centroid_a, id) on every axis -- exactly the
// order the reference's lexsort produces for that child.  O(n log n) work in total.
#include <cub/cub.cuh>

#include "lw_common.cuh"
#include "lw_host.h"

namespace lw {

__host__ __device__ long long lw_count_nodes(long long n) {
  if (n <= 4) return 1;
  long long s0 = n, c0 = 1, s1 = n + 1, c1 = 0, total = 0;
  while (c0 > 0 || c1 > 0) {
    total += c0 + c1;
    long long lo = s0 / 2, n0 = 0, n1 = 0;
    long long sz[2] = {s0, s1}, ct[2] = {c0, c1};
    for (int k = 0; k < 2; k++) {
      if (ct[k] == 0 || sz[k] <= 4) continue;
      long long h = sz[k] / 2, r = sz[k] - h;
      if (h == lo) n0 += ct[k]; else n1 += ct[k];
      if (r == lo) n0 += ct[k]; else n1 += ct[k];
    }
    s0 = lo;
    c0 = n0;
    s1 = lo + 1;
    c1 = n1;
  }
  return total;
}

int64_t bvh_node_count(int64_t ntris) { return ntris == 0 ? 1 : lw_count_nodes(ntris); }

__device__ __forceinline__ unsigned long long ord_of(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double from_ord(unsigned long long u) {
  unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
  return __longlong_as_double((long long)b);
}

__global__ void k_tri_prep(const double* __restrict__ v, long long n, double* __restrict__ tmin, double* __restrict__ tmax,
                           unsigned long long* __restrict__ keys, int* __restrict__ ids) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = v + 9 * i;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double lo = p[a], hi = p[a];
    if (p[3 + a] < lo) lo = p[3 + a];
    if (p[6 + a] < lo) lo = p[6 + a];
    if (p[3 + a] > hi) hi = p[3 + a];
    if (p[6 + a] > hi) hi = p[6 + a];
    tmin[a * n + i] = lo;
    tmax[a * n + i] = hi;
    double c = 0.5 * (lo + hi);
    if (c == 0.0) c = 0.0;  // np.lexsort treats -0.0 == 0.0: canonicalise before keying
    keys[a * n + i] = ord_of(c);
  }
  ids[i] = (int)i;
}

struct SegTable {
  int* start;
  int* size;
  int* node;
  int* paxis;
};

__global__ void k_seg_bounds_init(unsigned long long* bmin, unsigned long long* bmax, int nseg) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bmin[3 * s + a] = ~0ULL;
    bmax[3 * s + a] = 0ULL;
  }
}

// warp segmented min/max over runs of equal segment ids, one atomic per run and axis
__global__ void k_seg_bounds(const int* __restrict__ pos_seg, const int* __restrict__ list0, long long n,
                             const double* __restrict__ tmin, const double* __restrict__ tmax,
                             unsigned long long* __restrict__ bmin, unsigned long long* __restrict__ bmax) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int lane = threadIdx.x & 31;
  int s = -1;
  unsigned long long mn[3] = {~0ULL, ~0ULL, ~0ULL}, mx[3] = {0, 0, 0};
  if (i < n) {
    s = pos_seg[i];
    if (s >= 0) {
      int t = list0[i];
#pragma unroll
      for (int a = 0; a < 3; a++) {
        mn[a] = ord_of(tmin[a * n + t]);
        mx[a] = ord_of(tmax[a * n + t]);
      }
    }
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int so = __shfl_up_sync(0xffffffffu, s, off);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      unsigned long long vmn = __shfl_up_sync(0xffffffffu, mn[a], off);
      unsigned long long vmx = __shfl_up_sync(0xffffffffu, mx[a], off);
      if (lane >= off && so == s) {
        if (vmn < mn[a]) mn[a] = vmn;
        if (vmx > mx[a]) mx[a] = vmx;
      }
    }
  }
  int snext = __shfl_down_sync(0xffffffffu, s, 1);
  bool tail = (lane == 31) || (snext != s) || (i + 1 >= n);
  if (i < n && s >= 0 && tail) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      atomicMin(bmin + 3 * s + a, mn[a]);
      atomicMax(bmax + 3 * s + a, mx[a]);
    }
  }
}

__global__ void k_seg_split(SegTable cur, int nseg, const unsigned long long* __restrict__ bmin,
                            const unsigned long long* __restrict__ bmax, double* __restrict__ bounds,
                            long long* __restrict__ children, long long* __restrict__ order,
                            const int* __restrict__ l0, const int* __restrict__ l1, const int* __restrict__ l2,
                            int* __restrict__ seg_axis, int* __restrict__ seg_child, SegTable nxt,
                            int* __restrict__ nxt_count) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int start = cur.start[s], size = cur.size[s], node = cur.node[s];
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    lo[a] = from_ord(bmin[3 * s + a]);
    hi[a] = from_ord(bmax[3 * s + a]);
    bounds[6 * (long long)node + a] = lo[a];
    bounds[6 * (long long)node + 3 + a] = hi[a];
  }
  if (size <= 4) {
    children[2 * (long long)node] = -((long long)start + 1);
    children[2 * (long long)node + 1] = size;
    int pa = cur.paxis[s];
    const int* L = pa == 0 ? l0 : (pa == 1 ? l1 : l2);
    for (int j = 0; j < size; j++) order[start + j] = pa < 0 ? (long long)(start + j) : (long long)L[start + j];
    seg_axis[s] = -1;
    return;
  }
  double e0 = hi[0] - lo[0], e1 = hi[1] - lo[1], e2 = hi[2] - lo[2];
  int axis = 0;
  double best = e0;
  if (e1 > best) {
    axis = 1;
    best = e1;
  }
  if (e2 > best) axis = 2;
  int half = size / 2;
  int c = atomicAdd(nxt_count, 2);
  long long left_node = (long long)node + 1;
  long long right_node = left_node + lw_count_nodes(half);
  nxt.start[c] = start;
  nxt.size[c] = half;
  nxt.node[c] = (int)left_node;
  nxt.paxis[c] = axis;
  nxt.start[c + 1] = start + half;
  nxt.size[c + 1] = size - half;
  nxt.node[c + 1] = (int)right_node;
  nxt.paxis[c + 1] = axis;
  children[2 * (long long)node] = left_node;
  children[2 * (long long)node + 1] = right_node;
  seg_axis[s] = axis;
  seg_child[s] = c;
}

__global__ void k_mark_left(const int* __restrict__ pos_seg, long long n, SegTable cur, const int* __restrict__ seg_axis,
                            const int* __restrict__ l0, const int* __restrict__ l1, const int* __restrict__ l2,
                            unsigned char* __restrict__ left) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = pos_seg[i];
  if (s < 0) return;
  int ax = seg_axis[s];
  if (ax < 0) return;
  int j = (int)i - cur.start[s];
  const int* L = ax == 0 ? l0 : (ax == 1 ? l1 : l2);
  left[L[i]] = j < cur.size[s] / 2 ? 1 : 0;
}

__global__ void k_flags(const int* __restrict__ pos_seg, long long n, const int* __restrict__ seg_axis,
                        const int* __restrict__ L, const unsigned char* __restrict__ left, int* __restrict__ flag) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = pos_seg[i];
  flag[i] = (s >= 0 && seg_axis[s] >= 0) ? (int)left[L[i]] : 0;
}

__global__ void k_partition(const int* __restrict__ pos_seg, long long n, SegTable cur, const int* __restrict__ seg_axis,
                            const int* __restrict__ L, const unsigned char* __restrict__ left,
                            const int* __restrict__ scan, int* __restrict__ Lout) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = pos_seg[i];
  int t = L[i];
  if (s < 0 || seg_axis[s] < 0) {
    Lout[i] = t;
    return;
  }
  int start = cur.start[s], half = cur.size[s] / 2;
  int j = (int)i - start;
  int rl = scan[i] - scan[start];
  int np = left[t] ? start + rl : start + half + (j - rl);
  Lout[np] = t;
}

__global__ void k_next_seg(int* __restrict__ pos_seg, long long n, SegTable cur, const int* __restrict__ seg_axis,
                           const int* __restrict__ seg_child) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = pos_seg[i];
  if (s < 0) return;
  if (seg_axis[s] < 0) {
    pos_seg[i] = -1;
    return;
  }
  int j = (int)i - cur.start[s];
  pos_seg[i] = seg_child[s] + (j < cur.size[s] / 2 ? 0 : 1);
}

__global__ void k_root_init(SegTable t, int n, int* pos_seg_first) {
  t.start[0] = 0;
  t.size[0] = n;
  t.node[0] = 0;
  t.paxis[0] = -1;
}

#define TRY(x) LW_CUDA_TRY(x)

int bvh_build_device(const double* d_verts, int64_t n, cudaStream_t st, DeviceBVH& out) {
  int64_t nnodes = bvh_node_count(n);
  out.nnodes = nnodes;
  TRY(cudaMallocAsync(&out.bounds, sizeof(double) * 6 * nnodes, st));
  TRY(cudaMallocAsync(&out.children, sizeof(long long) * 2 * nnodes, st));
  TRY(cudaMallocAsync(&out.order, sizeof(long long) * (n > 0 ? n : 1), st));
  if (n == 0) {  // geometry.py:103-106
    TRY(cudaMemsetAsync(out.bounds, 0, sizeof(double) * 6, st));
    long long ch[2] = {-1, 0};
    TRY(cudaMemcpyAsync(out.children, ch, sizeof(ch), cudaMemcpyHostToDevice, st));
    TRY(cudaStreamSynchronize(st));
    return LW_OK;
  }
  LW_CHECK_ARG(n < (1LL << 28), "bvh build: at most 2^28 triangles");
  const int B = 256;
  int gn = (int)((n + B - 1) / B);
  DevBuf b_tmin, b_tmax, b_keys, b_keys_out, b_ids, b_lists, b_lists2, b_pos, b_left, b_flag, b_scan, b_cnt;
  TRY(b_tmin.alloc(sizeof(double) * 3 * n, st));
  TRY(b_tmax.alloc(sizeof(double) * 3 * n, st));
  TRY(b_keys.alloc(sizeof(unsigned long long) * 3 * n, st));
  TRY(b_keys_out.alloc(sizeof(unsigned long long) * n, st));
  TRY(b_ids.alloc(sizeof(int) * n, st));
  TRY(b_lists.alloc(sizeof(int) * 3 * n, st));
  TRY(b_lists2.alloc(sizeof(int) * 3 * n, st));
  TRY(b_pos.alloc(sizeof(int) * n, st));
  TRY(b_left.alloc(n, st));
  TRY(b_flag.alloc(sizeof(int) * n, st));
  TRY(b_scan.alloc(sizeof(int) * n, st));
  TRY(b_cnt.alloc(sizeof(int), st));
  k_tri_prep<<<gn, B, 0, st>>>(d_verts, n, b_tmin.as<double>(), b_tmax.as<double>(), b_keys.as<unsigned long long>(),
                               b_ids.as<int>());
  TRY(cudaGetLastError());
  // presort each axis list by (centroid key, id): stable radix sort of (key, id) pairs
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, b_keys.as<unsigned long long>(), b_keys_out.as<unsigned long long>(),
                                  b_ids.as<int>(), b_lists.as<int>(), (int)n, 0, 64, st);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, b_flag.as<int>(), b_scan.as<int>(), (int)n, st);
  DevBuf b_tmp;
  TRY(b_tmp.alloc(sort_bytes > scan_bytes ? sort_bytes : scan_bytes, st));
  int* lists[3];
  int* lists2[3];
  for (int a = 0; a < 3; a++) {
    lists[a] = b_lists.as<int>() + a * n;
    lists2[a] = b_lists2.as<int>() + a * n;
    size_t tb = b_tmp.bytes;
    TRY(cub::DeviceRadixSort::SortPairs(b_tmp.p, tb, b_keys.as<unsigned long long>() + a * n,
                                        b_keys_out.as<unsigned long long>(), b_ids.as<int>(), lists[a], (int)n, 0, 64,
                                        st));
  }
  // segment tables (double-buffered); capacity n + 2 segments per level
  int cap = (int)n + 2;
  DevBuf b_seg[2], b_bmin, b_bmax, b_axis, b_child;
  SegTable tab[2];
  for (int k = 0; k < 2; k++) {
    TRY(b_seg[k].alloc(sizeof(int) * 4 * cap, st));
    int* p = b_seg[k].as<int>();
    tab[k] = SegTable{p, p + cap, p + 2 * cap, p + 3 * cap};
  }
  TRY(b_bmin.alloc(sizeof(unsigned long long) * 3 * cap, st));
  TRY(b_bmax.alloc(sizeof(unsigned long long) * 3 * cap, st));
  TRY(b_axis.alloc(sizeof(int) * cap, st));
  TRY(b_child.alloc(sizeof(int) * cap, st));
  TRY(cudaMemsetAsync(b_pos.p, 0, sizeof(int) * n, st));
  k_root_init<<<1, 1, 0, st>>>(tab[0], (int)n, nullptr);
  int nseg = 1, cur = 0;
  int* d_cnt = b_cnt.as<int>();
  while (nseg > 0) {
    SegTable T = tab[cur], N = tab[cur ^ 1];
    int gs = (nseg + B - 1) / B;
    k_seg_bounds_init<<<gs, B, 0, st>>>(b_bmin.as<unsigned long long>(), b_bmax.as<unsigned long long>(), nseg);
    k_seg_bounds<<<gn, B, 0, st>>>(b_pos.as<int>(), lists[0], n, b_tmin.as<double>(), b_tmax.as<double>(),
                                   b_bmin.as<unsigned long long>(), b_bmax.as<unsigned long long>());
    TRY(cudaMemsetAsync(d_cnt, 0, sizeof(int), st));
    k_seg_split<<<gs, B, 0, st>>>(T, nseg, b_bmin.as<unsigned long long>(), b_bmax.as<unsigned long long>(), out.bounds,
                                  out.children, out.order, lists[0], lists[1], lists[2], b_axis.as<int>(),
                                  b_child.as<int>(), N, d_cnt);
    k_mark_left<<<gn, B, 0, st>>>(b_pos.as<int>(), n, T, b_axis.as<int>(), lists[0], lists[1], lists[2],
                                  b_left.as<unsigned char>());
    for (int a = 0; a < 3; a++) {
      k_flags<<<gn, B, 0, st>>>(b_pos.as<int>(), n, b_axis.as<int>(), lists[a], b_left.as<unsigned char>(),
                                b_flag.as<int>());
      size_t tb = b_tmp.bytes;
      TRY(cub::DeviceScan::ExclusiveSum(b_tmp.p, tb, b_flag.as<int>(), b_scan.as<int>(), (int)n, st));
      k_partition<<<gn, B, 0, st>>>(b_pos.as<int>(), n, T, b_axis.as<int>(), lists[a], b_left.as<unsigned char>(),
                                    b_scan.as<int>(), lists2[a]);
      int* t = lists[a];
      lists[a] = lists2[a];
      lists2[a] = t;
    }
    k_next_seg<<<gn, B, 0, st>>>(b_pos.as<int>(), n, T, b_axis.as<int>(), b_child.as<int>());
    TRY(cudaGetLastError());
    TRY(cudaMemcpyAsync(&nseg, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(cudaStreamSynchronize(st));
    cur ^= 1;
  }
  return LW_OK;
}

}  // namespace lw

using namespace lw;

extern "C" int lw_bvh_build(const double* verts, int64_t ntris, double* bounds, int64_t* children, int64_t* order,
                            int64_t* nnodes) {
  LW_CHECK_ARG(ntris >= 0 && (ntris == 0 || verts) && bounds && children && nnodes, "bad arguments");
  cudaStream_t st = cudaStreamPerThread;
  DevBuf b_v;
  LW_CUDA_TRY(b_v.alloc(sizeof(double) * 9 * (ntris > 0 ? ntris : 1), st));
  if (ntris > 0) LW_CUDA_TRY(cudaMemcpyAsync(b_v.p, verts, sizeof(double) * 9 * ntris, cudaMemcpyHostToDevice, st));
  DeviceBVH bvh;
  int rc = bvh_build_device(b_v.as<double>(), ntris, st, bvh);
  if (rc == LW_OK) {
    *nnodes = bvh.nnodes;
    cudaError_t e = cudaMemcpyAsync(bounds, bvh.bounds, sizeof(double) * 6 * bvh.nnodes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(children, bvh.children, sizeof(long long) * 2 * bvh.nnodes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && ntris > 0)
      e = cudaMemcpyAsync(order, bvh.order, sizeof(long long) * ntris, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("bvh download failed: %s", cudaGetErrorString(e));
      rc = LW_ERR_CUDA;
    }
  }
  cudaFree(bvh.bounds);
  cudaFree(bvh.children);
  cudaFree(bvh.order);
  return rc;
}
