// lw_lighttree.cuh -- probabilistic light hierarchy for many-light NEE.
//
// PAPER.md:215-253 / SPEC.md:180-221 (LightHierarchy, sample_light, light_pdf): a BVH over the
// emissive triangles is traversed probabilistically from the shading point; at every node the
// two children's contribution estimates (flux in the direction of the point, a conservative
// cosine at the point, inverse squared distance) set the branch probabilities, clamped to
// [1/64, 63/64] so no light gets probability zero; the same walk replayed along an emitter's
// stored path gives the selection probability for MIS.  Directional emission is captured by
// per-node flux bins over the 8 octants of the unit sphere ("subdivide the unit sphere into a
// small set of regions and store one representative value per region").
//
// Every operation is restated in oracle/lw_oracle.c (lt_*) in the same order, so sampled
// emitters, selection probabilities and images are bit-identical to the oracle.
#pragma once
#include "lw_common.cuh"

#define LW_LT_PMIN 0.015625  // 1/64

// 64-byte node.  Built (host, oracle) in depth-first order: left child = node + 1, right child =
// `right`; leaf: right = -(emitter + 1).  The estimates
// are heuristics (clamped branch probabilities keep the estimator unbiased), so the node data and
// the importance arithmetic are FP32: IEEE single operations with correctly rounded division and
// square root give the same bits on the host (oracle, -ffp-contract=off) and the device.
struct __align__(16) LwLightNode {
  float lo[3], hi[3];
  float tot;      // sum of emitter weights (luminance(L) * area) below the node
  float flux[8];  // per emission octant: sum of weight * max cos towards that octant
  int right;      // internal: right child index; leaf: -(emitter + 1)
};

// max over unit directions w in octant k (bit a set = negative axis a) of max(0, n . w) (FP64, build)
__host__ __device__ inline double lw_lt_octant_cos(int k, double nx, double ny, double nz) {
  double a = (k & 1) ? -nx : nx, b = (k & 2) ? -ny : ny, c = (k & 4) ? -nz : nz;
  a = a > 0.0 ? a : 0.0;
  b = b > 0.0 ? b : 0.0;
  c = c > 0.0 ? c : 0.0;
  return sqrt((a * a + b * b) + c * c);
}

// contribution estimate of a node at point x with (unit) normal n, as a fraction num / den
// (den > 0; FP32): pleft combines two fractions with a single division
__device__ __forceinline__ void lw_lt_importance(const LwLightNode& N, float x0, float x1, float x2, float n0, float n1,
                                                 float n2, float& num, float& den) {
  float cx = (N.lo[0] + N.hi[0]) * 0.5f, cy = (N.lo[1] + N.hi[1]) * 0.5f, cz = (N.lo[2] + N.hi[2]) * 0.5f;
  float dx = cx - x0, dy = cy - x1, dz = cz - x2;
  float d2 = (dx * dx + dy * dy) + dz * dz;
  float ex = N.hi[0] - N.lo[0], ey = N.hi[1] - N.lo[1], ez = N.hi[2] - N.lo[2];
  float r2 = ((ex * ex + ey * ey) + ez * ez) * 0.25f;
  float dist2 = d2 > r2 ? d2 : r2;
  bool inside = x0 >= N.lo[0] && x0 <= N.hi[0] && x1 >= N.lo[1] && x1 <= N.hi[1] && x2 >= N.lo[2] && x2 <= N.hi[2];
  if (inside || !(d2 > r2)) {
    num = N.tot;
    den = dist2 > 0.0f ? dist2 : 1.0f;
    return;
  }
  int oct = (dx > 0.0f ? 1 : 0) | (dy > 0.0f ? 2 : 0) | (dz > 0.0f ? 4 : 0);  // signs of x - c
  // cos(max(0, theta - alpha)) * d^2 with cos theta = dt / d, cos alpha = sqrt(d2 - r2) / d,
  // sin alpha = r / d: (dt sqrt(d2 - r2) + sqrt(d2 - dt^2) r) / d^2, 1 when theta <= alpha
  float dt = (n0 * dx + n1 * dy) + n2 * dz;
  float s1 = sqrtf(d2 - r2);
  if (dt >= s1) {
    num = N.flux[oct];
    den = dist2;
    return;
  }
  float s2 = d2 - dt * dt;
  float t = dt * s1 + sqrtf(s2 > 0.0f ? s2 : 0.0f) * sqrtf(r2);
  if (t < 0.0f) t = 0.0f;
  num = N.flux[oct] * t;
  den = d2 * dist2;
}

// The device keeps the tree in heap order (children of i at 2i + 1, 2i + 2; the median split makes
// it nearly complete, holes unused) so the top LW_LT_SMEM_NODES nodes -- the first nine levels,
// visited by every walk -- are one contiguous prefix that the shading kernels stage in shared
// memory; only the deepest levels come from L2.  Same values, same operation order as the
// oracle's depth-first layout, so samples and probabilities are unchanged.
#ifndef LW_LT_SMEM_NODES
#define LW_LT_SMEM_NODES 511
#endif

struct LwLightTree {
  const LwLightNode* nodes;  // heap order, global memory
  const LwLightNode* top;    // nodes [0, ntop) in shared memory (== nodes when not staged)
  int ntop;
  const unsigned long long* path;  // per emitter: branch bits (1 = right), depth
  const int* depth;
};

__device__ __forceinline__ const LwLightNode& lw_lt_node(const LwLightTree& T, int i) {
  return i < T.ntop ? T.top[i] : T.nodes[i];
}

// stage the top of the tree in shared memory (all threads of the block; nheap = heap slots)
__device__ __forceinline__ LwLightTree lw_lt_stage(LwLightTree T, int nheap, unsigned char* smem) {
  int n = nheap < LW_LT_SMEM_NODES ? nheap : LW_LT_SMEM_NODES;
  const int4* src = reinterpret_cast<const int4*>(T.nodes);
  int4* dst = reinterpret_cast<int4*>(smem);
  for (int k = threadIdx.x; k < n * 4; k += blockDim.x) dst[k] = src[k];
  __syncthreads();
  T.top = reinterpret_cast<const LwLightNode*>(smem);
  T.ntop = n;
  return T;
}

// probability of descending into the left child of internal heap node `k`
__device__ __forceinline__ double lw_lt_pleft(const LwLightTree& T, int k, v3 x, v3 n) {
  float x0 = (float)x.x, x1 = (float)x.y, x2 = (float)x.z, n0 = (float)n.x, n1 = (float)n.y, n2 = (float)n.z;
  float nl, dl, nr, dr;
  lw_lt_importance(lw_lt_node(T, 2 * k + 1), x0, x1, x2, n0, n1, n2, nl, dl);
  lw_lt_importance(lw_lt_node(T, 2 * k + 2), x0, x1, x2, n0, n1, n2, nr, dr);
  float il = nl * dr, ir = nr * dl;  // importances scaled by the common factor dl * dr
  float s = il + ir;
  float pl = s > 0.0f ? il / s : 0.5f;
  if (pl < (float)LW_LT_PMIN) pl = (float)LW_LT_PMIN;
  if (pl > 1.0f - (float)LW_LT_PMIN) pl = 1.0f - (float)LW_LT_PMIN;
  return (double)pl;
}

// sample_light: emitter index, selection probability, and the rescaled remaining uniform
__device__ __forceinline__ long long lw_lt_sample(const LwLightTree& T, v3 x, v3 n, double u, double& psel,
                                                  double& u_out) {
  int k = 0;
  double p = 1.0;
  while (lw_lt_node(T, k).right >= 0) {
    double pl = lw_lt_pleft(T, k, x, n);
    if (u < pl) {
      u = u / pl;
      p = p * pl;
      k = 2 * k + 1;
    } else {
      u = (u - pl) / (1.0 - pl);
      p = p * (1.0 - pl);
      k = 2 * k + 2;
    }
  }
  if (u >= 1.0) u = 0.9999999999999999;
  if (u < 0.0) u = 0.0;
  psel = p;
  u_out = u;
  return -(long long)lw_lt_node(T, k).right - 1;
}

// light_pdf's selection factor: the same walk along the emitter's stored path (bit l = branch
// taken at depth l, 1 = right); 0 for emitters outside the tree (zero weight)
__device__ __forceinline__ double lw_lt_pdf(const LwLightTree& T, long long e, v3 x, v3 n) {
  int dep = T.depth[e];
  if (dep < 0) return 0.0;
  unsigned long long bits = T.path[e];
  int k = 0;
  double p = 1.0;
  for (int l = 0; l < dep; l++) {
    double pl = lw_lt_pleft(T, k, x, n);
    if (((bits >> l) & 1ULL) == 0) {
      p = p * pl;
      k = 2 * k + 1;
    } else {
      p = p * (1.0 - pl);
      k = 2 * k + 2;
    }
  }
  return p;
}
