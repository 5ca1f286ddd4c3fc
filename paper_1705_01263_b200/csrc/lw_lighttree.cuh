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

// 128-byte node, depth-first order: left child = node + 1, right child = `right`
struct __align__(16) LwLightNode {
  double lo[3], hi[3];
  double tot;      // sum of emitter weights (luminance(L) * area) below the node
  double flux[8];  // per emission octant: sum of weight * max cos towards that octant
  int right;       // internal: right child index; leaf: -(emitter + 1)
  int pad;
};

// max over unit directions w in octant k (bit a set = negative axis a) of max(0, n . w)
__host__ __device__ inline double lw_lt_octant_cos(int k, double nx, double ny, double nz) {
  double a = (k & 1) ? -nx : nx, b = (k & 2) ? -ny : ny, c = (k & 4) ? -nz : nz;
  a = a > 0.0 ? a : 0.0;
  b = b > 0.0 ? b : 0.0;
  c = c > 0.0 ? c : 0.0;
  return sqrt((a * a + b * b) + c * c);
}

// contribution estimate of a node at point x with (unit) normal n
__device__ __forceinline__ double lw_lt_importance(const LwLightNode& N, v3 x, v3 n) {
  v3 c = mk3((N.lo[0] + N.hi[0]) * 0.5, (N.lo[1] + N.hi[1]) * 0.5, (N.lo[2] + N.hi[2]) * 0.5);
  v3 dx = c - x;
  double d2 = dot3(dx, dx);
  v3 ext = mk3(N.hi[0] - N.lo[0], N.hi[1] - N.lo[1], N.hi[2] - N.lo[2]);
  double r2 = dot3(ext, ext) * 0.25;
  double dist2 = d2 > r2 ? d2 : r2;
  bool inside = x.x >= N.lo[0] && x.x <= N.hi[0] && x.y >= N.lo[1] && x.y <= N.hi[1] && x.z >= N.lo[2] &&
                x.z <= N.hi[2];
  if (inside || !(d2 > r2)) return dist2 > 0.0 ? N.tot / dist2 : N.tot;
  int oct = (dx.x > 0.0 ? 1 : 0) | (dx.y > 0.0 ? 2 : 0) | (dx.z > 0.0 ? 4 : 0);  // signs of x - c
  double d = sqrt(d2);
  double cos_t = dot3(n, dx) / d;
  double sin2a = r2 / d2;
  double cos_a = sqrt(1.0 - sin2a);
  double cosb = 1.0;
  if (cos_t < cos_a) {
    double s2 = 1.0 - cos_t * cos_t;
    double sin_t = sqrt(s2 > 0.0 ? s2 : 0.0);
    cosb = cos_t * cos_a + sin_t * sqrt(sin2a);
    if (cosb < 0.0) cosb = 0.0;
  }
  return N.flux[oct] * cosb / dist2;
}

// probability of descending into the left child of internal node `k`
__device__ __forceinline__ double lw_lt_pleft(const LwLightNode* __restrict__ nodes, int k, v3 x, v3 n) {
  double il = lw_lt_importance(nodes[k + 1], x, n);
  double ir = lw_lt_importance(nodes[nodes[k].right], x, n);
  double s = il + ir;
  double pl = s > 0.0 ? il / s : 0.5;
  if (pl < LW_LT_PMIN) pl = LW_LT_PMIN;
  if (pl > 1.0 - LW_LT_PMIN) pl = 1.0 - LW_LT_PMIN;
  return pl;
}

// sample_light: emitter index, selection probability, and the rescaled remaining uniform
__device__ __forceinline__ long long lw_lt_sample(const LwLightNode* __restrict__ nodes, v3 x, v3 n, double u,
                                                  double& psel, double& u_out) {
  int k = 0;
  double p = 1.0;
  while (nodes[k].right >= 0) {
    double pl = lw_lt_pleft(nodes, k, x, n);
    if (u < pl) {
      u = u / pl;
      p = p * pl;
      k = k + 1;
    } else {
      u = (u - pl) / (1.0 - pl);
      p = p * (1.0 - pl);
      k = nodes[k].right;
    }
  }
  if (u >= 1.0) u = 0.9999999999999999;
  if (u < 0.0) u = 0.0;
  psel = p;
  u_out = u;
  return -(long long)nodes[k].right - 1;
}

// light_pdf's selection factor: the same walk along the emitter's stored path (bit l = branch
// taken at depth l, 1 = right); 0 for emitters outside the tree (zero weight)
__device__ __forceinline__ double lw_lt_pdf(const LwLightNode* __restrict__ nodes,
                                            const unsigned long long* __restrict__ path, const int* __restrict__ depth,
                                            long long e, v3 x, v3 n) {
  int dep = depth[e];
  if (dep < 0) return 0.0;
  unsigned long long bits = path[e];
  int k = 0;
  double p = 1.0;
  for (int l = 0; l < dep; l++) {
    double pl = lw_lt_pleft(nodes, k, x, n);
    if (((bits >> l) & 1ULL) == 0) {
      p = p * pl;
      k = k + 1;
    } else {
      p = p * (1.0 - pl);
      k = nodes[k].right;
    }
  }
  return p;
}
