// lw_traverse.cuh -- watertight FP64 ray/triangle test and BVH traversal.
//
// Reference semantics: _kernels.py:345-585.
//  * LwShear / lw_tri_test: the max-axis shear test (_tri_hit, 368-416) with the
//    reference's closest-hit tie rule (lower triangle id wins at equal t).  In compat
//    mode the unpermuted origin is subtracted from permuted vertex components (defect
//    D1, 378-386) exactly like the reference.
//  * lw_traverse_ref: _traverse_closest (422-545) over the reference layout
//    (bounds[N,6], children[N,2], order[T]) with its LIFO, right-child-first order and
//    cull rule; compat keeps the 1/0 -> 1e200 slab (defect D2), corrected tests slab
//    containment for zero direction components.
//  * RenderBVH: the render traversal over a child-box layout (two FP64 child boxes per
//    128-byte node), near-child-first, with a conservative 2^-40 relative slack on every
//    slab comparison; the oracle mirrors it operation for operation.
#pragma once
#include "lw_common.cuh"

struct LwShear {
  int kx, ky, kz;
  double sx, sy, sz;
  double op[3];  // origin as subtracted by the triangle test
};

__device__ __forceinline__ void lw_shear_setup(const double o[3], const double d[3], bool compat, LwShear& s) {
  double adx = fabs(d[0]), ady = fabs(d[1]), adz = fabs(d[2]);
  int kz = 0;
  if (ady > adx) {
    kz = 1;
    if (adz > ady) kz = 2;
  } else if (adz > adx) {
    kz = 2;
  }
  int kx = kz + 1;
  if (kx == 3) kx = 0;
  int ky = kx + 1;
  if (ky == 3) ky = 0;
  double dkz = kz == 0 ? d[0] : (kz == 1 ? d[1] : d[2]);
  if (dkz < 0.0) {
    int t = kx;
    kx = ky;
    ky = t;
  }
  double dkx = kx == 0 ? d[0] : (kx == 1 ? d[1] : d[2]);
  double dky = ky == 0 ? d[0] : (ky == 1 ? d[1] : d[2]);
  s.kx = kx;
  s.ky = ky;
  s.kz = kz;
  s.sz = 1.0 / dkz;
  s.sx = dkx * s.sz;
  s.sy = dky * s.sz;
  if (compat) {
    s.op[0] = o[0];
    s.op[1] = o[1];
    s.op[2] = o[2];
  } else {
    s.op[0] = kx == 0 ? o[0] : (kx == 1 ? o[1] : o[2]);
    s.op[1] = ky == 0 ? o[0] : (ky == 1 ? o[1] : o[2]);
    s.op[2] = kz == 0 ? o[0] : (kz == 1 ? o[1] : o[2]);
  }
}

struct LwHit {
  double t, bu, bv;
  long long tri;
};

// shear-space edge functions of one triangle; returns false if rejected, else t and (v, w), det.
// The barycentrics v/det, w/det are divided only once the closest hit is final (same ops,
// same bits as the reference, which divides on every accepted update).
// `v` points at the 9 vertex doubles in memory (global or shared): the per-ray axis permutation
// is applied through the load addresses, not with register selects.
__device__ __forceinline__ bool lw_tri_eval(const double* __restrict__ v, const LwShear& s, double& t, double& bu,
                                            double& bv, double& det_out) {
  double ax = v[s.kx] - s.op[0], ay = v[s.ky] - s.op[1], az = v[s.kz] - s.op[2];
  double bx = v[3 + s.kx] - s.op[0], by = v[3 + s.ky] - s.op[1], bz = v[3 + s.kz] - s.op[2];
  double cx = v[6 + s.kx] - s.op[0], cy = v[6 + s.ky] - s.op[1], cz = v[6 + s.kz] - s.op[2];
  double sax = ax - s.sx * az, say = ay - s.sy * az;
  double sbx = bx - s.sx * bz, sby = by - s.sy * bz;
  double scx = cx - s.sx * cz, scy = cy - s.sy * cz;
  double u = scx * sby - scy * sbx;
  double vv = sax * scy - say * scx;
  double w = sbx * say - sby * sax;
  if ((u < 0.0 || vv < 0.0 || w < 0.0) && (u > 0.0 || vv > 0.0 || w > 0.0)) return false;
  double det = u + vv + w;
  if (det == 0.0) return false;
  double t_scaled = u * (s.sz * az) + vv * (s.sz * bz) + w * (s.sz * cz);
  t = t_scaled / det;
  bu = vv;
  bv = w;
  det_out = det;
  return true;
}

// _tri_hit with the closest-hit update rule (t in (tmin, best], tie -> lower id)
__device__ __forceinline__ void lw_tri_test(const double* __restrict__ v, long long tri, const LwShear& s, double tmin,
                                            LwHit& h) {
  double t, bu, bv, det;
  if (!lw_tri_eval(v, s, t, bu, bv, det)) return;
  if (t <= tmin) return;
  if (t > h.t) return;
  if (t == h.t && h.tri >= 0 && tri >= h.tri) return;
  h.t = t;
  h.tri = tri;
  h.bu = bu / det;
  h.bv = bv / det;
}

__device__ __forceinline__ bool lw_tri_occludes(const double* __restrict__ v, const LwShear& s, double tmax) {
  double t, bu, bv, det;
  if (!lw_tri_eval(v, s, t, bu, bv, det)) return false;
  return t > 0.0 && t < tmax;
}

__device__ __forceinline__ double lw_safe_inv(double d) {
  if (d > 1e-200 || d < -1e-200) return 1.0 / d;
  if (d >= 0.0) return 1e200;
  return -1e200;
}

// _traverse_closest over the reference layout; stack holds node ids (LIFO, c1 popped first)
__device__ __forceinline__ void lw_traverse_ref(bool compat, const double* __restrict__ bounds,
                                                const long long* __restrict__ children,
                                                const long long* __restrict__ order, const double* __restrict__ verts,
                                                long long ntris, const double o[3], const double d[3], double tmax,
                                                LwHit& h) {
  h.t = tmax;
  h.tri = -1;
  h.bu = 0.0;
  h.bv = 0.0;
  if (ntris == 0) return;
  LwShear s;
  lw_shear_setup(o, d, compat, s);
  double inv[3] = {lw_safe_inv(d[0]), lw_safe_inv(d[1]), lw_safe_inv(d[2])};
  bool zero[3];
#pragma unroll
  for (int a = 0; a < 3; a++) zero[a] = !compat && (inv[a] == 1e200 || inv[a] == -1e200);
  int stack[128];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    int node = stack[--sp];
    const double* b = bounds + 6 * (size_t)node;
    double tn = -INFINITY, tf = INFINITY;
    bool culled = false;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double lo = __ldg(b + a), hi = __ldg(b + 3 + a);
      if (zero[a]) {
        if (o[a] < lo || o[a] > hi) culled = true;
        continue;
      }
      double t0 = (lo - o[a]) * inv[a];
      double t1 = (hi - o[a]) * inv[a];
      if (compat && a == 0) {
        if (t0 > t1) {
          tn = t1;
          tf = t0;
        } else {
          tn = t0;
          tf = t1;
        }
        continue;
      }
      if (t0 > t1) {
        if (t0 < tf) tf = t0;
        if (t1 > tn) tn = t1;
      } else {
        if (t1 < tf) tf = t1;
        if (t0 > tn) tn = t0;
      }
    }
    if (culled) continue;
    if (tn > tf || tn > h.t || tf < 0.0) continue;
    long long c0 = __ldg(children + 2 * (size_t)node), c1 = __ldg(children + 2 * (size_t)node + 1);
    if (c0 < 0) {
      long long start = -(c0 + 1);
      for (long long i = 0; i < c1; i++) {
        long long tri = __ldg(order + start + i);
        lw_tri_test(verts + 9 * tri, tri, s, 0.0, h);
      }
    } else if (sp < 126) {
      stack[sp++] = (int)c0;
      stack[sp++] = (int)c1;
    }
  }
}

// ---- render traversal ------------------------------------------------------------------

#define LW_CULL_M 9.094947017729282e-13  // 2^-40
#define LW_REF_NONE 0x7fffffff

// 128-byte node: child boxes (lo xyz, hi xyz) x 2, child refs; ref >= 0 internal, < 0 leaf
struct __align__(16) RNode {
  double box[12];
  int ref[2];
  int pad[6];
};

// 80-byte leaf-ordered triangle: vertices + original id
struct __align__(16) LTri {
  double v[9];
  long long id;
};

struct RenderBVH {
  const RNode* nodes;
  const LTri* tris;
  long long ntris;
  int root_ref;
  double root_box[6];
};

struct LwRay {
  double o[3], inv[3];
  bool zero[3];
  LwShear sh;
};

__device__ __forceinline__ void lw_ray_setup(LwRay& r, const double o[3], const double d[3]) {
#pragma unroll
  for (int a = 0; a < 3; a++) {
    r.o[a] = o[a];
    r.zero[a] = !(d[a] > 1e-200 || d[a] < -1e-200);
    r.inv[a] = r.zero[a] ? 0.0 : 1.0 / d[a];
  }
  lw_shear_setup(o, d, false, r.sh);
}

__device__ __forceinline__ bool lw_box_hit(const LwRay& r, const double* box, double best, double& tn_out) {
  double tn = -INFINITY, tf = INFINITY;
  bool miss = false;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double lo = box[a], hi = box[3 + a];
    if (r.zero[a]) {
      if (r.o[a] < lo || r.o[a] > hi) miss = true;
      continue;
    }
    double t0 = (lo - r.o[a]) * r.inv[a];
    double t1 = (hi - r.o[a]) * r.inv[a];
    double mn = t0 > t1 ? t1 : t0;
    double mx = t0 > t1 ? t0 : t1;
    if (mn > tn) tn = mn;
    if (mx < tf) tf = mx;
  }
  double tn_lo = tn - LW_CULL_M * fabs(tn);
  double tf_hi = tf + LW_CULL_M * fabs(tf);
  double best_hi = best + LW_CULL_M * fabs(best);
  tn_out = tn;
  return !miss && tn_lo <= tf_hi && tn_lo <= best_hi && tf_hi >= 0.0;
}

__device__ __forceinline__ bool lw_pop_keep(double tn, double best) {
  return tn - LW_CULL_M * fabs(tn) <= best + LW_CULL_M * fabs(best);
}

__device__ __forceinline__ void lw_load_node(const RNode* __restrict__ p, double box[12], int ref[2]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < 6; k++) {
    double2 t = q[k];
    box[2 * k] = t.x;
    box[2 * k + 1] = t.y;
  }
  int2 rr = *reinterpret_cast<const int2*>(&p->ref[0]);
  ref[0] = rr.x;
  ref[1] = rr.y;
}

__device__ __forceinline__ void lw_load_tri(const LTri* __restrict__ p, double v[9], long long& id) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    double2 t = q[k];
    v[2 * k] = t.x;
    v[2 * k + 1] = t.y;
  }
  double2 t = q[4];
  v[8] = t.x;
  id = __double_as_longlong(t.y);
}

#define LW_STACK 48

// work counters of the instrumented instantiation (node = one 128-byte node fetch,
// tri = one 80-byte triangle test)
struct LwTraceCount {
  unsigned nodes = 0, tris = 0;
};

// closest hit, t in (0, tmax], near-child-first
template <bool COUNT = false>
__device__ __forceinline__ void lw_trace_closest(const RenderBVH& bvh, const double o[3], const double d[3],
                                                 double tmax, LwHit& h, LwTraceCount* cnt = nullptr) {
  h.t = tmax;
  h.tri = -1;
  h.bu = 0.0;
  h.bv = 0.0;
  if (bvh.ntris == 0) return;
  LwRay r;
  lw_ray_setup(r, o, d);
  double tn;
  if (!lw_box_hit(r, bvh.root_box, h.t, tn)) return;
  int stack_ref[LW_STACK];
  double stack_tn[LW_STACK];
  int sp = 0;
  int ref = bvh.root_ref;
  double best_det = 1.0;
  for (;;) {
    while (ref >= 0 && ref != LW_REF_NONE) {
      double box[12];
      int cr[2];
      lw_load_node(bvh.nodes + ref, box, cr);
      if (COUNT) cnt->nodes++;
      double tn0, tn1;
      bool h0 = lw_box_hit(r, box, h.t, tn0);
      bool h1 = lw_box_hit(r, box + 6, h.t, tn1);
      if (h0 && h1) {
        bool swap = tn1 < tn0;
        stack_ref[sp] = swap ? cr[0] : cr[1];
        stack_tn[sp] = swap ? tn0 : tn1;
        sp++;
        ref = swap ? cr[1] : cr[0];
      } else if (h0) {
        ref = cr[0];
      } else if (h1) {
        ref = cr[1];
      } else {
        ref = LW_REF_NONE;
      }
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        double t, bu, bv, det;
        if (!lw_tri_eval(bvh.tris[k].v, r.sh, t, bu, bv, det) || t <= 0.0 || t > h.t) continue;
        long long id = bvh.tris[k].id;
        if (t == h.t && h.tri >= 0 && id >= h.tri) continue;
        h.t = t;
        h.tri = id;
        h.bu = bu;  // undivided v, w; divided by det once traversal ends
        h.bv = bv;
        best_det = det;
      }
    }
    ref = LW_REF_NONE;
    while (sp > 0) {
      sp--;
      if (lw_pop_keep(stack_tn[sp], h.t)) {
        ref = stack_ref[sp];
        break;
      }
    }
    if (ref == LW_REF_NONE) break;
  }
  if (h.tri >= 0) {
    h.bu = h.bu / best_det;
    h.bv = h.bv / best_det;
  }
}

// any hit with 0 < t < tmax
template <bool COUNT = false>
__device__ __forceinline__ bool lw_trace_any(const RenderBVH& bvh, const double o[3], const double d[3], double tmax,
                                             LwTraceCount* cnt = nullptr) {
  if (bvh.ntris == 0) return false;
  LwRay r;
  lw_ray_setup(r, o, d);
  double tn;
  if (!lw_box_hit(r, bvh.root_box, tmax, tn)) return false;
  int stack_ref[LW_STACK];
  int sp = 0;
  int ref = bvh.root_ref;
  for (;;) {
    while (ref >= 0 && ref != LW_REF_NONE) {
      double box[12];
      int cr[2];
      lw_load_node(bvh.nodes + ref, box, cr);
      if (COUNT) cnt->nodes++;
      double tn0, tn1;
      bool h0 = lw_box_hit(r, box, tmax, tn0);
      bool h1 = lw_box_hit(r, box + 6, tmax, tn1);
      if (h0 && h1) {
        stack_ref[sp++] = cr[1];
        ref = cr[0];
      } else if (h0) {
        ref = cr[0];
      } else if (h1) {
        ref = cr[1];
      } else {
        ref = LW_REF_NONE;
      }
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        if (lw_tri_occludes(bvh.tris[k].v, r.sh, tmax)) return true;
      }
    }
    if (sp == 0) return false;
    ref = stack_ref[--sp];
  }
}
