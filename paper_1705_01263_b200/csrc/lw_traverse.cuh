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
//
// 4-wide BVH with FP32 child boxes rounded outward (WNode, one 128-byte line).  The box test
// is conservative by construction: every plane distance is computed from an origin shifted by
// delta_a = 2^-18 (M_a + |o_a|) against the ray (M_a = scene extent on axis a), which exceeds
// the worst-case FP32 rounding of the slab arithmetic (< 2^-22 (M_a + |o_a|) |inv_a|) by 16x,
// so a box is never culled while it can hold a triangle whose FP64 hit t is <= the current
// best.  Triangles are tested in FP64 on the exact vertices with the (t, lower id) rule, so the
// closest hit equals exhaustive search -- the result the oracle's binary FP64 traversal also
// returns -- whatever the tree shape or visit order (tests/test_gpu_render.py checks bits).

#define LW_REF_NONE 0x7fffffff

// 4-wide node: per-axis child bounds as float4 (x = child 0 ... w = child 3), child refs;
// ref >= 0 internal node, < 0 leaf -(1 + (start << 3 | count)), LW_REF_NONE empty slot
struct __align__(128) WNode {
  float4 lo[3];
  float4 hi[3];
  int4 ref;
  int4 pad;
};

// 80-byte leaf-ordered triangle: vertices + original id
struct __align__(16) LTri {
  double v[9];
  long long id;
};

struct RenderBVH {
  const WNode* nodes;
  int nstride;  // bytes between nodes: 128 in global memory, LW_SNODE when staged in shared memory
  const LTri* tris;
  long long ntris;
  int root_ref;
  double root_box[6];
  double absmax[3];  // max |coordinate| of the scene per axis (box-test margin)
};

// per-ray constants of the FP32 box test
struct LwRayF {
  float inv[3];  // clamped reciprocal direction
  float olo[3];  // offset of the lo planes: near-plane offset -(o + delta) * inv when inv >= 0,
  float ohi[3];  // far-plane offset -(o - delta) * inv otherwise (ohi: the other one)
  LwShear sh;
};

__device__ __forceinline__ void lw_rayf_setup(LwRayF& r, const RenderBVH& bvh, const double o[3], const double d[3]) {
  double dmax = fmax(fabs(d[0]), fmax(fabs(d[1]), fabs(d[2])));
  bool ok = dmax >= 0x1p-60 && dmax <= 0x1p60;  // else every box passes (exhaustive, still exact)
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double da = d[a];
    double inv = fabs(da) > dmax * 0x1p-40 ? 1.0 / da : copysign(0x1p40 / dmax, da);
    if (!ok) inv = 0.0;
    float invf = (float)inv;
    bool neg = invf < 0.0f || (invf == 0.0f && signbit(invf));
    double delta = (bvh.absmax[a] + fabs(o[a])) * 0x1p-18;
    double o_n = neg ? o[a] - delta : o[a] + delta;
    double o_f = neg ? o[a] + delta : o[a] - delta;
    float on = (float)(-(o_n * (double)invf)), of = (float)(-(o_f * (double)invf));
    r.inv[a] = invf;
    r.olo[a] = neg ? of : on;
    r.ohi[a] = neg ? on : of;
  }
  lw_shear_setup(o, d, false, r.sh);
}

// slab test of one child from its lo / hi planes.  The near plane's entry distance is the smaller
// of the two (lo * inv + olo <= hi * inv + ohi for inv >= 0 and the reverse for inv < 0, exactly:
// lo <= hi, the offsets are ordered and rounding is monotone), so min / max pick near and far
// without per-ray plane indices (fewer live registers in the node loop).
__device__ __forceinline__ bool lw_slab(const LwRayF& r, float lx, float ly, float lz, float hx, float hy, float hz,
                                        float best, float& tn) {
  float a0 = __fmaf_rn(lx, r.inv[0], r.olo[0]), b0 = __fmaf_rn(hx, r.inv[0], r.ohi[0]);
  float a1 = __fmaf_rn(ly, r.inv[1], r.olo[1]), b1 = __fmaf_rn(hy, r.inv[1], r.ohi[1]);
  float a2 = __fmaf_rn(lz, r.inv[2], r.olo[2]), b2 = __fmaf_rn(hz, r.inv[2], r.ohi[2]);
  float lo = fmaxf(fmaxf(fminf(a0, b0), fminf(a1, b1)), fmaxf(fminf(a2, b2), 0.0f));
  float hi = fminf(fminf(fmaxf(a0, b0), fmaxf(a1, b1)), fminf(fmaxf(a2, b2), best));
  tn = lo;
  return lo <= hi;
}

// tests the four child boxes of a node against [0, best]; returns the hit mask and the entry
// distances (conservative lower bounds)
__device__ __forceinline__ unsigned lw_node_hit(const LwRayF& r, const WNode* __restrict__ nd, float best, float tn[4],
                                                int ref[4]) {
  float4 lx = nd->lo[0], ly = nd->lo[1], lz = nd->lo[2], hx = nd->hi[0], hy = nd->hi[1], hz = nd->hi[2];
  int4 rf = nd->ref;
  ref[0] = rf.x;
  ref[1] = rf.y;
  ref[2] = rf.z;
  ref[3] = rf.w;
  unsigned mask = 0;
  if (lw_slab(r, lx.x, ly.x, lz.x, hx.x, hy.x, hz.x, best, tn[0]) && ref[0] != LW_REF_NONE) mask |= 1u;
  if (lw_slab(r, lx.y, ly.y, lz.y, hx.y, hy.y, hz.y, best, tn[1]) && ref[1] != LW_REF_NONE) mask |= 2u;
  if (lw_slab(r, lx.z, ly.z, lz.z, hx.z, hy.z, hz.z, best, tn[2]) && ref[2] != LW_REF_NONE) mask |= 4u;
  if (lw_slab(r, lx.w, ly.w, lz.w, hx.w, hy.w, hz.w, best, tn[3]) && ref[3] != LW_REF_NONE) mask |= 8u;
  return mask;
}

// 256-bit read-only loads (sm_100 LDG.E.ENL2.256): a 128-byte node in four load instructions
// (3 x 32 B planes + the refs) instead of seven 16-byte ones; the trace kernels are bound by L1TEX
// wavefronts, which scale with load instructions of divergent lanes
__device__ __forceinline__ void lw_ldg256(const void* p, float v[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

__device__ __forceinline__ unsigned lw_node_hit_g(const LwRayF& r, const WNode* __restrict__ nd, float best, float tn[4],
                                                  int ref[4]) {
  float w[24];  // w[4 a + c] = lo[a].c, w[12 + 4 a + c] = hi[a].c
  lw_ldg256(reinterpret_cast<const char*>(nd), w);
  lw_ldg256(reinterpret_cast<const char*>(nd) + 32, w + 8);
  lw_ldg256(reinterpret_cast<const char*>(nd) + 64, w + 16);
  int4 rf = __ldg(&nd->ref);
  ref[0] = rf.x;
  ref[1] = rf.y;
  ref[2] = rf.z;
  ref[3] = rf.w;
  unsigned mask = 0;
#pragma unroll
  for (int c = 0; c < 4; c++)
    if (lw_slab(r, w[c], w[4 + c], w[8 + c], w[12 + c], w[16 + c], w[20 + c], best, tn[c]) && ref[c] != LW_REF_NONE)
      mask |= 1u << c;
  return mask;
}

__device__ __forceinline__ const WNode* lw_node_at(const RenderBVH& bvh, int ref) {
  return reinterpret_cast<const WNode*>(reinterpret_cast<const char*>(bvh.nodes) + (size_t)ref * bvh.nstride);
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

// traversal stack depth (entries); the builder rejects trees whose worst path needs more
#define LW_STACK 64

// work counters of the instrumented instantiation (node = one 128-byte node fetch,
// tri = one 80-byte triangle test)
struct LwTraceCount {
  unsigned nodes = 0, tris = 0, lit = 0;  // lit: shadow rays that reached their light
};

__device__ __forceinline__ unsigned long long lw_stk_pack(int ref, float tn) {
  return ((unsigned long long)__float_as_uint(tn) << 32) | (unsigned)ref;
}

// order the hit children by entry distance (misses last): 5 compare-exchanges
__device__ __forceinline__ void lw_cswap(float& ta, int& ra, float& tb, int& rb) {
  bool s = tb < ta;
  float t = s ? tb : ta;
  tb = s ? ta : tb;
  ta = t;
  int q = s ? rb : ra;
  rb = s ? ra : rb;
  ra = q;
}

// The traversals are flat loops over scalar locals: only the stack is an addressable array.
// (Written as a resumable object with init()/step() the whole object -- ray constants, hit
// record, stack pointer -- lived in local memory and was re-read on every node visit, and a
// dynamically indexed child array forced a local store per node: ~3x the L1TEX requests of the
// node fetches themselves.)  The wavefront engine's persistent lane-refill kernels
// (lw_render.cu k_trace_ext_p / k_trace_shadow_p) run the same loops with a yield after every leaf.

// node placement of the trace: LW_NODES_ANY decides per node fetch (stateless / megakernel paths),
// the wavefront trace kernels are instantiated for one placement so only that path is compiled
#define LW_NODES_ANY 0
#define LW_NODES_GLOBAL 1
#define LW_NODES_SMEM 2
template <int NODES>
__device__ __forceinline__ unsigned lw_node_test(const RenderBVH& bvh, const LwRayF& r, int ref, float best, float tn[4],
                                                 int cr[4]) {
  if (NODES == LW_NODES_GLOBAL) return lw_node_hit_g(r, lw_node_at(bvh, ref), best, tn, cr);
  if (NODES == LW_NODES_SMEM) return lw_node_hit(r, lw_node_at(bvh, ref), best, tn, cr);
  return bvh.nstride == (int)sizeof(WNode) ? lw_node_hit_g(r, lw_node_at(bvh, ref), best, tn, cr)
                                           : lw_node_hit(r, lw_node_at(bvh, ref), best, tn, cr);
}

// the single hit child of mask m (no dynamic register-array index)
__device__ __forceinline__ int lw_pick(unsigned m, const int cr[4]) {
  return (m & 1u) ? cr[0] : (m & 2u) ? cr[1] : (m & 4u) ? cr[2] : cr[3];
}

// next stack entry whose entry distance is within the current best (LW_REF_NONE when exhausted)
__device__ __forceinline__ int lw_pop_cull(const unsigned long long* stk, int& sp, float best) {
  while (sp > 0) {
    unsigned long long e = stk[--sp];
    if (__uint_as_float((unsigned)(e >> 32)) <= best) return (int)(unsigned)e;
  }
  return LW_REF_NONE;
}

// closest hit, t in (0, tmax], nearest child first
// SPEC: speculative traversal (Aila & Laine 2009) -- a lane that reaches a leaf postpones it and
// keeps descending until every active lane of the warp holds a leaf; same hit, fuller warps.
template <bool COUNT = false, int NODES = LW_NODES_ANY, bool SPEC = false>
__device__ __forceinline__ void lw_trace_closest(const RenderBVH& bvh, const double o[3], const double d[3],
                                                 double tmax, LwHit& h, LwTraceCount* cnt = nullptr) {
  LwRayF r;
  lw_rayf_setup(r, bvh, o, d);
  double ht = tmax, hu = 0.0, hv = 0.0, best_det = 1.0;
  long long htri = -1;
  float best = __double2float_ru(tmax);
  int ref = bvh.ntris == 0 ? LW_REF_NONE : bvh.root_ref;
  int sp = 0;
  unsigned long long stk[LW_STACK];
  if (SPEC) {
    while (ref != LW_REF_NONE) {
      int leaf = LW_REF_NONE;
      if (ref < 0) {
        leaf = ref;
        ref = lw_pop_cull(stk, sp, best);
      }
      while (ref >= 0 && ref != LW_REF_NONE) {
        float tn[4];
        int cr[4];
        unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
        if (COUNT) cnt->nodes++;
        int nh = __popc(m);
        if (nh <= 1) {
          ref = nh == 0 ? lw_pop_cull(stk, sp, best) : lw_pick(m, cr);
        } else {
#pragma unroll
          for (int c = 0; c < 4; c++)
            if (!(m & (1u << c))) tn[c] = INFINITY;
          lw_cswap(tn[0], cr[0], tn[1], cr[1]);
          lw_cswap(tn[2], cr[2], tn[3], cr[3]);
          lw_cswap(tn[0], cr[0], tn[2], cr[2]);
          lw_cswap(tn[1], cr[1], tn[3], cr[3]);
          lw_cswap(tn[1], cr[1], tn[2], cr[2]);
          if (nh > 3) stk[sp++] = lw_stk_pack(cr[3], tn[3]);
          if (nh > 2) stk[sp++] = lw_stk_pack(cr[2], tn[2]);
          stk[sp++] = lw_stk_pack(cr[1], tn[1]);
          ref = cr[0];
        }
        if (ref < 0 && leaf == LW_REF_NONE) {
          leaf = ref;
          ref = lw_pop_cull(stk, sp, best);
        }
        if (!__any_sync(__activemask(), leaf == LW_REF_NONE)) break;
      }
      if (leaf == LW_REF_NONE && ref < 0) {
        leaf = ref;
        ref = lw_pop_cull(stk, sp, best);
      }
      if (leaf == LW_REF_NONE) continue;
      int v = -leaf - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        double t, bu, bv, det;
        if (!lw_tri_eval(bvh.tris[k].v, r.sh, t, bu, bv, det) || t <= 0.0 || t > ht) continue;
        long long id = bvh.tris[k].id;
        if (t == ht && htri >= 0 && id >= htri) continue;
        ht = t;
        htri = id;
        hu = bu;
        hv = bv;
        best_det = det;
        best = __double2float_ru(t);
      }
    }
  }
  while (!SPEC && ref != LW_REF_NONE) {
    while (ref >= 0) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) cnt->nodes++;
      int nh = __popc(m);
      if (nh <= 1) {
        ref = nh == 0 ? LW_REF_NONE : lw_pick(m, cr);
        if (nh == 0) break;
        continue;
      }
#pragma unroll
      for (int c = 0; c < 4; c++)
        if (!(m & (1u << c))) tn[c] = INFINITY;
      lw_cswap(tn[0], cr[0], tn[1], cr[1]);
      lw_cswap(tn[2], cr[2], tn[3], cr[3]);
      lw_cswap(tn[0], cr[0], tn[2], cr[2]);
      lw_cswap(tn[1], cr[1], tn[3], cr[3]);
      lw_cswap(tn[1], cr[1], tn[2], cr[2]);
      if (nh > 3) stk[sp++] = lw_stk_pack(cr[3], tn[3]);
      if (nh > 2) stk[sp++] = lw_stk_pack(cr[2], tn[2]);
      stk[sp++] = lw_stk_pack(cr[1], tn[1]);
      ref = cr[0];
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        double t, bu, bv, det;
        if (!lw_tri_eval(bvh.tris[k].v, r.sh, t, bu, bv, det) || t <= 0.0 || t > ht) continue;
        long long id = bvh.tris[k].id;
        if (t == ht && htri >= 0 && id >= htri) continue;
        ht = t;
        htri = id;
        hu = bu;  // undivided v, w; divided by det once the hit is final
        hv = bv;
        best_det = det;
        best = __double2float_ru(t);
      }
    }
    ref = LW_REF_NONE;
    while (sp > 0) {
      unsigned long long e = stk[--sp];
      if (__uint_as_float((unsigned)(e >> 32)) <= best) {
        ref = (int)(unsigned)e;
        break;
      }
    }
  }
  h.t = ht;
  h.tri = htri;
  h.bu = htri >= 0 ? hu / best_det : 0.0;
  h.bv = htri >= 0 ? hv / best_det : 0.0;
}

// any hit with 0 < t < tmax
template <bool COUNT = false, int NODES = LW_NODES_ANY, bool SPEC = false>
__device__ __forceinline__ bool lw_trace_any(const RenderBVH& bvh, const double o[3], const double d[3], double tmax,
                                             LwTraceCount* cnt = nullptr) {
  LwRayF r;
  lw_rayf_setup(r, bvh, o, d);
  float best = __double2float_ru(tmax);
  int ref = bvh.ntris == 0 ? LW_REF_NONE : bvh.root_ref;
  int sp = 0;
  int stk[LW_STACK];
  if (SPEC) {
    while (ref != LW_REF_NONE) {
      int leaf = LW_REF_NONE;
      if (ref < 0) {
        leaf = ref;
        ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
      }
      while (ref >= 0 && ref != LW_REF_NONE) {
        float tn[4];
        int cr[4];
        unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
        if (COUNT) cnt->nodes++;
        if (m == 0) {
          ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
        } else {
          ref = lw_pick(m, cr);
          m &= m - 1;
#pragma unroll
          for (int c = 1; c < 4; c++)
            if (m & (1u << c)) stk[sp++] = cr[c];
        }
        if (ref < 0 && leaf == LW_REF_NONE) {
          leaf = ref;
          ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
        }
        if (!__any_sync(__activemask(), leaf == LW_REF_NONE)) break;
      }
      if (leaf == LW_REF_NONE && ref < 0) {
        leaf = ref;
        ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
      }
      if (leaf == LW_REF_NONE) continue;
      int v = -leaf - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        if (lw_tri_occludes(bvh.tris[k].v, r.sh, tmax)) return true;
      }
    }
    return false;
  }
  while (ref != LW_REF_NONE) {
    while (ref >= 0) {
      float tn[4];
      int cr[4];
      unsigned m = lw_node_test<NODES>(bvh, r, ref, best, tn, cr);
      if (COUNT) cnt->nodes++;
      if (m == 0) {
        ref = LW_REF_NONE;
        break;
      }
      ref = lw_pick(m, cr);
      m &= m - 1;
#pragma unroll
      for (int c = 1; c < 4; c++)
        if (m & (1u << c)) stk[sp++] = cr[c];
    }
    if (ref != LW_REF_NONE) {
      int v = -ref - 1;
      int start = v >> 3, count = v & 7;
      for (int k = start; k < start + count; k++) {
        if (COUNT) cnt->tris++;
        if (lw_tri_occludes(bvh.tris[k].v, r.sh, tmax)) return true;
      }
    }
    ref = sp > 0 ? stk[--sp] : LW_REF_NONE;
  }
  return false;
}
