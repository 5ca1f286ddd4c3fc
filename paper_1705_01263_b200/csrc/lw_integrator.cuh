// lw_integrator.cuh -- path-tracing stages shared by the wavefront engine and the megakernel.
//
// Implements the SPEC-only render path (SPEC.md:366-506 integrator, 309-317/351-355
// materials, 195-230 light/env selection) as defined in DESIGN.md §4, split into the
// wavefront stage functions of SPEC.md:508-567 (generate -> trace -> material/NEE ->
// shadow trace -> accumulate).  Every arithmetic step matches oracle/lw_oracle.c
// (trace_path) in operation order, so a (pixel, iteration) sample produces the same
// bits on the CPU oracle, in the megakernel, and in the wavefront engine.
#pragma once
#include "lw_common.cuh"
#include "lw_detmath.cuh"
#include "lw_envpyr.cuh"
#include "lw_lighttree.cuh"
#include "lw_qmc.cuh"
#include "lw_traverse.cuh"

struct DevScene {
  RenderBVH bvh;
  const double* verts;    // [ntris*9] original triangle order
  const double* normals;  // [ntris*9]
  const int* material;    // [ntris]
  const lw_material* materials;
  const int* emit_of_tri;  // [ntris] emitter index or -1
  long long nemit;
  const long long* emit_tri;
  const double* emit_rad;  // [nemit*3]
  const int* emit_two;
  const double* emit_area;
  const double* emit_prob;
  const double* emit_pdf;
  const int* emit_alias;
  // light hierarchy (light_mode == LW_LIGHTS_TREE)
  LwLightTree lt;
  int lt_nheap;  // heap slots of lt.nodes
  int light_mode;
  // environment pyramid (env_mode == LW_LIGHTS_ENV_PYRAMID)
  LwEnvPyr env_pyr;
  int env_mode;
  int env_kind;
  int env_w, env_h;
  const float* env_img;
  const double* env_prob;   // per texel: Vose table of its row (column | row)
  const double* env_pdf;    // per texel: p(row) * p(column | row)
  const int* env_alias;     // per texel: alias column
  const double* env_rprob;  // per row: Vose table over the row sums
  const int* env_ralias;
  double env_const[3];
  double env_scale;
  double p_env, p_tri;
  double cam_pos[3], cam_fwd[3], cam_right[3], cam_up[3];
  double tan_half;
  int W, H, max_depth, rr_start;
  int estimator;  // LW_EST_* (MIS in the renderer; NEE-only / BSDF-only for estimator-equivalence checks)
  int compact;    // compressed path state: oct-16 ray directions, FP32 throughput,
                  // radiance and pdf, quantised where the state is produced (both engines, the oracle)
  const QmcDim* qdims;
  const uint16_t* qperm;
};

// Scene classes: the shading kernels are compiled per class of the uploaded scene (the
// JIT-compiled material code of PAPER.md:416-418; the layered BSDF itself stays generic, one code
// path for every thread).  Each bit folds a scene-wide property to a constant:
//   LW_MC_DIFFUSE  every material is one uncoated diffuse layer (layer count / kind / coat);
//   LW_MC_NOENV    no environment (env_kind == LW_ENV_NONE);
//   LW_MC_ALIAS    emitters chosen by the alias table (light_mode != LW_LIGHTS_TREE);
//   LW_MC_NOTRI    no emissive triangles (nemit == 0);
//   LW_MC_ENVCONST no image environment (env_kind is constant or none);
//   LW_MC_L2       no material has more than two layers (the layer loops stop at 2).
// The arithmetic executed is the same, so results are identical; the dead code and its registers
// disappear.  0 (LW_MC_ANY) evaluates anything.  (A class for "diffuse + glossy layers only"
// spilled more than LW_MC_ANY and was dropped.)
#define LW_MC_ANY 0
#define LW_MC_DIFFUSE 1
#define LW_MC_NOENV 2
#define LW_MC_ALIAS 4
#define LW_MC_NOTRI 8
#define LW_MC_ENVCONST 16
#define LW_MC_L2 32
// compile-time bound of the layer loops of class MC
template <int MC>
struct LwLayers {
  static constexpr int max = (MC & LW_MC_DIFFUSE) ? 1 : (MC & LW_MC_L2) ? 2 : LW_MAX_LAYERS;
};
template <int MC>
__device__ __forceinline__ int lw_mat_nlayers(const lw_material& m) { return (MC & LW_MC_DIFFUSE) ? 1 : m.nlayers; }
template <int MC>
__device__ __forceinline__ int lw_layer_kind(const lw_layer& L) { return (MC & LW_MC_DIFFUSE) ? LW_BSDF_DIFFUSE : L.kind; }
template <int MC>
__device__ __forceinline__ int lw_env_kind(const DevScene& S) {
  if (MC & LW_MC_NOENV) return LW_ENV_NONE;
  if (MC & LW_MC_ENVCONST) return S.env_kind == LW_ENV_CONSTANT ? LW_ENV_CONSTANT : LW_ENV_NONE;
  return S.env_kind;
}
template <int MC>
__device__ __forceinline__ long long lw_nemit(const DevScene& S) { return (MC & LW_MC_NOTRI) ? 0 : S.nemit; }
template <int MC>
__device__ __forceinline__ int lw_light_mode(const DevScene& S) { return (MC & LW_MC_ALIAS) ? LW_LIGHTS_ALIAS : S.light_mode; }


struct PathState {
  v3 o, d;
  v3 beta, L;
  double pdf_prev;
  long long index;
  int bounce;
  int spec_prev;
  int nprev;  // octahedral-packed facing geometric normal of the previous vertex (light-tree MIS)
  int lpe;    // light-path-expression automaton state (megakernel with layers)
  unsigned doct;  // compact state: octahedral code of d (d == lw_oct_dir(doct))
};

struct ShadowRay {
  v3 o, d;
  double tmax;
  v3 contrib;
  int valid;
  v3 c_diffuse, c_glossy;  // LPE: the contribution's diffuse / glossy parts
  int term;                // LPE: terminal event (LW_EV_L / LW_EV_E)
  int lpe;                 // LPE: automaton state at the NEE vertex
};

// light-path-expression layers (megakernel engine): product DFA + layer framebuffers
struct LwLpe {
  const short* trans;           // [nstates * LW_EV_COUNT]
  const unsigned char* accept;  // [nstates] bit k: layer k accepts
  int start, nlayers;
  unsigned long long* fb;       // [nlayers][npix * 3] int64 fixed point
  long long npix;
};

__device__ __forceinline__ int lw_lpe_step(const LwLpe* lpe, int state, int ev) {
  return lpe->trans[state * LW_EV_COUNT + ev];
}

// add one contribution to every layer accepting `state` (same fixed-point rule as the beauty, per
// contribution: clamp to [0, 2^32], non-finite -> 0, round(v * 2^20))
__device__ __forceinline__ void lw_lpe_route(const LwLpe* lpe, int state, long long pix, v3 c) {
  int m = lpe->accept[state];
  if (!m) return;
  double v[3] = {c.x, c.y, c.z};
  long long q[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    double x = v[k];
    if (!(x == x) || x == INFINITY || x == -INFINITY || x < 0.0) x = 0.0;
    if (x > LW_FB_SAMPLE_CLAMP) x = LW_FB_SAMPLE_CLAMP;
    q[k] = __double2ll_rn(x * 1048576.0);
  }
  for (int l = 0; l < lpe->nlayers; l++) {
    if (!((m >> l) & 1)) continue;
    unsigned long long* f = lpe->fb + (size_t)l * lpe->npix * 3 + 3 * pix;
#pragma unroll
    for (int k = 0; k < 3; k++)
      if (q[k]) atomicAdd(f + k, (unsigned long long)q[k]);
  }
}

__device__ __forceinline__ double lw_qmc_s(const DevScene& S, int dim, long long index) {
  return lw_halton(S.qdims, S.qperm, dim, index);
}

__device__ __forceinline__ v3 lw_ld3(const double* p) { return mk3(p[0], p[1], p[2]); }

// ---- compressed path state (oracle: q32 / dir_q) ----------------------------
// Directions are stored as the 2x16-bit octahedral code of the reference's codec (_kernels.py:
// 233-299) and used as its decoded, normalised vector; throughput, radiance and the BSDF pdf as
// FP32.  Quantisation happens where a value is produced, identically in both engines and the
// oracle, so the compact render is as deterministic (and bit-identical across engines) as the
// FP64 one.
__device__ __forceinline__ double lw_q32(double x) { return (double)__double2float_rn(x); }
__device__ __forceinline__ v3 lw_q32v(v3 a) { return mk3(lw_q32(a.x), lw_q32(a.y), lw_q32(a.z)); }
__device__ __forceinline__ v3 lw_oct_dir(unsigned code) { return normalize3(lw_oct_decode((long long)code)); }

// DESIGN.md §4.1 (oracle camera_ray)
__device__ __forceinline__ void lw_camera_ray(const DevScene& S, long long index, v3& o, v3& d) {
  long long W = S.W, H = S.H, P = W * H;
  long long pix = index % P;
  long long x = pix % W, y = pix / W;
  double dx = lw_gauss_filter_offset(lw_qmc_s(S, 0, index));
  double dy = lw_gauss_filter_offset(lw_qmc_s(S, 1, index));
  double fx = (((double)x + 0.5) + dx) / (double)W;
  double fy = (((double)y + 0.5) + dy) / (double)H;
  double sx = fx * 2.0 - 1.0;
  double sy = 1.0 - fy * 2.0;
  double aspect = (double)W / (double)H;
  double ax = sx * (S.tan_half * aspect);
  double ay = sy * S.tan_half;
  v3 f = lw_ld3(S.cam_fwd), r = lw_ld3(S.cam_right), u = lw_ld3(S.cam_up);
  v3 dd = mk3((f.x + ax * r.x) + ay * u.x, (f.y + ax * r.y) + ay * u.y, (f.z + ax * r.z) + ay * u.z);
  d = normalize3(dd);
  o = lw_ld3(S.cam_pos);
}

__device__ __forceinline__ v3 lw_offset_origin(v3 p, v3 n, v3 dir) {
  double m = fabs(p.x);
  if (fabs(p.y) > m) m = fabs(p.y);
  if (fabs(p.z) > m) m = fabs(p.z);
  if (m < 1.0) m = 1.0;
  double eps = 1e-9 * m;
  double sgn = dot3(n, dir) >= 0.0 ? eps : -eps;
  return mk3(p.x + n.x * sgn, p.y + n.y * sgn, p.z + n.z * sgn);
}

// nprev: packed facing normal of the vertex the ray left (selects the pyramid's top levels)
template <int MC = LW_MC_ANY>
__device__ __forceinline__ v3 lw_env_eval(const DevScene& S, v3 d, int nprev, double& pdf) {
  const int env_kind = lw_env_kind<MC>(S);
  if (env_kind == LW_ENV_CONSTANT) {
    pdf = S.p_env * LW_INV_FOUR_PI;
    return mk3(S.env_const[0] * S.env_scale, S.env_const[1] * S.env_scale, S.env_const[2] * S.env_scale);
  }
  if (env_kind == LW_ENV_IMAGE) {
    double phi = lw_atan2(d.z, d.x);
    if (phi < 0.0) phi = phi + LW_TWO_PI;
    double sin_t = sqrt(d.x * d.x + d.z * d.z);
    double theta = lw_atan2(sin_t, d.y);
    long long W = S.env_w, H = S.env_h;
    long long col = (long long)(phi / LW_TWO_PI * (double)W);
    long long row = (long long)(theta / LW_PI * (double)H);
    if (col >= W) col = W - 1;
    if (row >= H) row = H - 1;
    if (col < 0) col = 0;
    if (row < 0) row = 0;
    long long j = row * W + col;
    double pt = S.env_mode == LW_LIGHTS_ENV_PYRAMID ? lw_ep_pdf(S.env_pyr, lw_ep_bin(nprev), row, col)
                                                     : __ldg(S.env_pdf + j);
    pdf = sin_t > 0.0 ? S.p_env * pt * (double)(W * H) / (LW_TWO_PI_SQ * sin_t) : 0.0;
    const float* px = S.env_img + 3 * j;
    return mk3((double)__ldg(px) * S.env_scale, (double)__ldg(px + 1) * S.env_scale, (double)__ldg(px + 2) * S.env_scale);
  }
  pdf = 0.0;
  return mk3(0.0, 0.0, 0.0);
}

// balance heuristic: weight of the strategy with pdf `a` against the one with `b`
__host__ __device__ __forceinline__ double lw_mis_balance(double a, double b) { return a / (a + b); }

// weight of radiance reached by BSDF sampling after a non-specular vertex (pdf_bsdf) whose
// light-sampling pdf is pdf_light
__device__ __forceinline__ double lw_bsdf_hit_weight(const DevScene& S, double pdf_bsdf, double pdf_light) {
  return S.estimator == LW_EST_MIS ? lw_mis_balance(pdf_bsdf, pdf_light) : (S.estimator == LW_EST_BSDF ? 1.0 : 0.0);
}

// ---- BSDF (oracle: make_frame .. bsdf_sample) --------------------------------------------

struct LwFrame {
  v3 t, b, n;
};

__device__ __forceinline__ LwFrame lw_make_frame(v3 n) {
  LwFrame f;
  double sgn = n.z >= 0.0 ? 1.0 : -1.0;
  double a = -1.0 / (sgn + n.z);
  double b = n.x * n.y * a;
  f.t = mk3(1.0 + sgn * n.x * n.x * a, sgn * b, -sgn * n.x);
  f.b = mk3(b, sgn + n.y * n.y * a, -n.y);
  f.n = n;
  return f;
}
__device__ __forceinline__ v3 lw_to_local(const LwFrame& f, v3 v) { return mk3(dot3(v, f.t), dot3(v, f.b), dot3(v, f.n)); }
__device__ __forceinline__ v3 lw_to_world(const LwFrame& f, v3 v) {
  return mk3((v.x * f.t.x + v.y * f.b.x) + v.z * f.n.x, (v.x * f.t.y + v.y * f.b.y) + v.z * f.n.y,
             (v.x * f.t.z + v.y * f.b.z) + v.z * f.n.z);
}

struct LayerW {
  double a[LW_MAX_LAYERS];
  double sum_a, inv_sum;
  int nonspec;
};

__device__ __forceinline__ double lw_schlick(double cosv, double ior) {
  double r0 = (ior - 1.0) / (ior + 1.0);
  double f0 = r0 * r0;
  double m = 1.0 - cosv;
  double m2 = m * m;
  return f0 + (1.0 - f0) * (m2 * m2 * m);
}

// (the scene class MC and its accessors are defined with DevScene above)
template <int MC>
__device__ __forceinline__ int lw_layer_coat(const lw_layer& L) { return (MC & LW_MC_DIFFUSE) ? 0 : L.coat; }

template <int MC = LW_MC_ANY>
__device__ __forceinline__ void lw_layer_weights(const lw_material& m, double cos_o, LayerW& lw) {
  double r = 1.0;
  lw.sum_a = 0.0;
  lw.nonspec = 0;
#pragma unroll
  for (int l = 0; l < LwLayers<MC>::max; l++) {
    lw.a[l] = 0.0;
    if (l >= lw_mat_nlayers<MC>(m)) continue;
    const lw_layer& L = m.layers[l];
    const int kind = lw_layer_kind<MC>(L);
    double a = lw_layer_coat<MC>(L) ? r * (L.weight * lw_schlick(cos_o, m.ior)) : r * L.weight;
    lw.a[l] = a;
    r = r - a;
    lw.sum_a = lw.sum_a + a;
    if (a > 0.0 && (kind == LW_BSDF_DIFFUSE || kind == LW_BSDF_GLOSSY)) lw.nonspec = 1;
  }
  lw.inv_sum = lw.sum_a > 0.0 ? 1.0 / lw.sum_a : 0.0;
}

__device__ __forceinline__ double lw_ggx_d(double alpha, double cos_h) {
  double a2 = alpha * alpha;
  double t = cos_h * cos_h * (a2 - 1.0) + 1.0;
  return a2 / (LW_PI * (t * t));
}
__device__ __forceinline__ double lw_ggx_g1(double alpha, double cos_v) {
  double a2 = alpha * alpha;
  return 2.0 * cos_v / (cos_v + sqrt(a2 + (1.0 - a2) * (cos_v * cos_v)));
}
__device__ __forceinline__ double lw_alpha_of(const lw_layer& L) {
  double a = L.roughness;
  if (a < 1e-4) a = 1e-4;
  if (a > 1.0) a = 1.0;
  return a;
}

template <int MC = LW_MC_ANY>
__device__ __forceinline__ v3 lw_bsdf_eval(const lw_material& m, const LayerW& lw, v3 wo, v3 wi, double& pdf) {
  v3 f = mk3(0.0, 0.0, 0.0);
  pdf = 0.0;
  if (wi.z <= 0.0 || wo.z <= 0.0 || !(lw.sum_a > 0.0)) return f;
#pragma unroll
  for (int l = 0; l < LwLayers<MC>::max; l++) {
    if (l >= lw_mat_nlayers<MC>(m)) break;
    const lw_layer& L = m.layers[l];
    const int kind = lw_layer_kind<MC>(L);
    double a = lw.a[l];
    if (!(a > 0.0)) continue;
    double sel = a * lw.inv_sum;
    if (kind == LW_BSDF_DIFFUSE) {
      double k = a * LW_INV_PI;
      f = f + mk3(L.tint[0] * k, L.tint[1] * k, L.tint[2] * k);
      pdf = pdf + sel * (wi.z * LW_INV_PI);
    } else if (kind == LW_BSDF_GLOSSY) {
      double al = lw_alpha_of(L);
      v3 h = normalize3(wo + wi);
      double D = lw_ggx_d(al, h.z);
      double G = lw_ggx_g1(al, wo.z) * lw_ggx_g1(al, wi.z);
      double k = a * (D * G / (4.0 * wo.z * wi.z));
      f = f + mk3(L.tint[0] * k, L.tint[1] * k, L.tint[2] * k);
      double oh = dot3(wo, h);
      if (oh > 0.0) pdf = pdf + sel * (D * h.z / (4.0 * oh));
    }
  }
  return f;
}

// the diffuse and glossy parts of lw_bsdf_eval's f (LPE routing of NEE contributions)
template <int MC = LW_MC_ANY>
__device__ __forceinline__ void lw_bsdf_eval_split(const lw_material& m, const LayerW& lw, v3 wo, v3 wi, v3& fd,
                                                   v3& fg) {
  fd = mk3(0.0, 0.0, 0.0);
  fg = mk3(0.0, 0.0, 0.0);
  if (wi.z <= 0.0 || wo.z <= 0.0 || !(lw.sum_a > 0.0)) return;
#pragma unroll
  for (int l = 0; l < LwLayers<MC>::max; l++) {
    if (l >= lw_mat_nlayers<MC>(m)) break;
    const lw_layer& L = m.layers[l];
    const int kind = lw_layer_kind<MC>(L);
    double a = lw.a[l];
    if (!(a > 0.0)) continue;
    if (kind == LW_BSDF_DIFFUSE) {
      double k = a * LW_INV_PI;
      fd = fd + mk3(L.tint[0] * k, L.tint[1] * k, L.tint[2] * k);
    } else if (kind == LW_BSDF_GLOSSY) {
      double al = lw_alpha_of(L);
      v3 h = normalize3(wo + wi);
      double D = lw_ggx_d(al, h.z);
      double G = lw_ggx_g1(al, wo.z) * lw_ggx_g1(al, wi.z);
      double k = a * (D * G / (4.0 * wo.z * wi.z));
      fg = fg + mk3(L.tint[0] * k, L.tint[1] * k, L.tint[2] * k);
    }
  }
}

__device__ __forceinline__ double lw_fresnel_dielectric(double cos_i, double eta) {
  double sin2t = eta * eta * (1.0 - cos_i * cos_i);
  if (sin2t >= 1.0) return 1.0;
  double cos_t = sqrt(1.0 - sin2t);
  double rs = (eta * cos_i - cos_t) / (eta * cos_i + cos_t);
  double rp = (cos_i - eta * cos_t) / (cos_i + eta * cos_t);
  return 0.5 * (rs * rs + rp * rp);
}

struct BSample {
  v3 wi, weight;
  double pdf;
  int delta, transmit;
  int event;  // LPE event of the sampled lobe (LW_EV_RD / RG / RS / TS)
};

template <int MC = LW_MC_ANY>
__device__ __forceinline__ bool lw_bsdf_sample(const lw_material& m, const LayerW& lw, v3 wo, bool front, double u,
                                               double v, BSample& bs) {
  if (!(lw.sum_a > 0.0) || wo.z <= 0.0) return false;
  double x = u * lw.sum_a;
  int pick = -1;
  double cum = 0.0, prev = 0.0, a_pick = 0.0;
  bool done = false;
#pragma unroll
  for (int l = 0; l < LwLayers<MC>::max; l++) {
    if (done || l >= lw_mat_nlayers<MC>(m) || !(lw.a[l] > 0.0)) continue;
    prev = cum;
    cum = cum + lw.a[l];
    pick = l;
    a_pick = lw.a[l];
    if (x < cum) done = true;
  }
  if (pick < 0) return false;
  double ur = (x - prev) / a_pick;
  if (ur < 0.0) ur = 0.0;
  if (ur >= 1.0) ur = 0.9999999999999999;
  const lw_layer& L = m.layers[pick];
  const int kind = lw_layer_kind<MC>(L);
  bs.delta = 0;
  bs.transmit = 0;
  bs.event = kind == LW_BSDF_DIFFUSE ? LW_EV_RD : (kind == LW_BSDF_GLOSSY ? LW_EV_RG : LW_EV_RS);
  if (kind == LW_BSDF_DIFFUSE) {
    double r = sqrt(ur), sp, cp;
    lw_sincos2pi(v, &sp, &cp);
    double z = 1.0 - ur;
    bs.wi = mk3(r * cp, r * sp, sqrt(z > 0.0 ? z : 0.0));
  } else if (kind == LW_BSDF_GLOSSY) {
    double al = lw_alpha_of(L);
    double tan2 = al * al * ur / (1.0 - ur);
    double ch = 1.0 / sqrt(1.0 + tan2);
    double sh2 = 1.0 - ch * ch;
    double sh = sqrt(sh2 > 0.0 ? sh2 : 0.0);
    double sp, cp;
    lw_sincos2pi(v, &sp, &cp);
    v3 h = mk3(sh * cp, sh * sp, ch);
    double oh = dot3(wo, h);
    bs.wi = h * (2.0 * oh) - wo;
  } else if (kind == LW_BSDF_SPECULAR_REFLECT) {
    bs.wi = mk3(-wo.x, -wo.y, wo.z);
    bs.delta = 1;
    bs.weight = mk3(lw.sum_a * L.tint[0], lw.sum_a * L.tint[1], lw.sum_a * L.tint[2]);
    bs.pdf = 0.0;
    return true;
  } else {
    double eta = front ? 1.0 / m.ior : m.ior;
    double F = lw_fresnel_dielectric(wo.z, eta);
    bs.delta = 1;
    bs.pdf = 0.0;
    if (ur < F) {
      bs.wi = mk3(-wo.x, -wo.y, wo.z);
      bs.weight = mk3(lw.sum_a * L.tint[0], lw.sum_a * L.tint[1], lw.sum_a * L.tint[2]);
    } else {
      double sin2t = eta * eta * (1.0 - wo.z * wo.z);
      double cos_t = sqrt(1.0 - sin2t);
      bs.wi = mk3(-eta * wo.x, -eta * wo.y, -cos_t);
      bs.transmit = 1;
      bs.event = LW_EV_TS;
      double k = lw.sum_a * (eta * eta);
      bs.weight = mk3(k * L.tint[0], k * L.tint[1], k * L.tint[2]);
    }
    return true;
  }
  if (bs.wi.z <= 0.0) return false;
  double pdf;
  v3 f = lw_bsdf_eval<MC>(m, lw, wo, bs.wi, pdf);
  if (!(pdf > 0.0)) return false;
  double k = bs.wi.z / pdf;
  bs.weight = mk3(f.x * k, f.y * k, f.z * k);
  bs.pdf = pdf;
  return true;
}

__device__ __forceinline__ long long lw_alias_sample(const double* __restrict__ prob, const int* __restrict__ alias,
                                                     long long n, double u, double& u_out) {
  double x = u * (double)n;
  double fi = floor(x);
  long long i = (long long)fi;
  if (i >= n) i = n - 1;
  double f = x - (double)i;
  double pr = __ldg(prob + i);
  if (f < pr) {
    u_out = f / pr;
    return i;
  }
  u_out = (f - pr) / (1.0 - pr);
  if (u_out >= 1.0) u_out = 0.9999999999999999;
  return __ldg(alias + i);
}

// ---- stages ---------------------------------------------------------------------------

// CMP: compressed path state (S.compact), a compile-time choice of the calling kernel
template <bool CMP = false>
__device__ __forceinline__ void lw_path_init(const DevScene& S, long long index, PathState& ps) {
  lw_camera_ray(S, index, ps.o, ps.d);
  ps.doct = 0;
  if (CMP) {
    ps.doct = (unsigned)lw_oct_encode(ps.d.x, ps.d.y, ps.d.z);
    ps.d = lw_oct_dir(ps.doct);
  }
  ps.beta = mk3(1.0, 1.0, 1.0);
  ps.L = mk3(0.0, 0.0, 0.0);
  ps.pdf_prev = 0.0;
  ps.index = index;
  ps.bounce = 0;
  ps.spec_prev = 1;
  ps.nprev = 0;
  ps.lpe = 0;
}

// reference point and normal of the light-hierarchy estimates at a vertex: the reflection-side
// offset point (the origin of NEE and of reflected continuation rays) and the facing geometric
// normal rounded through the octahedral packing, which is what the next vertex sees for MIS
__device__ __forceinline__ v3 lw_lt_ref_normal(int packed) { return normalize3(lw_oct_decode((long long)packed)); }

// ---- material / NEE stage (oracle trace_path loop body), split into reusable parts ----------
// The megakernel calls lw_path_shade (all parts in order); the wavefront runs lw_shade_nee and
// lw_shade_material as two kernels.  Both orders evaluate the same expressions on the same
// inputs, so results are identical.

struct ShadeGeom {
  v3 p, ng, ngf, wol;
  LwFrame fr;
  bool front;
  const lw_material* m;
  LayerW lw;
};

// hit point, geometric normal, facing (needed for emission)
__device__ __forceinline__ void lw_shade_hit(const DevScene& S, v3 d, const LwHit& h, ShadeGeom& g, double& w) {
  const double* vv = S.verts + 9 * h.tri;
  v3 v0 = lw_ld3(vv), v1 = lw_ld3(vv + 3), v2 = lw_ld3(vv + 6);
  w = (1.0 - h.bu) - h.bv;
  g.p = bary3(v0, v1, v2, w, h.bu, h.bv);
  g.ng = normalize3(cross3(v1 - v0, v2 - v0));
  g.front = dot3(g.ng, d) < 0.0;
}

// shading frame, material and layer weights (vertices with a scattering event)
template <int MC = LW_MC_ANY>
__device__ __forceinline__ void lw_shade_frame(const DevScene& S, v3 d, const LwHit& h, double w, ShadeGeom& g) {
  const double* nn = S.normals + 9 * h.tri;
  v3 ns = bary3(lw_ld3(nn), lw_ld3(nn + 3), lw_ld3(nn + 6), w, h.bu, h.bv);
  double nl = dot3(ns, ns);
  ns = nl > 0.0 ? ns * (1.0 / sqrt(nl)) : g.ng;
  v3 wo = neg3(d);
  g.ngf = g.front ? g.ng : neg3(g.ng);
  if (dot3(ns, g.ngf) < 0.0) ns = neg3(ns);
  if (dot3(ns, wo) <= 0.0) ns = g.ngf;
  g.fr = lw_make_frame(ns);
  g.wol = lw_to_local(g.fr, wo);
  g.m = &S.materials[S.material[h.tri]];  // read in place (no local-memory copy)
  lw_layer_weights<MC>(*g.m, g.wol.z, g.lw);
}

// light half of next-event estimation (SPEC.md:204-230 sample_light / sample_env): from the point p
// with facing geometric normal ngf and the NEE uniforms (ul, vl), choose the environment (p_env) or
// an emitter and a direction wi towards it; Le its radiance, pl the solid-angle pdf of wi (selection
// probabilities included), tmax the shadow-ray length (INFINITY for the environment), e the emitter
// (-1: environment).  Returns false when the sample carries no light (back side, sin(theta) = 0).
template <int MC = LW_MC_ANY>
__device__ __forceinline__ bool lw_nee_light_sample(const DevScene& S, v3 p, v3 ngf, double ul, double vl,
                                                    const LwLightTree* lt, v3& wi, v3& Le, double& pl,
                                                    double& tmax_sh, long long& e_out) {
  wi = mk3(0.0, 0.0, 0.0);
  Le = mk3(0.0, 0.0, 0.0);
  pl = 0.0;
  tmax_sh = INFINITY;
  e_out = -1;
  bool ok = false;
  const int env_kind = lw_env_kind<MC>(S);
  if (env_kind != LW_ENV_NONE && ul < S.p_env) {
    double ue = lw_nemit<MC>(S) > 0 ? ul / S.p_env : ul;
    if (env_kind == LW_ENV_CONSTANT) {
      double z = 1.0 - 2.0 * ue;
      double r2 = 1.0 - z * z;
      double r = sqrt(r2 > 0.0 ? r2 : 0.0), sp, cp;
      lw_sincos2pi(vl, &sp, &cp);
      wi = mk3(r * cp, z, r * sp);
      pl = S.p_env * LW_INV_FOUR_PI;
      Le = mk3(S.env_const[0] * S.env_scale, S.env_const[1] * S.env_scale, S.env_const[2] * S.env_scale);
      ok = true;
    } else {
      double ur, vr, pt;
      long long nt = (long long)S.env_w * S.env_h;
      long long j, row, col;
      if (S.env_mode == LW_LIGHTS_ENV_PYRAMID) {
        lw_ep_sample(S.env_pyr, lw_ep_bin(lw_oct_encode(ngf.x, ngf.y, ngf.z)), ue, vl, row, col, pt, ur, vr);
        j = row * S.env_w + col;
      } else {
        // two-level alias table (built on the GPU at upload): row from the marginal table, column
        // from the row's table with the rescaled remainder of the same uniform
        double u1;
        row = lw_alias_sample(S.env_rprob, S.env_ralias, S.env_h, ue, u1);
        col = lw_alias_sample(S.env_prob + row * S.env_w, S.env_alias + row * S.env_w, S.env_w, u1, ur);
        j = row * S.env_w + col;
        vr = vl;
        pt = __ldg(S.env_pdf + j);
      }
      double uu = ((double)col + ur) / (double)S.env_w;
      double vv2 = ((double)row + vr) / (double)S.env_h;
      double st, ct, sp, cp;
      lw_sincos2pi(vv2 * 0.5, &st, &ct);
      lw_sincos2pi(uu, &sp, &cp);
      wi = mk3(st * cp, ct, st * sp);
      if (st > 0.0) {
        pl = S.p_env * pt * (double)nt / (LW_TWO_PI_SQ * st);
        const float* px = S.env_img + 3 * j;
        Le = mk3((double)__ldg(px) * S.env_scale, (double)__ldg(px + 1) * S.env_scale,
                 (double)__ldg(px + 2) * S.env_scale);
        ok = true;
      }
    }
  } else if (lw_nemit<MC>(S) > 0) {
    double ut = env_kind != LW_ENV_NONE ? (ul - S.p_env) / (1.0 - S.p_env) : ul;
    double ur, psel;
    long long le;
    if (lw_light_mode<MC>(S) == LW_LIGHTS_TREE) {
      v3 xr = lw_offset_origin(p, ngf, ngf);
      v3 nr = lw_lt_ref_normal((int)lw_oct_encode(ngf.x, ngf.y, ngf.z));
      le = lw_lt_sample(lt ? *lt : S.lt, xr, nr, ut, psel, ur);
    } else {
      le = lw_alias_sample(S.emit_prob, S.emit_alias, S.nemit, ut, ur);
      psel = S.emit_pdf[le];
    }
    e_out = le;
    const double* lv = S.verts + 9 * S.emit_tri[le];
    v3 l0 = lw_ld3(lv), l1 = lw_ld3(lv + 3), l2 = lw_ld3(lv + 6);
    double su = sqrt(ur);
    double b0 = 1.0 - su, b1 = vl * su;
    double b2 = (1.0 - b0) - b1;
    v3 q = bary3(l0, l1, l2, b0, b1, b2);
    v3 dl = q - p;
    double dist2 = dot3(dl, dl);
    double dist = sqrt(dist2);
    double inv_dist = 1.0 / dist;
    wi = mk3(dl.x * inv_dist, dl.y * inv_dist, dl.z * inv_dist);
    v3 ngl = normalize3(cross3(l1 - l0, l2 - l0));
    double cos_l = -dot3(ngl, wi);
    if (S.emit_two[le]) cos_l = fabs(cos_l);
    if (cos_l > 0.0 && dist > 0.0) {
      pl = (S.p_tri * psel / S.emit_area[le]) * dist2 / cos_l;
      Le = lw_ld3(S.emit_rad + 3 * le);
      tmax_sh = dist * (1.0 - 1e-7);
      ok = true;
    }
  }
  return ok;
}

// solid-angle light-sampling pdf of emitter e reached by a ray from `o` (leaving a vertex whose
// packed facing normal is nprev) that hits it at distance t with geometric normal ng along d: the
// MIS counterpart of lw_nee_light_sample for BSDF-sampled emitter hits (SPEC.md:213-221 light_pdf)
template <int MC = LW_MC_ANY>
__device__ __forceinline__ double lw_emitter_hit_pdf(const DevScene& S, long long e, v3 o, int nprev, v3 ng, v3 d,
                                                     double t, const LwLightTree* lt) {
  double cos_l = fabs(dot3(ng, d));
  double psel = lw_light_mode<MC>(S) == LW_LIGHTS_TREE ? lw_lt_pdf(lt ? *lt : S.lt, e, o, lw_lt_ref_normal(nprev))
                                               : S.emit_pdf[e];
  double pdf_area = S.p_tri * psel / S.emit_area[e];
  return pdf_area * (t * t) / cos_l;
}

// next-event estimation: fills sh (valid = 0 if no contribution)
// lt: the light hierarchy with its top staged in shared memory (nullptr: S.lt, global memory)
template <int MC = LW_MC_ANY>
__device__ __forceinline__ void lw_shade_nee(const DevScene& S, const PathState& ps, const ShadeGeom& g, ShadowRay& sh,
                                             const LwLpe* lpe = nullptr, const LwLightTree* lt = nullptr) {
  sh.valid = 0;
  const lw_material& m = *g.m;
  const LayerW& lw = g.lw;
  if (!(lw.nonspec && (lw_nemit<MC>(S) > 0 || lw_env_kind<MC>(S) != LW_ENV_NONE)) || S.estimator == LW_EST_BSDF) return;
  const int bd = 4 + 8 * ps.bounce;
  double ul, vl;
  lw_halton2(S.qdims, S.qperm, bd + 2, bd + 3, ps.index, ul, vl);
  v3 wi, Le;
  double pl, tmax_sh;
  long long le;
  bool ok = lw_nee_light_sample<MC>(S, g.p, g.ngf, ul, vl, lt, wi, Le, pl, tmax_sh, le);
  if (ok && pl > 0.0 && dot3(g.ngf, wi) > 0.0) {
    v3 wil = lw_to_local(g.fr, wi);
    double pb;
    v3 f = lw_bsdf_eval<MC>(m, lw, g.wol, wil, pb);
    if (f.x > 0.0 || f.y > 0.0 || f.z > 0.0) {
      double wm = S.estimator == LW_EST_NEE ? 1.0 : lw_mis_balance(pl, pb);
      double k = (wil.z * wm) / pl;
      sh.contrib = mk3(ps.beta.x * f.x * Le.x * k, ps.beta.y * f.y * Le.y * k, ps.beta.z * f.z * Le.z * k);
      sh.o = lw_offset_origin(g.p, g.ngf, wi);
      sh.d = wi;
      sh.tmax = tmax_sh;
      sh.valid = 1;
      if (lpe) {  // the diffuse and glossy parts, routed after the shadow test
        v3 fd, fg;
        lw_bsdf_eval_split<MC>(m, lw, g.wol, wil, fd, fg);
        sh.c_diffuse = mk3(ps.beta.x * fd.x * Le.x * k, ps.beta.y * fd.y * Le.y * k, ps.beta.z * fd.z * Le.z * k);
        sh.c_glossy = mk3(ps.beta.x * fg.x * Le.x * k, ps.beta.y * fg.y * Le.y * k, ps.beta.z * fg.z * Le.z * k);
        sh.term = tmax_sh == INFINITY ? LW_EV_E : LW_EV_L;
        sh.lpe = ps.lpe;
      }
    }
  }
}

// miss / emission part: returns false if the path ends before any scattering
// lpe (megakernel with LPE layers): routes the emission to the layers accepting ... L / ... E
template <bool CMP = false, int MC = LW_MC_ANY>
__device__ __forceinline__ bool lw_shade_emission(const DevScene& S, PathState& ps, const LwHit& h, ShadeGeom& g,
                                                  double& w, const LwLpe* lpe = nullptr, long long pix = 0,
                                                  const LwLightTree* lt = nullptr) {
  v3 d = ps.d;
  if (h.tri < 0) {
    if (lw_env_kind<MC>(S) != LW_ENV_NONE) {
      double pe;
      v3 Le = lw_env_eval<MC>(S, d, ps.nprev, pe);
      double wm = ps.spec_prev ? 1.0 : lw_bsdf_hit_weight(S, ps.pdf_prev, pe);
      v3 c = mk3(ps.beta.x * Le.x * wm, ps.beta.y * Le.y * wm, ps.beta.z * Le.z * wm);
      ps.L = CMP ? lw_q32v(ps.L + c) : ps.L + c;
      if (lpe) lw_lpe_route(lpe, lw_lpe_step(lpe, ps.lpe, LW_EV_E), pix, c);
    }
    return false;
  }
  lw_shade_hit(S, d, h, g, w);
  int e = S.emit_of_tri[h.tri];
  if (e >= 0 && lw_nemit<MC>(S) > 0 && (g.front || S.emit_two[e])) {
    v3 Le = lw_ld3(S.emit_rad + 3 * e);
    double wm = 1.0;
    if (!ps.spec_prev) wm = lw_bsdf_hit_weight(S, ps.pdf_prev, lw_emitter_hit_pdf<MC>(S, e, ps.o, ps.nprev, g.ng, d, h.t, lt));
    v3 c = mk3(ps.beta.x * Le.x * wm, ps.beta.y * Le.y * wm, ps.beta.z * Le.z * wm);
    ps.L = CMP ? lw_q32v(ps.L + c) : ps.L + c;
    if (lpe) lw_lpe_route(lpe, lw_lpe_step(lpe, ps.lpe, LW_EV_L), pix, c);
  }
  return ps.bounce != S.max_depth - 1;
}

// BSDF sampling, Russian roulette and the next ray; returns true if the path continues
template <bool CMP = false, int MC = LW_MC_ANY>
__device__ __forceinline__ bool lw_shade_material(const DevScene& S, PathState& ps, const ShadeGeom& g,
                                                  const LwLpe* lpe = nullptr) {
  const int b = ps.bounce;
  const int bd = 4 + 8 * b;
  BSample bs;
  double ub, vb;
  lw_halton2(S.qdims, S.qperm, bd + 0, bd + 1, ps.index, ub, vb);
  if (!lw_bsdf_sample<MC>(*g.m, g.lw, g.wol, g.front, ub, vb, bs)) return false;
  if (lpe) ps.lpe = lw_lpe_step(lpe, ps.lpe, bs.event);
  v3 wi = lw_to_world(g.fr, bs.wi);
  unsigned code = 0;
  if (CMP) {  // the next ray runs along the stored (quantised) direction
    code = (unsigned)lw_oct_encode(wi.x, wi.y, wi.z);
    wi = lw_oct_dir(code);
  }
  double gside = dot3(g.ngf, wi);
  if (bs.transmit ? !(gside < 0.0) : !(gside > 0.0)) return false;
  ps.beta = mk3(ps.beta.x * bs.weight.x, ps.beta.y * bs.weight.y, ps.beta.z * bs.weight.z);
  ps.spec_prev = bs.delta;
  ps.pdf_prev = CMP ? lw_q32(bs.pdf) : bs.pdf;
  if (b >= S.rr_start) {
    double q = ps.beta.x;
    if (ps.beta.y > q) q = ps.beta.y;
    if (ps.beta.z > q) q = ps.beta.z;
    if (q > 1.0) q = 1.0;
    double ur = lw_qmc_s(S, bd + 4, ps.index);
    if (!(ur < q)) return false;
    double inv_q = 1.0 / q;
    ps.beta = mk3(ps.beta.x * inv_q, ps.beta.y * inv_q, ps.beta.z * inv_q);
  }
  if (CMP) ps.beta = lw_q32v(ps.beta);
  ps.o = lw_offset_origin(g.p, g.ngf, wi);
  ps.d = wi;
  ps.doct = code;
  ps.bounce = b + 1;
  ps.nprev = (int)lw_oct_encode(g.ngf.x, g.ngf.y, g.ngf.z);
  return true;
}

// whole stage in the oracle's order (megakernel): emission, NEE, BSDF sampling
template <bool CMP = false>
__device__ __forceinline__ bool lw_path_shade(const DevScene& S, PathState& ps, const LwHit& h, ShadowRay& sh,
                                              const LwLpe* lpe = nullptr, long long pix = 0) {
  sh.valid = 0;
  ShadeGeom g;
  double w;
  if (!lw_shade_emission<CMP>(S, ps, h, g, w, lpe, pix)) return false;
  lw_shade_frame(S, ps.d, h, w, g);
  lw_shade_nee(S, ps, g, sh, lpe);
  return lw_shade_material<CMP>(S, ps, g, lpe);
}

// fixed-point accumulation (oracle accumulate); returns 1 if a channel was non-finite
__device__ __forceinline__ int lw_accumulate(unsigned long long* fb, long long pix, v3 L) {
  double c[3] = {L.x, L.y, L.z};
  int bad = 0;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    double v = c[k];
    if (!(v == v) || v == INFINITY || v == -INFINITY) {
      bad = 1;
      v = 0.0;
    }
    if (v < 0.0) v = 0.0;
    if (v > LW_FB_SAMPLE_CLAMP) v = LW_FB_SAMPLE_CLAMP;
    long long q = __double2ll_rn(v * 1048576.0);
    if (q) atomicAdd(fb + 3 * pix + k, (unsigned long long)q);
  }
  return bad;
}
