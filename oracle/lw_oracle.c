/*
 * lw_oracle.c -- CPU restatement oracle (TEST INFRASTRUCTURE ONLY; see lw_oracle.h).
 *
 * Compile with -ffp-contract=off: every expression below is evaluated as written
 * in IEEE binary64 with round-to-nearest, like the reference's Cython output
 * (which contains no FMA) and like the device code (built with -fmad=false).
 * libm `log` is called directly in the pixel filter exactly as the reference does.
 */
#include "lw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ========================================================================== */
/* QMC: scrambled radical inverse, _kernels.py:160-208                        */
/* ========================================================================== */

/* radical_inverse_scrambled, _kernels.py:160-178 (cdivision=False; index > 0 loop) */
static double ri_scrambled(int64_t base, const int64_t* perm, int64_t perm_off, int64_t index) {
  double rev = 0.0, scale = 1.0, b = (double)base;
  while (index > 0) {
    int64_t digit = index % base;
    index = index / base;
    rev = rev * b + (double)perm[perm_off + digit];
    scale = scale * b;
  }
  return rev / scale;
}

/* radical_inverse_base2, _kernels.py:181-192 */
static double ri_base2(int64_t index) {
  double rev = 0.0, scale = 1.0;
  while (index > 0) {
    rev = rev * 2.0 + (double)(index & 1);
    scale = scale * 2.0;
    index = index >> 1;
  }
  return rev / scale;
}

/* halton_dim, _kernels.py:195-208 */
double lwo_halton_dim(const int64_t* bases, const int64_t* perm_flat, const int64_t* perm_offset, int64_t dim,
                      int64_t index) {
  int64_t b = bases[dim];
  if (b == 2) return ri_base2(index);
  return ri_scrambled(b, perm_flat, perm_offset[dim], index);
}

/* halton_batch, _kernels.py:211-222 */
void lwo_halton_batch(const int64_t* bases, const int64_t* perm_flat, const int64_t* perm_offset, int64_t dim,
                      const int64_t* indices, int64_t n, double* out) {
  for (int64_t i = 0; i < n; i++) out[i] = lwo_halton_dim(bases, perm_flat, perm_offset, dim, indices[i]);
}

/* ========================================================================== */
/* Pixel filter, _kernels.py:82-134                                           */
/* ========================================================================== */

/* Acklam inverse normal CDF, _kernels.py:87-109 (libm log + sqrt in the tails) */
static double norm_inv_cdf(double p) {
  double q, r;
  if (p <= 0.0) return -38.0;
  if (p >= 1.0) return 38.0;
  if (p < 0.02425) {
    q = sqrt(-2.0 * log(p));
    return (((((-7.784894002430293e-03 * q - 3.223964580411365e-01) * q - 2.400758277161838e00) * q -
              2.549732539343734e00) * q + 4.374664141464968e00) * q + 2.938163982698783e00) /
           ((((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e00) * q +
             3.754408661907416e00) * q + 1.0);
  }
  if (p > 1.0 - 0.02425) {
    q = sqrt(-2.0 * log(1.0 - p));
    return -(((((-7.784894002430293e-03 * q - 3.223964580411365e-01) * q - 2.400758277161838e00) * q -
               2.549732539343734e00) * q + 4.374664141464968e00) * q + 2.938163982698783e00) /
           ((((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e00) * q +
             3.754408661907416e00) * q + 1.0);
  }
  q = p - 0.5;
  r = q * q;
  return (((((-3.969683028665376e01 * r + 2.209460984245205e02) * r - 2.759285104469687e02) * r +
            1.383577518672690e02) * r - 3.066479806614716e01) * r + 2.506628277459239e00) * q /
         (((((-5.447609879822406e01 * r + 1.615858368580409e02) * r - 1.556989798598866e02) * r +
            6.680131188771972e01) * r - 1.328068155288572e01) * r + 1.0);
}

#define PHI_NEG3 0.0013498980316300933 /* _kernels.py:114 */
#define PHI_POS3 0.9986501019683699    /* _kernels.py:115 */

/* gauss_filter_offset, _kernels.py:121-129 */
double lwo_gauss_filter_offset(double u) {
  double p = PHI_NEG3 + u * (PHI_POS3 - PHI_NEG3);
  double x = norm_inv_cdf(p);
  if (x < -3.0) x = -3.0;
  if (x > 3.0) x = 3.0;
  return 0.5 * x;
}

void lwo_pixel_offset_batch(const double* u, int64_t n, double* out) {
  for (int64_t i = 0; i < 2 * n; i++) out[i] = lwo_gauss_filter_offset(u[i]);
}

/* ========================================================================== */
/* Octahedral compression, _kernels.py:233-342                                */
/* ========================================================================== */

int64_t lwo_oct_encode(double x, double y, double z) {
  double ax = fabs(x), ay = fabs(y), az = fabs(z);
  double norm = ax + ay + az;
  if (norm <= 0.0) return 0;
  double u = x / norm, v = y / norm;
  if (z < 0.0) {
    double fu = (1.0 - fabs(v)) * (u >= 0.0 ? 1.0 : -1.0);
    double fv = (1.0 - fabs(u)) * (v >= 0.0 ? 1.0 : -1.0);
    u = fu;
    v = fv;
  }
  int64_t eu = (int64_t)floor((u + 1.0) * 0.5 * 65535.0 + 0.5);
  int64_t ev = (int64_t)floor((v + 1.0) * 0.5 * 65535.0 + 0.5);
  if (eu < 0) eu = 0;
  if (eu > 65535) eu = 65535;
  if (ev < 0) ev = 0;
  if (ev > 65535) ev = 65535;
  return (eu << 16) | ev;
}

void lwo_oct_decode(int64_t packed, double* o) {
  int64_t eu = (packed >> 16) & 0xFFFF, ev = packed & 0xFFFF;
  double u = (double)eu / 65535.0 * 2.0 - 1.0;
  double v = (double)ev / 65535.0 * 2.0 - 1.0;
  double z = 1.0 - fabs(u) - fabs(v);
  double x = u, y = v;
  if (z < 0.0) {
    x = (1.0 - fabs(v)) * (u >= 0.0 ? 1.0 : -1.0);
    y = (1.0 - fabs(u)) * (v >= 0.0 ? 1.0 : -1.0);
  }
  o[0] = x;
  o[1] = y;
  o[2] = z;
}

/* oct_roundtrip_batch, _kernels.py:321-342 (rows with zero length are left untouched) */
void lwo_oct_roundtrip_batch(const double* vecs, int64_t n, double* out) {
  for (int64_t i = 0; i < n; i++) {
    double d[3];
    lwo_oct_decode(lwo_oct_encode(vecs[3 * i], vecs[3 * i + 1], vecs[3 * i + 2]), d);
    double ln = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (ln > 0.0) {
      out[3 * i] = d[0] / ln;
      out[3 * i + 1] = d[1] / ln;
      out[3 * i + 2] = d[2] / ln;
    }
  }
}

/* ========================================================================== */
/* Watertight triangle test and BVH traversal, _kernels.py:345-585            */
/* ========================================================================== */

typedef struct {
  double t, bu, bv;
  int64_t tri;
} hitrec;

typedef struct {
  int kx, ky, kz;
  double sx, sy, sz;
  double o[3];  /* original origin */
  double op[3]; /* origin passed to the triangle test: unpermuted (D1) or permuted */
} shear;

/* _kernels.py:439-477 */
static void shear_setup(const double* o, const double* d, int compat, shear* s) {
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
  if (d[kz] < 0.0) {
    int t = kx;
    kx = ky;
    ky = t;
  }
  s->kx = kx;
  s->ky = ky;
  s->kz = kz;
  s->sz = 1.0 / d[kz];
  s->sx = d[kx] * s->sz;
  s->sy = d[ky] * s->sz;
  for (int a = 0; a < 3; a++) s->o[a] = o[a];
  if (compat) { /* D1: _tri_hit receives (ox, oy, oz) and subtracts them from permuted components */
    s->op[0] = o[0];
    s->op[1] = o[1];
    s->op[2] = o[2];
  } else {
    s->op[0] = o[kx];
    s->op[1] = o[ky];
    s->op[2] = o[kz];
  }
}

/* _tri_hit, _kernels.py:368-416.  accept_tie: closest-hit tie rule; returns 1 on update. */
static int tri_test(const double* v, int64_t tri, const shear* s, double tmin, hitrec* r) {
  double ax = v[0 + s->kx] - s->op[0], ay = v[0 + s->ky] - s->op[1], az = v[0 + s->kz] - s->op[2];
  double bx = v[3 + s->kx] - s->op[0], by = v[3 + s->ky] - s->op[1], bz = v[3 + s->kz] - s->op[2];
  double cx = v[6 + s->kx] - s->op[0], cy = v[6 + s->ky] - s->op[1], cz = v[6 + s->kz] - s->op[2];
  double sax = ax - s->sx * az, say = ay - s->sy * az;
  double sbx = bx - s->sx * bz, sby = by - s->sy * bz;
  double scx = cx - s->sx * cz, scy = cy - s->sy * cz;
  double u = scx * sby - scy * sbx;
  double vv = sax * scy - say * scx;
  double w = sbx * say - sby * sax;
  if ((u < 0.0 || vv < 0.0 || w < 0.0) && (u > 0.0 || vv > 0.0 || w > 0.0)) return 0;
  double det = u + vv + w;
  if (det == 0.0) return 0;
  double t_scaled = u * (s->sz * az) + vv * (s->sz * bz) + w * (s->sz * cz);
  double t = t_scaled / det;
  if (t <= tmin) return 0;
  if (t > r->t) return 0;
  if (t == r->t && r->tri >= 0 && tri >= r->tri) return 0;
  r->t = t;
  r->tri = tri;
  r->bu = vv / det;
  r->bv = w / det;
  return 1;
}

/* any-hit variant: strict tmin < t < tmax */
static int tri_occludes(const double* v, const shear* s, double tmax) {
  double ax = v[0 + s->kx] - s->op[0], ay = v[0 + s->ky] - s->op[1], az = v[0 + s->kz] - s->op[2];
  double bx = v[3 + s->kx] - s->op[0], by = v[3 + s->ky] - s->op[1], bz = v[3 + s->kz] - s->op[2];
  double cx = v[6 + s->kx] - s->op[0], cy = v[6 + s->ky] - s->op[1], cz = v[6 + s->kz] - s->op[2];
  double sax = ax - s->sx * az, say = ay - s->sy * az;
  double sbx = bx - s->sx * bz, sby = by - s->sy * bz;
  double scx = cx - s->sx * cz, scy = cy - s->sy * cz;
  double u = scx * sby - scy * sbx;
  double vv = sax * scy - say * scx;
  double w = sbx * say - sby * sax;
  if ((u < 0.0 || vv < 0.0 || w < 0.0) && (u > 0.0 || vv > 0.0 || w > 0.0)) return 0;
  double det = u + vv + w;
  if (det == 0.0) return 0;
  double t_scaled = u * (s->sz * az) + vv * (s->sz * bz) + w * (s->sz * cz);
  double t = t_scaled / det;
  return t > 0.0 && t < tmax;
}

/* _safe_inv, _kernels.py:357-362 */
static double safe_inv(double d) {
  if (d > 1e-200 || d < -1e-200) return 1.0 / d;
  if (d >= 0.0) return 1e200;
  return -1e200;
}

/* _traverse_closest, _kernels.py:422-545 (compat = pristine; otherwise D1/D2 corrected) */
static void traverse_ref(int compat, const double* bounds, const int64_t* children, const int64_t* order,
                         const double* verts, int64_t ntris, const double* o, const double* d, double tmin,
                         double tmax, hitrec* r, int64_t* stack) {
  r->t = tmax;
  r->tri = -1;
  r->bu = 0.0;
  r->bv = 0.0;
  if (ntris == 0) return;
  shear s;
  shear_setup(o, d, compat, &s);
  double inv[3] = {safe_inv(d[0]), safe_inv(d[1]), safe_inv(d[2])};
  int zero[3];
  for (int a = 0; a < 3; a++) zero[a] = !compat && (inv[a] == 1e200 || inv[a] == -1e200);
  int64_t sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    int64_t node = stack[--sp];
    const double* b = bounds + 6 * node;
    double tn = -INFINITY, tf = INFINITY;
    int culled = 0;
    for (int a = 0; a < 3; a++) {
      if (zero[a]) { /* D2 fix: a ray parallel to the slab is inside it or misses */
        if (o[a] < b[a] || o[a] > b[3 + a]) culled = 1;
        continue;
      }
      double t0 = (b[a] - o[a]) * inv[a];
      double t1 = (b[3 + a] - o[a]) * inv[a];
      if (compat && a == 0) { /* _kernels.py:500-507 */
        if (t0 > t1) {
          tn = t1;
          tf = t0;
        } else {
          tn = t0;
          tf = t1;
        }
        continue;
      }
      if (t0 > t1) { /* _kernels.py:510-531 */
        if (t0 < tf) tf = t0;
        if (t1 > tn) tn = t1;
      } else {
        if (t1 < tf) tf = t1;
        if (t0 > tn) tn = t0;
      }
    }
    if (culled) continue;
    if (tn > tf || tn > r->t || tf < tmin) continue; /* _kernels.py:532 */
    int64_t c0 = children[2 * node], c1 = children[2 * node + 1];
    if (c0 < 0) {
      int64_t start = -(c0 + 1);
      for (int64_t i = 0; i < c1; i++) {
        int64_t tri = order[start + i];
        tri_test(verts + 9 * tri, tri, &s, tmin, r);
      }
    } else {
      stack[sp++] = c0;
      stack[sp++] = c1;
    }
  }
}

void lwo_intersect_batch(int mode, const double* bounds, const int64_t* children, const int64_t* order,
                         const double* verts, int64_t ntris, const double* origins, const double* dirs,
                         const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri, double* out_bary) {
  int64_t stack[256];
  for (int64_t i = 0; i < n; i++) {
    hitrec r;
    const double* o = origins + 3 * i;
    const double* d = dirs + 3 * i;
    if (mode == LW_TRAVERSE_BRUTE) {
      r.t = tmaxs[i];
      r.tri = -1;
      r.bu = r.bv = 0.0;
      shear s;
      shear_setup(o, d, 0, &s);
      for (int64_t k = 0; k < ntris; k++) tri_test(verts + 9 * k, k, &s, 0.0, &r);
    } else {
      traverse_ref(mode == LW_TRAVERSE_COMPAT, bounds, children, order, verts, ntris, o, d, 0.0, tmaxs[i], &r,
                   stack);
    }
    if (r.tri >= 0) { /* _kernels.py:576-585 */
      out_t[i] = r.t;
      out_tri[i] = r.tri;
      out_bary[2 * i] = r.bu;
      out_bary[2 * i + 1] = r.bv;
    } else {
      out_t[i] = 1e308;
      out_tri[i] = -1;
      out_bary[2 * i] = 0.0;
      out_bary[2 * i + 1] = 0.0;
    }
  }
}

/* ========================================================================== */
/* BVH build, geometry.py:100-148                                             */
/* ========================================================================== */

typedef struct {
  const double* tri_min;
  const double* tri_max;
  const double* centroid;
  double* bounds;
  int64_t* children;
  int64_t* order;
  int64_t nnodes;
  int64_t norder;
} bvh_build_ctx;

static const double* g_sort_keys; /* centroid column for the comparator (oracle is single-threaded here) */
static int g_sort_axis;

/* np.lexsort((idx, centroid[idx, axis])): primary centroid, secondary triangle index */
static int cmp_centroid(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  double ka = g_sort_keys[3 * a + g_sort_axis], kb = g_sort_keys[3 * b + g_sort_axis];
  if (ka < kb) return -1;
  if (ka > kb) return 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* emit(), geometry.py:116-134 */
static int64_t bvh_emit(bvh_build_ctx* c, int64_t* idx, int64_t n) {
  int64_t node = c->nnodes++;
  double bmin[3], bmax[3];
  for (int a = 0; a < 3; a++) {
    bmin[a] = c->tri_min[3 * idx[0] + a];
    bmax[a] = c->tri_max[3 * idx[0] + a];
  }
  for (int64_t i = 1; i < n; i++)
    for (int a = 0; a < 3; a++) {
      double lo = c->tri_min[3 * idx[i] + a], hi = c->tri_max[3 * idx[i] + a];
      if (lo < bmin[a]) bmin[a] = lo;
      if (hi > bmax[a]) bmax[a] = hi;
    }
  for (int a = 0; a < 3; a++) {
    c->bounds[6 * node + a] = bmin[a];
    c->bounds[6 * node + 3 + a] = bmax[a];
  }
  if (n <= 4) { /* LEAF_SIZE, geometry.py:20, 122-125 */
    c->children[2 * node] = -(c->norder + 1);
    c->children[2 * node + 1] = n;
    for (int64_t i = 0; i < n; i++) c->order[c->norder++] = idx[i];
    return node;
  }
  int axis = 0; /* np.argmax: first maximum */
  double ext0 = bmax[0] - bmin[0], ext1 = bmax[1] - bmin[1], ext2 = bmax[2] - bmin[2];
  if (ext1 > ext0) axis = 1;
  if (ext2 > (axis == 1 ? ext1 : ext0)) axis = 2;
  g_sort_keys = c->centroid;
  g_sort_axis = axis;
  qsort(idx, (size_t)n, sizeof(int64_t), cmp_centroid);
  int64_t half = n / 2;
  int64_t left = bvh_emit(c, idx, half);
  int64_t right = bvh_emit(c, idx + half, n - half);
  c->children[2 * node] = left;
  c->children[2 * node + 1] = right;
  return node;
}

int64_t lwo_build_bvh(const double* verts, int64_t n, double* bounds, int64_t* children, int64_t* order) {
  if (n == 0) { /* geometry.py:103-106 */
    for (int a = 0; a < 6; a++) bounds[a] = 0.0;
    children[0] = -1;
    children[1] = 0;
    return 1;
  }
  double* tmin = (double*)malloc(sizeof(double) * 3 * n);
  double* tmax = (double*)malloc(sizeof(double) * 3 * n);
  double* cen = (double*)malloc(sizeof(double) * 3 * n);
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; i++) {
    const double* v = verts + 9 * i;
    for (int a = 0; a < 3; a++) {
      double lo = v[a], hi = v[a];
      if (v[3 + a] < lo) lo = v[3 + a];
      if (v[6 + a] < lo) lo = v[6 + a];
      if (v[3 + a] > hi) hi = v[3 + a];
      if (v[6 + a] > hi) hi = v[6 + a];
      tmin[3 * i + a] = lo;
      tmax[3 * i + a] = hi;
      cen[3 * i + a] = 0.5 * (lo + hi);
    }
    idx[i] = i;
  }
  bvh_build_ctx c = {tmin, tmax, cen, bounds, children, order, 0, 0};
  bvh_emit(&c, idx, n);
  free(tmin);
  free(tmax);
  free(cen);
  free(idx);
  return c.nnodes;
}

/* ========================================================================== */
/* Deterministic math (basic IEEE ops only; restated in lw_detmath.cuh)       */
/* ========================================================================== */

#define LW_PI 3.141592653589793
#define LW_TWO_PI 6.283185307179586
#define LW_HALF_PI 1.5707963267948966
#define LW_QUARTER_PI 0.7853981633974483
#define LW_INV_PI 0.3183098861837907
#define LW_INV_FOUR_PI 0.07957747154594767
#define LW_TWO_PI_SQ 19.739208802178716

/* sin(2*pi*u), cos(2*pi*u): quadrant reduction, Taylor series on [-pi/4, pi/4] */
void lwo_sincos2pi(double u, double* s, double* c) {
  double k = floor(u * 4.0 + 0.5);
  double r = u - k * 0.25;
  double x = r * LW_TWO_PI;
  double x2 = x * x;
  double sp = x * (1.0 + x2 * (-1.6666666666666666e-01 + x2 * (8.3333333333333332e-03 + x2 * (-1.9841269841269841e-04 +
             x2 * (2.7557319223985893e-06 + x2 * (-2.5052108385441720e-08 + x2 * (1.6059043836821613e-10 +
             x2 * (-7.6471637318198164e-13 + x2 * 2.8114572543455206e-15))))))));
  double cp = 1.0 + x2 * (-0.5 + x2 * (4.1666666666666664e-02 + x2 * (-1.3888888888888889e-03 + x2 * (2.4801587301587302e-05 +
             x2 * (-2.7557319223985888e-07 + x2 * (2.0876756987868100e-09 + x2 * (-1.1470745597729725e-11 +
             x2 * 4.7794773323873853e-14)))))));
  int q = ((int)k) & 3;
  if (q == 0) {
    *s = sp;
    *c = cp;
  } else if (q == 1) {
    *s = cp;
    *c = -sp;
  } else if (q == 2) {
    *s = -sp;
    *c = -cp;
  } else {
    *s = -cp;
    *c = sp;
  }
}

/* atan for t in [0, 1]: two argument halvings (tan(a/4) <= tan(pi/16)), then the odd Taylor series */
static const double ATAN_C[12] = {1.0, -1.0 / 3.0, 1.0 / 5.0, -1.0 / 7.0, 1.0 / 9.0, -1.0 / 11.0,
                                  1.0 / 13.0, -1.0 / 15.0, 1.0 / 17.0, -1.0 / 19.0, 1.0 / 21.0, -1.0 / 23.0};
static double det_atan01(double t) {
  double h = t / (1.0 + sqrt(1.0 + t * t));
  h = h / (1.0 + sqrt(1.0 + h * h));
  double h2 = h * h;
  double p = ATAN_C[11];
  for (int k = 10; k >= 0; k--) p = p * h2 + ATAN_C[k];
  return 4.0 * (h * p);
}

double lwo_atan2(double y, double x) {
  double ax = fabs(x), ay = fabs(y);
  int swap = ay > ax;
  double num = swap ? ax : ay, den = swap ? ay : ax;
  double t = den == 0.0 ? 0.0 : num / den;
  double r = det_atan01(t);
  if (swap) r = LW_HALF_PI - r;
  if (x < 0.0) r = LW_PI - r;
  if (y < 0.0) r = -r;
  return r;
}

/* ========================================================================== */
/* Alias tables (Vose)                                        */
/* ========================================================================== */

int lwo_alias_build(const double* w, int64_t n, double* prob, int32_t* alias, double* pdf) {
  if (n <= 0) return 1;
  double total = 0.0;
  for (int64_t i = 0; i < n; i++) {
    if (!(w[i] >= 0.0) || w[i] == INFINITY) return 1;
    total += w[i];
  }
  if (!(total > 0.0)) return 1;
  double* scaled = (double*)malloc(sizeof(double) * n);
  int64_t* small = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* large = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t ns = 0, nl = 0;
  double dn = (double)n;
  for (int64_t i = 0; i < n; i++) {
    pdf[i] = w[i] / total;
    scaled[i] = pdf[i] * dn;
    if (scaled[i] < 1.0)
      small[ns++] = i;
    else
      large[nl++] = i;
  }
  while (ns > 0 && nl > 0) {
    int64_t s = small[--ns];
    int64_t l = large[--nl];
    prob[s] = scaled[s];
    alias[s] = (int32_t)l;
    scaled[l] = (scaled[l] + scaled[s]) - 1.0;
    if (scaled[l] < 1.0)
      small[ns++] = l;
    else
      large[nl++] = l;
  }
  while (nl > 0) {
    int64_t l = large[--nl];
    prob[l] = 1.0;
    alias[l] = (int32_t)l;
  }
  while (ns > 0) {
    int64_t s = small[--ns];
    prob[s] = 1.0;
    alias[s] = (int32_t)s;
  }
  free(scaled);
  free(small);
  free(large);
  return 0;
}

/* sample: returns the entry and remaps u to a fresh uniform in [0,1) */
static int64_t alias_sample(const double* prob, const int32_t* alias, int64_t n, double u, double* u_out) {
  double x = u * (double)n;
  double fi = floor(x);
  int64_t i = (int64_t)fi;
  if (i >= n) i = n - 1;
  double f = x - (double)i;
  double pr = prob[i];
  if (f < pr) {
    *u_out = f / pr;
    return i;
  }
  *u_out = (f - pr) / (1.0 - pr);
  if (*u_out >= 1.0) *u_out = 0.9999999999999999;
  return alias[i];
}

/* ========================================================================== */
/* Render scene: render BVH (child-box layout), lights, materials             */
/* ========================================================================== */

typedef struct {
  double box[2][6]; /* lo xyz, hi xyz of child 0 / child 1 */
  int32_t ref[2];   /* >= 0 internal node index; < 0 leaf: -(1 + (start << 3 | count)) */
} rnode;

/* light hierarchy node (device: LwLightNode): FP32 record of FP64 build sums */
typedef struct {
  float lo[3], hi[3];
  float tot;
  float flux[8];
  int32_t right;
} lt_node;

typedef struct {
  double lo[3], hi[3], tot, flux[8];
} lt_acc;

struct lwo_scene {
  lw_scene_desc d;
  int64_t ntris;
  double* verts;  /* [ntris*9] original order */
  double* normals;
  int32_t* material;
  lw_material* materials;
  /* reference-layout BVH */
  int64_t nnodes;
  double* bounds;
  int64_t* children;
  int64_t* order;
  /* render BVH */
  int64_t nrnodes;
  rnode* rnodes;
  int32_t root_ref;
  double root_box[6];
  double* lverts; /* leaf-ordered verts [ntris*9] */
  int64_t* ltri;  /* leaf slot -> original triangle id */
  /* emitters */
  int64_t nemit;
  int64_t* emit_of_tri; /* [ntris] emitter index or -1 */
  int64_t* emit_tri;
  double* emit_rad;
  int32_t* emit_two;
  double* emit_area;
  double* emit_prob;
  int32_t* emit_alias;
  double* emit_pdf;
  /* environment */
  int env_kind;
  int env_w, env_h;
  float* env_img;
  double* env_prob;   /* per texel: alias table of its row (conditional over the columns) */
  int32_t* env_alias; /* per texel: alias column within the row */
  double* env_pdf;    /* per texel: p(row) * p(column | row) */
  double* env_rprob;  /* per row: alias table over the row sums (marginal) */
  int32_t* env_ralias;
  double p_env, p_tri;
  /* environment pyramid (light_sampler & LW_LIGHTS_ENV_PYRAMID) */
  int ep_on, ep_nl, ep_ntop;
  double* ep_lvl;
  double* ep_top;
  int64_t ep_off[24], ep_toff[24], ep_stride;
  /* light hierarchy (light_sampler & LW_LIGHTS_TREE) */
  int64_t lt_n;
  lt_node* lt;
  uint64_t* lt_path;
  int32_t* lt_depth;
};

static int32_t leaf_ref(int64_t start, int64_t count) { return (int32_t)(-(1 + ((start << 3) | count))); }

static void build_render_bvh(lwo_scene* s) {
  int64_t nn = s->nnodes;
  int64_t* map = (int64_t*)malloc(sizeof(int64_t) * nn);
  int64_t ni = 0;
  for (int64_t k = 0; k < nn; k++) map[k] = s->children[2 * k] >= 0 ? ni++ : -1;
  s->nrnodes = ni;
  s->rnodes = (rnode*)calloc(ni > 0 ? ni : 1, sizeof(rnode));
  for (int64_t k = 0; k < nn; k++) {
    if (map[k] < 0) continue;
    rnode* r = s->rnodes + map[k];
    for (int c = 0; c < 2; c++) {
      int64_t ch = s->children[2 * k + c];
      memcpy(r->box[c], s->bounds + 6 * ch, sizeof(double) * 6);
      if (s->children[2 * ch] >= 0)
        r->ref[c] = (int32_t)map[ch];
      else
        r->ref[c] = leaf_ref(-(s->children[2 * ch] + 1), s->children[2 * ch + 1]);
    }
  }
  memcpy(s->root_box, s->bounds, sizeof(double) * 6);
  s->root_ref = s->children[0] >= 0 ? 0 : leaf_ref(-(s->children[0] + 1), s->children[1]);
  s->lverts = (double*)malloc(sizeof(double) * 9 * (s->ntris > 0 ? s->ntris : 1));
  s->ltri = (int64_t*)malloc(sizeof(int64_t) * (s->ntris > 0 ? s->ntris : 1));
  for (int64_t k = 0; k < s->ntris; k++) {
    memcpy(s->lverts + 9 * k, s->verts + 9 * s->order[k], sizeof(double) * 9);
    s->ltri[k] = s->order[k];
  }
  free(map);
}

/* Binned-SAH render tree, restating the specification of DESIGN.md §3.2 (the device builds
 * it in csrc/lw_sah.cu): FIFO segment order, 16 centroid bins per axis, first strict minimum of
 * A(L)nL + A(R)nR, split when n > 7 or A(B) + cost < n A(B), halve coincident centroids. */
#define SAH_BINS 16
#define SAH_MAXLEAF 7

typedef struct {
  int64_t start, n, parent;
  int side;
} sah_seg;

static double sah_area(const double* lo, const double* hi) {
  double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return 2.0 * ((dx * dy + dy * dz) + dz * dx);
}

static void bb_reset(double* lo, double* hi) {
  for (int a = 0; a < 3; a++) {
    lo[a] = INFINITY;
    hi[a] = -INFINITY;
  }
}

static void bb_add(double* lo, double* hi, const double* l2, const double* h2) {
  for (int a = 0; a < 3; a++) {
    if (l2[a] < lo[a]) lo[a] = l2[a];
    if (h2[a] > hi[a]) hi[a] = h2[a];
  }
}

static int sah_bin(double c, double cmin, double scale) {
  int b = (int)((c - cmin) * scale);
  return b > SAH_BINS - 1 ? SAH_BINS - 1 : b;
}

static void build_render_bvh_sah(lwo_scene* s) {
  int64_t n = s->ntris;
  s->ltri = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  s->lverts = (double*)malloc(sizeof(double) * 9 * (n > 0 ? n : 1));
  s->rnodes = (rnode*)calloc(n > 0 ? n : 1, sizeof(rnode));
  s->nrnodes = 0;
  s->root_ref = leaf_ref(0, 0);
  memset(s->root_box, 0, sizeof(s->root_box));
  if (n == 0) return;
  double *lo = (double*)malloc(sizeof(double) * 3 * n), *hi = (double*)malloc(sizeof(double) * 3 * n);
  double* ce = (double*)malloc(sizeof(double) * 3 * n);
  int64_t* spill = (int64_t*)malloc(sizeof(int64_t) * n);
  sah_seg* q = (sah_seg*)malloc(sizeof(sah_seg) * (2 * n + 2));
  for (int64_t i = 0; i < n; i++) {
    for (int a = 0; a < 3; a++) {
      const double* v = s->verts + 9 * i;
      double l = v[a], h = v[a];
      if (v[3 + a] < l) l = v[3 + a];
      if (v[6 + a] < l) l = v[6 + a];
      if (v[3 + a] > h) h = v[3 + a];
      if (v[6 + a] > h) h = v[6 + a];
      if (l == 0.0) l = 0.0; /* canonical +0: exact min/max are then order independent */
      if (h == 0.0) h = 0.0;
      double c = 0.5 * (l + h);
      if (c == 0.0) c = 0.0;
      lo[3 * i + a] = l;
      hi[3 * i + a] = h;
      ce[3 * i + a] = c;
    }
    s->ltri[i] = i;
  }
  int64_t qh = 0, qt = 0;
  q[qt++] = (sah_seg){0, n, -1, 0};
  while (qh < qt) {
    sah_seg g = q[qh++];
    int64_t* ids = s->ltri + g.start;
    double Blo[3], Bhi[3], Clo[3], Chi[3];
    bb_reset(Blo, Bhi);
    bb_reset(Clo, Chi);
    for (int64_t k = 0; k < g.n; k++) {
      bb_add(Blo, Bhi, lo + 3 * ids[k], hi + 3 * ids[k]);
      bb_add(Clo, Chi, ce + 3 * ids[k], ce + 3 * ids[k]);
    }
    if (g.parent < 0) {
      memcpy(s->root_box, Blo, sizeof(Blo));
      memcpy(s->root_box + 3, Bhi, sizeof(Bhi));
    }
    int bax = -1, bpl = -1;
    double bcost = INFINITY, blo[2][3], bhi[2][3];
    int64_t bnl = 0;
    for (int a = 0; a < 3 && g.n > 1; a++) {
      double ext = Chi[a] - Clo[a];
      if (!(ext > 0.0)) continue;
      double scale = (double)SAH_BINS / ext;
      int64_t cnt[SAH_BINS];
      double clo[SAH_BINS][3], chi[SAH_BINS][3];
      for (int b = 0; b < SAH_BINS; b++) {
        cnt[b] = 0;
        bb_reset(clo[b], chi[b]);
      }
      for (int64_t k = 0; k < g.n; k++) {
        int b = sah_bin(ce[3 * ids[k] + a], Clo[a], scale);
        cnt[b]++;
        bb_add(clo[b], chi[b], lo + 3 * ids[k], hi + 3 * ids[k]);
      }
      /* suffix boxes for the right side of plane p (bins p+1 .. 15) */
      double slo[SAH_BINS][3], shi[SAH_BINS][3];
      int64_t scnt[SAH_BINS];
      double rlo[3], rhi[3];
      bb_reset(rlo, rhi);
      int64_t rc = 0;
      for (int b = SAH_BINS - 1; b >= 1; b--) {
        bb_add(rlo, rhi, clo[b], chi[b]);
        rc += cnt[b];
        memcpy(slo[b], rlo, sizeof(rlo));
        memcpy(shi[b], rhi, sizeof(rhi));
        scnt[b] = rc;
      }
      double llo[3], lhi[3];
      bb_reset(llo, lhi);
      int64_t lc = 0;
      for (int p = 0; p + 1 < SAH_BINS; p++) {
        bb_add(llo, lhi, clo[p], chi[p]);
        lc += cnt[p];
        if (lc == 0 || scnt[p + 1] == 0) continue;
        double cost = sah_area(llo, lhi) * (double)lc + sah_area(slo[p + 1], shi[p + 1]) * (double)scnt[p + 1];
        if (cost < bcost) {
          bcost = cost;
          bax = a;
          bpl = p;
          bnl = lc;
          memcpy(blo[0], llo, sizeof(llo));
          memcpy(bhi[0], lhi, sizeof(lhi));
          memcpy(blo[1], slo[p + 1], sizeof(llo));
          memcpy(bhi[1], shi[p + 1], sizeof(lhi));
        }
      }
    }
    int split = 0, halve = 0;
    if (bax >= 0) {
      double aB = sah_area(Blo, Bhi);
      split = g.n > SAH_MAXLEAF || (aB + bcost) < (double)g.n * aB;
    } else if (g.n > SAH_MAXLEAF) {
      split = halve = 1;
    }
    if (!split) {
      int32_t r = leaf_ref(g.start, g.n);
      if (g.parent < 0)
        s->root_ref = r;
      else
        s->rnodes[g.parent].ref[g.side] = r;
      continue;
    }
    int64_t id = s->nrnodes++;
    if (g.parent < 0)
      s->root_ref = (int32_t)id;
    else
      s->rnodes[g.parent].ref[g.side] = (int32_t)id;
    if (halve) {
      bnl = g.n / 2;
      bb_reset(blo[0], bhi[0]);
      bb_reset(blo[1], bhi[1]);
      for (int64_t k = 0; k < g.n; k++) bb_add(blo[k < bnl ? 0 : 1], bhi[k < bnl ? 0 : 1], lo + 3 * ids[k], hi + 3 * ids[k]);
    } else {
      double scale = (double)SAH_BINS / (Chi[bax] - Clo[bax]);
      int64_t nl = 0, nr = 0;
      for (int64_t k = 0; k < g.n; k++) {
        int64_t t = ids[k];
        if (sah_bin(ce[3 * t + bax], Clo[bax], scale) <= bpl)
          ids[nl++] = t;
        else
          spill[nr++] = t;
      }
      memcpy(ids + nl, spill, sizeof(int64_t) * nr);
    }
    for (int c = 0; c < 2; c++) {
      memcpy(s->rnodes[id].box[c], blo[c], sizeof(double) * 3);
      memcpy(s->rnodes[id].box[c] + 3, bhi[c], sizeof(double) * 3);
    }
    q[qt++] = (sah_seg){g.start, bnl, id, 0};
    q[qt++] = (sah_seg){g.start + bnl, g.n - bnl, id, 1};
  }
  for (int64_t j = 0; j < n; j++) memcpy(s->lverts + 9 * j, s->verts + 9 * s->ltri[j], sizeof(double) * 9);
  free(lo);
  free(hi);
  free(ce);
  free(spill);
  free(q);
}

static double* dup_d(const double* p, int64_t n) {
  double* q = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  if (n > 0) memcpy(q, p, sizeof(double) * n);
  return q;
}

/* ---- light hierarchy: build (restating the library's light_tree_build) --------------------
 * Emitters of positive weight; median split (n/2 to the left) of the (centroid, emitter) order
 * along the axis of largest centroid extent (first on ties); single-emitter leaves; depth-first
 * node ids (left = node + 1, right = node + 2 * nleft).  Leaf: triangle box, tot = weight,
 * flux[k] = weight * max cos of the (two-sided: either) normal towards emission octant k. */
static double lt_octant_cos(int k, double nx, double ny, double nz) {
  double a = (k & 1) ? -nx : nx, b = (k & 2) ? -ny : ny, c = (k & 4) ? -nz : nz;
  a = a > 0.0 ? a : 0.0;
  b = b > 0.0 ? b : 0.0;
  c = c > 0.0 ? c : 0.0;
  return sqrt((a * a + b * b) + c * c);
}

typedef struct {
  const lw_scene_desc* d;
  double* cen;
  int64_t* items;
  lwo_scene* s;
} lt_ctx;

static const double* g_lt_cen; /* comparator key (oracle build is single-threaded) */
static int g_lt_axis;
static int lt_cmp(const void* pa, const void* pb) {
  int64_t x = *(const int64_t*)pa, y = *(const int64_t*)pb;
  double cx = g_lt_cen[3 * x + g_lt_axis], cy = g_lt_cen[3 * y + g_lt_axis];
  if (cx < cy) return -1;
  if (cx > cy) return 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static void lt_store(const lt_acc* A, int32_t right, lt_node* N) {
  for (int a = 0; a < 3; a++) {
    N->lo[a] = (float)A->lo[a];
    N->hi[a] = (float)A->hi[a];
  }
  N->tot = (float)A->tot;
  for (int k = 0; k < 8; k++) N->flux[k] = (float)A->flux[k];
  N->right = right;
}

static lt_acc lt_rec(lt_ctx* c, int64_t begin, int64_t end, int64_t node, uint64_t bits, int dep) {
  int64_t n = end - begin;
  lt_acc M;
  if (n == 1) {
    int64_t e = c->items[begin];
    const double* v = c->s->verts + 9 * c->d->emit_tri[e];
    for (int a = 0; a < 3; a++) {
      double lo = v[a], hi = v[a];
      if (v[3 + a] < lo) lo = v[3 + a];
      if (v[6 + a] < lo) lo = v[6 + a];
      if (v[3 + a] > hi) hi = v[3 + a];
      if (v[6 + a] > hi) hi = v[6 + a];
      M.lo[a] = lo;
      M.hi[a] = hi;
    }
    double e1x = v[3] - v[0], e1y = v[4] - v[1], e1z = v[5] - v[2];
    double e2x = v[6] - v[0], e2y = v[7] - v[1], e2z = v[8] - v[2];
    double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
    double inv = 1.0 / sqrt((cx * cx + cy * cy) + cz * cz);
    double nx = cx * inv, ny = cy * inv, nz = cz * inv;
    double w = c->d->emit_weight[e];
    M.tot = w;
    for (int k = 0; k < 8; k++) {
      double cc = lt_octant_cos(k, nx, ny, nz);
      if (c->d->emit_twosided[e]) {
        double c2 = lt_octant_cos(k, -nx, -ny, -nz);
        if (c2 > cc) cc = c2;
      }
      M.flux[k] = w * cc;
    }
    lt_store(&M, (int32_t)(-(e + 1)), c->s->lt + node);
    c->s->lt_path[e] = bits;
    c->s->lt_depth[e] = dep;
    return M;
  }
  double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = begin; i < end; i++)
    for (int a = 0; a < 3; a++) {
      double cv = c->cen[3 * c->items[i] + a];
      if (cv < cmin[a]) cmin[a] = cv;
      if (cv > cmax[a]) cmax[a] = cv;
    }
  int axis = 0;
  for (int a = 1; a < 3; a++)
    if (cmax[a] - cmin[a] > cmax[axis] - cmin[axis]) axis = a;
  g_lt_cen = c->cen;
  g_lt_axis = axis;
  qsort(c->items + begin, (size_t)n, sizeof(int64_t), lt_cmp);
  int64_t nl = n / 2;
  int64_t left = node + 1, right = node + 2 * nl;
  lt_acc L = lt_rec(c, begin, begin + nl, left, bits, dep + 1);
  lt_acc R = lt_rec(c, begin + nl, end, right, bits | (1ULL << dep), dep + 1);
  for (int a = 0; a < 3; a++) {
    M.lo[a] = L.lo[a] < R.lo[a] ? L.lo[a] : R.lo[a];
    M.hi[a] = L.hi[a] > R.hi[a] ? L.hi[a] : R.hi[a];
  }
  M.tot = L.tot + R.tot;
  for (int k = 0; k < 8; k++) M.flux[k] = L.flux[k] + R.flux[k];
  lt_store(&M, (int32_t)right, c->s->lt + node);
  return M;
}

static void lt_build(lwo_scene* s, const lw_scene_desc* d) {
  int64_t ne = d->nemit;
  lt_ctx c = {d, (double*)malloc(sizeof(double) * 3 * (ne > 0 ? ne : 1)),
              (int64_t*)malloc(sizeof(int64_t) * (ne > 0 ? ne : 1)), s};
  s->lt_path = (uint64_t*)calloc(ne > 0 ? ne : 1, sizeof(uint64_t));
  s->lt_depth = (int32_t*)malloc(sizeof(int32_t) * (ne > 0 ? ne : 1));
  int64_t m = 0;
  for (int64_t e = 0; e < ne; e++) {
    const double* v = s->verts + 9 * d->emit_tri[e];
    for (int a = 0; a < 3; a++) c.cen[3 * e + a] = ((v[a] + v[3 + a]) + v[6 + a]) / 3.0;
    s->lt_depth[e] = -1;
    if (d->emit_weight[e] > 0.0) c.items[m++] = e;
  }
  s->lt_n = m > 0 ? 2 * m - 1 : 0;
  s->lt = (lt_node*)calloc(s->lt_n > 0 ? s->lt_n : 1, sizeof(lt_node));
  if (m > 0) lt_rec(&c, 0, m, 0, 0ULL, 0);
  free(c.cen);
  free(c.items);
}

static void ep_build(lwo_scene* s, const lw_scene_desc* d);

/* Two-level environment alias table (device: k_env_rows / k_env_marginal / k_env_pdf in
 * lw_render.cu, built on the GPU at upload): per row, the Vose table of lwo_alias_build over the
 * row's texel weights (rows of zero weight: prob 1, self alias, pdf 0); over the rows, the Vose
 * table of the row sums (each summed in column order); texel pdf = p(row) * p(column | row).
 * Sampling draws the row with the NEE uniform and the column with the rescaled remainder. */
static int env_alias2_build(const double* w, int W, int H, double* prob, int32_t* alias, double* pdf, double* rprob,
                            int32_t* ralias) {
  double* rsum = (double*)malloc(sizeof(double) * H);
  double* rpdf = (double*)malloc(sizeof(double) * H);
  for (int r = 0; r < H; r++) {
    const double* wr = w + (int64_t)r * W;
    double t = 0.0;
    for (int c = 0; c < W; c++) t += wr[c];
    rsum[r] = t;
    if (lwo_alias_build(wr, W, prob + (int64_t)r * W, alias + (int64_t)r * W, pdf + (int64_t)r * W))
      for (int c = 0; c < W; c++) {
        prob[(int64_t)r * W + c] = 1.0;
        alias[(int64_t)r * W + c] = c;
        pdf[(int64_t)r * W + c] = 0.0;
      }
  }
  int bad = lwo_alias_build(rsum, H, rprob, ralias, rpdf);
  if (!bad)
    for (int r = 0; r < H; r++)
      for (int c = 0; c < W; c++) pdf[(int64_t)r * W + c] = rpdf[r] * pdf[(int64_t)r * W + c];
  free(rsum);
  free(rpdf);
  return bad;
}

lwo_scene* lwo_scene_create(const lw_scene_desc* d) {
  lwo_scene* s = (lwo_scene*)calloc(1, sizeof(lwo_scene));
  s->d = *d;
  s->ntris = d->ntris;
  s->verts = dup_d(d->verts, 9 * d->ntris);
  s->normals = dup_d(d->normals, 9 * d->ntris);
  s->material = (int32_t*)malloc(sizeof(int32_t) * (d->ntris > 0 ? d->ntris : 1));
  if (d->ntris) memcpy(s->material, d->material, sizeof(int32_t) * d->ntris);
  s->materials = (lw_material*)malloc(sizeof(lw_material) * (d->nmaterials > 0 ? d->nmaterials : 1));
  if (d->nmaterials) memcpy(s->materials, d->materials, sizeof(lw_material) * d->nmaterials);
  int64_t cap = d->ntris > 0 ? 2 * d->ntris : 1;
  s->bounds = (double*)malloc(sizeof(double) * 6 * cap);
  s->children = (int64_t*)malloc(sizeof(int64_t) * 2 * cap);
  s->order = (int64_t*)malloc(sizeof(int64_t) * (d->ntris > 0 ? d->ntris : 1));
  s->nnodes = lwo_build_bvh(s->verts, s->ntris, s->bounds, s->children, s->order);
  if (d->bvh_kind == LW_BVH_MEDIAN)
    build_render_bvh(s);
  else
    build_render_bvh_sah(s);
  /* emitters */
  s->nemit = d->nemit;
  s->emit_of_tri = (int64_t*)malloc(sizeof(int64_t) * (s->ntris > 0 ? s->ntris : 1));
  for (int64_t k = 0; k < s->ntris; k++) s->emit_of_tri[k] = -1;
  if (s->nemit > 0) {
    s->emit_tri = (int64_t*)malloc(sizeof(int64_t) * s->nemit);
    memcpy(s->emit_tri, d->emit_tri, sizeof(int64_t) * s->nemit);
    s->emit_rad = dup_d(d->emit_radiance, 3 * s->nemit);
    s->emit_two = (int32_t*)malloc(sizeof(int32_t) * s->nemit);
    memcpy(s->emit_two, d->emit_twosided, sizeof(int32_t) * s->nemit);
    s->emit_area = (double*)malloc(sizeof(double) * s->nemit);
    s->emit_prob = (double*)malloc(sizeof(double) * s->nemit);
    s->emit_alias = (int32_t*)malloc(sizeof(int32_t) * s->nemit);
    s->emit_pdf = (double*)malloc(sizeof(double) * s->nemit);
    for (int64_t e = 0; e < s->nemit; e++) {
      const double* v = s->verts + 9 * s->emit_tri[e];
      double e1[3] = {v[3] - v[0], v[4] - v[1], v[5] - v[2]};
      double e2[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
      double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
             cz = e1[0] * e2[1] - e1[1] * e2[0];
      s->emit_area[e] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
      s->emit_of_tri[s->emit_tri[e]] = e;
    }
    if (lwo_alias_build(d->emit_weight, s->nemit, s->emit_prob, s->emit_alias, s->emit_pdf)) s->nemit = 0;
  }
  if ((d->light_sampler & LW_LIGHTS_TREE) && s->nemit > 0) lt_build(s, d);
  s->env_kind = d->env_kind;
  s->env_w = d->env_width;
  s->env_h = d->env_height;
  if (s->env_kind == LW_ENV_IMAGE) {
    int64_t nt = (int64_t)s->env_w * s->env_h;
    s->env_img = (float*)malloc(sizeof(float) * 3 * nt);
    memcpy(s->env_img, d->env_image, sizeof(float) * 3 * nt);
    s->env_prob = (double*)malloc(sizeof(double) * nt);
    s->env_alias = (int32_t*)malloc(sizeof(int32_t) * nt);
    s->env_pdf = (double*)malloc(sizeof(double) * nt);
    s->env_rprob = (double*)malloc(sizeof(double) * s->env_h);
    s->env_ralias = (int32_t*)malloc(sizeof(int32_t) * s->env_h);
    if (env_alias2_build(d->env_weight, s->env_w, s->env_h, s->env_prob, s->env_alias, s->env_pdf, s->env_rprob,
                         s->env_ralias))
      s->env_kind = LW_ENV_NONE;
  }
  if (s->env_kind == LW_ENV_IMAGE && (d->light_sampler & LW_LIGHTS_ENV_PYRAMID)) ep_build(s, d);
  int has_env = s->env_kind != LW_ENV_NONE;
  int has_tri = s->nemit > 0;
  s->p_env = has_env ? (has_tri ? d->p_env : 1.0) : 0.0;
  s->p_tri = has_tri ? (has_env ? 1.0 - d->p_env : 1.0) : 0.0;
  return s;
}

void lwo_scene_destroy(lwo_scene* s) {
  if (!s) return;
  free(s->verts);
  free(s->normals);
  free(s->material);
  free(s->materials);
  free(s->bounds);
  free(s->children);
  free(s->order);
  free(s->rnodes);
  free(s->lverts);
  free(s->ltri);
  free(s->emit_of_tri);
  free(s->emit_tri);
  free(s->emit_rad);
  free(s->emit_two);
  free(s->emit_area);
  free(s->emit_prob);
  free(s->emit_alias);
  free(s->emit_pdf);
  free(s->env_img);
  free(s->env_prob);
  free(s->env_alias);
  free(s->env_pdf);
  free(s->env_rprob);
  free(s->env_ralias);
  free(s->ep_lvl);
  free(s->ep_top);
  free(s->lt);
  free(s->lt_path);
  free(s->lt_depth);
  free(s);
}

/* ---- render traversal: near-first over child boxes, conservative cull ----- */

#define CULL_M 9.094947017729282e-13 /* 2^-40 relative slack on every slab comparison */

typedef struct {
  double o[3], inv[3];
  int zero[3];
  shear sh;
} rray;

static void rray_setup(rray* r, const double* o, const double* d) {
  for (int a = 0; a < 3; a++) {
    r->o[a] = o[a];
    r->zero[a] = !(d[a] > 1e-200 || d[a] < -1e-200);
    r->inv[a] = r->zero[a] ? 0.0 : 1.0 / d[a];
  }
  shear_setup(o, d, 0, &r->sh);
}

/* returns 1 if the box may contain a hit in [0, best]; *tn_out = raw entry distance */
static int box_hit(const rray* r, const double* box, double best, double* tn_out) {
  double tn = -INFINITY, tf = INFINITY;
  for (int a = 0; a < 3; a++) {
    if (r->zero[a]) {
      if (r->o[a] < box[a] || r->o[a] > box[3 + a]) return 0;
      continue;
    }
    double t0 = (box[a] - r->o[a]) * r->inv[a];
    double t1 = (box[3 + a] - r->o[a]) * r->inv[a];
    if (t0 > t1) {
      double t = t0;
      t0 = t1;
      t1 = t;
    }
    if (t0 > tn) tn = t0;
    if (t1 < tf) tf = t1;
  }
  double tn_lo = tn - CULL_M * fabs(tn);
  double tf_hi = tf + CULL_M * fabs(tf);
  double best_hi = best + CULL_M * fabs(best);
  *tn_out = tn;
  return tn_lo <= tf_hi && tn_lo <= best_hi && tf_hi >= 0.0;
}

static int pop_keep(double tn, double best) { return tn - CULL_M * fabs(tn) <= best + CULL_M * fabs(best); }

static void leaf_decode(int32_t ref, int64_t* start, int64_t* count) {
  int64_t v = -(int64_t)ref - 1;
  *start = v >> 3;
  *count = v & 7;
}

/* closest hit; tie -> lower original triangle id */
static void trace_closest(const lwo_scene* s, const double* o, const double* d, double tmax, hitrec* h) {
  h->t = tmax;
  h->tri = -1;
  h->bu = h->bv = 0.0;
  if (s->ntris == 0) return;
  rray r;
  rray_setup(&r, o, d);
  double tn;
  if (!box_hit(&r, s->root_box, h->t, &tn)) return;
  int32_t stack_ref[64];
  double stack_tn[64];
  int sp = 0;
  int32_t ref = s->root_ref;
  for (;;) {
    while (ref >= 0) {
      const rnode* nd = s->rnodes + ref;
      double tn0, tn1;
      int h0 = box_hit(&r, nd->box[0], h->t, &tn0);
      int h1 = box_hit(&r, nd->box[1], h->t, &tn1);
      if (h0 && h1) {
        if (tn1 < tn0) {
          stack_ref[sp] = nd->ref[0];
          stack_tn[sp++] = tn0;
          ref = nd->ref[1];
        } else {
          stack_ref[sp] = nd->ref[1];
          stack_tn[sp++] = tn1;
          ref = nd->ref[0];
        }
      } else if (h0) {
        ref = nd->ref[0];
      } else if (h1) {
        ref = nd->ref[1];
      } else {
        ref = 0x7fffffff; /* nothing to descend into */
        break;
      }
    }
    if (ref != 0x7fffffff) {
      int64_t start, count;
      leaf_decode(ref, &start, &count);
      for (int64_t k = start; k < start + count; k++) tri_test(s->lverts + 9 * k, s->ltri[k], &r.sh, 0.0, h);
    }
    ref = 0x7fffffff;
    while (sp > 0) {
      sp--;
      if (pop_keep(stack_tn[sp], h->t)) {
        ref = stack_ref[sp];
        break;
      }
    }
    if (ref == 0x7fffffff) return;
  }
}

/* any hit with 0 < t < tmax */
static int trace_any(const lwo_scene* s, const double* o, const double* d, double tmax) {
  if (s->ntris == 0) return 0;
  rray r;
  rray_setup(&r, o, d);
  double tn;
  if (!box_hit(&r, s->root_box, tmax, &tn)) return 0;
  int32_t stack_ref[64];
  int sp = 0;
  int32_t ref = s->root_ref;
  for (;;) {
    while (ref >= 0) {
      const rnode* nd = s->rnodes + ref;
      double tn0, tn1;
      int h0 = box_hit(&r, nd->box[0], tmax, &tn0);
      int h1 = box_hit(&r, nd->box[1], tmax, &tn1);
      if (h0 && h1) {
        stack_ref[sp++] = nd->ref[1];
        ref = nd->ref[0];
      } else if (h0) {
        ref = nd->ref[0];
      } else if (h1) {
        ref = nd->ref[1];
      } else {
        ref = 0x7fffffff;
        break;
      }
    }
    if (ref != 0x7fffffff) {
      int64_t start, count;
      leaf_decode(ref, &start, &count);
      for (int64_t k = start; k < start + count; k++)
        if (tri_occludes(s->lverts + 9 * k, &r.sh, tmax)) return 1;
    }
    if (sp == 0) return 0;
    ref = stack_ref[--sp];
  }
}

void lwo_trace_closest_batch(const lwo_scene* s, const double* origins, const double* dirs, const double* tmaxs,
                             int64_t n, double* out_t, int64_t* out_tri, double* out_bary) {
  for (int64_t i = 0; i < n; i++) {
    hitrec h;
    trace_closest(s, origins + 3 * i, dirs + 3 * i, tmaxs[i], &h);
    if (h.tri >= 0) {
      out_t[i] = h.t;
      out_tri[i] = h.tri;
      out_bary[2 * i] = h.bu;
      out_bary[2 * i + 1] = h.bv;
    } else {
      out_t[i] = 1e308;
      out_tri[i] = -1;
      out_bary[2 * i] = out_bary[2 * i + 1] = 0.0;
    }
  }
}

void lwo_trace_any_batch(const lwo_scene* s, const double* origins, const double* dirs, const double* tmaxs,
                         int64_t n, int32_t* out) {
  for (int64_t i = 0; i < n; i++) out[i] = trace_any(s, origins + 3 * i, dirs + 3 * i, tmaxs[i]);
}

/* ========================================================================== */
/* Integrator                                 */
/* ========================================================================== */

typedef struct {
  double x, y, z;
} v3;

static v3 mk(double x, double y, double z) {
  v3 r = {x, y, z};
  return r;
}
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static v3 neg(v3 a) { return mk(-a.x, -a.y, -a.z); }
static double dot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static v3 cross(v3 a, v3 b) { return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static v3 normalize(v3 a) {
  double inv = 1.0 / sqrt(dot(a, a));
  return mk(a.x * inv, a.y * inv, a.z * inv);
}
static v3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
static v3 bary3(v3 a, v3 b, v3 c, double w, double bu, double bv) {
  return mk((w * a.x + bu * b.x) + bv * c.x, (w * a.y + bu * b.y) + bv * c.y, (w * a.z + bu * b.z) + bv * c.z);
}

typedef struct {
  const lwo_scene* s;
  const lw_render_params* p;
} rctx;

static double qmc(const rctx* c, int64_t dim, int64_t index) {
  return lwo_halton_dim(c->p->bases, c->p->perm_flat, c->p->perm_offset, dim, index);
}

/* camera ray */
static void camera_ray(const rctx* c, int64_t index, v3* o, v3* d) {
  const lw_scene_desc* sd = &c->s->d;
  int64_t W = c->p->width, H = c->p->height, P = W * H;
  int64_t pix = index % P;
  int64_t x = pix % W, y = pix / W;
  double dx = lwo_gauss_filter_offset(qmc(c, 0, index));
  double dy = lwo_gauss_filter_offset(qmc(c, 1, index));
  double fx = (((double)x + 0.5) + dx) / (double)W;
  double fy = (((double)y + 0.5) + dy) / (double)H;
  double sx = fx * 2.0 - 1.0;
  double sy = 1.0 - fy * 2.0;
  double aspect = (double)W / (double)H;
  double ax = sx * (sd->tan_half_fov * aspect);
  double ay = sy * sd->tan_half_fov;
  v3 f = ld3(sd->cam_fwd), r = ld3(sd->cam_right), u = ld3(sd->cam_up);
  v3 dd = mk((f.x + ax * r.x) + ay * u.x, (f.y + ax * r.y) + ay * u.y, (f.z + ax * r.z) + ay * u.z);
  *d = normalize(dd);
  *o = ld3(sd->cam_pos);
}

void lwo_camera_rays(const lwo_scene* s, const lw_render_params* p, const int64_t* idx, int64_t n, double* oo,
                     double* od) {
  rctx c = {s, p};
  for (int64_t i = 0; i < n; i++) {
    v3 o, d;
    camera_ray(&c, idx[i], &o, &d);
    oo[3 * i] = o.x;
    oo[3 * i + 1] = o.y;
    oo[3 * i + 2] = o.z;
    od[3 * i] = d.x;
    od[3 * i + 1] = d.y;
    od[3 * i + 2] = d.z;
  }
}

static v3 offset_origin(v3 p, v3 n, v3 dir) {
  double m = fabs(p.x);
  if (fabs(p.y) > m) m = fabs(p.y);
  if (fabs(p.z) > m) m = fabs(p.z);
  if (m < 1.0) m = 1.0;
  double eps = 1e-9 * m;
  double sgn = dot(n, dir) >= 0.0 ? eps : -eps;
  return mk(p.x + n.x * sgn, p.y + n.y * sgn, p.z + n.z * sgn);
}

/* ---- light hierarchy: sample_light / light_pdf (device: lw_lighttree.cuh) ---------------- */
#define LT_PMIN 0.015625 /* 1/64: branch probabilities clamped to [PMIN, 1 - PMIN] */

/* importance as a fraction num / den (den > 0); lt_pleft combines two fractions with one division */
static void lt_importance(const lt_node* N, float x0, float x1, float x2, float n0, float n1, float n2, float* num,
                          float* den) {
  float cx = (N->lo[0] + N->hi[0]) * 0.5f, cy = (N->lo[1] + N->hi[1]) * 0.5f, cz = (N->lo[2] + N->hi[2]) * 0.5f;
  float dx = cx - x0, dy = cy - x1, dz = cz - x2;
  float d2 = (dx * dx + dy * dy) + dz * dz;
  float ex = N->hi[0] - N->lo[0], ey = N->hi[1] - N->lo[1], ez = N->hi[2] - N->lo[2];
  float r2 = ((ex * ex + ey * ey) + ez * ez) * 0.25f;
  float dist2 = d2 > r2 ? d2 : r2;
  int inside = x0 >= N->lo[0] && x0 <= N->hi[0] && x1 >= N->lo[1] && x1 <= N->hi[1] && x2 >= N->lo[2] &&
               x2 <= N->hi[2];
  if (inside || !(d2 > r2)) {
    *num = N->tot;
    *den = dist2 > 0.0f ? dist2 : 1.0f;
    return;
  }
  int oct = (dx > 0.0f ? 1 : 0) | (dy > 0.0f ? 2 : 0) | (dz > 0.0f ? 4 : 0); /* signs of x - c */
  /* cos(max(0, theta - alpha)) * d^2 with cos theta = dt / d, cos alpha = sqrt(d2 - r2) / d,
   * sin alpha = r / d: (dt sqrt(d2 - r2) + sqrt(d2 - dt^2) r) / d^2, 1 when theta <= alpha */
  float dt = (n0 * dx + n1 * dy) + n2 * dz;
  float s1 = sqrtf(d2 - r2);
  if (dt >= s1) {
    *num = N->flux[oct];
    *den = dist2;
    return;
  }
  float s2 = d2 - dt * dt;
  float t = dt * s1 + sqrtf(s2 > 0.0f ? s2 : 0.0f) * sqrtf(r2);
  if (t < 0.0f) t = 0.0f;
  *num = N->flux[oct] * t;
  *den = d2 * dist2;
}

static double lt_pleft(const lwo_scene* s, int64_t k, v3 x, v3 n) {
  float x0 = (float)x.x, x1 = (float)x.y, x2 = (float)x.z, n0 = (float)n.x, n1 = (float)n.y, n2 = (float)n.z;
  float nl, dl, nr, dr;
  lt_importance(s->lt + k + 1, x0, x1, x2, n0, n1, n2, &nl, &dl);
  lt_importance(s->lt + s->lt[k].right, x0, x1, x2, n0, n1, n2, &nr, &dr);
  float il = nl * dr, ir = nr * dl; /* importances scaled by the common factor dl * dr */
  float sum = il + ir;
  float pl = sum > 0.0f ? il / sum : 0.5f;
  if (pl < (float)LT_PMIN) pl = (float)LT_PMIN;
  if (pl > 1.0f - (float)LT_PMIN) pl = 1.0f - (float)LT_PMIN;
  return (double)pl;
}

static int64_t lt_sample(const lwo_scene* s, v3 x, v3 n, double u, double* psel, double* u_out) {
  int64_t k = 0;
  double p = 1.0;
  while (s->lt[k].right >= 0) {
    double pl = lt_pleft(s, k, x, n);
    if (u < pl) {
      u = u / pl;
      p = p * pl;
      k = k + 1;
    } else {
      u = (u - pl) / (1.0 - pl);
      p = p * (1.0 - pl);
      k = s->lt[k].right;
    }
  }
  if (u >= 1.0) u = 0.9999999999999999;
  if (u < 0.0) u = 0.0;
  *psel = p;
  *u_out = u;
  return -(int64_t)s->lt[k].right - 1;
}

static double lt_pdf(const lwo_scene* s, int64_t e, v3 x, v3 n) {
  int dep = s->lt_depth[e];
  if (dep < 0) return 0.0;
  uint64_t bits = s->lt_path[e];
  int64_t k = 0;
  double p = 1.0;
  for (int l = 0; l < dep; l++) {
    double pl = lt_pleft(s, k, x, n);
    if (((bits >> l) & 1ULL) == 0) {
      p = p * pl;
      k = k + 1;
    } else {
      p = p * (1.0 - pl);
      k = s->lt[k].right;
    }
  }
  return p;
}

/* reference normal of the estimates: the facing geometric normal through the octahedral packing */
static v3 lt_ref_normal(int64_t packed) {
  double o[3];
  lwo_oct_decode(packed, o);
  return normalize(mk(o[0], o[1], o[2]));
}

int64_t lwo_light_tree(const lwo_scene* s, double* nodes15, int32_t* right, uint64_t* path, int32_t* depth) {
  if (!s->lt) return 0;
  for (int64_t k = 0; nodes15 && k < s->lt_n; k++) {
    const lt_node* N = s->lt + k;
    double* o = nodes15 + 15 * k;
    for (int a = 0; a < 3; a++) {
      o[a] = N->lo[a];
      o[3 + a] = N->hi[a];
    }
    o[6] = N->tot;
    for (int b = 0; b < 8; b++) o[7 + b] = N->flux[b];
    if (right) right[k] = N->right;
  }
  for (int64_t e = 0; path && e < s->d.nemit; e++) {
    path[e] = s->lt_path[e];
    depth[e] = s->lt_depth[e];
  }
  return s->lt_n;
}

void lwo_light_sample_batch(const lwo_scene* s, const double* x, const double* nrm, const double* u, int64_t n,
                            int64_t* out_e, double* out_psel, double* out_u) {
  for (int64_t i = 0; i < n; i++)
    out_e[i] = lt_sample(s, ld3(x + 3 * i), ld3(nrm + 3 * i), u[i], out_psel + i, out_u + i);
}

void lwo_light_pdf_batch(const lwo_scene* s, const int64_t* e, const double* x, const double* nrm, int64_t n,
                         double* out_psel) {
  for (int64_t i = 0; i < n; i++) out_psel[i] = lt_pdf(s, e[i], ld3(x + 3 * i), ld3(nrm + 3 * i));
}

/* ---- environment pyramid (device: lw_envpyr.cuh; library host build: env_pyramid_build) ----
 * Level 0 = texel weights (luminance * sin theta); level l+1 = sums of 2x2 children up to a 1 x 2
 * top; the top EP_TOP levels are replicated per normal bin (4 x 4 octahedral cells of the facing
 * geometric normal) with weights scaled by a conservative cosine bound floored at 1/64.
 * Sampling: column half with u, row half with v, both rescaled; pdf = product of conditionals. */
#define EP_BINS 16
#define EP_TOP 5
#define EP_CWMIN 0.015625

static int ep_bin(int64_t packed) { return (int)(((packed >> 30) & 3) * 4 + ((packed >> 14) & 3)); }

static v3 ep_dir(double phi_turns, double theta_turns) {
  double st, ct, sp, cp;
  lwo_sincos2pi(theta_turns, &st, &ct);
  lwo_sincos2pi(phi_turns, &sp, &cp);
  return mk(st * cp, ct, st * sp);
}

static v3 ep_decode_n(int64_t packed) {
  double o[3];
  lwo_oct_decode(packed, o);
  return normalize(mk(o[0], o[1], o[2]));
}

static void ep_bin_cone(int b, v3* axis, double* cosb) {
  int64_t bu = b / 4, bv = b % 4;
  *axis = ep_decode_n(((bu * 16384 + 8192) << 16) | (bv * 16384 + 8192));
  double m = 1.0;
  for (int k = 0; k <= 8; k++) {
    int64_t t = k * 2048;
    int64_t e0[4][2] = {{bu * 16384 + t, bv * 16384}, {bu * 16384 + t, bv * 16384 + 16384},
                        {bu * 16384, bv * 16384 + t}, {bu * 16384 + 16384, bv * 16384 + t}};
    for (int q = 0; q < 4; q++) {
      int64_t eu = e0[q][0] > 65535 ? 65535 : e0[q][0], ev = e0[q][1] > 65535 ? 65535 : e0[q][1];
      double c = dot(*axis, ep_decode_n((eu << 16) | ev));
      if (c < m) m = c;
    }
  }
  *cosb = m - 0.02;
}

static void ep_texel_cone(int64_t r, int64_t c, int64_t Hl, int64_t Wl, v3* ctr, double* cosg) {
  double f0 = (double)c / (double)Wl, f1 = (double)(c + 1) / (double)Wl;
  double t0 = (double)r / (double)Hl * 0.5, t1 = (double)(r + 1) / (double)Hl * 0.5;
  *ctr = ep_dir((f0 + f1) * 0.5, (t0 + t1) * 0.5);
  double m = 1.0;
  for (int k = 0; k <= 8; k++) {
    double a = (double)k / 8.0;
    double fk = f0 + (f1 - f0) * a, tk = t0 + (t1 - t0) * a;
    v3 sm[4] = {ep_dir(fk, t0), ep_dir(fk, t1), ep_dir(f0, tk), ep_dir(f1, tk)};
    for (int q = 0; q < 4; q++) {
      double cq = dot(*ctr, sm[q]);
      if (cq < m) m = cq;
    }
  }
  *cosg = m - 0.02;
}

static double ep_cos_bound(v3 axis, double cosb, v3 ctr, double cosg) {
  if (cosb <= 0.0 || cosg <= 0.0) return 1.0;
  double sinb = sqrt(1.0 - cosb * cosb), sing = sqrt(1.0 - cosg * cosg);
  double cosd = cosb * cosg - sinb * sing, sind = sinb * cosg + cosb * sing;
  if (sind <= 0.0) return 1.0;
  double cosa = dot(axis, ctr);
  if (cosa >= cosd) return 1.0;
  double s2 = 1.0 - cosa * cosa;
  double sina = sqrt(s2 > 0.0 ? s2 : 0.0);
  double cw = cosa * cosd + sina * sind;
  return cw > 0.0 ? cw : 0.0;
}

static void ep_build(lwo_scene* s, const lw_scene_desc* d) {
  int64_t W = d->env_width, H = d->env_height;
  if (!(H >= 1 && W == 2 * H && (H & (H - 1)) == 0)) return; /* library rejects the scene */
  int nl = 1;
  while ((H >> (nl - 1)) > 1) nl++;
  s->ep_nl = nl;
  int64_t tot = 0;
  for (int l = 0; l < nl; l++) {
    s->ep_off[l] = tot;
    tot += (H >> l) * (W >> l);
  }
  s->ep_lvl = (double*)malloc(sizeof(double) * tot);
  for (int64_t k = 0; k < W * H; k++) s->ep_lvl[k] = d->env_weight[k];
  for (int l = 1; l < nl; l++) {
    int64_t Hl = H >> l, Wl = W >> l, Wc = Wl * 2;
    const double* ch = s->ep_lvl + s->ep_off[l - 1];
    double* o = s->ep_lvl + s->ep_off[l];
    for (int64_t r = 0; r < Hl; r++)
      for (int64_t c = 0; c < Wl; c++)
        o[r * Wl + c] = ((ch[(2 * r) * Wc + 2 * c] + ch[(2 * r) * Wc + 2 * c + 1]) + ch[(2 * r + 1) * Wc + 2 * c]) +
                        ch[(2 * r + 1) * Wc + 2 * c + 1];
  }
  s->ep_ntop = nl < EP_TOP ? nl : EP_TOP;
  int64_t ts = 0;
  for (int l = nl - s->ep_ntop; l < nl; l++) {
    s->ep_toff[l] = ts;
    ts += (H >> l) * (W >> l);
  }
  s->ep_stride = ts;
  s->ep_top = (double*)malloc(sizeof(double) * EP_BINS * ts);
  for (int b = 0; b < EP_BINS; b++) {
    v3 axis;
    double cosb;
    ep_bin_cone(b, &axis, &cosb);
    for (int l = nl - s->ep_ntop; l < nl; l++) {
      int64_t Hl = H >> l, Wl = W >> l;
      for (int64_t r = 0; r < Hl; r++)
        for (int64_t c = 0; c < Wl; c++) {
          v3 ctr;
          double cosg;
          ep_texel_cone(r, c, Hl, Wl, &ctr, &cosg);
          double cw = ep_cos_bound(axis, cosb, ctr, cosg);
          if (cw < EP_CWMIN) cw = EP_CWMIN;
          s->ep_top[b * ts + s->ep_toff[l] + r * Wl + c] = s->ep_lvl[s->ep_off[l] + r * Wl + c] * cw;
        }
    }
  }
  s->ep_on = 1;
}

static double ep_w(const lwo_scene* s, int bin, int l, int64_t r, int64_t c) {
  int64_t wl = (int64_t)s->env_w >> l;
  if (l >= s->ep_nl - s->ep_ntop) return s->ep_top[bin * s->ep_stride + s->ep_toff[l] + r * wl + c];
  return s->ep_lvl[s->ep_off[l] + r * wl + c];
}

static void ep_sample(const lwo_scene* s, int bin, double u, double v, int64_t* row, int64_t* col, double* p_out,
                      double* u_out, double* v_out) {
  int l = s->ep_nl - 1;
  double w0 = ep_w(s, bin, l, 0, 0), w1 = ep_w(s, bin, l, 0, 1);
  double sm = w0 + w1;
  double p0 = sm > 0.0 ? w0 / sm : 0.5;
  int64_t r = 0, c;
  double p;
  if (u < p0) {
    u = u / p0;
    p = p0;
    c = 0;
  } else {
    u = (u - p0) / (1.0 - p0);
    p = 1.0 - p0;
    c = 1;
  }
  for (; l > 0; l--) {
    double a = ep_w(s, bin, l - 1, 2 * r, 2 * c), b = ep_w(s, bin, l - 1, 2 * r, 2 * c + 1);
    double cc = ep_w(s, bin, l - 1, 2 * r + 1, 2 * c), dd = ep_w(s, bin, l - 1, 2 * r + 1, 2 * c + 1);
    double top = a + b, bot = cc + dd;
    double st = top + bot;
    double pt = st > 0.0 ? top / st : 0.5;
    double left, right;
    if (v < pt) {
      v = v / pt;
      p = p * pt;
      r = 2 * r;
      left = a;
      right = b;
    } else {
      v = (v - pt) / (1.0 - pt);
      p = p * (1.0 - pt);
      r = 2 * r + 1;
      left = cc;
      right = dd;
    }
    double sl = left + right;
    double pl = sl > 0.0 ? left / sl : 0.5;
    if (u < pl) {
      u = u / pl;
      p = p * pl;
      c = 2 * c;
    } else {
      u = (u - pl) / (1.0 - pl);
      p = p * (1.0 - pl);
      c = 2 * c + 1;
    }
  }
  if (u >= 1.0) u = 0.9999999999999999;
  if (u < 0.0) u = 0.0;
  if (v >= 1.0) v = 0.9999999999999999;
  if (v < 0.0) v = 0.0;
  *row = r;
  *col = c;
  *p_out = p;
  *u_out = u;
  *v_out = v;
}

static double ep_pdf(const lwo_scene* s, int bin, int64_t row, int64_t col) {
  int l = s->ep_nl - 1;
  double w0 = ep_w(s, bin, l, 0, 0), w1 = ep_w(s, bin, l, 0, 1);
  double sm = w0 + w1;
  double p0 = sm > 0.0 ? w0 / sm : 0.5;
  int64_t r = 0, c = col >> l;
  double p = c == 0 ? p0 : 1.0 - p0;
  for (; l > 0; l--) {
    double a = ep_w(s, bin, l - 1, 2 * r, 2 * c), b = ep_w(s, bin, l - 1, 2 * r, 2 * c + 1);
    double cc = ep_w(s, bin, l - 1, 2 * r + 1, 2 * c), dd = ep_w(s, bin, l - 1, 2 * r + 1, 2 * c + 1);
    double top = a + b, bot = cc + dd;
    double st = top + bot;
    double pt = st > 0.0 ? top / st : 0.5;
    int64_t rb = (row >> (l - 1)) & 1, cb = (col >> (l - 1)) & 1;
    double left, right;
    if (rb == 0) {
      p = p * pt;
      left = a;
      right = b;
    } else {
      p = p * (1.0 - pt);
      left = cc;
      right = dd;
    }
    double sl = left + right;
    double pl = sl > 0.0 ? left / sl : 0.5;
    p = cb == 0 ? p * pl : p * (1.0 - pl);
    r = 2 * r + rb;
    c = 2 * c + cb;
  }
  return p;
}

int lwo_env_pyramid_info(const lwo_scene* s, int32_t* nlevels) {
  if (nlevels) *nlevels = s->ep_on ? s->ep_nl : 0;
  return s->ep_on;
}

void lwo_env_sample_batch(const lwo_scene* s, const int64_t* packed_normal, const double* uv, int64_t n,
                          int64_t* out_texel, double* out_p, double* out_uv) {
  for (int64_t i = 0; i < n; i++) {
    int64_t row, col;
    ep_sample(s, ep_bin(packed_normal[i]), uv[2 * i], uv[2 * i + 1], &row, &col, out_p + i, out_uv + 2 * i,
              out_uv + 2 * i + 1);
    out_texel[i] = row * s->env_w + col;
  }
}

void lwo_env_pdf_batch(const lwo_scene* s, const int64_t* packed_normal, const int64_t* texel, int64_t n,
                       double* out_p) {
  for (int64_t i = 0; i < n; i++)
    out_p[i] = ep_pdf(s, ep_bin(packed_normal[i]), texel[i] / s->env_w, texel[i] % s->env_w);
}

/* environment lookup: lat-long, y up, row 0 at +y */
static v3 env_eval(const lwo_scene* s, v3 d, int64_t nprev, double* pdf) {
  if (s->env_kind == LW_ENV_CONSTANT) {
    *pdf = s->p_env * LW_INV_FOUR_PI;
    return scl(ld3(s->d.env_constant), s->d.env_scale);
  }
  if (s->env_kind == LW_ENV_IMAGE) {
    double phi = lwo_atan2(d.z, d.x);
    if (phi < 0.0) phi = phi + LW_TWO_PI;
    double sin_t = sqrt(d.x * d.x + d.z * d.z);
    double theta = lwo_atan2(sin_t, d.y);
    int64_t W = s->env_w, H = s->env_h;
    int64_t col = (int64_t)(phi / LW_TWO_PI * (double)W);
    int64_t row = (int64_t)(theta / LW_PI * (double)H);
    if (col >= W) col = W - 1;
    if (row >= H) row = H - 1;
    if (col < 0) col = 0;
    if (row < 0) row = 0;
    int64_t j = row * W + col;
    double pt = s->ep_on ? ep_pdf(s, ep_bin(nprev), row, col) : s->env_pdf[j];
    *pdf = sin_t > 0.0 ? s->p_env * pt * (double)(W * H) / (LW_TWO_PI_SQ * sin_t) : 0.0;
    const float* px = s->env_img + 3 * j;
    return mk((double)px[0] * s->d.env_scale, (double)px[1] * s->d.env_scale, (double)px[2] * s->d.env_scale);
  }
  *pdf = 0.0;
  return mk(0, 0, 0);
}

/* ---- BSDF ------------------------------------------------- */

typedef struct {
  v3 t, b, n;
} frame;

static frame make_frame(v3 n) { /* Duff et al. 2017 */
  frame f;
  double sgn = n.z >= 0.0 ? 1.0 : -1.0;
  double a = -1.0 / (sgn + n.z);
  double b = n.x * n.y * a;
  f.t = mk(1.0 + sgn * n.x * n.x * a, sgn * b, -sgn * n.x);
  f.b = mk(b, sgn + n.y * n.y * a, -n.y);
  f.n = n;
  return f;
}
static v3 to_local(const frame* f, v3 v) { return mk(dot(v, f->t), dot(v, f->b), dot(v, f->n)); }
static v3 to_world(const frame* f, v3 v) {
  return mk((v.x * f->t.x + v.y * f->b.x) + v.z * f->n.x, (v.x * f->t.y + v.y * f->b.y) + v.z * f->n.y,
            (v.x * f->t.z + v.y * f->b.z) + v.z * f->n.z);
}

typedef struct {
  double a[LW_MAX_LAYERS]; /* layer mixture weights */
  double sum_a, inv_sum;
  int nonspec; /* any non-delta layer with a > 0 */
} layerw;

static double schlick(double cosv, double ior) {
  double r0 = (ior - 1.0) / (ior + 1.0);
  double f0 = r0 * r0;
  double m = 1.0 - cosv;
  double m2 = m * m;
  return f0 + (1.0 - f0) * (m2 * m2 * m);
}

static void layer_weights(const lw_material* m, double cos_o, layerw* lw) {
  double r = 1.0;
  lw->sum_a = 0.0;
  lw->nonspec = 0;
  for (int l = 0; l < LW_MAX_LAYERS; l++) {
    lw->a[l] = 0.0;
    if (l >= m->nlayers) continue;
    const lw_layer* L = m->layers + l;
    double a = L->coat ? r * (L->weight * schlick(cos_o, m->ior)) : r * L->weight;
    lw->a[l] = a;
    r = r - a;
    lw->sum_a = lw->sum_a + a;
    if (a > 0.0 && (L->kind == LW_BSDF_DIFFUSE || L->kind == LW_BSDF_GLOSSY)) lw->nonspec = 1;
  }
  lw->inv_sum = lw->sum_a > 0.0 ? 1.0 / lw->sum_a : 0.0;
}

static double ggx_d(double alpha, double cos_h) {
  double a2 = alpha * alpha;
  double t = cos_h * cos_h * (a2 - 1.0) + 1.0;
  return a2 / (LW_PI * (t * t));
}
static double ggx_g1(double alpha, double cos_v) {
  double a2 = alpha * alpha;
  return 2.0 * cos_v / (cos_v + sqrt(a2 + (1.0 - a2) * (cos_v * cos_v)));
}
static double alpha_of(const lw_layer* L) {
  double a = L->roughness;
  if (a < 1e-4) a = 1e-4;
  if (a > 1.0) a = 1.0;
  return a;
}

/* non-delta part of the layered BSDF: f (rgb) and mixture pdf (solid angle) */
static v3 bsdf_eval(const lw_material* m, const layerw* lw, v3 wo, v3 wi, double* pdf) {
  v3 f = mk(0, 0, 0);
  *pdf = 0.0;
  if (wi.z <= 0.0 || wo.z <= 0.0 || !(lw->sum_a > 0.0)) return f;
  for (int l = 0; l < m->nlayers; l++) {
    const lw_layer* L = m->layers + l;
    double a = lw->a[l];
    if (!(a > 0.0)) continue;
    double sel = a * lw->inv_sum;
    if (L->kind == LW_BSDF_DIFFUSE) {
      double k = a * LW_INV_PI;
      f = add(f, mk(L->tint[0] * k, L->tint[1] * k, L->tint[2] * k));
      *pdf = *pdf + sel * (wi.z * LW_INV_PI);
    } else if (L->kind == LW_BSDF_GLOSSY) {
      double al = alpha_of(L);
      v3 h = normalize(add(wo, wi));
      double D = ggx_d(al, h.z);
      double G = ggx_g1(al, wo.z) * ggx_g1(al, wi.z);
      double k = a * (D * G / (4.0 * wo.z * wi.z));
      f = add(f, mk(L->tint[0] * k, L->tint[1] * k, L->tint[2] * k));
      double oh = dot(wo, h);
      if (oh > 0.0) *pdf = *pdf + sel * (D * h.z / (4.0 * oh));
    }
  }
  return f;
}

/* the diffuse and glossy parts of bsdf_eval's f (LPE routing of NEE contributions) */
static void bsdf_eval_split(const lw_material* m, const layerw* lw, v3 wo, v3 wi, v3* fd, v3* fg) {
  *fd = mk(0, 0, 0);
  *fg = mk(0, 0, 0);
  if (wi.z <= 0.0 || wo.z <= 0.0 || !(lw->sum_a > 0.0)) return;
  for (int l = 0; l < m->nlayers; l++) {
    const lw_layer* L = m->layers + l;
    double a = lw->a[l];
    if (!(a > 0.0)) continue;
    if (L->kind == LW_BSDF_DIFFUSE) {
      double k = a * LW_INV_PI;
      *fd = add(*fd, mk(L->tint[0] * k, L->tint[1] * k, L->tint[2] * k));
    } else if (L->kind == LW_BSDF_GLOSSY) {
      double al = alpha_of(L);
      v3 h = normalize(add(wo, wi));
      double D = ggx_d(al, h.z);
      double G = ggx_g1(al, wo.z) * ggx_g1(al, wi.z);
      double k = a * (D * G / (4.0 * wo.z * wi.z));
      *fg = add(*fg, mk(L->tint[0] * k, L->tint[1] * k, L->tint[2] * k));
    }
  }
}

static double fresnel_dielectric(double cos_i, double eta) { /* eta = eta_i / eta_t */
  double sin2t = eta * eta * (1.0 - cos_i * cos_i);
  if (sin2t >= 1.0) return 1.0;
  double cos_t = sqrt(1.0 - sin2t);
  double rs = (eta * cos_i - cos_t) / (eta * cos_i + cos_t);
  double rp = (cos_i - eta * cos_t) / (cos_i + eta * cos_t);
  return 0.5 * (rs * rs + rp * rp);
}

typedef struct {
  v3 wi;       /* local */
  v3 weight;   /* f * cos / pdf */
  double pdf;  /* mixture pdf (non-delta) */
  int delta;
  int transmit;
  int event; /* LPE event of the sampled lobe */
} bsample;

/* returns 0 if no valid sample */
static int bsdf_sample(const lw_material* m, const layerw* lw, v3 wo, int front, double u, double v, bsample* bs) {
  if (!(lw->sum_a > 0.0) || wo.z <= 0.0) return 0;
  double x = u * lw->sum_a;
  int pick = -1;
  double cum = 0.0, prev = 0.0;
  for (int l = 0; l < m->nlayers; l++) {
    if (!(lw->a[l] > 0.0)) continue;
    prev = cum;
    cum = cum + lw->a[l];
    pick = l;
    if (x < cum) break;
  }
  if (pick < 0) return 0;
  double ur = (x - prev) / lw->a[pick];
  if (ur < 0.0) ur = 0.0;
  if (ur >= 1.0) ur = 0.9999999999999999;
  const lw_layer* L = m->layers + pick;
  bs->delta = 0;
  bs->transmit = 0;
  bs->event = L->kind == LW_BSDF_DIFFUSE ? LW_EV_RD : (L->kind == LW_BSDF_GLOSSY ? LW_EV_RG : LW_EV_RS);
  if (L->kind == LW_BSDF_DIFFUSE) {
    double r = sqrt(ur), sp, cp;
    lwo_sincos2pi(v, &sp, &cp);
    double z = 1.0 - ur;
    bs->wi = mk(r * cp, r * sp, sqrt(z > 0.0 ? z : 0.0));
  } else if (L->kind == LW_BSDF_GLOSSY) {
    double al = alpha_of(L);
    double tan2 = al * al * ur / (1.0 - ur);
    double ch = 1.0 / sqrt(1.0 + tan2);
    double sh2 = 1.0 - ch * ch;
    double sh = sqrt(sh2 > 0.0 ? sh2 : 0.0);
    double sp, cp;
    lwo_sincos2pi(v, &sp, &cp);
    v3 h = mk(sh * cp, sh * sp, ch);
    double oh = dot(wo, h);
    bs->wi = sub(scl(h, 2.0 * oh), wo);
  } else if (L->kind == LW_BSDF_SPECULAR_REFLECT) {
    bs->wi = mk(-wo.x, -wo.y, wo.z);
    bs->delta = 1;
    bs->weight = mk(lw->sum_a * L->tint[0], lw->sum_a * L->tint[1], lw->sum_a * L->tint[2]);
    bs->pdf = 0.0;
    return 1;
  } else { /* specular transmit: dielectric, choose reflect/refract by Fresnel */
    double eta = front ? 1.0 / m->ior : m->ior;
    double F = fresnel_dielectric(wo.z, eta);
    bs->delta = 1;
    bs->pdf = 0.0;
    if (ur < F) {
      bs->wi = mk(-wo.x, -wo.y, wo.z);
      bs->weight = mk(lw->sum_a * L->tint[0], lw->sum_a * L->tint[1], lw->sum_a * L->tint[2]);
    } else {
      double sin2t = eta * eta * (1.0 - wo.z * wo.z);
      double cos_t = sqrt(1.0 - sin2t);
      bs->wi = mk(-eta * wo.x, -eta * wo.y, -cos_t);
      bs->transmit = 1;
      bs->event = LW_EV_TS;
      double k = lw->sum_a * (eta * eta);
      bs->weight = mk(k * L->tint[0], k * L->tint[1], k * L->tint[2]);
    }
    return 1;
  }
  if (bs->wi.z <= 0.0) return 0;
  double pdf;
  v3 f = bsdf_eval(m, lw, wo, bs->wi, &pdf);
  if (!(pdf > 0.0)) return 0;
  double k = bs->wi.z / pdf;
  bs->weight = mk(f.x * k, f.y * k, f.z * k);
  bs->pdf = pdf;
  return 1;
}

static int has_light(const lwo_scene* s) { return s->nemit > 0 || s->env_kind != LW_ENV_NONE; }

static void accumulate(int64_t* fb, int64_t pix, v3 L, lw_render_stats* st) {
  double c[3] = {L.x, L.y, L.z};
  for (int k = 0; k < 3; k++) {
    double v = c[k];
    if (!(v == v) || v == INFINITY || v == -INFINITY) {
      if (st) st->nonfinite++;
      v = 0.0;
    }
    if (v < 0.0) v = 0.0;
    if (v > LW_FB_SAMPLE_CLAMP) v = LW_FB_SAMPLE_CLAMP;
    fb[3 * pix + k] += (int64_t)llrint(v * 1048576.0);
  }
}

/* one path, DESIGN.md §4 (SPEC.md:385-402 trace_eye_path / next_event) */
/* light-path-expression layers (lwo_render_lpe): product DFA + layer framebuffers */
typedef struct {
  const int16_t* trans;
  const uint8_t* accept;
  int start, nlayers;
  int64_t* fb;
  int64_t npix;
} lpe_ctx;

static int lpe_step(const lpe_ctx* x, int state, int ev) { return x->trans[state * LW_EV_COUNT + ev]; }

/* same per-contribution fixed-point rule as the device (lw_lpe_route) */
static void lpe_route(const lpe_ctx* x, int state, int64_t pix, v3 c) {
  int m = x->accept[state];
  if (!m) return;
  double v[3] = {c.x, c.y, c.z};
  int64_t q[3];
  for (int k = 0; k < 3; k++) {
    double y = v[k];
    if (!(y == y) || y == INFINITY || y == -INFINITY || y < 0.0) y = 0.0;
    if (y > LW_FB_SAMPLE_CLAMP) y = LW_FB_SAMPLE_CLAMP;
    q[k] = (int64_t)llrint(y * 1048576.0);
  }
  for (int l = 0; l < x->nlayers; l++)
    if ((m >> l) & 1)
      for (int k = 0; k < 3; k++) x->fb[(int64_t)l * x->npix * 3 + 3 * pix + k] += q[k];
}

/* light half of next-event estimation (device: lw_nee_light_sample): from p with
 * facing normal ngf and the NEE uniforms, the environment (p_env) or an emitter, the direction wi,
 * its radiance, solid-angle pdf (selection included) and the shadow-ray length; e_out the emitter
 * (-1 = environment).  Returns 0 when the sample carries no light. */
static int nee_light_sample(const lwo_scene* s, v3 p, v3 ngf, double ul, double vl, v3* wi, v3* Le, double* pl,
                            double* tmax_sh, int64_t* e_out) {
  *wi = mk(0, 0, 0);
  *Le = mk(0, 0, 0);
  *pl = 0.0;
  *tmax_sh = INFINITY;
  *e_out = -1;
  int ok = 0;
  if (s->env_kind != LW_ENV_NONE && ul < s->p_env) {
    double ue = s->nemit > 0 ? ul / s->p_env : ul;
    if (s->env_kind == LW_ENV_CONSTANT) {
      double z = 1.0 - 2.0 * ue;
      double r2 = 1.0 - z * z;
      double r = sqrt(r2 > 0.0 ? r2 : 0.0), sp, cp;
      lwo_sincos2pi(vl, &sp, &cp);
      *wi = mk(r * cp, z, r * sp);
      *pl = s->p_env * LW_INV_FOUR_PI;
      *Le = scl(ld3(s->d.env_constant), s->d.env_scale);
      ok = 1;
    } else {
      double ur, vr, pt;
      int64_t j, row, col;
      if (s->ep_on) {
        ep_sample(s, ep_bin(lwo_oct_encode(ngf.x, ngf.y, ngf.z)), ue, vl, &row, &col, &pt, &ur, &vr);
        j = row * s->env_w + col;
      } else {
        double u1;
        row = alias_sample(s->env_rprob, s->env_ralias, s->env_h, ue, &u1);
        col = alias_sample(s->env_prob + row * s->env_w, s->env_alias + row * s->env_w, s->env_w, u1, &ur);
        j = row * s->env_w + col;
        vr = vl;
        pt = s->env_pdf[j];
      }
      double uu = ((double)col + ur) / (double)s->env_w;
      double vv2 = ((double)row + vr) / (double)s->env_h;
      double st_, ct, sp, cp;
      lwo_sincos2pi(vv2 * 0.5, &st_, &ct);
      lwo_sincos2pi(uu, &sp, &cp);
      *wi = mk(st_ * cp, ct, st_ * sp);
      if (st_ > 0.0) {
        *pl = s->p_env * pt * (double)((int64_t)s->env_w * s->env_h) / (LW_TWO_PI_SQ * st_);
        const float* px = s->env_img + 3 * j;
        *Le = mk((double)px[0] * s->d.env_scale, (double)px[1] * s->d.env_scale, (double)px[2] * s->d.env_scale);
        ok = 1;
      }
    }
  } else if (s->nemit > 0) {
    double ut = s->env_kind != LW_ENV_NONE ? (ul - s->p_env) / (1.0 - s->p_env) : ul;
    double ur, psel;
    int64_t le;
    if (s->lt) {
      v3 xr = offset_origin(p, ngf, ngf);
      v3 nr = lt_ref_normal(lwo_oct_encode(ngf.x, ngf.y, ngf.z));
      le = lt_sample(s, xr, nr, ut, &psel, &ur);
    } else {
      le = alias_sample(s->emit_prob, s->emit_alias, s->nemit, ut, &ur);
      psel = s->emit_pdf[le];
    }
    *e_out = le;
    const double* lv = s->verts + 9 * s->emit_tri[le];
    v3 l0 = ld3(lv), l1 = ld3(lv + 3), l2 = ld3(lv + 6);
    double su = sqrt(ur);
    double b0 = 1.0 - su, b1 = vl * su;
    double b2 = (1.0 - b0) - b1;
    v3 q = bary3(l0, l1, l2, b0, b1, b2);
    v3 dl = sub(q, p);
    double dist2 = dot(dl, dl);
    double dist = sqrt(dist2);
    double inv_dist = 1.0 / dist;
    *wi = mk(dl.x * inv_dist, dl.y * inv_dist, dl.z * inv_dist);
    v3 ngl = normalize(cross(sub(l1, l0), sub(l2, l0)));
    double cos_l = -dot(ngl, *wi);
    if (s->emit_two[le]) cos_l = fabs(cos_l);
    if (cos_l > 0.0 && dist > 0.0) {
      *pl = (s->p_tri * psel / s->emit_area[le]) * dist2 / cos_l;
      *Le = ld3(s->emit_rad + 3 * le);
      *tmax_sh = dist * (1.0 - 1e-7);
      ok = 1;
    }
  }
  return ok;
}

/* solid-angle light-sampling pdf of emitter e hit at distance t from o along d (geometric normal ng;
 * nprev: packed facing normal of the vertex the ray left) -- device lw_emitter_hit_pdf */
static double emitter_hit_pdf(const lwo_scene* s, int64_t e, v3 o, int64_t nprev, v3 ng, v3 d, double t) {
  double cos_l = fabs(dot(ng, d));
  double psel = s->lt ? lt_pdf(s, e, o, lt_ref_normal(nprev)) : s->emit_pdf[e];
  double pdf_area = s->p_tri * psel / s->emit_area[e];
  return pdf_area * (t * t) / cos_l;
}

static v3 trace_path_lpe(const rctx* c, int64_t index, lw_render_stats* st, const lpe_ctx* lpe, int64_t pix);

/* compressed path state (lw_render_params.compact_state; device: lw_q32 /
 * lw_oct_dir in lw_integrator.cuh): FP32 throughput, radiance and pdf, directions through the
 * reference's octahedral codec (_kernels.py:233-299), quantised where each value is produced */
static double q32(double x) { return (double)(float)x; }
static v3 q32v(v3 a) { return mk(q32(a.x), q32(a.y), q32(a.z)); }
static v3 dir_q(v3 d) {
  double o[3];
  lwo_oct_decode(lwo_oct_encode(d.x, d.y, d.z), o);
  return normalize(mk(o[0], o[1], o[2]));
}

/* balance heuristic and the estimator switch of lw_render_params.estimator
 * (SPEC.md:400-402): weight of emission reached by BSDF sampling after a non-specular vertex */
static double mis_balance(double a, double b) { return a / (a + b); }
static double bsdf_hit_weight(int est, double pdf_bsdf, double pdf_light) {
  return est == LW_EST_MIS ? mis_balance(pdf_bsdf, pdf_light) : (est == LW_EST_BSDF ? 1.0 : 0.0);
}

static v3 trace_path(const rctx* c, int64_t index, lw_render_stats* st) { return trace_path_lpe(c, index, st, NULL, 0); }

static v3 trace_path_lpe(const rctx* c, int64_t index, lw_render_stats* st, const lpe_ctx* lpe, int64_t pix) {
  const lwo_scene* s = c->s;
  int depth = c->p->max_depth;
  v3 o, d;
  camera_ray(c, index, &o, &d);
  const int compact = c->p->compact_state != 0;
  if (compact) d = dir_q(d);
  v3 beta = mk(1, 1, 1), L = mk(0, 0, 0);
  int spec_prev = 1;
  double pdf_prev = 0.0;
  int64_t nprev = 0; /* packed facing normal of the previous vertex (light-tree MIS) */
  int lst = lpe ? lpe_step(lpe, lpe->start, LW_EV_C) : 0; /* LPE automaton state */
  for (int b = 0; b < depth; b++) {
    hitrec h;
    trace_closest(s, &o.x, &d.x, INFINITY, &h);
    if (st) st->rays_extension++;
    if (h.tri < 0) {
      if (s->env_kind != LW_ENV_NONE) {
        double pe;
        v3 Le = env_eval(s, d, nprev, &pe);
        double w = spec_prev ? 1.0 : bsdf_hit_weight(c->p->estimator, pdf_prev, pe);
        v3 cc = mk(beta.x * Le.x * w, beta.y * Le.y * w, beta.z * Le.z * w);
        L = compact ? q32v(add(L, cc)) : add(L, cc);
        if (lpe) lpe_route(lpe, lpe_step(lpe, lst, LW_EV_E), pix, cc);
      }
      break;
    }
    const double* vv = s->verts + 9 * h.tri;
    v3 v0 = ld3(vv), v1 = ld3(vv + 3), v2 = ld3(vv + 6);
    double w = (1.0 - h.bu) - h.bv;
    v3 p = bary3(v0, v1, v2, w, h.bu, h.bv);
    v3 e1 = sub(v1, v0), e2 = sub(v2, v0);
    v3 ng = normalize(cross(e1, e2));
    int front = dot(ng, d) < 0.0;
    /* emission with MIS against the light-sampling strategy */
    int64_t e = s->emit_of_tri[h.tri];
    if (e >= 0 && s->nemit > 0 && (front || s->emit_two[e])) {
      v3 Le = ld3(s->emit_rad + 3 * e);
      double wm = 1.0;
      if (!spec_prev) wm = bsdf_hit_weight(c->p->estimator, pdf_prev, emitter_hit_pdf(s, e, o, nprev, ng, d, h.t));
      v3 cc = mk(beta.x * Le.x * wm, beta.y * Le.y * wm, beta.z * Le.z * wm);
      L = compact ? q32v(add(L, cc)) : add(L, cc);
      if (lpe) lpe_route(lpe, lpe_step(lpe, lst, LW_EV_L), pix, cc);
    }
    if (b == depth - 1) break;
    /* shading frame */
    const double* nn = s->normals + 9 * h.tri;
    v3 ns = bary3(ld3(nn), ld3(nn + 3), ld3(nn + 6), w, h.bu, h.bv);
    double nl = dot(ns, ns);
    ns = nl > 0.0 ? scl(ns, 1.0 / sqrt(nl)) : ng;
    v3 wo = neg(d);
    v3 ngf = front ? ng : neg(ng);
    if (dot(ns, ngf) < 0.0) ns = neg(ns);
    if (dot(ns, wo) <= 0.0) ns = ngf;
    frame fr = make_frame(ns);
    v3 wol = to_local(&fr, wo);
    const lw_material* m = s->materials + s->material[h.tri];
    layerw lw;
    layer_weights(m, wol.z, &lw);
    int64_t bd = 4 + 8 * (int64_t)b;
    /* next-event estimation */
    if (lw.nonspec && has_light(s) && c->p->estimator != LW_EST_BSDF) {
      double ul = qmc(c, bd + 2, index), vl = qmc(c, bd + 3, index);
      v3 wi, Le;
      double pl, tmax_sh;
      int64_t le_;
      int ok = nee_light_sample(s, p, ngf, ul, vl, &wi, &Le, &pl, &tmax_sh, &le_);
      if (ok && pl > 0.0 && dot(ngf, wi) > 0.0) {
        v3 wil = to_local(&fr, wi);
        double pb;
        v3 f = bsdf_eval(m, &lw, wol, wil, &pb);
        if (f.x > 0.0 || f.y > 0.0 || f.z > 0.0) {
          double wm = c->p->estimator == LW_EST_NEE ? 1.0 : mis_balance(pl, pb);
          double k = (wil.z * wm) / pl;
          v3 contrib = mk(beta.x * f.x * Le.x * k, beta.y * f.y * Le.y * k, beta.z * f.z * Le.z * k);
          v3 so = offset_origin(p, ngf, wi);
          if (st) st->rays_shadow++;
          if (!trace_any(s, &so.x, &wi.x, tmax_sh)) {
            L = compact ? q32v(add(L, contrib)) : add(L, contrib);
            if (lpe) { /* diffuse and glossy parts, terminal L (triangle) or E (environment) */
              v3 fd, fg;
              bsdf_eval_split(m, &lw, wol, wil, &fd, &fg);
              int term = tmax_sh == INFINITY ? LW_EV_E : LW_EV_L;
              lpe_route(lpe, lpe_step(lpe, lpe_step(lpe, lst, LW_EV_RD), term), pix,
                        mk(beta.x * fd.x * Le.x * k, beta.y * fd.y * Le.y * k, beta.z * fd.z * Le.z * k));
              lpe_route(lpe, lpe_step(lpe, lpe_step(lpe, lst, LW_EV_RG), term), pix,
                        mk(beta.x * fg.x * Le.x * k, beta.y * fg.y * Le.y * k, beta.z * fg.z * Le.z * k));
            }
          }
        }
      }
    }
    /* BSDF sampling */
    bsample bs;
    double ub = qmc(c, bd + 0, index), vb = qmc(c, bd + 1, index);
    if (!bsdf_sample(m, &lw, wol, front, ub, vb, &bs)) break;
    if (lpe) lst = lpe_step(lpe, lst, bs.event);
    v3 wi = to_world(&fr, bs.wi);
    if (compact) wi = dir_q(wi);
    double gside = dot(ngf, wi);
    if (bs.transmit ? !(gside < 0.0) : !(gside > 0.0)) break;
    beta = mk(beta.x * bs.weight.x, beta.y * bs.weight.y, beta.z * bs.weight.z);
    spec_prev = bs.delta;
    pdf_prev = compact ? q32(bs.pdf) : bs.pdf;
    if (b >= c->p->rr_start) {
      double q = beta.x;
      if (beta.y > q) q = beta.y;
      if (beta.z > q) q = beta.z;
      if (q > 1.0) q = 1.0;
      double ur = qmc(c, bd + 4, index);
      if (!(ur < q)) break;
      double inv_q = 1.0 / q;
      beta = mk(beta.x * inv_q, beta.y * inv_q, beta.z * inv_q);
    }
    if (compact) beta = q32v(beta);
    o = offset_origin(p, ngf, wi);
    d = wi;
    nprev = lwo_oct_encode(ngf.x, ngf.y, ngf.z);
  }
  return L;
}

void lwo_render_lpe(const lwo_scene* s, const lw_render_params* p, int64_t pix_begin, int64_t pix_end,
                    int64_t it_begin, int64_t it_end, int64_t* fb, int nlayers, int nstates, const int16_t* trans,
                    const uint8_t* accept, int start, int64_t* layer_fb, int nthreads, lw_render_stats* stats) {
  rctx c = {s, p};
  int64_t P = (int64_t)p->width * p->height;
  lpe_ctx x = {trans, accept, start, nlayers, layer_fb, P};
  (void)nstates;
  int64_t ext = 0, shd = 0, nonf = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads) reduction(+ : ext, shd, nonf)
#endif
  for (int64_t pix = pix_begin; pix < pix_end; pix++) {
    lw_render_stats st;
    memset(&st, 0, sizeof(st));
    for (int64_t it = it_begin; it < it_end; it++) {
      v3 L = trace_path_lpe(&c, it * P + pix, &st, &x, pix);
      accumulate(fb, pix, L, &st);
    }
    ext += st.rays_extension;
    shd += st.rays_shadow;
    nonf += st.nonfinite;
  }
  (void)nthreads;
  if (stats) {
    stats->paths += (pix_end - pix_begin) * (it_end - it_begin);
    stats->rays_extension += ext;
    stats->rays_shadow += shd;
    stats->nonfinite += nonf;
  }
}

void lwo_render(const lwo_scene* s, const lw_render_params* p, int64_t pix_begin, int64_t pix_end, int64_t it_begin,
                int64_t it_end, int64_t* fb, int nthreads, lw_render_stats* stats) {
  rctx c = {s, p};
  int64_t P = (int64_t)p->width * p->height;
  int64_t ext = 0, shd = 0, nonf = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads) reduction(+ : ext, shd, nonf)
#endif
  for (int64_t pix = pix_begin; pix < pix_end; pix++) {
    lw_render_stats st;
    memset(&st, 0, sizeof(st));
    for (int64_t it = it_begin; it < it_end; it++) {
      v3 L = trace_path(&c, it * P + pix, &st);
      accumulate(fb, pix, L, &st);
    }
    ext += st.rays_extension;
    shd += st.rays_shadow;
    nonf += st.nonfinite;
  }
  (void)nthreads;
  if (stats) {
    stats->paths += (pix_end - pix_begin) * (it_end - it_begin);
    stats->rays_extension += ext;
    stats->rays_shadow += shd;
    stats->nonfinite += nonf;
  }
}

/* ---- known-answer surface of the render math (device: lw_bsdf_eval_batch, ...) ---------------- */

void lwo_bsdf_eval_batch(const lw_material* m, const double* wo, const double* wi, int64_t n, double* out_f,
                         double* out_pdf) {
  for (int64_t i = 0; i < n; i++) {
    v3 a = ld3(wo + 3 * i), b = ld3(wi + 3 * i);
    layerw lw;
    layer_weights(m, a.z, &lw);
    double pdf;
    v3 f = bsdf_eval(m, &lw, a, b, &pdf);
    out_f[3 * i] = f.x;
    out_f[3 * i + 1] = f.y;
    out_f[3 * i + 2] = f.z;
    out_pdf[i] = pdf;
  }
}

void lwo_bsdf_sample_batch(const lw_material* m, const double* wo, const int32_t* front, const double* uv, int64_t n,
                           double* out_wi, double* out_weight, double* out_pdf, int32_t* out_flags) {
  for (int64_t i = 0; i < n; i++) {
    v3 a = ld3(wo + 3 * i);
    layerw lw;
    layer_weights(m, a.z, &lw);
    bsample bs;
    memset(&bs, 0, sizeof(bs));
    int ok = bsdf_sample(m, &lw, a, front[i] != 0, uv[2 * i], uv[2 * i + 1], &bs);
    out_wi[3 * i] = bs.wi.x;
    out_wi[3 * i + 1] = bs.wi.y;
    out_wi[3 * i + 2] = bs.wi.z;
    out_weight[3 * i] = bs.weight.x;
    out_weight[3 * i + 1] = bs.weight.y;
    out_weight[3 * i + 2] = bs.weight.z;
    out_pdf[i] = bs.pdf;
    out_flags[i] = (ok ? 1 : 0) | (bs.delta ? 2 : 0) | (bs.transmit ? 4 : 0) | (bs.event << 8);
  }
}

void lwo_nee_light_sample_batch(const lwo_scene* s, const double* p, const double* ngf, const double* uv, int64_t n,
                                double* out_wi, double* out_le, double* out_pdf, double* out_tmax, int64_t* out_e) {
  for (int64_t i = 0; i < n; i++) {
    v3 wi, Le;
    double pl, tm;
    int64_t e;
    int ok = nee_light_sample(s, ld3(p + 3 * i), ld3(ngf + 3 * i), uv[2 * i], uv[2 * i + 1], &wi, &Le, &pl, &tm, &e);
    out_wi[3 * i] = wi.x;
    out_wi[3 * i + 1] = wi.y;
    out_wi[3 * i + 2] = wi.z;
    out_le[3 * i] = Le.x;
    out_le[3 * i + 1] = Le.y;
    out_le[3 * i + 2] = Le.z;
    out_pdf[i] = ok ? pl : 0.0;
    out_tmax[i] = tm;
    out_e[i] = e;
  }
}

void lwo_emission_pdf_batch(const lwo_scene* s, const double* o, const double* d, const int32_t* nprev, int64_t n,
                            double* out_le, double* out_pdf, int64_t* out_e) {
  for (int64_t i = 0; i < n; i++) {
    v3 oo = ld3(o + 3 * i), dd = ld3(d + 3 * i);
    hitrec h;
    trace_closest(s, &oo.x, &dd.x, INFINITY, &h);
    v3 Le = mk(0, 0, 0);
    double pdf = 0.0;
    int64_t e = -2;
    if (h.tri < 0) {
      e = -1;
      Le = env_eval(s, dd, nprev[i], &pdf);
    } else {
      const double* vv = s->verts + 9 * h.tri;
      v3 v0 = ld3(vv), v1 = ld3(vv + 3), v2 = ld3(vv + 6);
      v3 ng = normalize(cross(sub(v1, v0), sub(v2, v0)));
      int front = dot(ng, dd) < 0.0;
      int64_t k = s->emit_of_tri[h.tri];
      if (k >= 0 && s->nemit > 0 && (front || s->emit_two[k])) {
        e = k;
        Le = ld3(s->emit_rad + 3 * k);
        pdf = emitter_hit_pdf(s, k, oo, nprev[i], ng, dd, h.t);
      }
    }
    out_le[3 * i] = Le.x;
    out_le[3 * i + 1] = Le.y;
    out_le[3 * i + 2] = Le.z;
    out_pdf[i] = pdf;
    out_e[i] = e;
  }
}
