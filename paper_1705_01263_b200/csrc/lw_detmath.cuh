// lw_detmath.cuh -- deterministic device math.
//
//  * lw_glibc_log: operation-for-operation port of glibc 2.39's FMA log variant
//    (`__log_fma`, the ARM optimized-routines algorithm) that the reference's pixel
//    filter calls through libm (_kernels.py:95, 100).  Constants come from
//    lw_glibc_log_data.h (tools/extract_glibc_log.py).  The FMA placement below was
//    read off the variant's machine code; every other op is a plain IEEE op.
//  * lw_gauss_filter_offset: _kernels.py:87-129 (Acklam inverse CDF, 3-sigma clamp).
//  * lw_sincos2pi / lw_atan2: basic-op-only series restated from the oracle
//    (oracle/lw_oracle.c) so the render path is bit-identical on CPU and GPU.
#pragma once
#include "lw_common.cuh"
#include "lw_glibc_log_data.h"

__device__ const double lw_glibc_log_tab[256] = LW_GLIBC_LOG_TAB_INIT;

// log(x) for normal x outside [1-2^-4, 1+0x1.09p-4) (the reference only feeds
// p in [Phi(-3), 0.02425]); other inputs use CUDA's log.
__device__ __forceinline__ double lw_glibc_log(double x) {
  uint64_t ix = (uint64_t)__double_as_longlong(x);
  uint32_t top = (uint32_t)(ix >> 48);
  if (ix - 0x3fee000000000000ULL < 0x3090000000000ULL || top - 0x0010u >= 0x7ff0u - 0x0010u) return log(x);
  uint64_t tmp = ix - 0x3fe6000000000000ULL;
  int i = (int)((tmp >> 45) & 127);
  int k = (int)((int64_t)tmp >> 52);
  uint64_t iz = ix - (tmp & (0xfffULL << 52));
  double z = __longlong_as_double((long long)iz);
  double invc = __ldg(&lw_glibc_log_tab[2 * i]);
  double logc = __ldg(&lw_glibc_log_tab[2 * i + 1]);
  double kd = (double)k;
  double w = __fma_rn(kd, LW_GLIBC_LOG_LN2HI, logc);
  double r = __fma_rn(z, invc, -1.0);
  double hi = __dadd_rn(r, w);
  double r2 = __dmul_rn(r, r);
  double lo = __fma_rn(kd, LW_GLIBC_LOG_LN2LO, __dadd_rn(__dsub_rn(w, hi), r));
  double r3 = __dmul_rn(r, r2);
  double p = __fma_rn(__fma_rn(r, LW_GLIBC_LOG_A4, LW_GLIBC_LOG_A3), r2, __fma_rn(r, LW_GLIBC_LOG_A2, LW_GLIBC_LOG_A1));
  return __dadd_rn(__fma_rn(r3, p, __fma_rn(r2, LW_GLIBC_LOG_A0, lo)), hi);
}

// _kernels.py:87-109
__device__ __forceinline__ double lw_norm_inv_cdf(double p) {
  double q, r;
  if (p <= 0.0) return -38.0;
  if (p >= 1.0) return 38.0;
  if (p < 0.02425 || p > 1.0 - 0.02425) {
    double neg = p < 0.02425 ? 1.0 : -1.0;
    q = sqrt(-2.0 * lw_glibc_log(p < 0.02425 ? p : 1.0 - p));
    double num = ((((-7.784894002430293e-03 * q - 3.223964580411365e-01) * q - 2.400758277161838e00) * q -
                   2.549732539343734e00) * q + 4.374664141464968e00) * q + 2.938163982698783e00;
    double den = (((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e00) * q +
                  3.754408661907416e00) * q + 1.0;
    // -(num)/den == (-num)/den exactly (negation is exact)
    return (neg * num) / den;
  }
  q = p - 0.5;
  r = q * q;
  return (((((-3.969683028665376e01 * r + 2.209460984245205e02) * r - 2.759285104469687e02) * r +
            1.383577518672690e02) * r - 3.066479806614716e01) * r + 2.506628277459239e00) * q /
         (((((-5.447609879822406e01 * r + 1.615858368580409e02) * r - 1.556989798598866e02) * r +
            6.680131188771972e01) * r - 1.328068155288572e01) * r + 1.0);
}

// _kernels.py:121-129
__device__ __forceinline__ double lw_gauss_filter_offset(double u) {
  double p = 0.0013498980316300933 + u * (0.9986501019683699 - 0.0013498980316300933);
  double x = lw_norm_inv_cdf(p);
  if (x < -3.0) x = -3.0;
  if (x > 3.0) x = 3.0;
  return 0.5 * x;
}

#define LW_PI 3.141592653589793
#define LW_TWO_PI 6.283185307179586
#define LW_HALF_PI 1.5707963267948966
#define LW_INV_PI 0.3183098861837907
#define LW_INV_FOUR_PI 0.07957747154594767
#define LW_TWO_PI_SQ 19.739208802178716

// sin/cos of 2*pi*u (oracle: lwo_sincos2pi)
__host__ __device__ __forceinline__ void lw_sincos2pi(double u, double* s, double* c) {
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
  double ss = q == 0 ? sp : (q == 1 ? cp : (q == 2 ? -sp : -cp));
  double cc = q == 0 ? cp : (q == 1 ? -sp : (q == 2 ? -cp : sp));
  *s = ss;
  *c = cc;
}

// atan2 from two argument halvings and an odd series (oracle: lwo_atan2)
__device__ __forceinline__ double lw_atan2(double y, double x) {
  double ax = fabs(x), ay = fabs(y);
  bool swap = ay > ax;
  double num = swap ? ax : ay, den = swap ? ay : ax;
  double t = den == 0.0 ? 0.0 : num / den;
  double h = t / (1.0 + sqrt(1.0 + t * t));
  h = h / (1.0 + sqrt(1.0 + h * h));
  double h2 = h * h;
  double p = -1.0 / 23.0;
  p = p * h2 + 1.0 / 21.0;
  p = p * h2 + -1.0 / 19.0;
  p = p * h2 + 1.0 / 17.0;
  p = p * h2 + -1.0 / 15.0;
  p = p * h2 + 1.0 / 13.0;
  p = p * h2 + -1.0 / 11.0;
  p = p * h2 + 1.0 / 9.0;
  p = p * h2 + -1.0 / 7.0;
  p = p * h2 + 1.0 / 5.0;
  p = p * h2 + -1.0 / 3.0;
  p = p * h2 + 1.0;
  double rr = 4.0 * (h * p);
  if (swap) rr = LW_HALF_PI - rr;
  if (x < 0.0) rr = LW_PI - rr;
  if (y < 0.0) rr = -rr;
  return rr;
}

// octahedral packing, _kernels.py:233-299
__host__ __device__ __forceinline__ long long lw_oct_encode(double x, double y, double z) {
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
  long long eu = (long long)floor((u + 1.0) * 0.5 * 65535.0 + 0.5);
  long long ev = (long long)floor((v + 1.0) * 0.5 * 65535.0 + 0.5);
  eu = eu < 0 ? 0 : (eu > 65535 ? 65535 : eu);
  ev = ev < 0 ? 0 : (ev > 65535 ? 65535 : ev);
  return (eu << 16) | ev;
}

__host__ __device__ __forceinline__ v3 lw_oct_decode(long long packed) {
  long long eu = (packed >> 16) & 0xFFFF, ev = packed & 0xFFFF;
  double u = (double)eu / 65535.0 * 2.0 - 1.0;
  double v = (double)ev / 65535.0 * 2.0 - 1.0;
  double z = 1.0 - fabs(u) - fabs(v);
  double x = u, y = v;
  if (z < 0.0) {
    x = (1.0 - fabs(v)) * (u >= 0.0 ? 1.0 : -1.0);
    y = (1.0 - fabs(u)) * (v >= 0.0 ? 1.0 : -1.0);
  }
  return mk3(x, y, z);
}
