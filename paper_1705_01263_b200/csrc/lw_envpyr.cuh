// lw_envpyr.cuh -- environment importance pyramid with normal-binned top levels (SURVEY.md §8f
// row 2; PAPER.md:262-276, SPEC.md:185-188, 222-230 EnvPyramid / sample_env / env_pdf).
//
// Level 0 is the lat-long image's sampling weight (luminance * sin(theta), the same weights the
// alias table uses); level l+1 texel = sum of its 2x2 children, up to a 1 x 2 top level (images
// are 2H x H with H a power of two).  Sampling descends the quadtree choosing the row half with v
// and the column half with u (both rescaled), so a texel's probability is the product of the
// conditionals along its path; the same product recomputed from a direction's texel is the MIS
// pdf.  The top LW_EP_TOP levels exist once per normal bin (4 x 4 cells of the octahedral map of
// the facing geometric normal): their weights are multiplied by a conservative bound on the
// cosine between the bin's normals and the texel's directions, floored at 1/64 so no texel with
// radiance gets probability zero ("weighting for the top levels is done quite conservatively").
//
// Restated operation for operation in oracle/lw_oracle.c (ep_*): bit-identical samples and pdfs.
#pragma once
#include "lw_common.cuh"
#include "lw_detmath.cuh"

#define LW_EP_BINS 16
#define LW_EP_TOP 5
#define LW_EP_MAXLEV 24
#define LW_EP_CWMIN 0.015625  // 1/64

struct LwEnvPyr {
  const double* lvl;  // all levels, level l at off[l], row-major (H >> l) x (W >> l)
  const double* top;  // per bin: the top levels [nl - ntop, nl), bin b at b * top_stride
  long long off[LW_EP_MAXLEV];
  long long toff[LW_EP_MAXLEV];  // offset of level l inside a bin block (levels >= nl - ntop)
  long long top_stride;
  int nl, ntop, W, H;
};

// normal bin of an octahedral-packed normal: top two bits of each 16-bit coordinate
__host__ __device__ __forceinline__ int lw_ep_bin(long long packed) {
  return (int)(((packed >> 30) & 3) * 4 + ((packed >> 14) & 3));
}

__device__ __forceinline__ double lw_ep_w(const LwEnvPyr& P, int bin, int l, long long r, long long c) {
  long long wl = (long long)P.W >> l;
  if (l >= P.nl - P.ntop) return __ldg(P.top + bin * P.top_stride + P.toff[l] + r * wl + c);
  return __ldg(P.lvl + P.off[l] + r * wl + c);
}

// sample_env: base texel (row, col), its probability, and the in-texel remainders of (u, v)
__device__ __forceinline__ void lw_ep_sample(const LwEnvPyr& P, int bin, double u, double v, long long& row,
                                             long long& col, double& p, double& u_out, double& v_out) {
  int l = P.nl - 1;
  double w0 = lw_ep_w(P, bin, l, 0, 0), w1 = lw_ep_w(P, bin, l, 0, 1);
  double s = w0 + w1;
  double p0 = s > 0.0 ? w0 / s : 0.5;
  long long r = 0, c;
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
    double a = lw_ep_w(P, bin, l - 1, 2 * r, 2 * c), b = lw_ep_w(P, bin, l - 1, 2 * r, 2 * c + 1);
    double cc = lw_ep_w(P, bin, l - 1, 2 * r + 1, 2 * c), d = lw_ep_w(P, bin, l - 1, 2 * r + 1, 2 * c + 1);
    double top = a + b, bot = cc + d;
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
      right = d;
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
  row = r;
  col = c;
  u_out = u;
  v_out = v;
}

// env_pdf's texel probability: the same conditionals along the path of base texel (row, col)
__device__ __forceinline__ double lw_ep_pdf(const LwEnvPyr& P, int bin, long long row, long long col) {
  int l = P.nl - 1;
  double w0 = lw_ep_w(P, bin, l, 0, 0), w1 = lw_ep_w(P, bin, l, 0, 1);
  double s = w0 + w1;
  double p0 = s > 0.0 ? w0 / s : 0.5;
  long long r = 0, c = col >> l;
  double p = c == 0 ? p0 : 1.0 - p0;
  for (; l > 0; l--) {
    double a = lw_ep_w(P, bin, l - 1, 2 * r, 2 * c), b = lw_ep_w(P, bin, l - 1, 2 * r, 2 * c + 1);
    double cc = lw_ep_w(P, bin, l - 1, 2 * r + 1, 2 * c), d = lw_ep_w(P, bin, l - 1, 2 * r + 1, 2 * c + 1);
    double top = a + b, bot = cc + d;
    double st = top + bot;
    double pt = st > 0.0 ? top / st : 0.5;
    long long rb = (row >> (l - 1)) & 1, cb = (col >> (l - 1)) & 1;
    double left, right;
    if (rb == 0) {
      p = p * pt;
      left = a;
      right = b;
    } else {
      p = p * (1.0 - pt);
      left = cc;
      right = d;
    }
    double sl = left + right;
    double pl = sl > 0.0 ? left / sl : 0.5;
    p = cb == 0 ? p * pl : p * (1.0 - pl);
    r = 2 * r + rb;
    c = 2 * c + cb;
  }
  return p;
}
