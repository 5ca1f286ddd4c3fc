// lw_capi.cu -- library plumbing and the stateless kernel entry points of include/lw_b200.h.
//
// Each entry replaces one function of the reference's Cython kernel module
// (lumenwave/core/_kernels.py), keeping its argument meaning: caller-owned
// C-contiguous buffers, misses encoded as data, no exceptions.  The host-buffer
// variants copy in, launch one sm_100a kernel, and copy out on cudaStreamPerThread.
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "lw_common.cuh"
#include "lw_detmath.cuh"
#include "lw_host.h"
#include "lw_qmc.cuh"
#include "lw_traverse.cuh"

namespace lw {

static thread_local std::string g_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
}

// qmc.py:153-164 construction, for `bits`-wide operands
static void fast_divisor(uint64_t d, int bits, uint64_t& magic, int& shift, int& add) {
  if ((d & (d - 1)) == 0) {
    magic = 0;
    shift = 63 - __builtin_clzll(d);
    add = 0;
    return;
  }
  int ell = 64 - __builtin_clzll(d - 1);
  unsigned __int128 num = ((unsigned __int128)1) << (bits + ell);
  unsigned __int128 m = (num + d - 1) / d;
  unsigned __int128 lim = ((unsigned __int128)1) << bits;
  if (m < lim) {
    magic = (uint64_t)m;
    shift = ell;
    add = 0;
  } else {
    magic = (uint64_t)(m - lim);
    shift = ell - 1;
    add = 1;
  }
}

int pack_qmc_tables(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                    const int64_t* perm_offset, std::vector<QmcDim>& dims, std::vector<uint16_t>& perm) {
  LW_CHECK_ARG(ndims > 0 && bases && perm_offset, "qmc tables: empty dimension table");
  dims.resize(ndims);
  perm.resize(perm_len > 0 ? perm_len : 1);
  for (int64_t i = 0; i < perm_len; i++) {
    LW_CHECK_ARG(perm_flat[i] >= 0 && perm_flat[i] < 65536, "qmc tables: permutation digit out of range");
    perm[i] = (uint16_t)perm_flat[i];
  }
  for (int64_t k = 0; k < ndims; k++) {
    int64_t b = bases[k];
    LW_CHECK_ARG(b >= 2 && b < (1LL << 31), "qmc tables: base must be in [2, 2^31)");
    LW_CHECK_ARG(b == 2 || (perm_offset[k] >= 0 && perm_offset[k] + b <= perm_len),
                 "qmc tables: permutation slice out of range");
    QmcDim& q = dims[k];
    memset(&q, 0, sizeof(q));
    q.base = (uint32_t)b;
    q.perm_off = (uint32_t)(b == 2 ? 0 : perm_offset[k]);
    uint64_t m;
    int s, a;
    fast_divisor((uint64_t)b, 32, m, s, a);
    q.magic32 = (uint32_t)m;
    q.shift32 = (uint8_t)s;
    q.add32 = (uint8_t)a;
    fast_divisor((uint64_t)b, 64, m, s, a);
    q.magic64 = m;
    q.shift64 = (uint8_t)s;
    q.add64 = (uint8_t)a;
    q.exact_limit = ((1ULL << 53) - 1) / (uint64_t)b;
    // digit count of 2^32-1; padding with zero digits needs sigma(0) == 0 (Faure tables have it)
    uint32_t nd = 0;
    for (uint64_t v = 0xffffffffULL; v; v /= (uint64_t)b) nd++;
    q.digits32 = (b != 2 && perm_flat[perm_offset[k]] == 0) ? nd : 0;
  }
  return LW_OK;
}

// ---- environment pyramid (oracle ep_build) -------------------------------------------------
namespace {
v3 ep_dir(double phi_turns, double theta_turns) {
  double st, ct, sp, cp;
  lw_sincos2pi(theta_turns, &st, &ct);
  lw_sincos2pi(phi_turns, &sp, &cp);
  return mk3(st * cp, ct, st * sp);
}

// axis and conservative cos(half-angle) of normal bin b (4 x 4 cells of the octahedral map)
void ep_bin_cone(int b, v3& axis, double& cosb) {
  long long bu = b / 4, bv = b % 4;
  axis = normalize3(lw_oct_decode(((bu * 16384 + 8192) << 16) | (bv * 16384 + 8192)));
  double m = 1.0;
  for (int k = 0; k <= 8; k++) {
    long long t = k * 2048;
    long long e0[4][2] = {{bu * 16384 + t, bv * 16384}, {bu * 16384 + t, bv * 16384 + 16384},
                          {bu * 16384, bv * 16384 + t}, {bu * 16384 + 16384, bv * 16384 + t}};
    for (int q = 0; q < 4; q++) {
      long long eu = e0[q][0] > 65535 ? 65535 : e0[q][0], ev = e0[q][1] > 65535 ? 65535 : e0[q][1];
      double c = dot3(axis, normalize3(lw_oct_decode((eu << 16) | ev)));
      if (c < m) m = c;
    }
  }
  cosb = m - 0.02;
}

// center direction and conservative cos(half-angle) of texel (r, c) of a (Hl x Wl) level
void ep_texel_cone(long long r, long long c, long long Hl, long long Wl, v3& ctr, double& cosg) {
  double f0 = (double)c / (double)Wl, f1 = (double)(c + 1) / (double)Wl;
  double t0 = (double)r / (double)Hl * 0.5, t1 = (double)(r + 1) / (double)Hl * 0.5;
  ctr = ep_dir((f0 + f1) * 0.5, (t0 + t1) * 0.5);
  double m = 1.0;
  for (int k = 0; k <= 8; k++) {
    double a = (double)k / 8.0;
    double fk = f0 + (f1 - f0) * a, tk = t0 + (t1 - t0) * a;
    v3 s[4] = {ep_dir(fk, t0), ep_dir(fk, t1), ep_dir(f0, tk), ep_dir(f1, tk)};
    for (int q = 0; q < 4; q++) {
      double cq = dot3(ctr, s[q]);
      if (cq < m) m = cq;
    }
  }
  cosg = m - 0.02;
}

// upper bound of max(0, n . w) over normals in the bin cone and directions in the texel cone
double ep_cos_bound(v3 axis, double cosb, v3 ctr, double cosg) {
  if (cosb <= 0.0 || cosg <= 0.0) return 1.0;
  double sinb = sqrt(1.0 - cosb * cosb), sing = sqrt(1.0 - cosg * cosg);
  double cosd = cosb * cosg - sinb * sing, sind = sinb * cosg + cosb * sing;
  if (sind <= 0.0) return 1.0;  // combined half-angle beyond pi
  double cosa = dot3(axis, ctr);
  if (cosa >= cosd) return 1.0;
  double s2 = 1.0 - cosa * cosa;
  double sina = sqrt(s2 > 0.0 ? s2 : 0.0);
  double cw = cosa * cosd + sina * sind;
  return cw > 0.0 ? cw : 0.0;
}
}  // namespace

int env_pyramid_build(int W, int H, const double* w, std::vector<double>& lvl, std::vector<double>& top,
                      LwEnvPyr& P) {
  LW_CHECK_ARG(H >= 1 && W == 2 * H && (H & (H - 1)) == 0, "environment pyramid: image must be 2H x H, H a power of 2");
  memset(&P, 0, sizeof(P));
  int nl = 1;
  while ((H >> (nl - 1)) > 1) nl++;
  LW_CHECK_ARG(nl <= LW_EP_MAXLEV, "environment pyramid: image too large");
  P.nl = nl;
  P.W = W;
  P.H = H;
  long long tot = 0;
  for (int l = 0; l < nl; l++) {
    P.off[l] = tot;
    tot += (long long)(H >> l) * (W >> l);
  }
  lvl.assign(tot, 0.0);
  for (long long k = 0; k < (long long)W * H; k++) lvl[k] = w[k];
  for (int l = 1; l < nl; l++) {
    long long Hl = H >> l, Wl = W >> l, Wc = Wl * 2;
    const double* ch = lvl.data() + P.off[l - 1];
    double* o = lvl.data() + P.off[l];
    for (long long r = 0; r < Hl; r++)
      for (long long c = 0; c < Wl; c++)
        o[r * Wl + c] = ((ch[(2 * r) * Wc + 2 * c] + ch[(2 * r) * Wc + 2 * c + 1]) + ch[(2 * r + 1) * Wc + 2 * c]) +
                        ch[(2 * r + 1) * Wc + 2 * c + 1];
  }
  P.ntop = nl < LW_EP_TOP ? nl : LW_EP_TOP;
  long long ts = 0;
  for (int l = nl - P.ntop; l < nl; l++) {
    P.toff[l] = ts;
    ts += (long long)(H >> l) * (W >> l);
  }
  P.top_stride = ts;
  top.assign((size_t)LW_EP_BINS * ts, 0.0);
  for (int b = 0; b < LW_EP_BINS; b++) {
    v3 axis;
    double cosb;
    ep_bin_cone(b, axis, cosb);
    for (int l = nl - P.ntop; l < nl; l++) {
      long long Hl = H >> l, Wl = W >> l;
      for (long long r = 0; r < Hl; r++)
        for (long long c = 0; c < Wl; c++) {
          v3 ctr;
          double cosg;
          ep_texel_cone(r, c, Hl, Wl, ctr, cosg);
          double cw = ep_cos_bound(axis, cosb, ctr, cosg);
          if (cw < LW_EP_CWMIN) cw = LW_EP_CWMIN;
          top[b * ts + P.toff[l] + r * Wl + c] = lvl[P.off[l] + r * Wl + c] * cw;
        }
    }
  }
  return LW_OK;
}

// ---- light hierarchy (oracle lt_build) ------------------------------------------------------
namespace {
struct LtBuild {
  const double* verts;
  const int64_t* tri;
  const double* w;
  const int32_t* two;
  std::vector<double> cen;  // [nemit*3]
  std::vector<int64_t> items;
  std::vector<LwLightNode>* nodes;
  std::vector<unsigned long long>* path;
  std::vector<int>* depth;
};

// FP64 accumulation, FP32 node record (rounded to nearest once)
struct LtAcc {
  double lo[3], hi[3], tot, flux[8];
};

void lt_leaf(LtBuild& b, int64_t e, LtAcc& A) {
  const double* v = b.verts + 9 * b.tri[e];
  for (int a = 0; a < 3; a++) {
    double lo = v[a], hi = v[a];
    if (v[3 + a] < lo) lo = v[3 + a];
    if (v[6 + a] < lo) lo = v[6 + a];
    if (v[3 + a] > hi) hi = v[3 + a];
    if (v[6 + a] > hi) hi = v[6 + a];
    A.lo[a] = lo;
    A.hi[a] = hi;
  }
  double e1x = v[3] - v[0], e1y = v[4] - v[1], e1z = v[5] - v[2];
  double e2x = v[6] - v[0], e2y = v[7] - v[1], e2z = v[8] - v[2];
  double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
  double inv = 1.0 / sqrt((cx * cx + cy * cy) + cz * cz);
  double nx = cx * inv, ny = cy * inv, nz = cz * inv;
  A.tot = b.w[e];
  for (int k = 0; k < 8; k++) {
    double c = lw_lt_octant_cos(k, nx, ny, nz);
    if (b.two[e]) {
      double c2 = lw_lt_octant_cos(k, -nx, -ny, -nz);
      if (c2 > c) c = c2;
    }
    A.flux[k] = b.w[e] * c;
  }
}

void lt_store(const LtAcc& A, int right, LwLightNode& N) {
  for (int a = 0; a < 3; a++) {
    N.lo[a] = (float)A.lo[a];
    N.hi[a] = (float)A.hi[a];
  }
  N.tot = (float)A.tot;
  for (int k = 0; k < 8; k++) N.flux[k] = (float)A.flux[k];
  N.right = right;
}

LtAcc lt_rec(LtBuild& b, int64_t begin, int64_t end, int64_t node, unsigned long long bits, int dep) {
  int64_t n = end - begin;
  LtAcc M;
  if (n == 1) {
    int64_t e = b.items[begin];
    lt_leaf(b, e, M);
    lt_store(M, (int)(-(e + 1)), (*b.nodes)[node]);
    (*b.path)[e] = bits;
    (*b.depth)[e] = dep;
    return M;
  }
  double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = begin; i < end; i++)
    for (int a = 0; a < 3; a++) {
      double c = b.cen[3 * b.items[i] + a];
      if (c < cmin[a]) cmin[a] = c;
      if (c > cmax[a]) cmax[a] = c;
    }
  int axis = 0;
  for (int a = 1; a < 3; a++)
    if (cmax[a] - cmin[a] > cmax[axis] - cmin[axis]) axis = a;
  const double* cen = b.cen.data();
  std::sort(b.items.begin() + begin, b.items.begin() + end, [cen, axis](int64_t x, int64_t y) {
    double cx = cen[3 * x + axis], cy = cen[3 * y + axis];
    return cx < cy || (cx == cy && x < y);
  });
  int64_t nl = n / 2;
  int64_t left = node + 1, right = node + 2 * nl;
  LtAcc L = lt_rec(b, begin, begin + nl, left, bits, dep + 1);
  LtAcc R = lt_rec(b, begin + nl, end, right, bits | (1ULL << dep), dep + 1);
  for (int a = 0; a < 3; a++) {
    M.lo[a] = L.lo[a] < R.lo[a] ? L.lo[a] : R.lo[a];
    M.hi[a] = L.hi[a] > R.hi[a] ? L.hi[a] : R.hi[a];
  }
  M.tot = L.tot + R.tot;
  for (int k = 0; k < 8; k++) M.flux[k] = L.flux[k] + R.flux[k];
  lt_store(M, (int)right, (*b.nodes)[node]);
  return M;
}
}  // namespace

int light_tree_build(const double* verts, const int64_t* emit_tri, const double* weight, const int32_t* twosided,
                     int64_t nemit, std::vector<LwLightNode>& nodes, std::vector<unsigned long long>& path,
                     std::vector<int>& depth) {
  LtBuild b;
  b.verts = verts;
  b.tri = emit_tri;
  b.w = weight;
  b.two = twosided;
  b.cen.resize(3 * (size_t)(nemit > 0 ? nemit : 1));
  path.assign(nemit > 0 ? nemit : 1, 0ULL);
  depth.assign(nemit > 0 ? nemit : 1, -1);
  for (int64_t e = 0; e < nemit; e++) {
    const double* v = verts + 9 * emit_tri[e];
    for (int a = 0; a < 3; a++) b.cen[3 * e + a] = ((v[a] + v[3 + a]) + v[6 + a]) / 3.0;
    if (weight[e] > 0.0) b.items.push_back(e);
  }
  int64_t m = (int64_t)b.items.size();
  nodes.assign(m > 0 ? 2 * m - 1 : 0, LwLightNode());
  LW_CHECK_ARG(m < (1LL << 30), "light tree: too many emitters");
  b.nodes = &nodes;
  b.path = &path;
  b.depth = &depth;
  if (m > 0) lt_rec(b, 0, m, 0, 0ULL, 0);
  return LW_OK;
}

// Vose alias table, identical in operation order to oracle lwo_alias_build
int alias_build(const double* w, int64_t n, double* prob, int32_t* alias, double* pdf) {
  LW_CHECK_ARG(n > 0, "alias table: no entries");
  double total = 0.0;
  for (int64_t i = 0; i < n; i++) {
    LW_CHECK_ARG(w[i] >= 0.0 && w[i] != INFINITY, "alias table: weights must be finite and >= 0");
    total += w[i];
  }
  LW_CHECK_ARG(total > 0.0, "alias table: all weights are zero");
  std::vector<double> scaled(n);
  std::vector<int64_t> small(n), large(n);
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
  return LW_OK;
}

}  // namespace lw

using namespace lw;

// ---- kernels ------------------------------------------------------------------------------

__global__ void k_halton(const QmcDim* __restrict__ dims, const uint16_t* __restrict__ perm, int dim,
                         const long long* __restrict__ idx, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = lw_halton(dims, perm, dim, idx[i]);
}

__global__ void k_pixel_offset(const double* __restrict__ u, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = lw_gauss_filter_offset(u[i]);
}

// oct_roundtrip_batch (_kernels.py:321-342): rows whose decoded length is 0 are untouched
__global__ void k_oct_roundtrip(const double* __restrict__ v, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    v3 d = lw_oct_decode(lw_oct_encode(v[3 * i], v[3 * i + 1], v[3 * i + 2]));
    double ln = sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
    if (ln > 0.0) {
      out[3 * i] = d.x / ln;
      out[3 * i + 1] = d.y / ln;
      out[3 * i + 2] = d.z / ln;
    }
  }
}

__global__ void k_oct_encode(const double* __restrict__ v, long long n, long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = lw_oct_encode(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
}

__global__ void k_oct_decode(const long long* __restrict__ p, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    v3 d = lw_oct_decode(p[i]);
    out[3 * i] = d.x;
    out[3 * i + 1] = d.y;
    out[3 * i + 2] = d.z;
  }
}

__global__ void k_intersect_ref(int compat, const double* __restrict__ bounds, const long long* __restrict__ children,
                                const long long* __restrict__ order, const double* __restrict__ verts, long long ntris,
                                const double* __restrict__ origins, const double* __restrict__ dirs,
                                const double* __restrict__ tmaxs, long long n, double* __restrict__ out_t,
                                long long* __restrict__ out_tri, double* __restrict__ out_bary) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double o[3] = {origins[3 * i], origins[3 * i + 1], origins[3 * i + 2]};
  double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
  LwHit h;
  lw_traverse_ref(compat != 0, bounds, children, order, verts, ntris, o, d, tmaxs[i], h);
  if (h.tri >= 0) {
    out_t[i] = h.t;
    out_tri[i] = h.tri;
    out_bary[2 * i] = h.bu;
    out_bary[2 * i + 1] = h.bv;
  } else {
    out_t[i] = 1e308;
    out_tri[i] = -1;
    out_bary[2 * i] = 0.0;
    out_bary[2 * i + 1] = 0.0;
  }
}

__global__ void k_intersect_brute(const double* __restrict__ verts, long long ntris, const double* __restrict__ origins,
                                  const double* __restrict__ dirs, const double* __restrict__ tmaxs, long long n,
                                  double* __restrict__ out_t, long long* __restrict__ out_tri,
                                  double* __restrict__ out_bary) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double o[3] = {origins[3 * i], origins[3 * i + 1], origins[3 * i + 2]};
  double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
  LwShear s;
  lw_shear_setup(o, d, false, s);
  LwHit h;
  h.t = tmaxs[i];
  h.tri = -1;
  h.bu = h.bv = 0.0;
  for (long long k = 0; k < ntris; k++) lw_tri_test(verts + 9 * k, k, s, 0.0, h);
  if (h.tri >= 0) {
    out_t[i] = h.t;
    out_tri[i] = h.tri;
    out_bary[2 * i] = h.bu;
    out_bary[2 * i + 1] = h.bv;
  } else {
    out_t[i] = 1e308;
    out_tri[i] = -1;
    out_bary[2 * i] = 0.0;
    out_bary[2 * i + 1] = 0.0;
  }
}

// ---- C ABI --------------------------------------------------------------------------------

#define S_ cudaStreamPerThread

// stateless entry points allocate from the device's stream-ordered pool; keep freed blocks reserved
// (release threshold) so repeated batches neither re-map memory nor synchronise in cudaFree
static void keep_pool() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

template <class T>
static int upload(DevBuf& b, const T* host, int64_t count) {
  keep_pool();
  LW_CUDA_TRY(b.alloc(sizeof(T) * (count > 0 ? count : 1), S_));  // stream-ordered pool: no sync, no remap
  if (count > 0) LW_CUDA_TRY(cudaMemcpyAsync(b.p, host, sizeof(T) * count, cudaMemcpyHostToDevice, S_));
  return LW_OK;
}

extern "C" {

const char* lw_last_error(void) { return g_error.c_str(); }
int lw_abi_version(void) { return LW_ABI_VERSION; }

int lw_device_count(int* count) {
  LW_CHECK_ARG(count, "null count");
  LW_CUDA_TRY(cudaGetDeviceCount(count));
  return LW_OK;
}

int lw_set_device(int device) {
  LW_CUDA_TRY(cudaSetDevice(device));
  return LW_OK;
}

int lw_alias_build(const double* weights, int64_t n, double* prob, int32_t* alias, double* pdf) {
  LW_CHECK_ARG(weights && prob && alias && pdf, "null pointer");
  return alias_build(weights, n, prob, alias, pdf);
}

static int halton_impl(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                       const int64_t* perm_offset, int64_t dim, const long long* d_idx, int64_t n, double* d_out) {
  LW_CHECK_ARG(dim >= 0 && dim < ndims, "dim out of range");
  std::vector<QmcDim> dims;
  std::vector<uint16_t> perm;
  LW_STATUS_TRY(pack_qmc_tables(bases, ndims, perm_flat, perm_len, perm_offset, dims, perm));
  DevBuf b_dims, b_perm;
  LW_STATUS_TRY(upload(b_dims, dims.data(), (int64_t)dims.size()));
  LW_STATUS_TRY(upload(b_perm, perm.data(), (int64_t)perm.size()));
  if (n > 0) k_halton<<<grid_for(n, 256), 256, 0, S_>>>(b_dims.as<QmcDim>(), b_perm.as<uint16_t>(), (int)dim, d_idx, n, d_out);
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_halton_batch(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                    const int64_t* perm_offset, int64_t dim, const int64_t* indices, int64_t n, double* out) {
  LW_CHECK_ARG(n >= 0 && (n == 0 || (indices && out)), "bad batch");
  DevBuf b_idx, b_out;
  LW_STATUS_TRY(upload(b_idx, indices, n));
  LW_CUDA_TRY(b_out.alloc(sizeof(double) * (n > 0 ? n : 1), S_));
  LW_STATUS_TRY(halton_impl(bases, ndims, perm_flat, perm_len, perm_offset, dim, b_idx.as<long long>(), n, b_out.as<double>()));
  if (n > 0) LW_CUDA_TRY(cudaMemcpyAsync(out, b_out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_halton_batch_device(const int64_t* bases, int64_t ndims, const int64_t* perm_flat, int64_t perm_len,
                           const int64_t* perm_offset, int64_t dim, const int64_t* indices_device, int64_t n,
                           double* out_device) {
  return halton_impl(bases, ndims, perm_flat, perm_len, perm_offset, dim, (const long long*)indices_device, n, out_device);
}

int lw_pixel_offset_batch(const double* u, int64_t n, double* out) {
  LW_CHECK_ARG(n >= 0 && (n == 0 || (u && out)), "bad batch");
  if (n == 0) return LW_OK;
  DevBuf b_u, b_o;
  LW_STATUS_TRY(upload(b_u, u, 2 * n));
  LW_CUDA_TRY(b_o.alloc(sizeof(double) * 2 * n, S_));
  k_pixel_offset<<<grid_for(2 * n, 256), 256, 0, S_>>>(b_u.as<double>(), 2 * n, b_o.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out, b_o.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_oct_roundtrip_batch(const double* vecs, int64_t n, double* out) {
  LW_CHECK_ARG(n >= 0 && (n == 0 || (vecs && out)), "bad batch");
  if (n == 0) return LW_OK;
  DevBuf b_v, b_o;
  LW_STATUS_TRY(upload(b_v, vecs, 3 * n));
  LW_STATUS_TRY(upload(b_o, out, 3 * n));  // untouched rows keep the caller's values
  k_oct_roundtrip<<<grid_for(n, 256), 256, 0, S_>>>(b_v.as<double>(), n, b_o.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out, b_o.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_oct_encode_batch(const double* vecs, int64_t n, int64_t* out) {
  LW_CHECK_ARG(n >= 0 && (n == 0 || (vecs && out)), "bad batch");
  if (n == 0) return LW_OK;
  DevBuf b_v, b_o;
  LW_STATUS_TRY(upload(b_v, vecs, 3 * n));
  LW_CUDA_TRY(b_o.alloc(sizeof(long long) * n, S_));
  k_oct_encode<<<grid_for(n, 256), 256, 0, S_>>>(b_v.as<double>(), n, b_o.as<long long>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out, b_o.p, sizeof(long long) * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_oct_decode_batch(const int64_t* packed, int64_t n, double* out) {
  LW_CHECK_ARG(n >= 0 && (n == 0 || (packed && out)), "bad batch");
  if (n == 0) return LW_OK;
  DevBuf b_p, b_o;
  LW_STATUS_TRY(upload(b_p, packed, n));
  LW_CUDA_TRY(b_o.alloc(sizeof(double) * 3 * n, S_));
  k_oct_decode<<<grid_for(n, 256), 256, 0, S_>>>(b_p.as<long long>(), n, b_o.as<double>());
  LW_CUDA_TRY(cudaGetLastError());
  LW_CUDA_TRY(cudaMemcpyAsync(out, b_o.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

static int intersect_launch(int mode, const double* bounds, const int64_t* children, const int64_t* order,
                            const double* verts, int64_t ntris, const double* origins, const double* dirs,
                            const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri, double* out_bary) {
  LW_CHECK_ARG(mode == LW_TRAVERSE_COMPAT || mode == LW_TRAVERSE_CORRECTED || mode == LW_TRAVERSE_BRUTE,
               "unknown traversal mode");
  if (n == 0) return LW_OK;
  if (mode == LW_TRAVERSE_BRUTE)
    k_intersect_brute<<<(int)((n + 127) / 128), 128, 0, S_>>>(verts, ntris, origins, dirs, tmaxs, n, out_t,
                                                               (long long*)out_tri, out_bary);
  else
    k_intersect_ref<<<(int)((n + 127) / 128), 128, 0, S_>>>(mode == LW_TRAVERSE_COMPAT, bounds,
                                                             (const long long*)children, (const long long*)order, verts,
                                                             ntris, origins, dirs, tmaxs, n, out_t,
                                                             (long long*)out_tri, out_bary);
  LW_CUDA_TRY(cudaGetLastError());
  return LW_OK;
}

int lw_intersect_batch(int mode, const double* bounds, const int64_t* children, int64_t nnodes, const int64_t* order,
                       const double* verts, int64_t ntris, const double* origins, const double* dirs,
                       const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri, double* out_bary) {
  LW_CHECK_ARG(n >= 0 && ntris >= 0 && nnodes >= 1, "bad sizes");
  LW_CHECK_ARG(n == 0 || (origins && dirs && tmaxs && out_t && out_tri && out_bary), "null ray buffers");
  if (n == 0) return LW_OK;
  DevBuf b_bounds, b_children, b_order, b_verts, b_o, b_d, b_tm, b_t, b_tri, b_bary;
  LW_STATUS_TRY(upload(b_bounds, bounds, 6 * nnodes));
  LW_STATUS_TRY(upload(b_children, children, 2 * nnodes));
  LW_STATUS_TRY(upload(b_order, order, ntris));
  LW_STATUS_TRY(upload(b_verts, verts, 9 * ntris));
  LW_STATUS_TRY(upload(b_o, origins, 3 * n));
  LW_STATUS_TRY(upload(b_d, dirs, 3 * n));
  LW_STATUS_TRY(upload(b_tm, tmaxs, n));
  LW_CUDA_TRY(b_t.alloc(sizeof(double) * n, S_));
  LW_CUDA_TRY(b_tri.alloc(sizeof(int64_t) * n, S_));
  LW_CUDA_TRY(b_bary.alloc(sizeof(double) * 2 * n, S_));
  LW_STATUS_TRY(intersect_launch(mode, b_bounds.as<double>(), b_children.as<int64_t>(), b_order.as<int64_t>(),
                                 b_verts.as<double>(), ntris, b_o.as<double>(), b_d.as<double>(), b_tm.as<double>(), n,
                                 b_t.as<double>(), b_tri.as<int64_t>(), b_bary.as<double>()));
  LW_CUDA_TRY(cudaMemcpyAsync(out_t, b_t.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaMemcpyAsync(out_tri, b_tri.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaMemcpyAsync(out_bary, b_bary.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, S_));
  LW_CUDA_TRY(cudaStreamSynchronize(S_));
  return LW_OK;
}

int lw_intersect_batch_device(int mode, const double* bounds, const int64_t* children, int64_t nnodes,
                              const int64_t* order, const double* verts, int64_t ntris, const double* origins,
                              const double* dirs, const double* tmaxs, int64_t n, double* out_t, int64_t* out_tri,
                              double* out_bary) {
  LW_CHECK_ARG(n >= 0 && ntris >= 0 && nnodes >= 1, "bad sizes");
  return intersect_launch(mode, bounds, children, order, verts, ntris, origins, dirs, tmaxs, n, out_t, out_tri, out_bary);
}

}  // extern "C"
