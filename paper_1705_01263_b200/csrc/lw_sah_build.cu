// lw_sah_build.cu -- binned-SAH render BVH built on the GPU.
//
// Produces exactly the tree of the specification restated in oracle/lw_oracle.c
// (build_render_bvh_sah): segments processed breadth-first, internal nodes numbered in that
// order, 16 centroid bins per axis, first strict minimum of A(L)nL + A(R)nR over (axis, plane),
// split when n > 7 or A(B) + cost < n*A(B), coincident centroids halved in order, stable
// partition.  Per level:
//   1. bins of large segments (n > 32): ordered-u64 min/max + count atomics, privatised in
//      shared memory when a 1024-position chunk lies inside one segment;
//   2. one warp per segment (k_sah_decide_w; the per-thread k_sah_decide with LW_SAH_SERIAL=1,
//      LW_SAH_CHECK=1 runs both and reports differing decisions): lanes own bins, small segments
//      bin their triangles, prefix / suffix boxes by shuffles, first strict minimum of the plane
//      costs by a warp argmin, leaf / split decision (identical FP64 formulas on every path);
//   3. node ids = level base + rank among splitting segments (scan), child segments at 2r, 2r+1;
//   4. stable partition of the position list (scan + scatter) and the next position->segment map.
// Bounds are exact (min/max), so every path reproduces the sequential specification bit for bit.
#include <string.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "lw_common.cuh"
#include "lw_host.h"

namespace lw {

namespace {

#ifndef LW_SAH_BINS
#define LW_SAH_BINS 16
#endif
#ifndef LW_SAH_MAXLEAF
#define LW_SAH_MAXLEAF 7
#endif
#ifndef LW_SAH_CTRAV
#define LW_SAH_CTRAV 1.0
#endif
#ifndef LW_SAH_PRIV
#define LW_SAH_PRIV 1  // large-segment bins privatised in shared memory per 1024-position chunk
#endif
constexpr int kBins = LW_SAH_BINS;      // centroid bins per axis
constexpr int kMaxLeaf = LW_SAH_MAXLEAF; // segments above this size are always split (leaf count field: <= 7)
constexpr int kSmall = 32;   // segments up to this size are binned by one thread
constexpr int kChunk = 1024; // positions per block in the large-segment binning pass

struct SSeg {
  int start, n, parent, side;
  double B[6];  // triangle-bounds box lo xyz, hi xyz
  double C[6];  // centroid box
};

struct SSplit {
  int split;    // 0 leaf, 1 split
  int axis;     // -1 = halve
  int plane, nl;
  double L[6], R[6], CL[6], CR[6];
};

// 13 values per bin: count, triangle box (6), centroid box (6), as order-preserving u64
struct BinAcc {
  unsigned long long v[13];
};

__device__ __forceinline__ unsigned long long ordd(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double unordd(unsigned long long u) {
  unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ double area6(const double* b) {
  double dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
  return 2.0 * ((dx * dy + dy * dz) + dz * dx);
}

__device__ __forceinline__ void box_reset(double* b) {
  b[0] = b[1] = b[2] = INFINITY;
  b[3] = b[4] = b[5] = -INFINITY;
}

__device__ __forceinline__ void box_grow(double* b, const double* lo, const double* hi) {
#pragma unroll
  for (int a = 0; a < 3; a++) {
    if (lo[a] < b[a]) b[a] = lo[a];
    if (hi[a] > b[3 + a]) b[3 + a] = hi[a];
  }
}

__device__ __forceinline__ int bin_of(double c, double cmin, double scale) {
  int b = (int)((c - cmin) * scale);
  return b > kBins - 1 ? kBins - 1 : b;
}

__device__ __forceinline__ double canon(double x) { return x == 0.0 ? 0.0 : x; }

__global__ void k_sah_prep(const double* __restrict__ v, int n, double* __restrict__ tb, double* __restrict__ cen,
                           int* __restrict__ ids, int* __restrict__ pos_seg) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = v + 9 * (size_t)i;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double lo = p[a], hi = p[a];
    if (p[3 + a] < lo) lo = p[3 + a];
    if (p[6 + a] < lo) lo = p[6 + a];
    if (p[3 + a] > hi) hi = p[3 + a];
    if (p[6 + a] > hi) hi = p[6 + a];
    lo = canon(lo);
    hi = canon(hi);
    tb[6 * (size_t)i + a] = lo;
    tb[6 * (size_t)i + 3 + a] = hi;
    cen[3 * (size_t)i + a] = canon(0.5 * (lo + hi));
  }
  ids[i] = i;
  pos_seg[i] = 0;
}

// root boxes: block reduction then ordered atomics (12 values)
__global__ void k_sah_root_reduce(const double* __restrict__ tb, const double* __restrict__ cen, int n,
                                  unsigned long long* __restrict__ acc) {
  double v[12];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    v[k] = INFINITY;
    v[3 + k] = -INFINITY;
    v[6 + k] = INFINITY;
    v[9 + k] = -INFINITY;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      v[a] = fmin(v[a], tb[6 * (size_t)i + a]);
      v[3 + a] = fmax(v[3 + a], tb[6 * (size_t)i + 3 + a]);
      v[6 + a] = fmin(v[6 + a], cen[3 * (size_t)i + a]);
      v[9 + a] = fmax(v[9 + a], cen[3 * (size_t)i + a]);
    }
  }
#pragma unroll
  for (int k = 0; k < 12; k++) {
    unsigned long long u = ordd(v[k]);
    bool mn = (k % 6) < 3;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      unsigned long long o = __shfl_down_sync(0xffffffffu, u, off);
      u = mn ? (o < u ? o : u) : (o > u ? o : u);
    }
    if ((threadIdx.x & 31) == 0) {
      if (mn)
        atomicMin(acc + k, u);
      else
        atomicMax(acc + k, u);
    }
  }
}

__global__ void k_sah_root_init(unsigned long long* acc, SSeg* seg, int n) {
  SSeg s;
  s.start = 0;
  s.n = n;
  s.parent = -1;
  s.side = 0;
  for (int k = 0; k < 6; k++) {
    s.B[k] = unordd(acc[k]);
    s.C[k] = unordd(acc[6 + k]);
  }
  seg[0] = s;
}

__global__ void k_sah_bins_init(BinAcc* __restrict__ bins, int nbins) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbins) return;
  BinAcc b;
  b.v[0] = 0;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    b.v[1 + k] = ~0ULL;
    b.v[4 + k] = 0ULL;
    b.v[7 + k] = ~0ULL;
    b.v[10 + k] = 0ULL;
  }
  bins[i] = b;
}

__device__ __forceinline__ void bin_add(unsigned long long* b, const double* tb, const double* c, bool shared_mem) {
  // count, tri box, centroid box; atomics are exact, so the accumulation order is irrelevant
  atomicAdd(b, 1ULL);
#pragma unroll
  for (int a = 0; a < 3; a++) {
    atomicMin(b + 1 + a, ordd(tb[a]));
    atomicMax(b + 4 + a, ordd(tb[3 + a]));
    atomicMin(b + 7 + a, ordd(c[a]));
    atomicMax(b + 10 + a, ordd(c[a]));
  }
  (void)shared_mem;
}

// value k of a triangle's bin record (BinAcc v[1 + k]): k < 3 box min, < 6 box max, < 9 centroid
// min, < 12 centroid max, as ordered u64
__device__ __forceinline__ unsigned long long bin_val(int k, const double* tbt, const double* ct) {
  return k < 6 ? ordd(tbt[k]) : ordd(ct[(k - 6) % 3]);
}

// Large-segment bins.  A 1024-position chunk inside one segment accumulates privately in shared
// memory and flushes once with global atomics (native 64-bit min / max, REDG.E.MIN.64).  Shared
// 64-bit min / max would compile to CAS loops (ATOMS.CAST.SPIN.64) that serialise the threads of a
// bin, so the private minima / maxima are exact 64-bit results of two native 32-bit passes: the
// high words first, then the low words of the values whose high word won.
__global__ void __launch_bounds__(256) k_sah_bin_large(const int* __restrict__ pos_seg, const int* __restrict__ ids,
                                                       int n, const SSeg* __restrict__ seg,
                                                       const int* __restrict__ large_rank, const double* __restrict__ tb,
                                                       const double* __restrict__ cen, BinAcc* __restrict__ bins) {
  __shared__ unsigned s_cnt[3 * kBins], s_hi[3 * kBins][12], s_lo[3 * kBins][12];
  int c0 = blockIdx.x * kChunk;
  if (c0 >= n) return;
  int c1 = min(c0 + kChunk, n);
  int s_first = pos_seg[c0], s_last = pos_seg[c1 - 1];
  bool priv = LW_SAH_PRIV && s_first >= 0 && s_first == s_last && large_rank[s_first] >= 0;
  if (!priv) {
    for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      int s = pos_seg[i];
      if (s < 0) continue;
      int lr = large_rank[s];
      if (lr < 0) continue;
      int t = ids[i];
      const double* tbt = tb + 6 * (size_t)t;
      const double* ct = cen + 3 * (size_t)t;
      const SSeg& g = seg[s];
#pragma unroll
      for (int a = 0; a < 3; a++) {
        double ext = g.C[3 + a] - g.C[a];
        if (!(ext > 0.0)) continue;
        int b = bin_of(ct[a], g.C[a], (double)kBins / ext);
        bin_add(bins[(size_t)lr * 3 * kBins + a * kBins + b].v, tbt, ct, false);
      }
    }
    return;
  }
  for (int q = threadIdx.x; q < 3 * kBins; q += blockDim.x) {
    s_cnt[q] = 0;
#pragma unroll
    for (int k = 0; k < 12; k++) {
      bool mx = (k % 6) >= 3;
      s_hi[q][k] = mx ? 0u : ~0u;
      s_lo[q][k] = mx ? 0u : ~0u;
    }
  }
  __syncthreads();
  const SSeg& g = seg[s_first];
  double scale[3];
  bool live[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double ext = g.C[3 + a] - g.C[a];
    live[a] = ext > 0.0;
    scale[a] = (double)kBins / ext;
  }
  for (int pass = 0; pass < 2; pass++) {
    for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      int t = ids[i];
      const double* tbt = tb + 6 * (size_t)t;
      const double* ct = cen + 3 * (size_t)t;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        if (!live[a]) continue;
        int q = a * kBins + bin_of(ct[a], g.C[a], scale[a]);
        if (pass == 0) atomicAdd(&s_cnt[q], 1u);
#pragma unroll
        for (int k = 0; k < 12; k++) {
          unsigned long long v = bin_val(k, tbt, ct);
          unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
          bool mx = (k % 6) >= 3;
          if (pass == 0) {
            if (mx)
              atomicMax(&s_hi[q][k], hi);
            else
              atomicMin(&s_hi[q][k], hi);
          } else if (hi == s_hi[q][k]) {
            if (mx)
              atomicMax(&s_lo[q][k], lo);
            else
              atomicMin(&s_lo[q][k], lo);
          }
        }
      }
    }
    __syncthreads();
  }
  const int lr = large_rank[s_first];
  for (int q = threadIdx.x; q < 3 * kBins; q += blockDim.x) {
    if (s_cnt[q] == 0) continue;
    unsigned long long* d = bins[(size_t)lr * 3 * kBins + q].v;
    atomicAdd(d, (unsigned long long)s_cnt[q]);
#pragma unroll
    for (int k = 0; k < 12; k++) {
      unsigned long long v = ((unsigned long long)s_hi[q][k] << 32) | s_lo[q][k];
      if ((k % 6) >= 3)
        atomicMax(d + 1 + k, v);
      else
        atomicMin(d + 1 + k, v);
    }
  }
}

// one thread per segment: bin (small segments), sweep, decide
__global__ void k_sah_decide(const SSeg* __restrict__ seg, int nseg, const int* __restrict__ large_rank,
                             const BinAcc* __restrict__ bins, const int* __restrict__ ids,
                             const double* __restrict__ tb, const double* __restrict__ cen, SSplit* __restrict__ out,
                             int* __restrict__ split_flag) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const SSeg g = seg[s];
  SSplit r;
  r.split = 0;
  r.axis = -1;
  r.plane = -1;
  r.nl = 0;
  double best = INFINITY;
  if (g.n > 1) {
    for (int a = 0; a < 3; a++) {
      double ext = g.C[3 + a] - g.C[a];
      if (!(ext > 0.0)) continue;
      double scale = (double)kBins / ext;
      int cnt[kBins];
      double bb[kBins][6], cb[kBins][6];
      if (large_rank[s] >= 0) {
        const BinAcc* src = bins + (size_t)large_rank[s] * 3 * kBins + a * kBins;
        for (int b = 0; b < kBins; b++) {
          cnt[b] = (int)src[b].v[0];
          for (int k = 0; k < 6; k++) {
            bb[b][k] = unordd(src[b].v[1 + k]);
            cb[b][k] = unordd(src[b].v[7 + k]);
          }
        }
      } else {
        for (int b = 0; b < kBins; b++) {
          cnt[b] = 0;
          box_reset(bb[b]);
          box_reset(cb[b]);
        }
        for (int k = 0; k < g.n; k++) {
          int t = ids[g.start + k];
          const double* ct = cen + 3 * (size_t)t;
          int b = bin_of(ct[a], g.C[a], scale);
          cnt[b]++;
          box_grow(bb[b], tb + 6 * (size_t)t, tb + 6 * (size_t)t + 3);
          box_grow(cb[b], ct, ct);
        }
      }
      // suffix (right side of plane p = bins p+1..15)
      double rb[kBins][6], rc[kBins][6];
      int rn[kBins];
      double accb[6], accc[6];
      box_reset(accb);
      box_reset(accc);
      int an = 0;
      for (int b = kBins - 1; b >= 1; b--) {
        box_grow(accb, bb[b], bb[b] + 3);
        box_grow(accc, cb[b], cb[b] + 3);
        an += cnt[b];
        for (int k = 0; k < 6; k++) {
          rb[b][k] = accb[k];
          rc[b][k] = accc[k];
        }
        rn[b] = an;
      }
      box_reset(accb);
      box_reset(accc);
      an = 0;
      for (int p = 0; p < kBins - 1; p++) {
        box_grow(accb, bb[p], bb[p] + 3);
        box_grow(accc, cb[p], cb[p] + 3);
        an += cnt[p];
        int nr = rn[p + 1];
        if (an == 0 || nr == 0) continue;
        double cost = area6(accb) * (double)an + area6(rb[p + 1]) * (double)nr;
        if (cost < best) {
          best = cost;
          r.axis = a;
          r.plane = p;
          r.nl = an;
          for (int k = 0; k < 6; k++) {
            r.L[k] = accb[k];
            r.CL[k] = accc[k];
            r.R[k] = rb[p + 1][k];
            r.CR[k] = rc[p + 1][k];
          }
        }
      }
    }
  }
  if (r.axis >= 0) {
    double aB = area6(g.B);
    r.split = (g.n > kMaxLeaf || (LW_SAH_CTRAV * aB + best) < (double)g.n * aB) ? 1 : 0;
  } else if (g.n > kMaxLeaf) {
    r.split = 1;  // coincident centroids: halve in the current order
    r.axis = -1;
    r.nl = g.n / 2;
    box_reset(r.L);
    box_reset(r.R);
    box_reset(r.CL);
    box_reset(r.CR);
    for (int k = 0; k < g.n; k++) {
      int t = ids[g.start + k];
      double* B = k < r.nl ? r.L : r.R;
      double* Cc = k < r.nl ? r.CL : r.CR;
      box_grow(B, tb + 6 * (size_t)t, tb + 6 * (size_t)t + 3);
      box_grow(Cc, cen + 3 * (size_t)t, cen + 3 * (size_t)t);
    }
  }
  out[s] = r;
  split_flag[s] = r.split;
}

// k_sah_decide with one warp per segment (the per-thread version serialises 48 bins and two
// 16-bin sweeps through local memory: ~60 us per level even for a 36-triangle scene).  Lane
// b & 15 owns bin b of the current axis (both half-warps compute the same axis); prefix / suffix
// boxes come from shuffles.  min / max and integer counts are exact and order-free, and every
// cost is the same FP64 expression of the same boxes, so the first strict minimum over
// (axis, plane) -- taken as the lexicographic minimum of (cost, 15 * axis + plane) -- and the
// split are those of the sequential specification, bit for bit.
__device__ __forceinline__ double shfl_up_d(double v, int off) { return __shfl_up_sync(0xffffffffu, v, off, 16); }
__device__ __forceinline__ double shfl_down_d(double v, int off) { return __shfl_down_sync(0xffffffffu, v, off, 16); }

#ifndef LW_SAH_DEC_MINB
#define LW_SAH_DEC_MINB 4
#endif
// bin `bin` of axis a of segment g: count, triangle-bounds box, centroid box.  Large segments read
// the pre-binned accumulators; for small ones the warp's triangles sit in its shared-memory slice
// (tri[k] = triangle k's bounds and centroid, written once per segment); lane k computes triangle
// k's bin and a ballot per bin gives each lane the triangles of its own bin to fold in: min / max
// and counts are exact and order-free, so these are the boxes and counts of a sequential loop.  (Binning with ordered-u64 min / max
// atomics compiled to shared-memory CAS loops, ATOMS.CAST.SPIN.64, that serialised on the lanes
// sharing a bin.)  An empty large-segment bin decodes to NaN bounds, an empty small-segment bin to
// the reset box; box_grow ignores both.
__device__ __forceinline__ void sah_bin_data(const SSeg& g, int lr, int a, double scale, int bin,
                                             const BinAcc* __restrict__ bins, const double (*tri)[9], int& cnt,
                                             double bb[6], double cb[6]) {
  if (lr >= 0) {
    const BinAcc& src = bins[(size_t)lr * 3 * kBins + a * kBins + bin];
    cnt = (int)src.v[0];
#pragma unroll
    for (int k = 0; k < 6; k++) {
      bb[k] = unordd(src.v[1 + k]);
      cb[k] = unordd(src.v[7 + k]);
    }
    return;
  }
  // lane k bins triangle k once; one ballot per bin hands every lane the members of its bin
  const int lane = threadIdx.x & 31;
  const int mb = lane < g.n ? bin_of(tri[lane][6 + a], g.C[a], scale) : -1;
  unsigned members = 0;
#pragma unroll
  for (int j = 0; j < kBins; j++) {
    unsigned m = __ballot_sync(0xffffffffu, mb == j);
    if (j == bin) members = m;
  }
  cnt = __popc(members);
  box_reset(bb);
  box_reset(cb);
  while (members) {
    const double* t = tri[__ffs(members) - 1];
    members &= members - 1;
    box_grow(bb, t, t + 3);
    box_grow(cb, t + 6, t + 6);
  }
}

// inclusive prefix (bins 0..bin) and suffix (bins bin..15) of one box quantity over the half-warp,
// started from the empty box grown by the bin's box as the sequential sweep does
__device__ __forceinline__ void sah_scan_boxes(const double bx[6], int bin, double pb[6], double sb[6]) {
  box_reset(pb);
  box_grow(pb, bx, bx + 3);
#pragma unroll
  for (int k = 0; k < 6; k++) sb[k] = pb[k];
#pragma unroll
  for (int off = 1; off < kBins; off <<= 1) {
    double ub[6], db[6];
#pragma unroll
    for (int k = 0; k < 6; k++) {
      ub[k] = shfl_up_d(pb[k], off);
      db[k] = shfl_down_d(sb[k], off);
    }
    if (bin >= off) box_grow(pb, ub, ub + 3);
    if (bin + off < kBins) box_grow(sb, db, db + 3);
  }
}

__device__ __forceinline__ void sah_scan_counts(int cnt, int bin, int& pn, int& sn) {
  pn = sn = cnt;
#pragma unroll
  for (int off = 1; off < kBins; off <<= 1) {
    int un = __shfl_up_sync(0xffffffffu, pn, off, 16), dn = __shfl_down_sync(0xffffffffu, sn, off, 16);
    if (bin >= off) pn += un;
    if (bin + off < kBins) sn += dn;
  }
}

// Two passes keep the live state small (206 -> ~100 registers): pass 1 scans counts and bounds of
// every axis and keeps only (cost, key, nl) of each lane's best plane; after the warp argmin, pass 2
// recomputes the winning axis' bins and scans to produce the four boxes of the split.  Every value
// is the same expression of the same inputs as in the single pass, so the split is unchanged.
// the decision for segment s by one whole warp (sbw: the warp's shared-memory bin slice)
__device__ __forceinline__ void sah_decide_seg(int s, const SSeg* __restrict__ seg, const int* __restrict__ large_rank,
                                               const BinAcc* __restrict__ bins, const int* __restrict__ ids,
                                               const double* __restrict__ tb, const double* __restrict__ cen,
                                               SSplit* __restrict__ out, int* __restrict__ split_flag,
                                               double (*tri)[9], int lane) {
  const int bin = lane & 15;
  const SSeg g = seg[s];
  const int lr = large_rank[s];
  __syncwarp();  // the previous segment's reads of tri are done
  if (lr < 0 && lane < g.n) {
    int t = ids[g.start + lane];
#pragma unroll
    for (int k = 0; k < 6; k++) tri[lane][k] = tb[6 * (size_t)t + k];
#pragma unroll
    for (int k = 0; k < 3; k++) tri[lane][6 + k] = cen[3 * (size_t)t + k];
  }
  __syncwarp();
  double best = INFINITY;
  int bkey = 1 << 30, bnl = 0;
  if (g.n > 1) {
    for (int a = 0; a < 3; a++) {
      double ext = g.C[3 + a] - g.C[a];
      if (!(ext > 0.0)) continue;
      double scale = (double)kBins / ext;
      int cnt, pn, sn;
      double bb[6], cb[6], pb[6], sb[6];
      sah_bin_data(g, lr, a, scale, bin, bins, tri, cnt, bb, cb);
      sah_scan_counts(cnt, bin, pn, sn);
      sah_scan_boxes(bb, bin, pb, sb);
      // right side of plane p = bin: the suffix of bin + 1
      int rn = __shfl_down_sync(0xffffffffu, sn, 1, 16);
      double rb[6];
#pragma unroll
      for (int k = 0; k < 6; k++) rb[k] = shfl_down_d(sb[k], 1);
      if (bin < kBins - 1 && pn != 0 && rn != 0) {
        double cost = area6(pb) * (double)pn + area6(rb) * (double)rn;
        if (cost < best) {
          best = cost;
          bkey = a * (kBins - 1) + bin;
          bnl = pn;
        }
      }
    }
  }
  // warp argmin of (cost, key)
  double wc = best;
  int wk = bkey;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double oc = __shfl_xor_sync(0xffffffffu, wc, off);
    int ok = __shfl_xor_sync(0xffffffffu, wk, off);
    if (oc < wc || (oc == wc && ok < wk)) {
      wc = oc;
      wk = ok;
    }
  }
  SSplit r;
  r.split = 0;
  r.axis = -1;
  r.plane = -1;
  r.nl = 0;
  if (wk < (1 << 30)) {
    // pass 2: the winning axis again, now with the centroid boxes (whole warp, uniform)
    const int a = wk / (kBins - 1), plane = wk % (kBins - 1);
    double scale = (double)kBins / (g.C[3 + a] - g.C[a]);
    int cnt;
    double bb[6], cb[6], pb[6], sb[6], pc[6], sc[6];
    sah_bin_data(g, lr, a, scale, bin, bins, tri, cnt, bb, cb);
    sah_scan_boxes(bb, bin, pb, sb);
    sah_scan_boxes(cb, bin, pc, sc);
    double rb[6], rc[6];
#pragma unroll
    for (int k = 0; k < 6; k++) {
      rb[k] = shfl_down_d(sb[k], 1);
      rc[k] = shfl_down_d(sc[k], 1);
    }
    if (lane != plane) return;  // the owning lane of group 0 writes the split
    r.axis = a;
    r.plane = plane;
    r.nl = bnl;
#pragma unroll
    for (int k = 0; k < 6; k++) {
      r.L[k] = pb[k];
      r.CL[k] = pc[k];
      r.R[k] = rb[k];
      r.CR[k] = rc[k];
    }
    double aB = area6(g.B);
    r.split = (g.n > kMaxLeaf || (LW_SAH_CTRAV * aB + wc) < (double)g.n * aB) ? 1 : 0;
  } else {
    if (lane != 0) return;
    if (g.n > kMaxLeaf) {
      r.split = 1;  // coincident centroids: halve in the current order
      r.axis = -1;
      r.nl = g.n / 2;
      box_reset(r.L);
      box_reset(r.R);
      box_reset(r.CL);
      box_reset(r.CR);
      for (int k = 0; k < g.n; k++) {
        int t = ids[g.start + k];
        double* B = k < r.nl ? r.L : r.R;
        double* Cc = k < r.nl ? r.CL : r.CR;
        box_grow(B, tb + 6 * (size_t)t, tb + 6 * (size_t)t + 3);
        box_grow(Cc, cen + 3 * (size_t)t, cen + 3 * (size_t)t);
      }
    }
  }
  out[s] = r;
  split_flag[s] = r.split;
}

__global__ void __launch_bounds__(128, LW_SAH_DEC_MINB) k_sah_decide_w(const SSeg* __restrict__ seg, int nseg, const int* __restrict__ large_rank,
                               const BinAcc* __restrict__ bins, const int* __restrict__ ids,
                               const double* __restrict__ tb, const double* __restrict__ cen,
                               SSplit* __restrict__ out, int* __restrict__ split_flag) {
  __shared__ double tri[4][32][9];
  const int s = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31, wib = (threadIdx.x >> 5) & 3;
  if (s >= nseg) return;  // uniform per warp
  sah_decide_seg(s, seg, large_rank, bins, ids, tb, cen, out, split_flag, tri[wib], lane);
}

__device__ __forceinline__ int leaf_ref32(long long start, long long count) {
  return (int)(-(1 + ((start << 3) | count)));
}

// node ids, parent refs, node boxes and the next level's segment table
__device__ __forceinline__ void sah_emit_seg(int s, const SSeg* __restrict__ seg, const SSplit* __restrict__ sp,
                                             const int* __restrict__ split_rank, int node_base,
                                             SahNode* __restrict__ nodes, int* __restrict__ root_ref,
                                             SSeg* __restrict__ next) {
  const SSeg g = seg[s];
  const SSplit& r = sp[s];
  int ref;
  if (!r.split) {
    ref = leaf_ref32(g.start, g.n);
  } else {
    int rank = split_rank[s];
    int id = node_base + rank;
    ref = id;
    SahNode& nd = nodes[id];
    for (int k = 0; k < 6; k++) {
      nd.box[k] = r.L[k];
      nd.box[6 + k] = r.R[k];
    }
    SSeg L, R;
    L.start = g.start;
    L.n = r.nl;
    L.parent = id;
    L.side = 0;
    R.start = g.start + r.nl;
    R.n = g.n - r.nl;
    R.parent = id;
    R.side = 1;
    for (int k = 0; k < 6; k++) {
      L.B[k] = r.L[k];
      L.C[k] = r.CL[k];
      R.B[k] = r.R[k];
      R.C[k] = r.CR[k];
    }
    next[2 * rank] = L;
    next[2 * rank + 1] = R;
  }
  if (g.parent < 0)
    *root_ref = ref;
  else
    nodes[g.parent].ref[g.side] = ref;
}

__global__ void k_sah_emit(const SSeg* __restrict__ seg, int nseg, const SSplit* __restrict__ sp,
                           const int* __restrict__ split_rank, int node_base, SahNode* __restrict__ nodes,
                           int* __restrict__ root_ref, SSeg* __restrict__ next) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) sah_emit_seg(s, seg, sp, split_rank, node_base, nodes, root_ref, next);
}

__device__ __forceinline__ int sah_left_of(int i, const int* __restrict__ pos_seg, const int* __restrict__ ids,
                                           const SSeg* __restrict__ seg, const SSplit* __restrict__ sp,
                                           const double* __restrict__ cen) {
  int s = pos_seg[i];
  int f = 0;
  if (s >= 0 && sp[s].split) {
    const SSeg& g = seg[s];
    const SSplit& r = sp[s];
    if (r.axis < 0) {
      f = (i - g.start) < r.nl;
    } else {
      double ext = g.C[3 + r.axis] - g.C[r.axis];
      int b = bin_of(cen[3 * (size_t)ids[i] + r.axis], g.C[r.axis], (double)kBins / ext);
      f = b <= r.plane;
    }
  }
  return f;
}

__global__ void k_sah_flags(const int* __restrict__ pos_seg, const int* __restrict__ ids, int n,
                            const SSeg* __restrict__ seg, const SSplit* __restrict__ sp, const double* __restrict__ cen,
                            int* __restrict__ left) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) left[i] = sah_left_of(i, pos_seg, ids, seg, sp, cen);
}

__device__ __forceinline__ void sah_scatter_pos(int i, const int* __restrict__ pos_seg, const int* __restrict__ ids,
                                                const SSeg* __restrict__ seg, const SSplit* __restrict__ sp,
                                                const int* __restrict__ split_rank, const int* __restrict__ left,
                                                const int* __restrict__ scan, int* __restrict__ ids_out,
                                                int* __restrict__ pos_out) {
  int s = pos_seg[i];
  if (s < 0 || !sp[s].split) {
    ids_out[i] = ids[i];
    pos_out[i] = -1;
    return;
  }
  const SSeg& g = seg[s];
  int nl = sp[s].nl;
  int j = i - g.start;
  int rl = scan[i] - scan[g.start];
  bool l = left[i] != 0;
  int np = l ? g.start + rl : g.start + nl + (j - rl);
  ids_out[np] = ids[i];
  pos_out[np] = 2 * split_rank[s] + (l ? 0 : 1);
}

__global__ void k_sah_scatter(const int* __restrict__ pos_seg, const int* __restrict__ ids, int n,
                              const SSeg* __restrict__ seg, const SSplit* __restrict__ sp,
                              const int* __restrict__ split_rank, const int* __restrict__ left,
                              const int* __restrict__ scan, int* __restrict__ ids_out, int* __restrict__ pos_out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) sah_scatter_pos(i, pos_seg, ids, seg, sp, split_rank, left, scan, ids_out, pos_out);
}

__global__ void k_large_flags(const SSeg* __restrict__ seg, int nseg, int* __restrict__ flag) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) flag[s] = seg[s].n > kSmall ? 1 : 0;
}

__global__ void k_large_rank(const int* __restrict__ flag, const int* __restrict__ scan, int nseg, int* __restrict__ rank) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) rank[s] = flag[s] ? scan[s] : -1;
}

// ---- small scenes: the whole level loop in one thread block ------------------------------------
// The level-synchronous build above reads two counts back per level (segments to bin, nodes
// emitted), ~100 us of launches and round trips per level: 0.8 ms for the 36-triangle Cornell box,
// whose whole render pass is 16 ms.  Up to kSmallBuildMax triangles one block runs the same
// per-level steps -- large-segment binning with the same exact atomics, the warp decision
// (sah_decide_seg), node emission, stable partition -- with block-wide scans in place of the
// device-wide ones: the same tree, one launch, one read-back.
constexpr int kSmallBuildThreads = 256;
constexpr int kSmallBuildMax = 4096;

struct SmallBuildResult {
  int nnodes, levels, root_ref, pad;
};

// exclusive scan of in[0, m) into out[0, m], out[m] = total (returned); the whole block calls it
__device__ int block_exscan(const int* __restrict__ in, int* __restrict__ out, int m) {
  using BlockScan = cub::BlockScan<int, kSmallBuildThreads>;
  __shared__ typename BlockScan::TempStorage ts;
  __shared__ int carry;
  __syncthreads();  // in[] complete
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < m; base += kSmallBuildThreads) {
    int i = base + threadIdx.x;
    int v = i < m ? in[i] : 0, x, agg;
    BlockScan(ts).ExclusiveSum(v, x, agg);
    int c = carry;
    if (i < m) out[i] = c + x;
    __syncthreads();  // carry read and temp storage reuse
    if (threadIdx.x == 0) carry = c + agg;
    __syncthreads();
  }
  int total = carry;
  if (threadIdx.x == 0) out[m] = total;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kSmallBuildThreads) k_sah_small(
    int n, const double* __restrict__ tb, const double* __restrict__ cen, int* __restrict__ ids, int* __restrict__ ids2,
    int* pos_a, int* pos_b, SSeg* seg_a, SSeg* seg_b, SSplit* __restrict__ split, int* __restrict__ sflag,
    int* __restrict__ srank, int* __restrict__ lflag, int* __restrict__ lscan, int* __restrict__ lrank,
    int* __restrict__ left, int* __restrict__ scan, BinAcc* __restrict__ bins, SahNode* __restrict__ nodes,
    int* __restrict__ root_ref, SmallBuildResult* __restrict__ res) {
  __shared__ double tri[kSmallBuildThreads / 32][32][9];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kSmallBuildThreads / 32;
  SSeg* seg = seg_a;
  SSeg* nxt = seg_b;
  int* pos = pos_a;
  int* pos2 = pos_b;
  int nseg = 1, node_base = 0, levels = 0;
  while (nseg > 0) {
    // large segments: ranks, then their bins over all positions (exact order-free atomics)
    for (int q = tid; q < nseg; q += kSmallBuildThreads) lflag[q] = seg[q].n > kSmall ? 1 : 0;
    const int nlarge = block_exscan(lflag, lscan, nseg);
    for (int q = tid; q < nseg; q += kSmallBuildThreads) lrank[q] = lflag[q] ? lscan[q] : -1;
    for (int q = tid; q < nlarge * 3 * kBins; q += kSmallBuildThreads) {
      unsigned long long* b = bins[q].v;
      b[0] = 0;
#pragma unroll
      for (int k = 0; k < 3; k++) {
        b[1 + k] = ~0ULL;
        b[4 + k] = 0ULL;
        b[7 + k] = ~0ULL;
        b[10 + k] = 0ULL;
      }
    }
    __syncthreads();
    if (nlarge > 0) {
      for (int i = tid; i < n; i += kSmallBuildThreads) {
        int sg = pos[i];
        if (sg < 0) continue;
        int lr = lrank[sg];
        if (lr < 0) continue;
        int t = ids[i];
        const double* tbt = tb + 6 * (size_t)t;
        const double* ct = cen + 3 * (size_t)t;
        const SSeg& g = seg[sg];
#pragma unroll
        for (int a = 0; a < 3; a++) {
          double ext = g.C[3 + a] - g.C[a];
          if (!(ext > 0.0)) continue;
          int b = bin_of(ct[a], g.C[a], (double)kBins / ext);
          bin_add(bins[(size_t)lr * 3 * kBins + a * kBins + b].v, tbt, ct, false);
        }
      }
    }
    __syncthreads();
    // split decisions, one warp per segment
    for (int q = warp; q < nseg; q += nw) sah_decide_seg(q, seg, lrank, bins, ids, tb, cen, split, sflag, tri[warp], lane);
    const int nsplit = block_exscan(sflag, srank, nseg);
    for (int q = tid; q < nseg; q += kSmallBuildThreads) sah_emit_seg(q, seg, split, srank, node_base, nodes, root_ref, nxt);
    // stable partition of the positions
    for (int i = tid; i < n; i += kSmallBuildThreads) left[i] = sah_left_of(i, pos, ids, seg, split, cen);
    block_exscan(left, scan, n);
    for (int i = tid; i < n; i += kSmallBuildThreads) sah_scatter_pos(i, pos, ids, seg, split, srank, left, scan, ids2, pos2);
    __syncthreads();
    for (int i = tid; i < n; i += kSmallBuildThreads) ids[i] = ids2[i];
    __syncthreads();
    int* tp = pos;
    pos = pos2;
    pos2 = tp;
    SSeg* ts = seg;
    seg = nxt;
    nxt = ts;
    node_base += nsplit;
    nseg = 2 * nsplit;
    levels++;
  }
  if (tid == 0) {
    res->nnodes = node_base;
    res->levels = levels;
    res->root_ref = *root_ref;
  }
}

}  // namespace

#define TRY(x) LW_CUDA_TRY(x)

int sah_build_device(const double* d_verts, int64_t n64, cudaStream_t st, DeviceSah& out) {
  out.nnodes = 0;
  out.root_ref = leaf_ref32_host(0, 0);
  for (int a = 0; a < 6; a++) out.root_box[a] = 0.0;
  int n = (int)n64;
  LW_CHECK_ARG(n64 >= 0 && n64 < (1LL << 28), "sah build: at most 2^28 triangles");
  TRY(cudaMallocAsync(&out.nodes, sizeof(SahNode) * (n > 1 ? n - 1 : 1), st));
  TRY(cudaMallocAsync(&out.order, sizeof(int) * (n > 0 ? n : 1), st));
  if (n == 0) return LW_OK;
  const int B = 256;
  int gn = (n + B - 1) / B;
  DevBuf b_tb, b_cen, b_ids2, b_pos, b_pos2, b_left, b_scan, b_acc, b_root;
  TRY(b_tb.alloc(sizeof(double) * 6 * (size_t)n, st));
  TRY(b_cen.alloc(sizeof(double) * 3 * (size_t)n, st));
  TRY(b_ids2.alloc(sizeof(int) * n, st));
  TRY(b_pos.alloc(sizeof(int) * n, st));
  TRY(b_pos2.alloc(sizeof(int) * n, st));
  TRY(b_left.alloc(sizeof(int) * n, st));
  TRY(b_scan.alloc(sizeof(int) * (n + 1), st));
  TRY(b_acc.alloc(sizeof(unsigned long long) * 12, st));
  TRY(b_root.alloc(sizeof(int), st));
  int* ids = out.order;
  int* ids2 = b_ids2.as<int>();
  int* pos = b_pos.as<int>();
  int* pos2 = b_pos2.as<int>();
  k_sah_prep<<<gn, B, 0, st>>>(d_verts, n, b_tb.as<double>(), b_cen.as<double>(), ids, pos);
  unsigned long long init[12];
  for (int k = 0; k < 12; k++) init[k] = ((k % 6) < 3) ? ~0ULL : 0ULL;
  TRY(cudaMemcpyAsync(b_acc.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  k_sah_root_reduce<<<std::min(gn, 1184), B, 0, st>>>(b_tb.as<double>(), b_cen.as<double>(), n,
                                                      b_acc.as<unsigned long long>());
  // segment tables (current / next); a level has at most n segments
  DevBuf b_seg[2], b_split, b_sflag, b_srank, b_lflag, b_lscan, b_lrank, b_bins, b_tmp;
  TRY(b_seg[0].alloc(sizeof(SSeg) * n, st));
  TRY(b_seg[1].alloc(sizeof(SSeg) * n, st));
  TRY(b_split.alloc(sizeof(SSplit) * n, st));
  TRY(b_sflag.alloc(sizeof(int) * (n + 1), st));
  TRY(b_srank.alloc(sizeof(int) * (n + 1), st));
  TRY(b_lflag.alloc(sizeof(int) * (n + 1), st));
  TRY(b_lscan.alloc(sizeof(int) * (n + 1), st));
  TRY(b_lrank.alloc(sizeof(int) * (n + 1), st));
  int max_large = n / (kSmall + 1) + 1;
  TRY(b_bins.alloc(sizeof(BinAcc) * 3 * kBins * (size_t)max_large, st));
  k_sah_root_init<<<1, 1, 0, st>>>(b_acc.as<unsigned long long>(), b_seg[0].as<SSeg>(), n);
  size_t tb1 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb1, b_left.as<int>(), b_scan.as<int>(), n + 1, st);
  TRY(b_tmp.alloc(tb1, st));
  if (n <= kSmallBuildMax && !getenv("LW_SAH_LEVELS") && !getenv("LW_SAH_SERIAL") && !getenv("LW_SAH_CHECK")) {
    DevBuf b_res;
    TRY(b_res.alloc(sizeof(SmallBuildResult), st));
    k_sah_small<<<1, kSmallBuildThreads, 0, st>>>(
        n, b_tb.as<double>(), b_cen.as<double>(), ids, ids2, pos, pos2, b_seg[0].as<SSeg>(), b_seg[1].as<SSeg>(),
        b_split.as<SSplit>(), b_sflag.as<int>(), b_srank.as<int>(), b_lflag.as<int>(), b_lscan.as<int>(),
        b_lrank.as<int>(), b_left.as<int>(), b_scan.as<int>(), b_bins.as<BinAcc>(), out.nodes, b_root.as<int>(),
        b_res.as<SmallBuildResult>());
    TRY(cudaGetLastError());
    SmallBuildResult hr;
    unsigned long long acc[12];
    TRY(cudaMemcpyAsync(&hr, b_res.p, sizeof(hr), cudaMemcpyDeviceToHost, st));
    TRY(cudaMemcpyAsync(acc, b_acc.p, sizeof(acc), cudaMemcpyDeviceToHost, st));
    TRY(cudaStreamSynchronize(st));
    out.nnodes = hr.nnodes;
    out.levels = hr.levels;
    out.root_ref = hr.root_ref;
    for (int k = 0; k < 6; k++) {
      unsigned long long u = acc[k];
      unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
      double d;
      memcpy(&d, &b, sizeof(d));
      out.root_box[k] = d;
    }
    return LW_OK;
  }
  int nseg = 1, cur = 0, node_base = 0;
  int h_counts[2];
  while (nseg > 0) {
    SSeg* seg = b_seg[cur].as<SSeg>();
    SSeg* nxt = b_seg[cur ^ 1].as<SSeg>();
    int gs = (nseg + B - 1) / B;
    // large-segment ranks and bins
    k_large_flags<<<gs, B, 0, st>>>(seg, nseg, b_lflag.as<int>());
    size_t t = b_tmp.bytes;
    TRY(cub::DeviceScan::ExclusiveSum(b_tmp.p, t, b_lflag.as<int>(), b_lscan.as<int>(), nseg + 1, st));
    k_large_rank<<<gs, B, 0, st>>>(b_lflag.as<int>(), b_lscan.as<int>(), nseg, b_lrank.as<int>());
    TRY(cudaMemcpyAsync(&h_counts[0], b_lscan.as<int>() + nseg, sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(cudaStreamSynchronize(st));
    int nlarge = h_counts[0];
    if (nlarge > 0) {
      int nb = nlarge * 3 * kBins;
      k_sah_bins_init<<<(nb + B - 1) / B, B, 0, st>>>(b_bins.as<BinAcc>(), nb);
      k_sah_bin_large<<<(n + kChunk - 1) / kChunk, B, 0, st>>>(pos, ids, n, seg, b_lrank.as<int>(), b_tb.as<double>(),
                                                              b_cen.as<double>(), b_bins.as<BinAcc>());
    }
    if (getenv("LW_SAH_CHECK")) {
      std::vector<SSplit> h1(nseg), h2(nseg);
      k_sah_decide<<<(nseg + 63) / 64, 64, 0, st>>>(seg, nseg, b_lrank.as<int>(), b_bins.as<BinAcc>(), ids,
                                                    b_tb.as<double>(), b_cen.as<double>(), b_split.as<SSplit>(),
                                                    b_sflag.as<int>());
      cudaMemcpyAsync(h1.data(), b_split.p, sizeof(SSplit) * nseg, cudaMemcpyDeviceToHost, st);
      k_sah_decide_w<<<(nseg + 3) / 4, 128, 0, st>>>(seg, nseg, b_lrank.as<int>(), b_bins.as<BinAcc>(), ids,
                                                     b_tb.as<double>(), b_cen.as<double>(), b_split.as<SSplit>(),
                                                     b_sflag.as<int>());
      cudaMemcpyAsync(h2.data(), b_split.p, sizeof(SSplit) * nseg, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      int bad = 0;
      for (int q = 0; q < nseg && bad < 5; q++) {
        const SSplit &x = h1[q], &y = h2[q];
        bool same = x.split == y.split && x.axis == y.axis && x.plane == y.plane && x.nl == y.nl;
        if (same && x.split) same = memcmp(x.L, y.L, sizeof(x.L)) == 0 && memcmp(x.R, y.R, sizeof(x.R)) == 0;
        if (!same) {
          bad++;
          fprintf(stderr, "seg %d/%d: serial split %d axis %d plane %d nl %d | warp split %d axis %d plane %d nl %d\n", q,
                  nseg, x.split, x.axis, x.plane, x.nl, y.split, y.axis, y.plane, y.nl);
        }
      }
    }
    if (getenv("LW_SAH_SERIAL"))
      k_sah_decide<<<(nseg + 63) / 64, 64, 0, st>>>(seg, nseg, b_lrank.as<int>(), b_bins.as<BinAcc>(), ids,
                                                    b_tb.as<double>(), b_cen.as<double>(), b_split.as<SSplit>(),
                                                    b_sflag.as<int>());
    else
      k_sah_decide_w<<<(nseg + 3) / 4, 128, 0, st>>>(seg, nseg, b_lrank.as<int>(), b_bins.as<BinAcc>(), ids,
                                                     b_tb.as<double>(), b_cen.as<double>(), b_split.as<SSplit>(),
                                                     b_sflag.as<int>());
    t = b_tmp.bytes;
    TRY(cub::DeviceScan::ExclusiveSum(b_tmp.p, t, b_sflag.as<int>(), b_srank.as<int>(), nseg + 1, st));
    k_sah_emit<<<gs, B, 0, st>>>(seg, nseg, b_split.as<SSplit>(), b_srank.as<int>(), node_base, out.nodes,
                                 b_root.as<int>(), nxt);
    k_sah_flags<<<gn, B, 0, st>>>(pos, ids, n, seg, b_split.as<SSplit>(), b_cen.as<double>(), b_left.as<int>());
    t = b_tmp.bytes;
    TRY(cub::DeviceScan::ExclusiveSum(b_tmp.p, t, b_left.as<int>(), b_scan.as<int>(), n, st));
    k_sah_scatter<<<gn, B, 0, st>>>(pos, ids, n, seg, b_split.as<SSplit>(), b_srank.as<int>(), b_left.as<int>(),
                                    b_scan.as<int>(), ids2, pos2);
    TRY(cudaGetLastError());
    TRY(cudaMemcpyAsync(ids, ids2, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    std::swap(pos, pos2);
    TRY(cudaMemcpyAsync(&h_counts[1], b_srank.as<int>() + nseg, sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(cudaStreamSynchronize(st));
    int nsplit = h_counts[1];
    node_base += nsplit;
    nseg = 2 * nsplit;
    cur ^= 1;
    out.levels++;
  }
  out.nnodes = node_base;
  int rr = 0;
  unsigned long long acc[12];
  TRY(cudaMemcpyAsync(&rr, b_root.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY(cudaMemcpyAsync(acc, b_acc.p, sizeof(acc), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  out.root_ref = rr;
  for (int k = 0; k < 6; k++) {
    unsigned long long u = acc[k];
    unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
    double d;
    memcpy(&d, &b, sizeof(d));
    out.root_box[k] = d;
  }
  return LW_OK;
}

}  // namespace lw
