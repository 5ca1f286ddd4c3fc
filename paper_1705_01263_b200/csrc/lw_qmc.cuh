// lw_qmc.cuh -- scrambled Halton sampler on the device (_kernels.py:160-208, qmc.py:112-135).
//
// Per dimension the host packs {base, perm offset, 32- and 64-bit magic dividers}
// (qmc.py:153-164 construction).  Digits come from strength-reduced division
// (__umulhi / __umul64hi) instead of hardware division.  Two evaluation regimes give
// results bit-identical to the reference kernel:
//   * base*index < 2^53: every intermediate of the reference's double accumulation is an
//     exact integer, so the digit reversal is accumulated in uint64 and rounded once by
//     the final IEEE division (the reference's single rounding);
//   * otherwise: the reference's double operations are replayed one by one.
#pragma once
#include "lw_common.cuh"

struct QmcDim {
  uint32_t base;
  uint32_t perm_off;
  uint32_t magic32;
  uint8_t shift32, add32, shift64, add64;
  uint64_t magic64;
  uint64_t exact_limit;  // largest index with base*index < 2^53
  uint32_t digits32;     // digits of 2^32-1 in this base if perm[0] == 0, else 0 (no padding)
  uint32_t pad_;
};

__device__ __forceinline__ uint32_t lw_div32(uint32_t n, const QmcDim& d) {
  uint32_t q = __umulhi(n, d.magic32);
  if (d.add32) return (((n - q) >> 1) + q) >> d.shift32;
  return q >> d.shift32;
}

__device__ __forceinline__ uint64_t lw_div64(uint64_t n, const QmcDim& d) {
  uint64_t q = __umul64hi(n, d.magic64);
  if (d.add64) return (((n - q) >> 1) + q) >> d.shift64;
  return q >> d.shift64;
}

// radical_inverse_base2, _kernels.py:181-192
__device__ __forceinline__ double lw_ri_base2(long long index) {
  if (index <= 0) return 0.0;
  uint64_t n = (uint64_t)index;
  int nbits = 64 - __clzll((long long)n);
  if (n < (1ULL << 53)) {
    uint64_t rev = __brevll(n) >> (64 - nbits);
    return (double)rev / (double)(1ULL << nbits);
  }
  double rev = 0.0, scale = 1.0;
  while (n > 0) {
    rev = rev * 2.0 + (double)(n & 1);
    scale = scale * 2.0;
    n >>= 1;
  }
  return rev / scale;
}

// halton_dim, _kernels.py:195-208
__device__ __forceinline__ double lw_halton(const QmcDim* __restrict__ dims, const uint16_t* __restrict__ perm,
                                            int dim, long long index) {
  QmcDim d = dims[dim];
  if (d.base == 2) return lw_ri_base2(index);
  if (index <= 0) return 0.0;
  uint64_t n = (uint64_t)index;
  const uint16_t* p = perm + d.perm_off;
  const uint32_t b = d.base;
  if (n <= d.exact_limit) {
    uint64_t rev = 0, scale = 1;
    while (n >> 32) {
      uint64_t q = lw_div64(n, d);
      uint32_t digit = (uint32_t)(n - q * b);
      rev = rev * b + __ldg(p + digit);
      scale *= b;
      n = q;
    }
    uint32_t m = (uint32_t)n;
    if (d.digits32 && scale == 1) {
      // fixed digit count: sigma(0) == 0, so zero digits above the top one scale rev and scale
      // alike and the exact ratio (hence its correctly rounded quotient) is unchanged; with no
      // data-dependent exit the table loads of all digits are independent and overlap
#pragma unroll 4
      for (uint32_t k = 0; k < d.digits32; k++) {
        uint32_t q = lw_div32(m, d);
        uint32_t digit = m - q * b;
        rev = rev * b + __ldg(p + digit);
        scale *= b;
        m = q;
      }
      return (double)rev / (double)scale;
    }
    while (m) {
      uint32_t q = lw_div32(m, d);
      uint32_t digit = m - q * b;
      rev = rev * b + __ldg(p + digit);
      scale *= b;
      m = q;
    }
    return (double)rev / (double)scale;
  }
  double rev = 0.0, scale = 1.0, bd = (double)b;
  while (n > 0) {
    uint64_t q = lw_div64(n, d);
    uint32_t digit = (uint32_t)(n - q * b);
    rev = rev * bd + (double)__ldg(p + digit);
    scale = scale * bd;
    n = q;
  }
  return rev / scale;
}

// Two dimensions of the same index with interleaved digit loops: the two dependent
// divide-and-accumulate chains run side by side (instruction-level parallelism for the
// latency-bound shading kernels).  Same integers and the same final divisions as lw_halton, so
// the same bits; falls back to lw_halton outside the fixed-digit 32-bit regime.
__device__ __forceinline__ void lw_halton2(const QmcDim* __restrict__ dims, const uint16_t* __restrict__ perm, int dimA,
                                           int dimB, long long index, double& a, double& b) {
  QmcDim A = dims[dimA], B = dims[dimB];
  uint64_t n = (uint64_t)index;
  if (index <= 0 || A.base == 2 || B.base == 2 || !A.digits32 || !B.digits32 || (n >> 32) || n > A.exact_limit ||
      n > B.exact_limit) {
    a = lw_halton(dims, perm, dimA, index);
    b = lw_halton(dims, perm, dimB, index);
    return;
  }
  const uint16_t *pa = perm + A.perm_off, *pb = perm + B.perm_off;
  uint32_t ma = (uint32_t)n, mb = (uint32_t)n;
  uint64_t ra = 0, sa = 1, rb = 0, sb = 1;
  const uint32_t kmax = A.digits32 > B.digits32 ? A.digits32 : B.digits32;
#pragma unroll 2
  for (uint32_t k = 0; k < kmax; k++) {
    if (k < A.digits32) {
      uint32_t q = lw_div32(ma, A);
      uint32_t digit = ma - q * A.base;
      ra = ra * A.base + __ldg(pa + digit);
      sa *= A.base;
      ma = q;
    }
    if (k < B.digits32) {
      uint32_t q = lw_div32(mb, B);
      uint32_t digit = mb - q * B.base;
      rb = rb * B.base + __ldg(pb + digit);
      sb *= B.base;
      mb = q;
    }
  }
  a = (double)ra / (double)sa;
  b = (double)rb / (double)sb;
}
