// lw_common.cuh -- error plumbing and small vector helpers shared by every TU of liblw_b200.so.
//
// All device arithmetic in this library is IEEE binary64 evaluated exactly as written:
// the library is compiled with -fmad=false (no contraction of mul+add into FMA), and
// divisions / square roots use the correctly rounded defaults (-prec-div, -prec-sqrt).
// This is what makes every result bit-identical to the CPU oracle (built with
// -ffp-contract=off) and, on the reference-defined paths, to the reference itself.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/lw_b200.h"

namespace lw {

void set_error(const char* fmt, ...);

#define LW_CUDA_TRY(expr)                                                                      \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      ::lw::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return _e == cudaErrorMemoryAllocation ? LW_ERR_NOMEM : LW_ERR_CUDA;                     \
    }                                                                                          \
  } while (0)

#define LW_CHECK_ARG(cond, msg)      \
  do {                               \
    if (!(cond)) {                   \
      ::lw::set_error("%s", msg);    \
      return LW_ERR_INVALID;         \
    }                                \
  } while (0)

#define LW_STATUS_TRY(expr)  \
  do {                       \
    int _s = (expr);         \
    if (_s != LW_OK) return _s; \
  } while (0)

// RAII device buffer.  alloc(n) is a plain cudaMalloc (stateless entry points); alloc(n, stream)
// is stream-ordered (cudaMallocAsync from the device's default pool, whose release threshold the
// render context raises), so builder temporaries cost neither a driver allocation nor the
// implicit device synchronisation of cudaFree.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool async = false;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (!p) return;
    if (async)
      cudaFreeAsync(p, st);
    else
      cudaFree(p);
  }
  cudaError_t alloc(size_t n) {
    bytes = n;
    return cudaMalloc(&p, n > 0 ? n : 16);
  }
  cudaError_t alloc(size_t n, cudaStream_t stream) {
    bytes = n;
    async = true;
    st = stream;
    return cudaMallocAsync(&p, n > 0 ? n : 16, stream);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline int grid_for(int64_t n, int block, int max_blocks = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

}  // namespace lw

// ---- device vector helpers (plain IEEE ops, evaluation order fixed) -------------------
struct v3 {
  double x, y, z;
};

__host__ __device__ __forceinline__ v3 mk3(double x, double y, double z) {
  v3 r;
  r.x = x;
  r.y = y;
  r.z = z;
  return r;
}
__host__ __device__ __forceinline__ v3 operator+(v3 a, v3 b) { return mk3(a.x + b.x, a.y + b.y, a.z + b.z); }
__host__ __device__ __forceinline__ v3 operator-(v3 a, v3 b) { return mk3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ __forceinline__ v3 operator*(v3 a, double s) { return mk3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ __forceinline__ v3 neg3(v3 a) { return mk3(-a.x, -a.y, -a.z); }
__host__ __device__ __forceinline__ double dot3(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ __forceinline__ v3 cross3(v3 a, v3 b) {
  return mk3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ v3 normalize3(v3 a) {
  double inv = 1.0 / sqrt(dot3(a, a));
  return mk3(a.x * inv, a.y * inv, a.z * inv);
}
__host__ __device__ __forceinline__ v3 bary3(v3 a, v3 b, v3 c, double w, double bu, double bv) {
  return mk3((w * a.x + bu * b.x) + bv * c.x, (w * a.y + bu * b.y) + bv * c.y, (w * a.z + bu * b.z) + bv * c.z);
}
