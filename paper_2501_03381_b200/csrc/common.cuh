// Shared device/host helpers for libhoib200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <atomic>

#include "../../include/hoi_b200.h"

namespace hoib {

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int check_launch(const char *what);
void count_launch(int n = 1);

#define HOI_CHECK_ARG(cond, msg)                 \
  do {                                           \
    if (!(cond)) return ::hoib::fail(HOI_INVALID_ARG, msg); \
  } while (0)

// -------------------------------------------------------------- binomials --
// C(n, m) for 0 <= n, m <= 64 in constant memory (saturated at UINT64_MAX when
// it does not fit; callers restrict themselves to ranges that fit).
constexpr int kBinomN = 65;
uint64_t host_binom(int n, int m);
void fill_binomials(uint64_t *h);   // host table, kBinomN^2 entries
// Without relocatable device code every translation unit owns its own copy
// of the constant table, so the uploader is instantiated per unit too.
static __constant__ uint64_t c_binom[kBinomN * kBinomN];
// Global copy for lookups whose indices differ across a warp (constant
// memory serialises divergent addresses; this one goes through L1).
static __device__ uint64_t g_binom_l1[kBinomN * kBinomN];
static inline void upload_binomials() {
  static thread_local int uploaded_for = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (uploaded_for == dev) return;
  uint64_t h[kBinomN * kBinomN];
  fill_binomials(h);
  cudaMemcpyToSymbol(c_binom, h, sizeof(h));
  cudaMemcpyToSymbol(g_binom_l1, h, sizeof(h));
  uploaded_for = dev;
}

__device__ __forceinline__ uint64_t binom(int n, int m) {
  return (m < 0 || n < 0 || m > n) ? 0ull : c_binom[n * kBinomN + m];
}
__device__ __forceinline__ uint64_t binom_l1(int n, int m) {
  return (m < 0 || n < 0 || m > n) ? 0ull : __ldg(g_binom_l1 + n * kBinomN + m);
}

// ------------------------------------------------- floating-point helpers --
// Running product with a split-off binary exponent: the mantissa is only
// renormalised when it leaves [1e-150, 1e150], so products of up to ~64
// factors never overflow/underflow while exact products (an identity
// matrix gives exactly 1) keep an exact log of 0.  One log per product.
struct LogProd {
  double m;
  int e;
  __device__ __forceinline__ void init() { m = 1.0; e = 0; }
  __device__ __forceinline__ void mul(double x) { m *= x; }
  // Fold the exponent into e when |m| leaves [2^-498, 2^499) (frexp's
  // exact normalisation to [0.5, 1); round 1 used the thresholds 1e-150 and
  // 1e150 and a branch).  Branch-free: the per-n-plet kernels call it inside
  // their unrolled factorisations, where a branch splits the straight-line
  // code the scheduler interleaves.  Denormals are first scaled by 2^54
  // (exact); zero, inf and NaN pass through unchanged.
  __device__ __forceinline__ void renorm() {
    const int ex0 = (int)((__double_as_longlong(m) >> 52) & 0x7FF);
    const double ms = ex0 == 0 ? m * 18014398509481984.0 : m;   // 2^54
    const long long b = __double_as_longlong(ms);
    const int ex = (int)((b >> 52) & 0x7FF);
    const bool out = ex != 0 && ex != 0x7FF && (ex < 1023 - 498 || ex > 1023 + 498);
    const double mn = __longlong_as_double((b & ~(0x7FFll << 52)) | (1022ll << 52));
    m = out ? mn : m;
    e += out ? ex - 1022 - (ex0 == 0 ? 54 : 0) : 0;
  }
  __device__ __forceinline__ double log_value() const {
    double l = log(m);
    return e == 0 ? l : l + (double)e * 0.69314718055994530942;
  }
};

// Order-preserving map of a double onto uint64 (-0.0 canonicalised to +0.0,
// which is how value comparisons, and hence scipy's rankdata, treat it).
__device__ __forceinline__ uint64_t orderable_key(double v) {
  if (v == 0.0) v = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (int)(g < 1 ? 1 : g);
}

// Stream-ordered scratch from the device's default pool.  The pool's release
// threshold defaults to 0, which hands freed memory back to the driver at
// every synchronize and makes the next call map pages again (milliseconds
// per call); keep up to 256 MB cached instead.
inline cudaError_t stream_alloc(void **p, size_t bytes, cudaStream_t s) {
  static const bool pooled = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 256ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return true;
  }();
  (void)pooled;
  return cudaMallocAsync(p, bytes, s);
}

}  // namespace hoib
