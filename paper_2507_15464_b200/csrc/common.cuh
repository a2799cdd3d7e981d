// Shared helpers for the tidas_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/tidas_b200.h"

namespace tidas {

// ---------------------------------------------------------------- errors

void set_error(const char* fmt, ...);

#define TIDAS_REQUIRE(cond, ...)          \
  do {                                    \
    if (!(cond)) {                        \
      ::tidas::set_error(__VA_ARGS__);    \
      return TIDAS_EINVAL;                \
    }                                     \
  } while (0)

#define TIDAS_CUDA_CHECK(expr)                                              \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::tidas::set_error("%s: %s", #expr, cudaGetErrorString(_e));          \
      return TIDAS_ECUDA;                                                   \
    }                                                                       \
  } while (0)

#define TIDAS_LAUNCH_CHECK()                                                \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) {                                                \
      ::tidas::set_error("kernel launch: %s", cudaGetErrorString(_e));      \
      return TIDAS_ECUDA;                                                   \
    }                                                                       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- complex

template <typename R> struct cplx_t;
template <> struct cplx_t<float> { using type = float2; };
template <> struct cplx_t<double> { using type = double2; };
template <typename R> using cplx = typename cplx_t<R>::type;

template <typename C> __host__ __device__ __forceinline__ C cmake(double re, double im) {
  C r; r.x = re; r.y = im; return r;
}
// FP32 complex arithmetic on the packed sm_100 pipes (FADD2 / FMUL2 / FFMA2):
// one instruction per complex add, two per complex multiply (a.x b + a.y (i b):
// one product rounded, the other fused, as the scalar form contracts). The
// swaps and signs of a multiplication by +-i fold into FADD2's operand
// modifiers when the translation unit is built without -ftz (analytic.cu,
// _build.py); with -ftz the compiler materialises negated copies instead.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
}
// a * (c + i s) for a constant twiddle given as (c, s) and its rotation (-s, c)
__device__ __forceinline__ float2 cmul_k(float2 a, float2 cs, float2 rot) {
  return __ffma2_rn(make_float2(a.x, a.x), cs, __fmul2_rn(make_float2(a.y, a.y), rot));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename C, typename R> __device__ __forceinline__ C cscale(C a, R s) {
  C r; r.x = a.x * s; r.y = a.y * s; return r;
}
// multiply by -i (fwd) or +i (inv)
template <bool INV, typename C> __device__ __forceinline__ C mul_mi(C a) {
  C r;
  if (INV) { r.x = -a.y; r.y = a.x; } else { r.x = a.y; r.y = -a.x; }
  return r;
}
__device__ __forceinline__ float cabs_(float2 a) { return sqrtf(a.x * a.x + a.y * a.y); }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }

}  // namespace tidas
