// Shared types and device helpers for the B200 middle-MPO engine.
//
// Complex numbers are stored interleaved (re, im) exactly like numpy's
// complex128 / complex64, so a site tensor (l, top, bottom, r) in row-major
// order is byte-identical to the reference's ndarray linearization
// (reference tensor.py:1-8).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cmath>

namespace mb {

// Debug-only environment switches (shape/timing logs, matrix dumps, site
// checks) exist only in builds with -DMB_DEBUG_LOGS=1 (MB_DEBUG_BUILD=1 in
// _build.py); in release builds this returns nullptr at compile time and the
// synchronizing debug paths are dead code.
#ifndef MB_DEBUG_LOGS
#define MB_DEBUG_LOGS 0
#endif
inline const char* mb_debug_env(const char* name) {
#if MB_DEBUG_LOGS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

template <typename R>
struct alignas(2 * sizeof(R)) cx {
  R x, y;
};

template <typename R>
__host__ __device__ __forceinline__ cx<R> mk(R a, R b) { return cx<R>{a, b}; }
template <typename R>
__host__ __device__ __forceinline__ cx<R> cadd(cx<R> a, cx<R> b) { return {a.x + b.x, a.y + b.y}; }
template <typename R>
__host__ __device__ __forceinline__ cx<R> csub(cx<R> a, cx<R> b) { return {a.x - b.x, a.y - b.y}; }
template <typename R>
__host__ __device__ __forceinline__ cx<R> cmul(cx<R> a, cx<R> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// conj(a) * b
template <typename R>
__host__ __device__ __forceinline__ cx<R> cmulc(cx<R> a, cx<R> b) {
  return {a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x};
}
template <typename R>
__host__ __device__ __forceinline__ cx<R> cconj(cx<R> a) { return {a.x, -a.y}; }
template <typename R>
__host__ __device__ __forceinline__ cx<R> cscale(cx<R> a, R s) { return {a.x * s, a.y * s}; }
template <typename R>
__host__ __device__ __forceinline__ R cabs2(cx<R> a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
template <typename R>
__device__ __forceinline__ void cfma(cx<R>& acc, cx<R> a, cx<R> b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename R>
__device__ __forceinline__ void cfmac(cx<R>& acc, cx<R> a, cx<R> b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

template <typename R>
struct Eps;
template <>
struct Eps<double> {
  static constexpr double u = 1.1102230246251565e-16;
};
template <>
struct Eps<float> {
  static constexpr double u = 5.9604644775390625e-08;
};

}  // namespace mb
