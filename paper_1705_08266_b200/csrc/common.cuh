// common.cuh -- shared device helpers for the b2dwt kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define B2DWT_HD __host__ __device__

namespace b2dwt {

// One compiled term: out[target] (+)= coeff * in[src][n+dn, m+dm].  `unit`
// marks a coefficient that is exactly 1.0 in the built-in program (the host
// verifies it at plan time), so the kernel skips that multiply: x * 1.0 == x
// in IEEE arithmetic, which keeps strict mode bit-exact.
struct TermInfo {
  int src, dm, dn, unit;
};
// Vertical (up = max -dn, down = max dn) and horizontal reach of a sub-step.
struct Reach {
  int up, down, left, right;
};
// Per source component: used at all, max left / right column reach.
struct CompNeed {
  int used, left, right;
};

namespace progs {
#include "programs.inc"
}  // namespace progs

// Pixel parity of component c on each axis (engine.py:52).
B2DWT_HD constexpr int row_parity(int c) { return c >> 1; }
B2DWT_HD constexpr int col_parity(int c) { return c & 1; }

// Component index actually read at quad index i for a component of phase
// `parity` and length cs: whole-sample symmetric extension in pixel
// coordinates (engine.py:55-92).  Periodic, so tiny sizes fold repeatedly.
__device__ __forceinline__ int reflect(int i, int parity, int cs) {
  const int size = 2 * cs;  // >= 2
  const int period = 2 * size - 2;
  int r = (2 * i + parity) % period;
  if (r < 0) r += period;
  if (r >= size) r = period - r;
  return (r - parity) >> 1;
}

// Arithmetic policies.  Strict: separately rounded IEEE multiply and add in
// the compiled order -- NumPy's `acc = x*k; acc += x*k` (engine.py:350-362).
// Fast: fused multiply-add in the same order -- and ONLY there: the leading
// product and unit additions stay separately rounded, so the compiler cannot
// contract them differently in different kernels (stream, tile, two-level
// fused) and every fast kernel computes the same bits.
template <bool kStrict>
struct Arith;
template <>
struct Arith<true> {
  static __device__ __forceinline__ float mul(float x, float k) { return __fmul_rn(x, k); }
  static __device__ __forceinline__ double mul(double x, double k) { return __dmul_rn(x, k); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ float mac(float acc, float x, float k) { return __fadd_rn(acc, __fmul_rn(x, k)); }
  static __device__ __forceinline__ double mac(double acc, double x, double k) {
    return __dadd_rn(acc, __dmul_rn(x, k));
  }
};
template <>
struct Arith<false> {
  static __device__ __forceinline__ float mul(float x, float k) { return __fmul_rn(x, k); }
  static __device__ __forceinline__ double mul(double x, double k) { return __dmul_rn(x, k); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ float mac(float acc, float x, float k) { return fmaf(x, k, acc); }
  static __device__ __forceinline__ double mac(double acc, double x, double k) { return fma(x, k, acc); }
};

// Fast mode's one contraction, made explicit: when a target's first term is a
// product and its second a unit term, the pair is evaluated as one fused
// multiply-add, fma(x0, k0, x1) (what a contracting compiler would emit for
// x0 * k0 + x1, but fixed here so every kernel computes the same bits).
// defer(K, count, unit_K, unit_next): term K's product is deferred to K + 1.
template <bool kStrict>
struct FastJoin {
  B2DWT_HD static constexpr bool defer(int k, int count, bool unit_k, bool unit_next) {
    return !kStrict && k == 0 && count > 1 && !unit_k && unit_next;
  }
};

}  // namespace b2dwt
