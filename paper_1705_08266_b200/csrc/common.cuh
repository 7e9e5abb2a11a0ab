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
// Row address base + n * ldb (ldb: pitch in bytes) for the fused kernel's
// sinks.  Written as int64 arithmetic there, the compiler kept the operands'
// sign words in registers and emitted a 64 x 64 multiply (4 instructions per
// store address); as unsigned 32 x 32 -> 64 the loop got shorter (711 vs 739
// instructions) but slower.  Measured on C3 (tools/ab_lib.sh, same box):
// levels 0+1 406.6 -> 405.7 us fast, 445 -> 429 us strict with this form;
// 420 / 460 us unsigned.  (The stream kernel's int64 form already compiles to
// one IMAD.WIDE with the base as addend and keeps it.)
__device__ __forceinline__ char* row_addr(const void* base, int n, int ldb) {
  unsigned long long r;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(n), "r"(ldb), "l"(base));
  return reinterpret_cast<char*>(r);
}

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

// Evaluation order of a target's terms.  Strict: the compiled order
// (engine.py:267), separately rounded.  Fast: the target's unit term first
// (when it has exactly one: acc = x), then every product in compiled order as
// one fused multiply-add -- the contraction a compiler might apply to
// x0 * k0 + x1 made explicit and applied to every target, so each product is
// exactly one FMA and every fast kernel (stream, two-level fused, tile)
// computes the same bits.  at(base, count, k) = offset of the k-th evaluated term.
template <class P, bool kStrict>
struct TermOrder {
  B2DWT_HD static constexpr int unit_pos(int base, int count) {
    int u = -1, n = 0;
    for (int k = 0; k < count; ++k)
      if (P::term(base + k).unit) {
        u = k;
        ++n;
      }
    return n == 1 ? u : -1;
  }
  B2DWT_HD static constexpr int at(int base, int count, int k) {
    if (kStrict) return k;
    const int u = unit_pos(base, count);
    if (u < 0) return k;
    if (k == 0) return u;
    return k <= u ? k - 1 : k;
  }
};

}  // namespace b2dwt
