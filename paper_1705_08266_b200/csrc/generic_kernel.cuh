// generic_kernel.cuh -- per-sub-step stencil interpreter (any StencilProgram).
//
// Used for programs whose structure is not one of the built-in fused kernels
// (custom lifting plans with other supports, the reference tests' HAAR_LIKE /
// TRIVIAL plans) and as a cross-check of the fused kernel.  It is the direct
// GPU analogue of liftfuse's run_reference (engine.py:442-451): one launch
// per sub-step, gather from the full previous state through the reflection
// map (engine.py:82-92), out-of-place.  One thread per quad.
#pragma once

#include "common.cuh"

namespace b2dwt {

constexpr int kGenericMaxTerms = 192;

struct GenericTerm {
  int8_t src, dm, dn, tgt;
  float pad;
  double coeff;
};

template <class T>
struct PlaneView {
  T* p;
  int64_t rs, cs;  // element (n, m) = p[n * rs + m * cs]
};

struct GenericSubstep {
  int count[4];
  GenericTerm terms[kGenericMaxTerms];
};

template <class T, bool kStrict>
__global__ void __launch_bounds__(256)
    generic_substep_kernel(const __grid_constant__ GenericSubstep sub, PlaneView<const T> i0, PlaneView<const T> i1,
                           PlaneView<const T> i2, PlaneView<const T> i3, PlaneView<T> o0, PlaneView<T> o1,
                           PlaneView<T> o2, PlaneView<T> o3, int64_t in_bstride, int64_t out_bstride, int rows,
                           int cols) {
  using Ar = Arith<kStrict>;
  const PlaneView<const T> in[4] = {i0, i1, i2, i3};
  const PlaneView<T> out[4] = {o0, o1, o2, o3};
  const int64_t b = blockIdx.y;
  const int64_t total = static_cast<int64_t>(rows) * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(idx / cols);
    const int m = static_cast<int>(idx - static_cast<int64_t>(n) * cols);
    int k = 0;
    for (int t = 0; t < 4; ++t) {
      T acc = T(0);
      for (int j = 0; j < sub.count[t]; ++j, ++k) {
        const GenericTerm& g = sub.terms[k];
        const int s = g.src;
        // reflection (a periodic map with divisions) only for reads outside the image
        const int rn = n + g.dn, cm = m + g.dm;
        const int rr = static_cast<unsigned>(rn) < static_cast<unsigned>(rows) ? rn : reflect(rn, row_parity(s), rows);
        const int cc = static_cast<unsigned>(cm) < static_cast<unsigned>(cols) ? cm : reflect(cm, col_parity(s), cols);
        const T x = in[s].p[b * in_bstride + rr * in[s].rs + cc * in[s].cs];
        const T c = static_cast<T>(g.coeff);
        acc = (j == 0) ? Ar::mul(x, c) : Ar::mac(acc, x, c);
      }
      out[t].p[b * out_bstride + n * out[t].rs + m * out[t].cs] = acc;
    }
  }
}

}  // namespace b2dwt
