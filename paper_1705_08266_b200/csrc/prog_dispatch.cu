// prog_dispatch.cu -- per-program entry points used by b2dwt_host.cu: pick the
// variant (prog_variant.cu) for a launch request, report the program's cone.
// Compiled with -DB2DWT_PROG=<ident> -DB2DWT_PROG_INV=<0|1>; holds no kernels.
#include <cuda_runtime.h>

#include "launch.h"
#include "stream_kernel.cuh"

#define B2DWT_CAT2(a, b) a##b
#define B2DWT_CAT(a, b) B2DWT_CAT2(a, b)
#define B2DWT_CAT3_(a, b, c) a##b##_##c
#define B2DWT_CAT3(a, b, c) B2DWT_CAT3_(a, b, c)
#define B2DWT_V(k) B2DWT_CAT3(b2dwt_v_, B2DWT_PROG, k)

namespace b2dwt {

cudaError_t B2DWT_V(0)(const FusedLaunch&);
cudaError_t B2DWT_V(1)(const FusedLaunch&);
cudaError_t B2DWT_V(2)(const FusedLaunch&);
cudaError_t B2DWT_V(3)(const FusedLaunch&);
cudaError_t B2DWT_V(4)(const FusedLaunch&);
cudaError_t B2DWT_V(5)(const FusedLaunch&);
cudaError_t B2DWT_V(6)(const FusedLaunch&);
cudaError_t B2DWT_V(7)(const FusedLaunch&);

namespace {
constexpr int kMainIn = B2DWT_PROG_INV ? kLayoutPlanar : kLayoutInterleaved;
constexpr int kMainOut = B2DWT_PROG_INV ? kLayoutInterleaved : kLayoutPlanar;

cudaError_t try_variant(cudaError_t (*fn)(const FusedLaunch&), const FusedLaunch& r) {
  const cudaError_t e = fn(r);
  if (e == cudaErrorNotSupported) (void)cudaGetLastError();
  return e;
}
}  // namespace

// Returns cudaErrorNotSupported when no compiled variant can serve the request
// (the host then runs the generic interpreter).
cudaError_t B2DWT_CAT(b2dwt_fused_, B2DWT_PROG)(const FusedLaunch& r, bool* used_tma) {
  *used_tma = false;
  const bool main = r.lin == kMainIn && r.lout == kMainOut;
  const bool pp = r.lin == kLayoutPlanar && r.lout == kLayoutPlanar;
  if (r.dtype == 1) {
    if (main) return try_variant(&B2DWT_V(6), r);
    if (pp) return try_variant(&B2DWT_V(7), r);
    return cudaErrorNotSupported;
  }
  if (pp) return try_variant(r.strict ? &B2DWT_V(4) : &B2DWT_V(5), r);
  if (!main) return cudaErrorNotSupported;
  if (r.allow_tma) {
    const cudaError_t e = try_variant(r.strict ? &B2DWT_V(0) : &B2DWT_V(1), r);
    if (e != cudaErrorNotSupported) {
      *used_tma = true;
      return e;
    }
  }
  return try_variant(r.strict ? &B2DWT_V(2) : &B2DWT_V(3), r);
}

ConeInfo B2DWT_CAT(b2dwt_cone_, B2DWT_PROG)() {
  using C = Geo<progs::B2DWT_PROG>;
  return ConeInfo{C::up, C::down, C::left, C::right};
}

}  // namespace b2dwt
