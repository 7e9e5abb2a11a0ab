// prog_variant.cu -- ONE fused-kernel instantiation of ONE built-in program.
//
// Compiled with -DB2DWT_PROG=<ident> -DB2DWT_PROG_INV=<0|1> -DB2DWT_VID=<k>
// (see paper_1705_08266_b200/build.py); -DB2DWT_STUB compiles a placeholder
// that reports cudaErrorNotSupported (development builds of a subset).
//
//   VID  element  layout                      arithmetic  fill
//    0   f32      main (fwd I->P, inv P->I)   strict      TMA
//    1   f32      main                        fast (FMA)  TMA
//    2   f32      main                        strict      cp.async
//    3   f32      main                        fast        cp.async
//    4   f32      planar -> planar            strict      cp.async
//    5   f32      planar -> planar            fast        cp.async
//    6   f64      main                        strict      cp.async
//    7   f64      planar -> planar            strict      cp.async
#include "launch_impl.cuh"

#ifndef B2DWT_PROG
#error "compile with -DB2DWT_PROG=<program ident>"
#endif

#define B2DWT_CAT3_(a, b, c) a##b##_##c
#define B2DWT_CAT3(a, b, c) B2DWT_CAT3_(a, b, c)

namespace b2dwt {
namespace {

constexpr int kMainIn = B2DWT_PROG_INV ? kLayoutPlanar : kLayoutInterleaved;
constexpr int kMainOut = B2DWT_PROG_INV ? kLayoutInterleaved : kLayoutPlanar;

template <int V>
struct Variant;
template <>
struct Variant<0> { using T = float; static constexpr int kIn = kMainIn, kOut = kMainOut; static constexpr bool kStrict = true, kTma = true; };
template <>
struct Variant<1> { using T = float; static constexpr int kIn = kMainIn, kOut = kMainOut; static constexpr bool kStrict = false, kTma = true; };
template <>
struct Variant<2> { using T = float; static constexpr int kIn = kMainIn, kOut = kMainOut; static constexpr bool kStrict = true, kTma = false; };
template <>
struct Variant<3> { using T = float; static constexpr int kIn = kMainIn, kOut = kMainOut; static constexpr bool kStrict = false, kTma = false; };
template <>
struct Variant<4> { using T = float; static constexpr int kIn = kLayoutPlanar, kOut = kLayoutPlanar; static constexpr bool kStrict = true, kTma = false; };
template <>
struct Variant<5> { using T = float; static constexpr int kIn = kLayoutPlanar, kOut = kLayoutPlanar; static constexpr bool kStrict = false, kTma = false; };
template <>
struct Variant<6> { using T = double; static constexpr int kIn = kMainIn, kOut = kMainOut; static constexpr bool kStrict = true, kTma = false; };
template <>
struct Variant<7> { using T = double; static constexpr int kIn = kLayoutPlanar, kOut = kLayoutPlanar; static constexpr bool kStrict = true, kTma = false; };

}  // namespace

cudaError_t B2DWT_CAT3(b2dwt_v_, B2DWT_PROG, B2DWT_VID)(const FusedLaunch& r) {
#ifdef B2DWT_STUB
  (void)r;
  return cudaErrorNotSupported;
#else
  using V = Variant<B2DWT_VID>;
  return launch<progs::B2DWT_PROG, typename V::T, V::kIn, V::kOut, V::kStrict, V::kTma>(r);
#endif
}

}  // namespace b2dwt
