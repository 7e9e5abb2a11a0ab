// prog_tile.cu -- the 2-D tile kernel (tile_kernel.cuh) of ONE built-in program,
// main layout only (forward: interleaved image -> planes; inverse: planes ->
// interleaved image), in f32 strict / f32 fast / f64 strict.  Used for levels
// too small to fill the machine with the streaming kernel (pyramid levels >= 2
// of a 16384^2 image, small single images).
//
// Compiled with -DB2DWT_PROG=<ident> -DB2DWT_PROG_INV=<0|1>.
#include <mutex>

#include "launch.h"
#include "tile_kernel.cuh"

#define B2DWT_CAT2(a, b) a##b
#define B2DWT_CAT(a, b) B2DWT_CAT2(a, b)

namespace b2dwt {
namespace {

constexpr int kMainIn = B2DWT_PROG_INV ? kLayoutPlanar : kLayoutInterleaved;
constexpr int kMainOut = B2DWT_PROG_INV ? kLayoutInterleaved : kLayoutPlanar;
template <class P, class T, bool kStrict, int WR>
cudaError_t launch_tile_wr(const FusedLaunch& r) {
  using TG = TileGeo<P, WR>;
  auto kern = tile_kernel<P, T, kMainIn, kMainOut, kStrict, WR>;
  constexpr size_t kSmem = tile_smem_bytes<P, T, WR>();
  static PerDevice once;
  static cudaError_t attr_err[kMaxDevices] = {};
  const int dev = once.run([&](int d) {
    attr_err[d] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
  });
  if (dev < 0) return cudaErrorNotSupported;
  if (attr_err[dev] != cudaSuccess) return attr_err[dev];
  TileArgs<T> a{};
  a.in_img = static_cast<const T*>(r.in_img);
  for (int c = 0; c < 4; ++c) {
    a.in_pl[c] = static_cast<const T*>(r.in_pl[c]);
    a.out_pl[c] = static_cast<T*>(r.out_pl[c]);
    a.in_ld[c] = r.in_ld[c];
    a.out_ld[c] = r.out_ld[c];
  }
  a.in_bstride = r.in_bstride;
  a.out_img = static_cast<T*>(r.out_img);
  a.out_bstride = r.out_bstride;
  a.rows = r.rows;
  a.cols = r.cols;
  a.batch = r.batch;
  a.tiles_r = (r.rows + TG::kTR - 1) / TG::kTR;
  a.tiles_c = (r.cols + TG::kTC - 1) / TG::kTC;
  // 2-vector pixel-pair loads need an even row pitch / batch stride and an aligned base
  a.vec_in = kMainIn == kLayoutInterleaved && (reinterpret_cast<uintptr_t>(r.in_img) % (2 * sizeof(T))) == 0 &&
             r.in_ld[0] % 2 == 0 && (r.batch == 1 || r.in_bstride % 2 == 0);
  const int64_t n = static_cast<int64_t>(a.tiles_r) * a.tiles_c * r.batch;
  if (n > 0x7fffffff) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n));
  cfg.blockDim = dim3(kTileThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = r.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = r.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// Window rows: 32 (1.22x window re-read for CDF 9/7) when that still gives
// two CTAs per SM, else 16 (more, smaller tiles for the smallest levels).
template <class P, class T, bool kStrict>
cudaError_t launch_tile(const FusedLaunch& r) {
  using TG = TileGeo<P, 32>;
  const int64_t tiles = static_cast<int64_t>(r.batch) * ((r.rows + TG::kTR - 1) / TG::kTR) *
                        ((r.cols + TG::kTC - 1) / TG::kTC);
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
    return n;
  }();
  const int wr = r.tile_rows > 0 ? r.tile_rows : (tiles >= 2 * sms ? 32 : 16);
  // f64 keeps to 16 rows: its 32-row load phase would spill
  if constexpr (sizeof(T) == 4) {
    if (wr >= 32) return launch_tile_wr<P, T, kStrict, 32>(r);
  }
  return launch_tile_wr<P, T, kStrict, 16>(r);
}

}  // namespace

// cudaErrorNotSupported: no tile variant for this request (caller streams instead).
cudaError_t B2DWT_CAT(b2dwt_tile_, B2DWT_PROG)(const FusedLaunch& r) {
#ifdef B2DWT_STUB
  (void)r;
  return cudaErrorNotSupported;
#else
  using P = progs::B2DWT_PROG;
  if (r.lin != kMainIn || r.lout != kMainOut) return cudaErrorNotSupported;
  if (r.dtype == 1) return r.strict ? launch_tile<P, double, true>(r) : cudaErrorNotSupported;
  return r.strict ? launch_tile<P, float, true>(r) : launch_tile<P, float, false>(r);
#endif
}

}  // namespace b2dwt
