// prog_instance.cu -- fused-kernel instantiations for ONE built-in program.
//
// Compiled once per program structure with
//   -DB2DWT_PROG=<ident> -DB2DWT_PROG_INV=<0|1>
// (see paper_1705_08266_b200/build.py) so the 16 programs build in parallel.
// Exposes b2dwt_fused_<ident>() and b2dwt_cone_<ident>() to b2dwt_host.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "launch.h"
#include "stream_kernel.cuh"

#ifndef B2DWT_PROG
#error "compile with -DB2DWT_PROG=<program ident>"
#endif
#ifndef B2DWT_PROG_INV
#define B2DWT_PROG_INV 0
#endif

#define B2DWT_CAT2(a, b) a##b
#define B2DWT_CAT(a, b) B2DWT_CAT2(a, b)

namespace b2dwt {
namespace {

using Prog = progs::B2DWT_PROG;
constexpr int kQ = 2;

// Launch shape per element type: WARPS per CTA, ring STAGES, RPS quad rows
// per stage.  f32: 4 x 2 x 1 KB = 8 KB ring per warp (16 warps/SM = 128 KB).
template <class T>
struct Shape;
template <>
struct Shape<float> {
  static constexpr int kWarps = 4, kStages = 4, kRps = 2;
};
template <>
struct Shape<double> {
  static constexpr int kWarps = 4, kStages = 3, kRps = 2;
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D tiled map: x = elements along a row, y = rows, z = batch item.
template <class T>
bool make_map(CUtensorMap* map, const void* base, int64_t width, int64_t height, int64_t batch, int64_t ld,
              int64_t bstride, int box_x, int box_y) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const int64_t esz = sizeof(T);
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * esz) % 16 != 0) return false;
  int64_t bs = bstride;
  if (batch <= 1) bs = ((ld * height * esz + 15) / 16) * 16 / esz;
  if ((bs * esz) % 16 != 0) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(width), static_cast<cuuint64_t>(height),
                        static_cast<cuuint64_t>(std::max<int64_t>(batch, 1))};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * esz), static_cast<cuuint64_t>(bs * esz)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_x), static_cast<cuuint32_t>(box_y), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt =
      sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

template <class T, int LIN, int LOUT, bool kStrict, bool kTma>
cudaError_t launch(const FusedLaunch& r) {
  using S = Shape<T>;
  using Args = StreamArgs<T, (Prog::kNumTerms > 0 ? Prog::kNumTerms : 1)>;
  constexpr int kWarps = S::kWarps, kStages = S::kStages, kRps = S::kRps;
  auto kern = stream_kernel<Prog, T, kQ, LIN, LOUT, kStrict, kTma, kWarps, kStages, kRps>;
  constexpr size_t kRing = static_cast<size_t>(kWarps) * kStages * kRps * RowGeom<T, kQ>::kBytes;
  constexpr size_t kSmem = kRing + (kTma ? kWarps * kStages * sizeof(uint64_t) : 0);

  static int blocks_per_sm = 0;
  static std::once_flag once;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kWarps * kLaneCount, kSmem);
    if (blocks_per_sm <= 0) blocks_per_sm = 1;
  });

  Args a{};
  a.in_img = static_cast<const T*>(r.in_img);
  for (int c = 0; c < 4; ++c) {
    a.in_pl[c] = static_cast<const T*>(r.in_pl[c]);
    a.out_pl[c] = static_cast<T*>(r.out_pl[c]);
  }
  for (int c = 0; c < 4; ++c) {
    a.in_ld[c] = r.in_ld[c];
    a.out_ld[c] = r.out_ld[c];
  }
  a.in_bstride = r.in_bstride;
  a.in_row0 = r.in_row0;
  a.out_img = static_cast<T*>(r.out_img);
  a.out_bstride = r.out_bstride;
  a.out_row0 = r.out_row0;
  a.rows = r.rows;
  a.cols = r.cols;
  a.row_begin = r.row_begin;
  a.row_end = r.row_end;
  a.batch = r.batch;
  for (int i = 0; i < Prog::kNumTerms; ++i) a.k[i] = static_cast<T>(r.coeffs[i]);

  // strips: 32*Q quads loaded, the cone recomputed on both sides.  Strip
  // starts are kept 16-byte aligned in the input rows (a TMA box whose
  // innermost start is not 16 B aligned faults) and even (vector stores).
  using C = Cone<Prog>;
  constexpr int kQuadBytes = static_cast<int>(sizeof(T)) * (LIN == kLayoutInterleaved ? 2 : 1);
  constexpr int kAlign = std::max(2, 16 / kQuadBytes);
  const int halo_l = (C::left + kAlign - 1) / kAlign * kAlign;
  int strip_w = kLaneCount * kQ - halo_l - C::right;
  strip_w = strip_w / kAlign * kAlign;
  a.strip_w = strip_w;
  a.halo_l = halo_l;
  a.n_strips = (r.cols + strip_w - 1) / strip_w;
  // Work split: the flat (item, strip, row) space is divided evenly over at
  // most one full wave of resident warps (each warp >= min_rows rows so the
  // per-segment cone overhead stays bounded).
  const int64_t kMinRows = std::max(1, r.min_rows_per_warp);
  const int rows_out = r.row_end - r.row_begin;
  const int64_t resident = static_cast<int64_t>(num_sms()) * blocks_per_sm * kWarps;
  const int64_t total_rows = static_cast<int64_t>(r.batch) * a.n_strips * rows_out;
  const int64_t n_warps = std::max<int64_t>(1, std::min(resident, (total_rows + kMinRows - 1) / kMinRows));
  a.n_warps = static_cast<int>(n_warps);

  CUtensorMap maps[4];
  memset(maps, 0, sizeof(maps));
  if constexpr (kTma) {
    if (LIN == kLayoutInterleaved) {
      if (!make_map<T>(&maps[0], r.in_img, 2LL * r.cols, 2LL * r.in_rows, r.batch, r.in_ld[0], r.in_bstride,
                       2 * kQ * kLaneCount, 2 * kRps))
        return cudaErrorNotSupported;
    } else {
      for (int c = 0; c < 4; ++c)
        if (!make_map<T>(&maps[c], r.in_pl[c], r.cols, r.in_rows, r.batch, r.in_ld[c], r.in_bstride,
                         kQ * kLaneCount, kRps))
          return cudaErrorNotSupported;
    }
  }
  const unsigned grid = static_cast<unsigned>((n_warps + kWarps - 1) / kWarps);
  kern<<<grid, kWarps * kLaneCount, kSmem, r.stream>>>(a, maps[0], maps[1], maps[2], maps[3]);
  return cudaGetLastError();
}

template <class T, int LIN, int LOUT>
cudaError_t dispatch_fill(const FusedLaunch& r, bool* used_tma) {
  if (r.allow_tma) {
    const cudaError_t e = r.strict ? launch<T, LIN, LOUT, true, true>(r) : launch<T, LIN, LOUT, false, true>(r);
    if (e != cudaErrorNotSupported) {
      *used_tma = true;
      return e;
    }
    (void)cudaGetLastError();
  }
  *used_tma = false;
  return r.strict ? launch<T, LIN, LOUT, true, false>(r) : launch<T, LIN, LOUT, false, false>(r);
}

template <class T>
cudaError_t dispatch_layout(const FusedLaunch& r, bool* used_tma) {
#if B2DWT_PROG_INV
  if (r.lin == kLayoutPlanar && r.lout == kLayoutInterleaved)
    return dispatch_fill<T, kLayoutPlanar, kLayoutInterleaved>(r, used_tma);
#else
  if (r.lin == kLayoutInterleaved && r.lout == kLayoutPlanar)
    return dispatch_fill<T, kLayoutInterleaved, kLayoutPlanar>(r, used_tma);
#endif
  if (r.lin == kLayoutPlanar && r.lout == kLayoutPlanar)
    return dispatch_fill<T, kLayoutPlanar, kLayoutPlanar>(r, used_tma);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t B2DWT_CAT(b2dwt_fused_, B2DWT_PROG)(const FusedLaunch& r, bool* used_tma) {
  if (r.n_coeffs != Prog::kNumTerms) return cudaErrorInvalidValue;
  return r.dtype == 0 ? dispatch_layout<float>(r, used_tma) : dispatch_layout<double>(r, used_tma);
}

ConeInfo B2DWT_CAT(b2dwt_cone_, B2DWT_PROG)() {
  using C = Cone<Prog>;
  return ConeInfo{C::up, C::down, C::left, C::right};
}

}  // namespace b2dwt
