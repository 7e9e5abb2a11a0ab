// launch_impl.cuh -- host side of one fused-kernel instantiation: strip
// geometry, work split, TMA descriptors, launch.  Included by prog_variant.cu,
// which compiles exactly one (program, element type, layout, arithmetic, fill)
// kernel per translation unit so the build parallelises across CPU cores.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "launch.h"
#include "stream_kernel.cuh"

namespace b2dwt {
namespace {

// Launch shape per element type: WARPS per CTA, ring STAGES, RPS quad rows
// per stage.  f32: 4 x 2 x 1 KB = 8 KB ring per warp (16 warps/SM = 128 KB).
template <class T>
struct Shape;
template <>
struct Shape<float> {
#ifndef B2DWT_F32_Q
#define B2DWT_F32_Q 2
#endif
#ifndef B2DWT_F32_STAGES
#define B2DWT_F32_STAGES 4
#endif
#ifndef B2DWT_F32_RPS
#define B2DWT_F32_RPS 4
#endif
#ifndef B2DWT_F32_WARPS
#define B2DWT_F32_WARPS 4
#endif
  static constexpr int kQ = B2DWT_F32_Q;  // quads per lane
  static constexpr int kWarps = B2DWT_F32_WARPS, kStages = B2DWT_F32_STAGES, kRps = B2DWT_F32_RPS;
};
template <>
struct Shape<double> {
  static constexpr int kQ = 2;
  static constexpr int kWarps = 4, kStages = 3, kRps = 2;
};

// Per program: f32 programs whose tick period does not divide the ring's 4 rows
// per stage (the separable convolutions: vertical windows of 3 or 5 rows) get
// stages of `period` rows at the same ring bytes per warp, so the steady loop
// switches stages once per period instead of testing every row (CDF 9/7
// convolution: ~55 of 1153 loop instructions per 5 rows were that test and
// the TMA issue path).
template <class P, class T>
struct ShapeFor : Shape<T> {};
template <class P>
struct ShapeFor<P, float> : Shape<float> {
  static constexpr int kPer = Geo<P>::kPeriod;
  static constexpr bool kOdd = (Shape<float>::kRps % kPer) != 0 && kPer <= 8;
  static constexpr int kRps = kOdd ? kPer : Shape<float>::kRps;
  static constexpr int kStages =
      kOdd ? (Shape<float>::kStages * Shape<float>::kRps) / kPer : Shape<float>::kStages;
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
  // L2 promotion of the box reads (B2DWT_L2PROMO: 0, 64, 128, 256 bytes): box
  // rows start on 32-B boundaries, so large promotion over-fetches from DRAM
  // (measured 64 vs 256 B: C3 level 0 390 vs 393 us, C4 655 vs 653 Gpx/s)
  static const CUtensorMapL2promotion promo = [] {
    const char* e = std::getenv("B2DWT_L2PROMO");
    const int v = e ? std::atoi(e) : 64;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
           : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                      : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static PerDevice once;
  static int sms[kMaxDevices] = {};
  const int dev = once.run([](int d) {
    cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d);
    if (sms[d] <= 0) sms[d] = 148;
  });
  return dev < 0 ? 148 : sms[dev];
}

template <class Prog, class T, int LIN, int LOUT, bool kStrict, bool kTma>
cudaError_t launch(const FusedLaunch& r) {
  using S = ShapeFor<Prog, T>;
  using Args = StreamArgs<T, (Prog::kNumTerms > 0 ? Prog::kNumTerms : 1)>;
  constexpr int kWarps = S::kWarps, kStages = S::kStages, kRps = S::kRps, kQ = S::kQ;
  auto kern = stream_kernel<Prog, T, kQ, LIN, LOUT, kStrict, kTma, kWarps, kStages, kRps>;
  constexpr size_t kRing = static_cast<size_t>(kWarps) * kStages * kRps * RowGeom<T, kQ>::kBytes;
  constexpr size_t kSmem = kRing + (kTma ? kWarps * kStages * sizeof(uint64_t) : 0);

  static PerDevice once;
  static int bps[kMaxDevices] = {};
  const int dev = once.run([&](int d) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[d], kern, kWarps * kLaneCount, kSmem);
    if (bps[d] <= 0) bps[d] = 1;
  });
  if (dev < 0) return cudaErrorNotSupported;
  const int blocks_per_sm = bps[dev];

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
  a.in_row_end = r.in_row0 + r.in_rows;
  a.out_img = static_cast<T*>(r.out_img);
  a.out_bstride = r.out_bstride;
  a.out_row0 = r.out_row0;
  a.rows = r.rows;
  a.cols = r.cols;
  a.row_begin = r.row_begin;
  a.row_end = r.row_end;
  a.batch = r.batch;

  // strips: 32*Q quads loaded, the cone recomputed on both sides.  Geometry
  // keeps DRAM sectors whole: each strip's input box starts on a 32-B boundary
  // (TMA itself faults below 16 B) and each output row segment is a whole
  // number of 32-B sectors at a sector boundary -- partial sectors written by
  // two strips cost a DRAM read-modify-write (measured: 0.59 -> 0.48 ms at C3).
  // the kernel addresses output rows with 32-bit byte pitches
  for (int c = 0; c < (LOUT == kLayoutInterleaved ? 1 : 4); ++c)
    if (r.out_ld[c] < 0 || r.out_ld[c] * static_cast<int64_t>(sizeof(T)) > int64_t{0x7fffffff})
      return cudaErrorNotSupported;
  using C = Cone<Prog>;
  constexpr int kInQuadBytes = static_cast<int>(sizeof(T)) * (LIN == kLayoutInterleaved ? 2 : 1);
  constexpr int kOutQuadBytes = static_cast<int>(sizeof(T)) * (LOUT == kLayoutInterleaved ? 2 : 1);
  // B2DWT_STRIP_PACK=1 (experiment): strips packed at the cone (16-B box
  // starts, strip widths not sector multiples)
  static const bool pack = [] {
    const char* e = std::getenv("B2DWT_STRIP_PACK");
    return e && std::atoi(e) != 0;
  }();
  const int halo_align = pack ? std::max(2, 16 / kInQuadBytes)
                              : std::max({2, std::min(4, 32 / kInQuadBytes), 16 / kInQuadBytes, r.strip_align});
  const int width_align = pack ? halo_align : std::max(halo_align, 32 / kOutQuadBytes);
  const int halo_l = (C::left + halo_align - 1) / halo_align * halo_align;
  int strip_w = kLaneCount * kQ - halo_l - C::right;
  strip_w = strip_w / width_align * width_align;
  a.strip_w = strip_w;
  a.halo_l = halo_l;
  a.n_strips = (r.cols + strip_w - 1) / strip_w;
  // Work split: the flat (item, strip, row) space is divided evenly over at
  // most one full wave of resident warps (each warp >= min_rows rows so the
  // per-segment cone overhead stays bounded).
  const int64_t kMinRows = std::max(1, r.min_rows_per_warp);
  const int rows_out = r.row_end - r.row_begin;
  const int64_t n_super = (a.n_strips + kWarps - 1) / kWarps;
  const int64_t total_rows = static_cast<int64_t>(r.batch) * n_super * rows_out;
  int64_t ctas_per_sm = blocks_per_sm;
  if (r.full_rows > 0)
    ctas_per_sm = std::max<int64_t>(1, std::min<int64_t>(blocks_per_sm, total_rows / (int64_t{num_sms()} * r.full_rows)));
  const int64_t resident_ctas = static_cast<int64_t>(num_sms()) * ctas_per_sm;
  const int64_t n_ctas = std::max<int64_t>(1, std::min(resident_ctas, (total_rows + kMinRows - 1) / kMinRows));
  a.n_warps = static_cast<int>(n_ctas);
  a.edge_cost = std::max(8, r.edge_cost8);
  a.dbg = r.dbg;
  // Small levels (few rows per CTA) are latency-bound: chunking them only adds
  // prologues, so the tail shrinks with the per-CTA share and vanishes below it.
  const int64_t rows_per_cta = total_rows / n_ctas;
  a.tail_counter = rows_per_cta >= 64 ? r.tail_counter : nullptr;
  a.static_frac = std::min(1024, std::max(0, r.static_frac));
  a.tail_chunk = static_cast<int>(std::max<int64_t>(4, std::min<int64_t>(r.tail_rows, rows_per_cta / 8))) * 8;
  a.guided = r.guided;

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
  // Programmatic dependent launch: the kernel's prologue (barriers, descriptor
  // prefetch, work split) overlaps the tail of the previous kernel on the
  // stream; it waits (griddepcontrol.wait) before touching global memory.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n_ctas));
  cfg.blockDim = dim3(kWarps * kLaneCount);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = r.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = r.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, maps[0], maps[1], maps[2], maps[3]);
}

}  // namespace
}  // namespace b2dwt
