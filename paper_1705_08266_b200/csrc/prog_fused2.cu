// prog_fused2.cu -- host side of the two-level fused kernel (fused2_kernel.cuh)
// for ONE built-in forward program: geometry checks, work split, TMA map,
// launch.  Compiled with -DB2DWT_PROG=<ident> (forward lifting programs only;
// -DB2DWT_STUB compiles a placeholder that reports cudaErrorNotSupported).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "launch.h"
#ifndef B2DWT_STUB
#include "fused2_kernel.cuh"
#endif

#define B2DWT_CAT2(a, b) a##b
#define B2DWT_CAT(a, b) B2DWT_CAT2(a, b)

namespace b2dwt {

#ifndef B2DWT_STUB
namespace {

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

constexpr int kStages = 4, kRps = 4;

template <bool kStrict>
struct KernelInfo {
  int blocks_per_sm = 0;
  int sms = 0;
  cudaError_t attr = cudaSuccess;
};

template <bool kStrict>
cudaError_t launch(const Fused2Launch& r) {
  using P = progs::B2DWT_PROG;
  using T = float;
  auto kern = fused2_kernel<P, T, kStrict, kStages, kRps>;
  constexpr size_t kRing0 = static_cast<size_t>(4) * kStages * kRps * RowGeom<T, 2>::kBytes;
  constexpr size_t kSmem = kRing0 + 4 * kStages * sizeof(uint64_t) + kF2Ring * kF2J * 4 * sizeof(T) +
                           kF2Ring * 4 * sizeof(uint64_t);
  // per device: the smem opt-in and occupancy (attributes are per device)
  static PerDevice once;
  static KernelInfo<kStrict> info[kMaxDevices];
  const int dev = once.run([&](int d) {
    KernelInfo<kStrict>& k = info[d];
    k.attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    if (k.attr == cudaSuccess) k.attr = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.blocks_per_sm, kern, 128, kSmem);
    cudaDeviceGetAttribute(&k.sms, cudaDevAttrMultiProcessorCount, d);
    if (k.sms <= 0) k.sms = 148;
    if (k.blocks_per_sm <= 0) k.blocks_per_sm = 1;
  });
  if (dev < 0) return cudaErrorNotSupported;
  const KernelInfo<kStrict> ki = info[dev];
  if (ki.attr != cudaSuccess) return ki.attr;

  Fused2Args<T> a{};
  a.in_img = static_cast<const T*>(r.in_img);
  a.in_ld[0] = r.in_ld;
  a.in_row0 = 0;
  a.in_row_end = r.rows;
  for (int c = 0; c < 4; ++c) {
    a.out_pl[c] = static_cast<T*>(r.out0_pl[c]);
    a.out_ld[c] = r.out0_ld[c];
    a.out1_pl[c] = static_cast<T*>(r.out1_pl[c]);
    a.out1_ld[c] = r.out1_ld[c];
    a.out1_ldb[c] = static_cast<int>(r.out1_ld[c] * static_cast<int64_t>(sizeof(T)));
  }
  a.out_row0 = 0;
  a.rows = r.rows;
  a.cols = r.cols;
  a.k_begin = r.k_begin;
  a.k_end = r.k_end;
  a.n_super = (r.cols + kF2SuperW - 1) / kF2SuperW;
  const int64_t rows_out = r.k_end - r.k_begin;
  const int64_t total = static_cast<int64_t>(a.n_super) * rows_out;
  const int64_t resident = static_cast<int64_t>(ki.sms) * ki.blocks_per_sm;
  const int64_t min_rows = std::max(1, r.min_rows1);
  a.n_ctas = static_cast<int>(std::max<int64_t>(1, std::min(resident, (total + min_rows - 1) / min_rows)));
  const int64_t per_cta = total / a.n_ctas;
  // dynamic tail only when a CTA's share is long (small launches: all static,
  // edge units weighted in); B2DWT_F2_DYN_MIN overrides the 64-row threshold
  static const int dyn_min = [] {
    const char* e = std::getenv("B2DWT_F2_DYN_MIN");
    return e ? std::atoi(e) : 64;
  }();
  a.tail_counter = per_cta >= dyn_min ? r.tail_counter : nullptr;
  a.tail_chunk = static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(r.tail_rows1, per_cta / 4)));
  a.guided = r.guided;
  f2_work_space(a, std::min(1024, std::max(0, r.static_frac)), r.edge_rows1);

  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  {
    const int64_t es = sizeof(T);
    if ((reinterpret_cast<uintptr_t>(r.in_img) & 15) != 0 || (r.in_ld * es) % 16 != 0) return cudaErrorNotSupported;
    const int64_t bs = ((r.in_ld * 2 * r.rows * es + 15) / 16) * 16 / es;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * r.cols), static_cast<cuuint64_t>(2 * r.rows), 1};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(r.in_ld * es), static_cast<cuuint64_t>(bs * es)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(2 * 2 * kLaneCount), static_cast<cuuint32_t>(2 * kRps), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    // L2 promotion of the box reads (B2DWT_F2_L2PROMO: 0, 64, 128, 256 bytes).
    // The warps' 512-B box rows start on 32-B, not 256-B, boundaries: with 256-B
    // promotion every row pulls a third block from DRAM.  Measured on C3 levels
    // 0+1: DRAM reads 1.325 GB at 256 B vs 1.215 GB at 64 B, 440.6 vs 426.8 us.
    static const CUtensorMapL2promotion promo = [] {
      const char* e = std::getenv("B2DWT_F2_L2PROMO");
      const int v = e ? std::atoi(e) : 64;
      return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
             : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
             : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                        : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(r.in_img), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(a.n_ctas));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = r.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = r.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, map);
}

}  // namespace
#endif

cudaError_t B2DWT_CAT(b2dwt_fused2_, B2DWT_PROG)(const Fused2Launch& r) {
#ifdef B2DWT_STUB
  (void)r;
  return cudaErrorNotSupported;
#else
  // f32, interleaved image (TMA: 16-B pitch), wide enough that every halo
  // reflects at most once at both levels, even level-l grid
  if (r.dtype != 0 || r.cols < 128 || r.rows < 8 || (r.rows & 1) || (r.cols & 1)) return cudaErrorNotSupported;
  // 32-bit work space: super-strips x level-(l+1) rows
  if (int64_t{(r.cols + kF2SuperW - 1) / kF2SuperW} * (r.rows / 2) > int64_t{0x3fffffff}) return cudaErrorNotSupported;
  for (int c = 1; c < 4; ++c)
    if (r.out0_ld[c] * 4 > int64_t{0x7fffffff}) return cudaErrorNotSupported;
  for (int c = 0; c < 4; ++c)
    if (r.out1_ld[c] * 4 > int64_t{0x7fffffff}) return cudaErrorNotSupported;
  return r.strict ? launch<true>(r) : launch<false>(r);
#endif
}

}  // namespace b2dwt
