// launch.h -- internal host-side launch interface between the C ABI
// (b2dwt_host.cu) and the per-program fused-kernel translation units
// (prog_instance.cu, compiled once per built-in program structure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace b2dwt {

struct FusedLaunch {
  int dtype;           // 0 f32, 1 f64
  int lin, lout;       // kLayoutInterleaved / kLayoutPlanar
  bool strict;
  bool allow_tma;
  // input buffer: global quad row in_row0 is buffer row 0; in_rows rows held
  const void* in_img;
  const void* in_pl[4];
  int64_t in_ld[4];  // interleaved input uses in_ld[0]
  int64_t in_bstride;
  int in_row0, in_rows;
  // output buffer: global quad row out_row0 is buffer row 0
  void* out_pl[4];
  void* out_img;
  int64_t out_ld[4];  // interleaved output uses out_ld[0]
  int64_t out_bstride;
  int out_row0;
  // global quad grid and the rows to produce
  int rows, cols, row_begin, row_end, batch;
  const double* coeffs;
  int n_coeffs;
  int min_rows_per_warp;  // work split: lower bound on rows per warp (latency vs cone overhead)
  int edge_cost8;         // work split: cost of an image-edge strip row in 1/8 of an interior row
  long long* dbg;         // per-warp timing records (b2dwt_debug_*), usually null
  unsigned long long* tail_counter;  // zeroed device counter for the dynamic tail, or null
  int static_frac;        // share of the work split statically (1/1024)
  int tail_rows;          // rows per dynamic tail chunk (the smallest, when guided)
  int guided;             // guided self-scheduling of the tail: claims of remaining / (k x CTAs), k = guided (0: fixed chunks)
  int strip_align;        // strip start / width alignment in quads (>= 2)
  int full_rows;
  bool pdl;               // launch with programmatic stream serialization
  bool use_tile;          // run the 2-D tile kernel (tile_kernel.cuh) instead
  int tile_rows;          // its window rows (16 / 32), 0 = by level size
  cudaStream_t stream;
};

// Two pyramid levels in one launch (fused2_kernel.cuh): level l of an
// interleaved f32 image (rows x cols quads) and level l+1 of its LL band, which
// never leaves the SM.  Level l's HL/LH/HH go to out0_pl[1..3]; level l+1's
// LL/HL/LH/HH to out1_pl[0..3]; level-(l+1) quad rows [k_begin, k_end).
struct Fused2Launch {
  int dtype;  // 0 f32 (only)
  bool strict;
  const void* in_img;
  int64_t in_ld;
  int rows, cols;
  void* out0_pl[4];
  int64_t out0_ld[4];
  void* out1_pl[4];
  int64_t out1_ld[4];
  int k_begin, k_end;
  unsigned long long* tail_counter;
  int static_frac;
  int tail_rows1;
  int guided;
  int edge_rows1;  // level-(l+1) rows per checked unit at the image top / bottom
  int min_rows1;
  bool pdl;
  cudaStream_t stream;
};

// One-time setup per device (function attributes and occupancy are per
// device): run(f) calls f(device) the first time it is reached on each device.
constexpr int kMaxDevices = 64;
struct PerDevice {
  std::mutex mu;
  bool done[kMaxDevices] = {};
  template <class F>
  int run(F&& f) {  // the current device, or -1
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
    std::lock_guard<std::mutex> lock(mu);
    if (!done[dev]) {
      f(dev);
      done[dev] = true;
    }
    return dev;
  }
};

// RAII NVTX range (b2dwt_host.cu); a no-op unless B2DWT_NVTX is set.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
  bool active;
};

// Cone of a built-in program (quads): halo the caller must provide.
struct ConeInfo {
  int up, down, left, right;
};

// Returns cudaSuccess or the launch error; `used_tma` reports the fill path.
using FusedLauncher = cudaError_t (*)(const FusedLaunch&, bool* used_tma);
using TileLauncher = cudaError_t (*)(const FusedLaunch&);
using ConeGetter = ConeInfo (*)();
using Fused2Launcher = cudaError_t (*)(const Fused2Launch&);

}  // namespace b2dwt
