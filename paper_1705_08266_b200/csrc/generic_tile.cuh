// generic_tile.cuh -- fused interpreter for ANY StencilProgram (custom plans).
//
// The built-in programs have compile-time kernels (stream_kernel.cuh,
// tile_kernel.cuh).  A user's own lifting plan (the reference accepts any
// LiftingPlan, schemes.py:87-108) arrives as a runtime term table; the
// per-sub-step interpreter (generic_kernel.cuh) runs it with one launch and a
// full global-memory round trip per sub-step.  This kernel runs the whole
// program in one launch with the tile kernel's structure -- a CTA owns a
// 32 x 64-quad window (output tile + the program's cone), all sub-steps run
// in shared memory with one barrier each, image edges are ghost cells
// refilled from their mirror images before every sub-step (the reference's
// per-sub-step reflection, engine.py:312-347) -- but reads its terms from a
// small device-resident table (uniform loads, broadcast to the warp).  Same
// arithmetic contract: compiled term order, strict = separate IEEE multiply
// and add (bit-identical to run_reference).
#pragma once

#include "common.cuh"

namespace b2dwt {

constexpr int kGTileMaxSub = 32;
constexpr int kGTileMaxTerms = 512;
constexpr int kGTileWR = 32, kGTileWC = 64, kGTileThreads = 256;
constexpr int kGTilePlane = kGTileWR * kGTileWC;
constexpr int kGTilePer = kGTilePlane / kGTileThreads;
constexpr int kGTilePad = 4 * kGTileWC;  // reads up to |dn| <= 3, |dm| <= 63 past a plane
constexpr int kGTileMaxReach = 3;        // per-term |dn|, |dm| bound checked on the host

struct GTileProgram {
  int n_sub;
  int up, down, left, right;  // cone: sums of the sub-steps' reaches
  int16_t count[kGTileMaxSub][4];
  int16_t first[kGTileMaxSub][4];
  uint8_t identity[kGTileMaxSub][4];
  int16_t src[kGTileMaxTerms];
  int16_t off[kGTileMaxTerms];  // dn * 64 + dm
  uint8_t unit[kGTileMaxTerms];
  double coef[kGTileMaxTerms];
};

template <class T>
struct GTileArgs {
  const T* in_img;
  const T* in_pl[4];
  int64_t in_ld[4];
  int64_t in_bstride;
  T* out_pl[4];
  T* out_img;
  int64_t out_ld[4];
  int64_t out_bstride;
  int lin, lout;  // 0 interleaved image, 1 planes
  int rows, cols, batch, tiles_r, tiles_c, tr, tc;
};

constexpr size_t gtile_smem_bytes(size_t es) {
  return (8 * static_cast<size_t>(kGTilePlane) + 2 * kGTilePad) * es + 4 * (kGTileWR + kGTileWC) * sizeof(int);
}

template <class T, bool kStrict>
__global__ void __launch_bounds__(kGTileThreads)
    generic_tile_kernel(const __grid_constant__ GTileArgs<T> a, const GTileProgram* __restrict__ gp) {
  using Ar = Arith<kStrict>;
  constexpr int WR = kGTileWR, WC = kGTileWC;
  const GTileProgram& g = *gp;  // uniform reads: one transaction per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw) + kGTilePad;  // plane q at sm + q * kGTilePlane
  int* mrow = reinterpret_cast<int*>(smem_raw + (8 * kGTilePlane + 2 * kGTilePad) * sizeof(T));  // [2][WR]
  int* mcol = mrow + 2 * WR;                                                                      // [2][WC]

  int bid = blockIdx.x;
  const int tj = bid % a.tiles_c;
  bid /= a.tiles_c;
  const int ti = bid % a.tiles_r;
  const int item = bid / a.tiles_r;
  const int wr0 = ti * a.tr - g.up, wc0 = tj * a.tc - g.left;
  const int rows = a.rows, cols = a.cols;
  const bool ghosts = wr0 < 0 || wr0 + WR > rows || wc0 < 0 || wc0 + WC > cols;
  if (ghosts) {
    for (int i = threadIdx.x; i < 2 * (WR + WC); i += kGTileThreads) {
      if (i < 2 * WR) {
        const int par = i / WR, r = i % WR, gg = wr0 + r;
        mrow[i] = (gg >= 0 && gg < rows) ? r : min(max(reflect(gg, par, rows) - wr0, 0), WR - 1);
      } else {
        const int j = i - 2 * WR, par = j / WC, c = j % WC, gg = wc0 + c;
        mcol[j] = (gg >= 0 && gg < cols) ? c : min(max(reflect(gg, par, cols) - wc0, 0), WC - 1);
      }
    }
  }
  // 1. in-image part of the window -> planes of buffer 0
  const int c = threadIdx.x % WC;
  const int gc = wc0 + c;
  const bool cin = gc >= 0 && gc < cols;
  for (int k = 0; k < kGTilePer; ++k) {
    const int r = threadIdx.x / WC + k * (kGTileThreads / WC);
    const int gr = wr0 + r;
    if (!cin || gr < 0 || gr >= rows) continue;
    const int p = r * WC + c;
    for (int j = 0; j < 4; ++j) {
      T v;
      if (a.lin == 0)
        v = a.in_img[static_cast<int64_t>(item) * a.in_bstride + static_cast<int64_t>(2 * gr + (j >> 1)) * a.in_ld[0] +
                     2 * gc + (j & 1)];
      else
        v = a.in_pl[j][static_cast<int64_t>(item) * a.in_bstride + static_cast<int64_t>(gr) * a.in_ld[j] + gc];
      sm[j * kGTilePlane + p] = v;
    }
  }
  __syncthreads();

  // 2. sub-steps; buf bit c = which buffer holds component c
  int buf = 0;
#pragma unroll 1
  for (int s = 0; s < g.n_sub; ++s) {
    if (ghosts) {
      const int mc0 = mcol[c], mc1 = mcol[WC + c];
      for (int k = 0; k < kGTilePer; ++k) {
        const int r = threadIdx.x / WC + k * (kGTileThreads / WC);
        const int mr0 = mrow[r], mr1 = mrow[WR + r];
        if (mr0 == r && mc0 == c) continue;
        const int p = r * WC + c;
        for (int j = 0; j < 4; ++j) {
          T* pl = sm + (((buf >> j) & 1) * 4 + j) * kGTilePlane;
          pl[p] = pl[((j >> 1) ? mr1 : mr0) * WC + ((j & 1) ? mc1 : mc0)];
        }
      }
      __syncthreads();
    }
    // term-major: each (uniform) table entry is read once and applied to all
    // of the thread's positions, whose accumulators stay in registers
#pragma unroll 1
    for (int t = 0; t < 4; ++t) {
      if (g.identity[s][t]) continue;
      const int n = g.count[s][t], f = g.first[s][t];
      T acc[kGTilePer];
#pragma unroll
      for (int k = 0; k < kGTilePer; ++k) acc[k] = T(0);
#pragma unroll 1
      for (int q = 0; q < n; ++q) {
        const int src = g.src[f + q];
        const T* pl = sm + (((buf >> src) & 1) * 4 + src) * kGTilePlane + g.off[f + q] + threadIdx.x;
        const T kc = static_cast<T>(g.coef[f + q]);
        const bool unit = g.unit[f + q] != 0;
#pragma unroll
        for (int k = 0; k < kGTilePer; ++k) {
          const T x = pl[k * kGTileThreads];
          if (q == 0)
            acc[k] = unit ? x : Ar::mul(x, kc);
          else
            acc[k] = unit ? Ar::add(acc[k], x) : Ar::mac(acc[k], x, kc);
        }
      }
      T* dst = sm + ((((buf >> t) & 1) ^ 1) * 4 + t) * kGTilePlane + threadIdx.x;
#pragma unroll
      for (int k = 0; k < kGTilePer; ++k) dst[k * kGTileThreads] = acc[k];
    }
    for (int t = 0; t < 4; ++t)
      if (!g.identity[s][t]) buf ^= 1 << t;
    __syncthreads();
  }

  // 3. the output tile
  const bool cout = c >= g.left && c < g.left + a.tc && gc < cols;
  for (int k = 0; k < kGTilePer; ++k) {
    const int r = threadIdx.x / WC + k * (kGTileThreads / WC);
    const int gr = wr0 + r;
    if (!cout || r < g.up || r >= g.up + a.tr || gr >= rows) continue;
    const int p = r * WC + c;
    for (int j = 0; j < 4; ++j) {
      const T v = sm[(((buf >> j) & 1) * 4 + j) * kGTilePlane + p];
      if (a.lout == 0)
        a.out_img[static_cast<int64_t>(item) * a.out_bstride + static_cast<int64_t>(2 * gr + (j >> 1)) * a.out_ld[0] +
                  2 * gc + (j & 1)] = v;
      else
        a.out_pl[j][static_cast<int64_t>(item) * a.out_bstride + static_cast<int64_t>(gr) * a.out_ld[j] + gc] = v;
    }
  }
}

}  // namespace b2dwt
