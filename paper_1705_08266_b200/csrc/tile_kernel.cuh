// tile_kernel.cuh -- 2-D tiled fused DWT kernel for SMALL levels (sm_100a).
//
// The streaming kernel (stream_kernel.cuh) walks a warp down a column strip,
// one quad row per tick: ideal when a level holds enough rows to fill 148 SMs
// with long pipelines, but a 2048^2-pixel or smaller pyramid level leaves each
// warp a handful of rows plus the vertical cone, so its time is the latency of
// a few dependent ticks, not bytes.  Here a CTA owns a 2-D tile instead and
// runs the whole program on it in shared memory, every thread busy at once:
//
//   1. load the tile's WINDOW -- a fixed WR x 64-quad block: the output tile
//      plus the program's cone on every side -- from HBM/L2 into per-component
//      planes, de-interleaving the pixel quads on the way (engine.py:200-211),
//      all loads of a thread in flight at once;
//   2. run every compiled sub-step over the WHOLE window, one __syncthreads
//      per sub-step, with no per-position tests.  Positions near the window
//      border read past it (into padding or neighbouring planes) and become
//      garbage; the garbage front advances by the sub-step's reach, which is
//      exactly the cone, so the output tile stays exact (the paper's
//      overlapping blocks).  Targets whose term list is the
//      identity keep their plane; every other target writes the other plane of
//      a double buffer, so each sub-step reads only its input snapshot (the
//      reference's gather semantics, engine.py:349-362);
//   3. store the output tile (4 subband planes, or the interleaved image for
//      an inverse program) with coalesced row stores.
//
// Image edges: window positions outside the image are GHOST cells.  Before
// every sub-step a window that has any refills them from their mirror images
// in the CURRENT state -- the reference reflects the state entering each
// sub-step (engine.py:55-92, 312-347), per component parity -- so the compute
// loop itself never tests or reflects anything.  A ghost cell whose mirror is
// garbage is itself past the garbage front, so the invariant "positions
// farther than the accumulated reach from the window border are exact" holds
// for ghosts too.
//
// Thread mapping: the window is flattened row-major with a compile-time pitch
// of 64; thread t owns column t % 64 of rows t / 64 + 4k.  A term's
// shared-memory address is (the position) + (a compile-time offset for source
// plane, dn, dm): one LDS with an immediate offset and one FMUL/FFMA per term.
//
// Arithmetic is the stream kernel's term evaluation: the compiled (dm, dn,
// src) order, exact coefficients as immediates, strict = separately rounded
// multiply and add (bit-identical to run_reference), fast = FMA.
//
// Cost: the window is re-read by neighbouring tiles (WR x 64 loaded per
// (WR - up - down) x (64 - left - right) stored: 1.42x for CDF 9/7 at WR = 16,
// 1.22x at WR = 32), irrelevant at the sizes this kernel serves.
#pragma once

#include "stream_kernel.cuh"

namespace b2dwt {

constexpr int kTileWinCols = 64;   // window width (quads), the flattened pitch
constexpr int kTileThreads = 256;  // 8 warps; 4 window rows per pass

template <class T>
struct TileArgs {
  const T* in_img;    // interleaved image (LIN == kLayoutInterleaved)
  const T* in_pl[4];  // component planes (LIN == kLayoutPlanar)
  int64_t in_ld[4];
  int64_t in_bstride;
  T* out_pl[4];
  T* out_img;
  int64_t out_ld[4];
  int64_t out_bstride;
  int rows, cols, batch;  // quad grid
  int tiles_r, tiles_c;
  int vec_in;             // interleaved input rows may be read as 2-element vectors
};

// Compile-time tile geometry and buffer plan of a program.
template <class P, int WR>
struct TileGeo {
  using G = Geo<P>;
  static constexpr int kWC = kTileWinCols;
  static constexpr int kWR = WR;
  static constexpr int kPlane = WR * kWC;               // elements per component plane
  static constexpr int kTR = WR - G::up - G::down;      // output rows per tile
  static constexpr int kTC = kWC - G::left - G::right;  // output cols per tile
  static constexpr int kPer = kPlane / kTileThreads;    // window positions per thread
  static_assert(kTR >= 2 && kTC >= 2, "window too small for the program's cone");
  static_assert(kPlane % kTileThreads == 0, "window must be a whole number of passes");
  // every ghost cell inside the cone of the output tile mirrors a cell inside
  // the window (the tile's own image part reaches at least `up` + 1 rows past
  // the edge it shares with the image)
  static_assert(G::up + 1 >= G::down && G::down + 1 >= G::up && G::left + 1 >= G::right &&
                    G::right + 1 >= G::left,
                "tile kernel needs a near-symmetric cone");

  B2DWT_HD static constexpr int count(int s, int t) { return P::begin(s * 4 + t + 1) - P::begin(s * 4 + t); }
  // exactly one unit term reading the target itself at (0, 0): value unchanged
  B2DWT_HD static constexpr bool identity(int s, int t) {
    if (count(s, t) != 1) return false;
    const TermInfo ti = P::term(P::begin(s * 4 + t));
    return ti.src == t && ti.dm == 0 && ti.dn == 0 && ti.unit != 0;
  }
  // a sub-step reading any neighbour (dm, dn) != (0, 0): needs the exchange
  B2DWT_HD static constexpr bool stencil(int s) {
    for (int i = P::begin(s * 4); i < P::begin(s * 4 + 4); ++i)
      if (P::term(i).dm != 0 || P::term(i).dn != 0) return true;
    return false;
  }
  // component c is read at an offset in sub-step s: published to shared memory
  B2DWT_HD static constexpr bool published(int s, int c) {
    for (int i = P::begin(s * 4); i < P::begin(s * 4 + 4); ++i)
      if (P::term(i).src == c && (P::term(i).dm != 0 || P::term(i).dn != 0)) return true;
    return false;
  }
  // shared-memory buffer (0/1) of stencil sub-step s: alternates
  B2DWT_HD static constexpr int stencil_rank(int s) {
    int n = 0;
    for (int k = 0; k < s; ++k)
      if (stencil(k)) ++n;
    return n & 1;
  }
  // largest |offset| a term reads relative to its position
  B2DWT_HD static constexpr int max_offset() {
    int m = 0;
    for (int i = 0; i < P::kNumTerms; ++i) {
      const int o = P::term(i).dn * kWC + P::term(i).dm;
      m = o > m ? o : (-o > m ? -o : m);
    }
    return m;
  }
  // padding before the first and after the last plane (reads past the window)
  static constexpr int kPad = (max_offset() + 31) / 32 * 32;
  // plane of component c in exchange buffer b
  B2DWT_HD static constexpr int plane_of(int b, int c) { return kPad + (b * 4 + c) * kPlane; }
};

template <class P, class T, int WR>
B2DWT_HD constexpr size_t tile_smem_bytes() {
  using TG = TileGeo<P, WR>;
  return (static_cast<size_t>(8) * TG::kPlane + 2 * TG::kPad) * sizeof(T) + 4 * (WR + kTileWinCols) * sizeof(int);
}

template <class P, class T, bool kStrict, int WR>
struct TileStep {
  using TG = TileGeo<P, WR>;
  using Ar = Arith<kStrict>;
  static constexpr int WC = TG::kWC;
  static constexpr int K = TG::kPer;
  using State = T[TG::kPer][4];

  template <int S, int TGT, int KT>
  __device__ __forceinline__ static void term(T& acc, const State& v, const T* sm, int k) {
    constexpr int base = P::begin(S * 4 + TGT);
    constexpr int cnt = P::begin(S * 4 + TGT + 1) - base;
    constexpr int idx = base + TermOrder<P, kStrict>::at(base, cnt, KT);  // fast: unit term first (common.cuh)
    constexpr TermInfo ti = P::term(idx);
    constexpr T kc = static_cast<T>(P::coef(idx));  // liftfuse: dtype.type(coeff), engine.py:357
    T x;
    if constexpr (ti.dm == 0 && ti.dn == 0) {
      x = v[k][ti.src];  // own position: the register snapshot
    } else {
      x = sm[TG::plane_of(TG::stencil_rank(S), ti.src) + ti.dn * WC + ti.dm + threadIdx.x + k * kTileThreads];
    }
    if constexpr (KT == 0) {
      acc = ti.unit ? x : Ar::mul(x, kc);
    } else {
      acc = ti.unit ? Ar::add(acc, x) : Ar::mac(acc, x, kc);
    }
  }

  template <int S, int TGT, int... KT>
  __device__ __forceinline__ static T target(const State& v, const T* sm, int k, std::integer_sequence<int, KT...>) {
    T acc = T(0);
    (term<S, TGT, KT>(acc, v, sm, k), ...);
    return acc;
  }

  template <int S, int TGT>
  __device__ __forceinline__ static T eval(const State& v, const T* sm, int k) {
    constexpr int cnt = TG::count(S, TGT);
    if constexpr (cnt == 0) {
      return T(0);
    } else {
      return target<S, TGT>(v, sm, k, std::make_integer_sequence<int, cnt>{});
    }
  }

  // ghost cells of the published planes <- their mirror images
  template <int S>
  __device__ __forceinline__ static void fill_ghosts(T* sm, const int* mrow, const int* mcol) {
    const int c = threadIdx.x % WC;
    const int mc0 = mcol[c], mc1 = mcol[WC + c];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = threadIdx.x / WC + k * (kTileThreads / WC);
      const int mr0 = mrow[r], mr1 = mrow[WR + r];
      // mrow/mcol hold the position itself when it lies inside the image
      if (mr0 != r || mc0 != c) {
        const int p = r * WC + c;
        constexpr int R = TG::stencil_rank(S);
        if constexpr (TG::published(S, 0)) sm[TG::plane_of(R, 0) + p] = sm[TG::plane_of(R, 0) + mr0 * WC + mc0];
        if constexpr (TG::published(S, 1)) sm[TG::plane_of(R, 1) + p] = sm[TG::plane_of(R, 1) + mr0 * WC + mc1];
        if constexpr (TG::published(S, 2)) sm[TG::plane_of(R, 2) + p] = sm[TG::plane_of(R, 2) + mr1 * WC + mc0];
        if constexpr (TG::published(S, 3)) sm[TG::plane_of(R, 3) + p] = sm[TG::plane_of(R, 3) + mr1 * WC + mc1];
      }
    }
  }

  template <int S>
  __device__ __forceinline__ static void substep(State& v, T* sm, bool ghosts, const int* mrow, const int* mcol) {
    if constexpr (TG::stencil(S)) {
      // publish the components read at an offset (this stencil sub-step's
      // buffer; the previous stencil sub-step used the other one, so one
      // barrier per stencil sub-step orders both the RAW and the WAR hazards)
      constexpr int R = TG::stencil_rank(S);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int p = threadIdx.x + k * kTileThreads;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (TG::published(S, c)) sm[TG::plane_of(R, c) + p] = v[k][c];
      }
      __syncthreads();
      if (ghosts) {  // block-uniform
        fill_ghosts<S>(sm, mrow, mcol);
        __syncthreads();
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      // every target reads the input snapshot: evaluate all, then assign
      T n0 = TG::identity(S, 0) ? v[k][0] : eval<S, 0>(v, sm, k);
      T n1 = TG::identity(S, 1) ? v[k][1] : eval<S, 1>(v, sm, k);
      T n2 = TG::identity(S, 2) ? v[k][2] : eval<S, 2>(v, sm, k);
      T n3 = TG::identity(S, 3) ? v[k][3] : eval<S, 3>(v, sm, k);
      v[k][0] = n0;
      v[k][1] = n1;
      v[k][2] = n2;
      v[k][3] = n3;
    }
  }

  template <int... S>
  __device__ __forceinline__ static void program(State& v, T* sm, bool ghosts, const int* mrow, const int* mcol,
                                                 std::integer_sequence<int, S...>) {
    (substep<S>(v, sm, ghosts, mrow, mcol), ...);
  }
};

template <class T>
struct Vec2;
template <>
struct Vec2<float> {
  using type = float2;
};
template <>
struct Vec2<double> {
  using type = double2;
};

template <class P, class T, int LIN, int LOUT, bool kStrict, int WR>
__global__ void __launch_bounds__(kTileThreads) tile_kernel(const __grid_constant__ TileArgs<T> a) {
  using G = Geo<P>;
  using TG = TileGeo<P, WR>;
  constexpr int WC = TG::kWC;
  constexpr int kRowsPerPass = kTileThreads / WC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  // mirror tables: window row / column each position reads its value from, per parity
  int* mrow = reinterpret_cast<int*>(smem_raw + (8 * TG::kPlane + 2 * TG::kPad) * sizeof(T));  // [2][WR]
  int* mcol = mrow + 2 * WR;                                                                    // [2][WC]

  int bid = blockIdx.x;
  const int tj = bid % a.tiles_c;
  bid /= a.tiles_c;
  const int ti = bid % a.tiles_r;
  const int item = bid / a.tiles_r;
  const int wr0 = ti * TG::kTR - G::up, wc0 = tj * TG::kTC - G::left;
  const int rows = a.rows, cols = a.cols;
  const bool ghosts = wr0 < 0 || wr0 + WR > rows || wc0 < 0 || wc0 + WC > cols;
  if (ghosts) {
    for (int i = threadIdx.x; i < 2 * (WR + WC); i += kTileThreads) {
      if (i < 2 * WR) {
        const int par = i / WR, r = i % WR, g = wr0 + r;
        // clamped: a mirror outside the window only belongs to a ghost past the
        // garbage front (see TileGeo's cone assertion), whose value is unused
        mrow[i] = (g >= 0 && g < rows) ? r : min(max(reflect(g, par, rows) - wr0, 0), WR - 1);
      } else {
        const int j = i - 2 * WR, par = j / WC, c = j % WC, g = wc0 + c;
        mcol[j] = (g >= 0 && g < cols) ? c : min(max(reflect(g, par, cols) - wc0, 0), WC - 1);
      }
    }
  }

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // 1. the in-image part of the window -> registers (positions outside stay
  //    0 until their ghost values are published); every load of a thread is
  //    issued before any is consumed
  const int c = threadIdx.x % WC;
  const int gc = wc0 + c;
  const bool cin = gc >= 0 && gc < cols;
  T v[TG::kPer][4];
#pragma unroll
  for (int k = 0; k < TG::kPer; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) v[k][j] = T(0);
  if constexpr (LIN == kLayoutInterleaved) {
    // quad (r, c) = pixels (2r + i, 2c + j): one 2-vector per pixel row
    const T* img = a.in_img + static_cast<int64_t>(item) * a.in_bstride;
    const int64_t ld = a.in_ld[0];
    if (a.vec_in) {
      using V = typename Vec2<T>::type;
#pragma unroll
      for (int k = 0; k < TG::kPer; ++k) {
        const int gr = wr0 + threadIdx.x / WC + k * kRowsPerPass;
        if (cin && gr >= 0 && gr < rows) {
          const T* q = img + static_cast<int64_t>(2 * gr) * ld + 2 * gc;
          const V top = __ldg(reinterpret_cast<const V*>(q));
          const V bot = __ldg(reinterpret_cast<const V*>(q + ld));
          v[k][0] = top.x;
          v[k][1] = top.y;
          v[k][2] = bot.x;
          v[k][3] = bot.y;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < TG::kPer; ++k) {
        const int gr = wr0 + threadIdx.x / WC + k * kRowsPerPass;
        if (cin && gr >= 0 && gr < rows) {
          const T* q = img + static_cast<int64_t>(2 * gr) * ld + 2 * gc;
          v[k][0] = __ldg(q);
          v[k][1] = __ldg(q + 1);
          v[k][2] = __ldg(q + ld);
          v[k][3] = __ldg(q + ld + 1);
        }
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < TG::kPer; ++k) {
      const int gr = wr0 + threadIdx.x / WC + k * kRowsPerPass;
      if (cin && gr >= 0 && gr < rows) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[k][j] = __ldg(a.in_pl[j] + static_cast<int64_t>(item) * a.in_bstride +
                          static_cast<int64_t>(gr) * a.in_ld[j] + gc);
      }
    }
  }
  if (ghosts) __syncthreads();  // mirror tables

  // 2. the program, sub-step by sub-step (registers; shared memory only for
  //    the neighbour exchange of stencil sub-steps)
  TileStep<P, T, kStrict, WR>::program(v, sm, ghosts, mrow, mcol, std::make_integer_sequence<int, P::kNumSub>{});

  // 3. the output tile: window rows [up, up + TR) x cols [left, left + TC), in the image
  const bool cout = c >= G::left && c < G::left + TG::kTC && gc < cols;
  if constexpr (LOUT == kLayoutPlanar) {
#pragma unroll
    for (int k = 0; k < TG::kPer; ++k) {
      const int r = threadIdx.x / WC + k * kRowsPerPass;
      const int gr = wr0 + r;
      if (cout && r >= G::up && r < G::up + TG::kTR && gr < rows) {
        const int64_t o = static_cast<int64_t>(item) * a.out_bstride + gc;
#pragma unroll
        for (int j = 0; j < 4; ++j) a.out_pl[j][o + static_cast<int64_t>(gr) * a.out_ld[j]] = v[k][j];
      }
    }
  } else {
    T* img = a.out_img + static_cast<int64_t>(item) * a.out_bstride;
    const int64_t ld = a.out_ld[0];
#pragma unroll
    for (int k = 0; k < TG::kPer; ++k) {
      const int r = threadIdx.x / WC + k * kRowsPerPass;
      const int gr = wr0 + r;
      if (cout && r >= G::up && r < G::up + TG::kTR && gr < rows) {
        T* q = img + static_cast<int64_t>(2 * gr) * ld + 2 * gc;
        q[0] = v[k][0];
        q[1] = v[k][1];
        q[ld] = v[k][2];
        q[ld + 1] = v[k][3];
      }
    }
  }
}

}  // namespace b2dwt
