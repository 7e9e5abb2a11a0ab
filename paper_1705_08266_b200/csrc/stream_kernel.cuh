// stream_kernel.cuh -- fused single-pass 2-D DWT kernel for sm_100a.
//
// Replaces the reference's pass loop (liftfuse/engine.py:404-439 run_tiled ->
// :376 _run_pass_on_tile -> :288 _apply_substep) with ONE kernel per level that
// reads every pixel once from HBM and writes every subband sample once.
//
// Work decomposition
//   A warp owns a column STRIP of 32*Q quads (Q quads per lane, adjacent) and a
//   SEGMENT of quad rows, and walks down the rows one "tick" per quad row.
//   Every sub-step of the program is a stage of a software pipeline held in
//   registers:
//     - vertical neighbours (dn != 0) live in a per-stage window of the
//       stage's INPUT rows n-up .. n+down; row r sits in slot r mod NW, and
//       the tick loop is unrolled by a period P (a multiple of every NW), so
//       every slot index is a compile-time constant: no register moves;
//     - horizontal neighbours (dm != 0) come from the adjacent lane with one
//       __shfl per needed value ("ext" rows with left/right halo slots).
//   Each stage reads only its own input window, so the gather semantics of the
//   reference (every target reads the sub-step's input snapshot,
//   engine.py:349-362) hold by construction.
//   The dependency cone of the whole program (sum of reaches) is recomputed
//   redundantly at strip / segment borders -- the paper's overlapping blocks
//   (PAPER.md:287).  Only the valid interior is stored.
//
// Boundary semantics (engine.py:55-92, 312-347): reflection is applied to the
// state entering EVERY sub-step.  A segment runs a few CHECKED ticks at its
// start and end (row-range tests, top/bottom window remap through extend())
// around an unchecked steady loop.  Strips that touch the left/right image
// edge run a steady loop instantiated with the halo-slot reflection map; all
// other strips run one with none of it.
//
// Loads are staged through a per-warp shared-memory ring (TMA tiles when the
// row pitch allows it, per-lane cp.async otherwise); stores go straight from
// registers as coalesced 8/16-byte vectors.
#pragma once

#include <cuda.h>

#include <utility>

#include "common.cuh"

namespace b2dwt {

constexpr int kLaneCount = 32;

enum : int { kLayoutInterleaved = 0, kLayoutPlanar = 1 };

template <class T, int NT>
struct StreamArgs {
  // input (buffer row 0 == global quad row in_row0)
  const T* in_img;     // interleaved image (LIN == kLayoutInterleaved)
  const T* in_pl[4];   // component planes (LIN == kLayoutPlanar)
  int64_t in_ld[4];    // elements per image row ([0]) / per plane row
  int64_t in_bstride;  // elements per batch item
  int in_row0;
  int in_row_end;      // one past the last global quad row the input buffer holds
  // output (buffer row 0 == global quad row out_row0)
  T* out_pl[4];
  T* out_img;
  int64_t out_ld[4];
  int64_t out_bstride;
  int out_row0;
  // global quad grid + work decomposition
  int rows, cols;
  int row_begin, row_end;  // quad rows to produce
  int strip_w;             // valid quads per strip
  int halo_l;              // strip's first quad = strip * strip_w - halo_l
  int n_strips, batch;
  int n_warps;              // CTAs sharing the (item, super-strip, row) space
  int edge_cost;            // cost of an image-edge strip row, in 1/8 of an interior row
  long long* dbg;           // optional per-warp timing record (debug builds of the split), or null
  unsigned long long* tail_counter;  // [0] claimed tail units, [1] CTAs done, [2] (fused kernel) edge
                                     // tickets; null: fully static split.  The last CTA out resets them,
                                     // so the slot is reusable
  int static_frac;          // share of the cost split statically, in 1/1024
  int tail_chunk;           // cost units per dynamic tail chunk (the smallest, when guided)
  int guided;               // tail claims: guided, a 1/k share of the rest (k > 0), or fixed chunks (0)
};

__host__ __device__ constexpr int cmod(int x, int m) { return ((x % m) + m) % m; }
__host__ __device__ constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

// Compile-time geometry of a program.
template <class P>
struct Geo {
  static constexpr int nw(int s) { return P::reach(s).up + P::reach(s).down + 1; }
  // input row of stage s at tick t is t - lag_in(s)
  static constexpr int lag_in(int s) {
    int x = 0;
    for (int k = 0; k < s; ++k) x += P::reach(k).down;
    return x;
  }
  static constexpr int sum(int which) {
    int s = 0;
    for (int i = 0; i < P::kNumSub; ++i) {
      const Reach r = P::reach(i);
      s += which == 0 ? r.up : which == 1 ? r.down : which == 2 ? r.left : r.right;
    }
    return s;
  }
  static constexpr int max_up() {
    int m = 0;
    for (int i = 0; i < P::kNumSub; ++i) m = P::reach(i).up > m ? P::reach(i).up : m;
    return m;
  }
  static constexpr int period() {
    int p = 1;
    for (int i = 0; i < P::kNumSub; ++i) p = p / cgcd(p, nw(i)) * nw(i);
    return p;
  }
  static constexpr int up = sum(0), down = sum(1), left = sum(2), right = sum(3);
  static constexpr int kPeriod = period();
  static constexpr int kMaxUp = max_up();
};

// Kept for the host: cone of a program.
template <class P>
using Cone = Geo<P>;

// ---------------------------------------------------------------------------
// Per-warp runtime context shared by all pipeline stages.
struct Ctx {
  int rows, cols;
  bool fold1;    // cols large enough that every halo read reflects at most once
  bool hedge;    // this strip's columns leave [0, cols)
  int first;     // first quad row any stage computes (segment start - cone)
  int n0, n1;    // rows stored
  int m_lane;    // global quad column of this lane's slot 0
  int m_strip;   // global quad column of lane 0's slot 0
};

// Single-fold whole-sample reflection of component index i (valid when i is
// less than one component length outside [0, cs)): engine.py:55-92 unrolled.
__device__ __forceinline__ int reflect1(int i, int parity, int cs) {
  return i < 0 ? -i - parity : (i >= cs ? 2 * cs - 1 - parity - i : i);
}

template <class T>
__device__ __forceinline__ T shfl_idx(T v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
template <class T>
__device__ __forceinline__ T shfl_up1(T v) {
  return __shfl_up_sync(0xffffffffu, v, 1);
}
template <class T>
__device__ __forceinline__ T shfl_down1(T v) {
  return __shfl_down_sync(0xffffffffu, v, 1);
}

// ---------------------------------------------------------------------------
// Pipeline stage S (sub-step S of program P).
template <class P, class T, int Q, bool kStrict, int S, bool kEnd = (S == P::kNumSub)>
struct Stage;

template <class P, class T, int Q, bool kStrict, int S>
struct Stage<P, T, Q, kStrict, S, false> {
  static constexpr Reach kR = P::reach(S);
  static constexpr int U = kR.up, D = kR.down, L = kR.left, R = kR.right;
  static constexpr int NW = U + D + 1;
  static constexpr int E = L + Q + R;
  static constexpr int kLag = Geo<P>::lag_in(S);
  static_assert(L <= Q && R <= Q, "horizontal reach must not exceed the lane width");
  static_assert(Geo<P>::kPeriod % NW == 0, "period must be a multiple of every window");
  using Ar = Arith<kStrict>;
  using Next = Stage<P, T, Q, kStrict, S + 1>;

  T w[NW][4][E];  // input row r (with halo) lives in slot r mod NW
  Next next;

  // One tick: append input row (t - kLag), compute row n = t - kLag - D.
  // HEDGE: 0 interior strip, 1 image-edge strip, 2 decided at run time (checked ticks).
  template <int PH, bool CHECK, int HEDGE, class Args, class Sink>
  __device__ __forceinline__ void tick(const T (&in)[4][Q], int t, const Ctx& cx, const Args& a, Sink& sink) {
    constexpr int kSlotIn = cmod(PH - kLag, NW);
    if constexpr (HEDGE == 2) {
      if (cx.hedge)
        append<2>(in, w[kSlotIn], cx);
      else
        append<0>(in, w[kSlotIn], cx);
    } else {
      append<HEDGE>(in, w[kSlotIn], cx);
    }
    constexpr int kOff = cmod(PH - kLag - D, NW);  // slot of row n
    T out[4][Q];
    if constexpr (!CHECK) {
      eval<kOff>(w, out, a);
      next.template tick<PH, false, HEDGE>(out, t, cx, a, sink);
    } else {
      // Rows past the bottom edge are not computed, but the tick is still
      // forwarded so later stages with lookahead can finish their last rows
      // (they reflect instead of reading the placeholder).
      const int n = t - kLag - D;
      if (n >= cx.first) {
        if (n < cx.rows) {
          if ((U > 0 || D > 0) && (n - U < 0 || n + D >= cx.rows)) {
            T vw[NW][4][E];
            remap_rows(n, cx, vw);
            eval<U>(vw, out, a);  // logical order: slot(dn) = U + dn
          } else {
            eval<kOff>(w, out, a);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < Q; ++q) out[c][q] = T(0);
        }
        next.template tick<PH, true, HEDGE>(out, t, cx, a, sink);
      }
    }
  }

  // Window row = input row plus left/right halo from the neighbour lanes.
  // HEDGE: 0 interior strip, 1 image-edge strip of a wide image (single fold;
  // the unchecked loop), 2 any image-edge strip (checked ticks only).
  template <int HEDGE>
  __device__ __forceinline__ static void append(const T (&in)[4][Q], T (&x)[4][E], const Ctx& cx) {
    append_comp<0, HEDGE>(in, x[0], cx);
    append_comp<1, HEDGE>(in, x[1], cx);
    append_comp<2, HEDGE>(in, x[2], cx);
    append_comp<3, HEDGE>(in, x[3], cx);
  }

  template <int C, int HEDGE>
  __device__ __forceinline__ static void append_comp(const T (&in)[4][Q], T (&x)[E], const Ctx& cx) {
    constexpr CompNeed nd = P::need(S, C);
    if constexpr (nd.used) {
#pragma unroll
      for (int q = 0; q < Q; ++q) x[L + q] = in[C][q];
      if constexpr (!HEDGE) {
#pragma unroll
        for (int e = 0; e < L; ++e)
          if (L - e <= nd.left) x[e] = shfl_up1(in[C][Q - L + e]);
#pragma unroll
        for (int e = 0; e < R; ++e)
          if (e < nd.right) x[L + Q + e] = shfl_down1(in[C][e]);
      } else {
        // Image-edge strip.  Wide images: do the interior exchange, then the one
        // lane whose window crosses column 0 and the lanes whose window crosses
        // column cols fold their out-of-image slots onto the mirrored in-image
        // slots of the SAME window (single-fold whole-sample symmetry,
        // engine.py:55-92) -- predicated selects, no extra shuffles.
        if (HEDGE == 1 || cx.fold1) {
#pragma unroll
          for (int e = 0; e < L; ++e)
            if (L - e <= nd.left) x[e] = shfl_up1(in[C][Q - L + e]);
#pragma unroll
          for (int e = 0; e < R; ++e)
            if (e < nd.right) x[L + Q + e] = shfl_down1(in[C][e]);
          constexpr int p = col_parity(C);
          // left edge: window column d = e - L < 0 mirrors to -d - p
          const bool at_left = cx.m_lane == 0;
#pragma unroll
          for (int e = 0; e < L; ++e) {
            constexpr_if_fold(x, at_left, e, L - (e - L) - p);
          }
          // right edge: k = cols - m_lane in-image slots; column d >= k mirrors to 2k-1-p-d
          const int k = cx.cols - cx.m_lane;
#pragma unroll
          for (int kk = 1; kk < Q + R; ++kk) {
#pragma unroll
            for (int d = kk; d < Q + R; ++d) {
              const int dm = 2 * kk - 1 - p - d;  // mirrored column offset
              if (dm >= -L && dm < kk) constexpr_if_fold(x, k == kk, L + d, L + dm);
            }
          }
        } else if constexpr (HEDGE == 2) {
          // Narrow images: generic gather through the full (periodic) map.
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const bool needed = (nd.left > 0 || nd.right > 0) && e >= L - nd.left && e < L + Q + nd.right;
            if (!needed) continue;
            const int col = reflect(cx.m_lane - L + e, col_parity(C), cx.cols);
            const int rel = col - cx.m_strip;
            int src = rel / Q;
            const int slot = rel - src * Q;
            src = src < 0 ? 0 : (src > kLaneCount - 1 ? kLaneCount - 1 : src);
            T v = shfl_idx(in[C][0], src);
#pragma unroll
            for (int j = 1; j < Q; ++j) {
              const T tt = shfl_idx(in[C][j], src);
              v = (slot == j) ? tt : v;
            }
            x[e] = v;
          }
        }
      }
    }
  }

  // x[dst] = x[src] where `pred` (indices are compile-time after unrolling).
  __device__ __forceinline__ static void constexpr_if_fold(T (&x)[E], bool pred, int dst, int src) {
    if (dst >= 0 && dst < E && src >= 0 && src < E) x[dst] = pred ? x[src] : x[dst];
  }

  // Top / bottom rows: rebuild the window in logical order through the row
  // reflection map (reflected rows are always inside the window).
  __device__ __forceinline__ void remap_rows(int n, const Ctx& cx, T (&vw)[NW][4][E]) const {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int rp = row_parity(c);
#pragma unroll
      for (int p = 0; p < NW; ++p) {
        const int src = reflect(n - U + p, rp, cx.rows) % NW;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          T v = w[0][c][e];
#pragma unroll
          for (int j = 1; j < NW; ++j) v = (src == j) ? w[j][c][e] : v;
          vw[p][c][e] = v;
        }
      }
    }
  }

  template <int OFF, int TGT, int K, class Args>
  __device__ __forceinline__ static void term(const T (&win)[NW][4][E], T (&acc)[Q], const Args& a) {
    constexpr int base = P::begin(S * 4 + TGT);
    constexpr int cnt = P::begin(S * 4 + TGT + 1) - base;
    constexpr int idx = base + TermOrder<P, kStrict>::at(base, cnt, K);  // fast: unit term first
    constexpr TermInfo ti = P::term(idx);
    constexpr int slot = cmod(OFF + ti.dn, NW);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const T x = win[slot][ti.src][L + q + ti.dm];
      constexpr T kc = static_cast<T>(P::coef(idx));  // liftfuse: dtype.type(coeff), engine.py:357
      if constexpr (K == 0) {
        acc[q] = ti.unit ? x : Ar::mul(x, kc);
      } else {
        acc[q] = ti.unit ? Ar::add(acc[q], x) : Ar::mac(acc[q], x, kc);
      }
    }
  }

  template <int OFF, int TGT, class Args, int... K>
  __device__ __forceinline__ static void target(const T (&win)[NW][4][E], T (&acc)[Q], const Args& a,
                                                std::integer_sequence<int, K...>) {
    (term<OFF, TGT, K>(win, acc, a), ...);
  }

  template <int OFF, int TGT, class Args>
  __device__ __forceinline__ static void eval_target(const T (&win)[NW][4][E], T (&out)[4][Q], const Args& a) {
    constexpr int cnt = P::begin(S * 4 + TGT + 1) - P::begin(S * 4 + TGT);
    if constexpr (cnt == 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) out[TGT][q] = T(0);
    } else {
      target<OFF, TGT>(win, out[TGT], a, std::make_integer_sequence<int, cnt>{});
    }
  }

  template <int OFF, class Args>
  __device__ __forceinline__ static void eval(const T (&win)[NW][4][E], T (&out)[4][Q], const Args& a) {
#ifdef B2DWT_EXPERIMENT_COPY
    // data-movement ceiling experiment: pass the input through untouched
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < Q; ++q) out[c][q] = win[cmod(OFF, NW)][c][L + q];
    return;
#endif
    eval_target<OFF, 0>(win, out, a);
    eval_target<OFF, 1>(win, out, a);
    eval_target<OFF, 2>(win, out, a);
    eval_target<OFF, 3>(win, out, a);
  }
};

// End of the pipeline: hand the finished row (t - sum of lookaheads) to the sink.
template <class P, class T, int Q, bool kStrict, int S>
struct Stage<P, T, Q, kStrict, S, true> {
  template <int PH, bool CHECK, int HEDGE, class Args, class Sink>
  __device__ __forceinline__ void tick(const T (&in)[4][Q], int t, const Ctx& cx, const Args& a, Sink& sink) {
    // unchecked segments run whole periods past both ends of their rows: the
    // row mask is the store predicate
    const int n = t - Geo<P>::down;
    // the interior steady path only ever has full, aligned lanes or idle lanes
    sink.template store<CHECK || HEDGE != 0>(in, n, n >= cx.n0 && n < cx.n1);
  }
};

// ---------------------------------------------------------------------------
// Output sinks: per-lane base pointers precomputed once per warp.
template <class T, int Q, int LOUT>
struct StoreSink;

// Predicated vector store of one lane's Q values (no branch: the row-range and
// lane masks become the instruction predicate).
template <class T, int Q>
__device__ __forceinline__ void st_pred(char* p, const T (&v)[Q], bool ok) {
  if constexpr (Q == 2 && sizeof(T) == 4) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n@p st.global.v2.f32 [%0], {%1, %2};\n}\n" ::"l"(p),
                 "f"(v[0]), "f"(v[1]), "r"(static_cast<int>(ok))
                 : "memory");
  } else if constexpr (Q == 4 && sizeof(T) == 4) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n@p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(p),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "r"(static_cast<int>(ok))
                 : "memory");
  } else if constexpr (Q == 2 && sizeof(T) == 8) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n@p st.global.v2.f64 [%0], {%1, %2};\n}\n" ::"l"(p),
                 "d"(v[0]), "d"(v[1]), "r"(static_cast<int>(ok))
                 : "memory");
  } else {
    if (ok) {
#pragma unroll
      for (int q = 0; q < Q; ++q) reinterpret_cast<T*>(p)[q] = v[q];
    }
  }
}

// Four planes, Q consecutive quads per lane.  Row addresses are byte pointers
// plus 32-bit byte pitches (one wide multiply-add per plane and row).
template <class T, int Q>
struct StoreSink<T, Q, kLayoutPlanar> {
  char* base[4];   // plane c at row 0 of the global grid, this lane's column
  int ldb[4];      // row pitch in bytes
  bool full, vec;  // all Q slots stored / vector store legal
  bool any_scalar; // some lane of the warp stores slot by slot
  unsigned mask;   // per-slot store mask when !full

  template <class Args>
  __device__ __forceinline__ void init(const Args& a, int64_t boff, int m_lane, int vlo, int vhi) {
    bool v = true;
    mask = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (m_lane + q >= vlo && m_lane + q < vhi) mask |= 1u << q;
    full = mask == (1u << Q) - 1;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ldb[c] = static_cast<int>(a.out_ld[c] * static_cast<int64_t>(sizeof(T)));
      T* p = a.out_pl[c] + boff - static_cast<int64_t>(a.out_row0) * a.out_ld[c] + m_lane;
      base[c] = reinterpret_cast<char*>(p);
      v = v && (a.out_ld[c] % Q == 0) && (reinterpret_cast<uintptr_t>(p) % (sizeof(T) * Q) == 0);
    }
    vec = v;
    any_scalar = __any_sync(0xffffffffu, mask != 0 && !(full && vec));
  }

  // Store row n if `in_range` (the caller's row mask).
  template <bool kScalar>
  __device__ __forceinline__ void store(const T (&v)[4][Q], int n, bool in_range) {
#ifdef B2DWT_EXPERIMENT_NOSTORE
    // load-path ceiling experiment: keep the values alive, store (almost) nothing
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < Q; ++q) acc += v[c][q];
    if (acc == T(-12345)) reinterpret_cast<T*>(base[0])[n] = acc;
    return;
#endif
    const bool vok = in_range && full && vec;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#ifdef B2DWT_EXPERIMENT_L2STORE
      // write-path experiment: same instructions, all rows folded into 64 rows (L2 resident)
      char* p = base[c] + static_cast<int64_t>(n & 63) * ldb[c];
#else
      char* p = base[c] + static_cast<int64_t>(n) * ldb[c];
#endif
      st_pred<T, Q>(p, v[c], vok);
      if (kScalar && any_scalar) {  // warp-uniform: only warps that own ragged / unaligned lanes
        if (in_range && !(full && vec)) {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (mask & (1u << q)) reinterpret_cast<T*>(p)[q] = v[c][q];
        }
      }
    }
  }
};

// Interleaved image: quad (n, m) -> pixels (2n, 2m) .. (2n+1, 2m+1).
template <class T, int Q>
struct StoreSink<T, Q, kLayoutInterleaved> {
  char* base;
  int ldb;  // image row pitch in bytes
  bool full, vec, any_scalar;
  unsigned mask;

  template <class Args>
  __device__ __forceinline__ void init(const Args& a, int64_t boff, int m_lane, int vlo, int vhi) {
    mask = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (m_lane + q >= vlo && m_lane + q < vhi) mask |= 1u << q;
    full = mask == (1u << Q) - 1;
    const int64_t ld = a.out_ld[0];
    ldb = static_cast<int>(ld * static_cast<int64_t>(sizeof(T)));
    T* p = a.out_img + boff - 2 * static_cast<int64_t>(a.out_row0) * ld + 2 * m_lane;
    base = reinterpret_cast<char*>(p);
    vec = (ld * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(p) % 16) == 0;
    any_scalar = __any_sync(0xffffffffu, mask != 0 && !(full && vec));
  }

  template <bool kScalar>
  __device__ __forceinline__ void store(const T (&v)[4][Q], int n, bool in_range) {
    const bool vok = in_range && full && vec;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      char* p = base + static_cast<int64_t>(2 * n + h) * ldb;
      T px[2 * Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        px[2 * q] = v[2 * h][q];
        px[2 * q + 1] = v[2 * h + 1][q];
      }
      constexpr int kVec = 16 / static_cast<int>(sizeof(T));
#pragma unroll
      for (int i = 0; i < 2 * Q; i += kVec) {
        T chunk[kVec];
#pragma unroll
        for (int e = 0; e < kVec; ++e) chunk[e] = px[i + e];
        st_pred<T, kVec>(p + i * sizeof(T), chunk, vok);
      }
      if (kScalar && any_scalar) {
        if (in_range && !(full && vec)) {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (mask & (1u << q)) {
              reinterpret_cast<T*>(p)[2 * q] = px[2 * q];
              reinterpret_cast<T*>(p)[2 * q + 1] = px[2 * q + 1];
            }
        }
      }
    }
  }
};

// ---------------------------------------------------------------------------
// cp.async / TMA primitives.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy BYTES (multiple of 4, <= 32) with the widest cp.async the alignment allows.
template <int BYTES>
__device__ __forceinline__ void cp_chunk(char* s, const char* g) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(g);
  if constexpr (BYTES % 16 == 0) {
    if ((al & 15) == 0) {
#pragma unroll
      for (int i = 0; i < BYTES; i += 16) cp_async16(s + i, g + i);
      return;
    }
  }
  if constexpr (BYTES % 8 == 0) {
    if ((al & 7) == 0) {
#pragma unroll
      for (int i = 0; i < BYTES; i += 8) cp_async8(s + i, g + i);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < BYTES; i += 4) cp_async4(s + i, g + i);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
// The same wait with a value the caller needs right after it as an asm input,
// so it is materialised (e.g. reloaded from a spill slot) BEFORE the wait.
__device__ __forceinline__ void mbar_wait_keep(uint64_t* bar, unsigned parity, int keep) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity), "r"(keep)
      : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(b), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// L2 prefetch of a TMA box (no shared memory, no completion): warms L2 for a
// ring stage that will be loaded later.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

#ifndef B2DWT_L2_PREFETCH
#define B2DWT_L2_PREFETCH 0  // ring stages beyond the ring's own look-ahead prefetched into L2
#endif

// ---------------------------------------------------------------------------
// Per-warp shared-memory ring.  One stage = RPS quad rows of 4*Q*32 elements,
// laid out exactly like the TMA box that fills it:
//   interleaved input: [2*RPS image rows][64*Q pixels]
//   planar input:      [4 planes][RPS rows][32*Q quads]
// so the cp.async fill path writes the same layout and one reader serves both.
template <class T, int Q>
struct RowGeom {
  static constexpr int kElems = 4 * Q * kLaneCount;
  static constexpr int kBytes = kElems * static_cast<int>(sizeof(T));
};

template <int Q, int LIN, int RPS>
__device__ __forceinline__ constexpr int stage_offset(int j, int hc) {
  return LIN == kLayoutInterleaved ? (2 * j + hc) * (2 * Q * kLaneCount) : (hc * RPS + j) * (Q * kLaneCount);
}

template <class T, int Q, int LIN, int RPS>
__device__ __forceinline__ void read_row(const T* stage, int j, int lane, T (&r)[4][Q]) {
  if constexpr (LIN == kLayoutInterleaved) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const T* p = stage + stage_offset<Q, LIN, RPS>(j, h) + 2 * Q * lane;
      T px[2 * Q];
#pragma unroll
      for (int i = 0; i < 2 * Q; i += 16 / static_cast<int>(sizeof(T))) {
        if constexpr (sizeof(T) == 4) {
          const float4 f = *reinterpret_cast<const float4*>(p + i);
          px[i] = f.x;
          px[i + 1] = f.y;
          px[i + 2] = f.z;
          px[i + 3] = f.w;
        } else {
          const double2 f = *reinterpret_cast<const double2*>(p + i);
          px[i] = f.x;
          px[i + 1] = f.y;
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        r[2 * h][q] = px[2 * q];
        r[2 * h + 1][q] = px[2 * q + 1];
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const T* p = stage + stage_offset<Q, LIN, RPS>(j, c) + Q * lane;
#pragma unroll
      for (int q = 0; q < Q; ++q) r[c][q] = p[q];
    }
  }
}

template <class T, int Q, int LIN, int RPS, class Args>
__device__ __forceinline__ void fill_row_cpasync(T* stage, int j, int gr, int64_t boff, int lane, int m_lane,
                                                 int cols, const Args& a) {
  const int64_t br = gr - a.in_row0;  // buffer quad row
  const bool full = m_lane >= 0 && m_lane + Q <= cols;
  if constexpr (LIN == kLayoutInterleaved) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const T* g = a.in_img + boff + (2 * br + h) * a.in_ld[0] + 2 * m_lane;
      T* s = stage + stage_offset<Q, LIN, RPS>(j, h) + 2 * Q * lane;
      if (full) {
        cp_chunk<2 * Q * sizeof(T)>(reinterpret_cast<char*>(s), reinterpret_cast<const char*>(g));
      } else {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int m = m_lane + q;
          if (m >= 0 && m < cols)
            cp_chunk<2 * sizeof(T)>(reinterpret_cast<char*>(s + 2 * q), reinterpret_cast<const char*>(g + 2 * q));
        }
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const T* g = a.in_pl[c] + boff + br * a.in_ld[c] + m_lane;
      T* s = stage + stage_offset<Q, LIN, RPS>(j, c) + Q * lane;
      if (full) {
        cp_chunk<Q * sizeof(T)>(reinterpret_cast<char*>(s), reinterpret_cast<const char*>(g));
      } else {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int m = m_lane + q;
          if (m >= 0 && m < cols)
            cp_chunk<sizeof(T)>(reinterpret_cast<char*>(s + q), reinterpret_cast<const char*>(g + q));
        }
      }
    }
  }
}

// Streams quad rows first .. last_load of one (strip, segment) through the ring.
// Ring stages cover global rows [k*RPS, (k+1)*RPS): the first stage starts at
// the multiple of RPS at or below `first` (TMA zero-fills rows outside the
// buffer; cp.async skips rows before `first`), so stage switches fall on the
// same global rows in every segment and an unrolled tick loop whose period
// divides RPS meets them only at its first tick.
template <class T, int Q, int LIN, bool kTma, int STAGES, int RPS>
struct RowSource {
  static constexpr int kStageElems = RPS * RowGeom<T, Q>::kElems;
  static constexpr int kStageRows = RPS;
  T* ring;
  uint64_t* bars;
  int first, last_load, n_stages;
  int row0;   // global row of the segment's first ring stage (multiple of RPS)
  int k, j;   // current stage within the segment, row within the stage
  int base;   // stages consumed by earlier segments (mbarrier phase continuity)
  const T* slot;
  int lane, m_lane, m_strip, cols, b;
  int64_t boff;

  template <class Args>
  __device__ __forceinline__ void issue(int kk, const Args& a, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                        const CUtensorMap* tm2, const CUtensorMap* tm3) {
#ifdef B2DWT_EXPERIMENT_NOLOAD
    return;  // store-path ceiling experiment: compute on whatever the ring holds
#endif
    const int g = base + kk;
    T* s = ring + (g % STAGES) * kStageElems;
    if constexpr (kTma) {
      if (lane == 0) {
        uint64_t* bar = bars + (g % STAGES);
        mbar_expect_tx(bar, kStageElems * sizeof(T));
        const int r0 = row0 + kk * RPS - a.in_row0;
        if constexpr (LIN == kLayoutInterleaved) {
          tma_load_3d(s, tm0, bar, 2 * m_strip, 2 * r0, b);
          if constexpr (B2DWT_L2_PREFETCH > 0) {
            if (kk + B2DWT_L2_PREFETCH < n_stages) tma_prefetch_3d(tm0, 2 * m_strip, 2 * (r0 + B2DWT_L2_PREFETCH * RPS), b);
          }
        } else {
          constexpr int kPlane = RPS * Q * kLaneCount;
          tma_load_3d(s + 0 * kPlane, tm0, bar, m_strip, r0, b);
          tma_load_3d(s + 1 * kPlane, tm1, bar, m_strip, r0, b);
          tma_load_3d(s + 2 * kPlane, tm2, bar, m_strip, r0, b);
          tma_load_3d(s + 3 * kPlane, tm3, bar, m_strip, r0, b);
        }
      }
    } else {
      if (kk < n_stages) {
#pragma unroll 1
        for (int jj = 0; jj < RPS; ++jj) {
          const int gr = row0 + kk * RPS + jj;
          if (gr >= first && gr <= last_load) fill_row_cpasync<T, Q, LIN, RPS>(s, jj, gr, boff, lane, m_lane, cols, a);
        }
      }
      cp_async_commit();
    }
  }

  __device__ __forceinline__ void init_barriers(const CUtensorMap* tm0, const CUtensorMap* tm1,
                                                const CUtensorMap* tm2, const CUtensorMap* tm3) {
    base = 0;
    if constexpr (kTma) {
      if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1);
        fence_mbar_init();
        // warm the descriptor cache: every stage's TMA names these maps
        prefetch_tensormap(tm0);
        if constexpr (LIN == kLayoutPlanar) {
          prefetch_tensormap(tm1);
          prefetch_tensormap(tm2);
          prefetch_tensormap(tm3);
        }
      }
      __syncwarp();
    }
  }

  // Switch to the next ring stage: wait for it, refill the slot freed by the
  // previous one.
  template <class Args>
  __device__ __forceinline__ void advance(const Args& a, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                          const CUtensorMap* tm2, const CUtensorMap* tm3) {
    ++k;
    const int g = base + k;
    if constexpr (kTma) {
      // decided before the wait: under register pressure n_stages may live in
      // local memory, and its load then overlaps the wait instead of following it
      const bool refill = k + STAGES - 1 < n_stages;
#ifndef B2DWT_EXPERIMENT_NOLOAD
      mbar_wait_keep(bars + (g % STAGES), (g / STAGES) & 1, refill);
#endif
      __syncwarp();
      if (refill) {
        if (lane == 0) fence_proxy_async();
        issue(k + STAGES - 1, a, tm0, tm1, tm2, tm3);
      }
    } else {
      cp_async_wait<STAGES - 2>();
      issue(k + STAGES - 1, a, tm0, tm1, tm2, tm3);
    }
    slot = ring + (g % STAGES) * kStageElems;
  }

  // Begin a segment: rows first .. last_load will be consumed in order.
  template <class Args>
  __device__ __forceinline__ void start(const Args& a, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                        const CUtensorMap* tm2, const CUtensorMap* tm3) {
    row0 = first - first % RPS;
    n_stages = (last_load - row0 + RPS) / RPS;
    if constexpr (kTma) {
      __syncwarp();  // every lane is done reading the previous segment's slots
      if (lane == 0) fence_proxy_async();
      for (int kk = 0; kk < STAGES - 1 && kk < n_stages; ++kk) issue(kk, a, tm0, tm1, tm2, tm3);
    } else {
      for (int kk = 0; kk < STAGES - 1; ++kk) issue(kk, a, tm0, tm1, tm2, tm3);
    }
    k = -1;
    advance(a, tm0, tm1, tm2, tm3);
    j = first - row0 - 1;
  }

  // End a segment (all its stages were consumed).
  __device__ __forceinline__ void finish() {
    base += n_stages;
    if constexpr (!kTma) cp_async_wait<0>();
  }

  // Next quad row (rows are consumed strictly in order).
  template <class Args>
  __device__ __forceinline__ void next(T (&row)[4][Q], const Args& a, const CUtensorMap* tm0,
                                       const CUtensorMap* tm1, const CUtensorMap* tm2, const CUtensorMap* tm3) {
    if (++j == RPS) {
      j = 0;
      advance(a, tm0, tm1, tm2, tm3);
    }
    read_row<T, Q, LIN, RPS>(slot, j, lane, row);
  }

  // Split form for loops whose period divides RPS: one stage check per
  // period (at a global row that is a multiple of the period), then rows
  // without checks.
  template <class Args>
  __device__ __forceinline__ void advance_if_due(const Args& a, const CUtensorMap* tm0, const CUtensorMap* tm1,
                                                 const CUtensorMap* tm2, const CUtensorMap* tm3) {
    if (j == RPS - 1) {
      j = -1;
      advance(a, tm0, tm1, tm2, tm3);
    }
  }
  __device__ __forceinline__ void next_row(T (&row)[4][Q]) {
    ++j;
    read_row<T, Q, LIN, RPS>(slot, j, lane, row);
  }
};

// ---------------------------------------------------------------------------
// Tick helpers (everything force-inlined: the pipeline must stay in registers).
template <int PH, bool CHECK, int HEDGE, class Pipe, class T, int Q, class Args, class Sink>
__device__ __forceinline__ void run_tick(Pipe& pipe, const T (&row)[4][Q], int t, const Ctx& cx, const Args& a,
                                         Sink& sink) {
  pipe.template tick<PH, CHECK, HEDGE>(row, t, cx, a, sink);
}

// Checked tick at runtime phase t % P (edge flag read at run time).
template <int P, class Pipe, class T, int Q, class Args, class Sink, int... I>
__device__ __forceinline__ void checked_tick(Pipe& pipe, const T (&row)[4][Q], int t, const Ctx& cx, const Args& a,
                                             Sink& sink, std::integer_sequence<int, I...>) {
  const int ph = t % P;
  ((ph == I ? run_tick<I, true, 2>(pipe, row, t, cx, a, sink) : void()), ...);
}

// P unchecked ticks t .. t+P-1 (t % P == 0).
template <int HEDGE, class T, int Q, class Pipe, class Src, class Args, class Sink, int... I>
__device__ __forceinline__ void steady_chunk(Pipe& pipe, Src& src, int t, const Ctx& cx, const Args& a, Sink& sink,
                                             const CUtensorMap* m0, const CUtensorMap* m1, const CUtensorMap* m2,
                                             const CUtensorMap* m3, std::integer_sequence<int, I...>) {
  T row[sizeof...(I)][4][Q];
  // One row at a time: load, then push through every stage.
  if constexpr (Src::kStageRows % static_cast<int>(sizeof...(I)) == 0) {
    src.advance_if_due(a, m0, m1, m2, m3);  // t is a multiple of the period: the only possible stage switch
    ((src.next_row(row[I]), run_tick<I, false, HEDGE>(pipe, row[I], t + I, cx, a, sink)), ...);
  } else {
    ((src.next(row[I], a, m0, m1, m2, m3), run_tick<I, false, HEDGE>(pipe, row[I], t + I, cx, a, sink)), ...);
  }
}

// ---------------------------------------------------------------------------
// Dynamic tail: the next range of the cost space [0, span) past the static
// share, claimed by one thread for its CTA.  Guided self-scheduling (guided =
// k > 0): a k-th of a fair share of what remains (remaining / (k x CTAs)), at
// least `min_chunk` units, so early claims are long (few cone re-reads and ring
// restarts) and the last ones short (balance).  guided == 0: fixed min_chunk
// tickets.  Returns the claim's offset, or `span` when nothing is left.
__device__ __forceinline__ int64_t claim_guided(unsigned long long* pos, int64_t span, int64_t min_chunk,
                                                int n_ctas, int guided, int64_t* size) {
  int64_t sz = min_chunk;
  if (guided > 0) {
    // size from a plain (possibly stale) read, then ONE fetch-add: a CAS loop
    // serialised the ~444 CTAs that finish their static shares together
    // (measured 4x slower); a stale size only makes that claim a little long
    const int64_t rem = span - static_cast<int64_t>(*reinterpret_cast<volatile unsigned long long*>(pos));
    if (rem <= 0) return span;
    const int64_t g = rem / (static_cast<int64_t>(guided) * n_ctas);
    sz = g > min_chunk ? g : min_chunk;
  }
  const int64_t f = static_cast<int64_t>(atomicAdd(pos, static_cast<unsigned long long>(sz)));
  if (f >= span) return span;
  *size = sz < span - f ? sz : span - f;
  return f;
}

// ---------------------------------------------------------------------------
// The kernel.
//   P        program structure (programs.inc)
//   T        float | double
//   Q        quads per lane
//   LIN/LOUT input / output layout
//   kTma     fill the ring with TMA (requires 16 B pitches) instead of cp.async
// f32: cap registers at 168/thread so 3 CTAs (12 warps) fit per SM; without
// the hint ptxas spends ~200 and only 2 CTAs fit.
#ifndef B2DWT_WARP_CLAIM
#define B2DWT_WARP_CLAIM 1
#endif
#ifndef B2DWT_UNROLL
#define B2DWT_UNROLL 1
#endif
#ifndef B2DWT_MIN_CTAS_PER_SM
#define B2DWT_MIN_CTAS_PER_SM 3
#endif
template <class P, class T, int Q, int LIN, int LOUT, bool kStrict, bool kTma, int WARPS, int STAGES, int RPS>
__global__ void __launch_bounds__(WARPS* kLaneCount, (sizeof(T) == 4 ? B2DWT_MIN_CTAS_PER_SM : 1))
    stream_kernel(const __grid_constant__ StreamArgs<T, (P::kNumTerms > 0 ? P::kNumTerms : 1)> a,
                  const __grid_constant__ CUtensorMap tmap0, const __grid_constant__ CUtensorMap tmap1,
                  const __grid_constant__ CUtensorMap tmap2, const __grid_constant__ CUtensorMap tmap3) {
  using G = Geo<P>;
  using Src = RowSource<T, Q, LIN, kTma, STAGES, RPS>;
  using Sink = StoreSink<T, Q, LOUT>;
  using Pipe = Stage<P, T, Q, kStrict, 0>;
  constexpr int kP = G::kPeriod;
  using Phases = std::make_integer_sequence<int, kP>;
  // steady loop: B2DWT_UNROLL periods per iteration (more ticks in one basic
  // block: the scheduler overlaps a tick's late stages with the next tick's early ones)
  constexpr int kPS = kP * B2DWT_UNROLL;
  using SteadyPhases = std::make_integer_sequence<int, kPS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];

  const int warp = threadIdx.x / kLaneCount;
  const int lane = threadIdx.x % kLaneCount;
  const int cta = blockIdx.x;
  if (cta >= a.n_warps) return;  // (n_warps counts CTAs here) block-uniform
  const long long clk0 = clock64();
  int dbg_rows = 0, dbg_edge_rows = 0;
  __shared__ long long s_claim[2];  // dynamic tail: offset, size

  // Work unit = (item, SUPER-strip of WARPS adjacent strips, row range); warp k
  // of the CTA takes strip WARPS*ss + k over the same rows.  Adjacent strips'
  // stores then reach DRAM together as wide row segments (measured write
  // bandwidth 3.8 -> 5.6 TB/s for this pattern) and their shared halo columns
  // hit in L2.  Cost units: an interior super-strip row costs 8, one containing
  // a strip that touches the left/right image edge costs edge_cost.
  const int rows_out = a.row_end - a.row_begin;
  const int qspan = Q * kLaneCount;
  const int n_super = (a.n_strips + WARPS - 1) / WARPS;
  // strips [0, h0) and [h1, n_strips) touch an image edge -> super-strips [0, s0) and [s1, n_super)
  const int h0 = a.halo_l > 0 ? 1 : 0;
  int h1 = a.n_strips;
  while (h1 > h0 && (h1 - 1) * a.strip_w - a.halo_l + qspan > a.cols) --h1;
  const int s0 = (h0 + WARPS - 1) / WARPS;
  const int s1 = h1 / WARPS > s0 ? h1 / WARPS : s0;
  const int64_t we = a.edge_cost, wi = 8;
  auto super_cost0 = [&](int s) -> int64_t {  // cost of super-strips [0, s) of one item, per row
    const int64_t e = (s < s0 ? s : s0) + (s > s1 ? s - s1 : 0);
    return e * we + (s - e) * wi;
  };
  // Batches with uniform strip cost: super-strips run over the flattened
  // (item, strip) sequence, so an image's last, partial super-strip is topped
  // up with the next image's first strips instead of idling warps (2048^2
  // images: 19 strips per item = 4 full super-strips + 3 strips).
  const bool span = a.batch > 1 && we == wi;
  const int64_t n_gstrips = static_cast<int64_t>(a.batch) * a.n_strips;
  const int64_t item_cost = span ? wi * rows_out * ((n_gstrips + WARPS - 1) / WARPS)
                                 : super_cost0(n_super) * rows_out;
  const int64_t total = span ? item_cost : item_cost * a.batch;
  // Two tiers: [0, static_end) is split evenly over the resident CTAs (long
  // pipelines, no atomics); the tail is claimed in small chunks per CTA through
  // an atomic counter, so SMs that run faster absorb more of it.
  const int64_t static_end = a.tail_counter != nullptr ? total * a.static_frac / 1024 : total;
  int64_t f = static_end * cta / a.n_warps;
  int64_t f_end = static_end * (cta + 1) / a.n_warps;

  Src src;
  src.ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(warp) * STAGES * Src::kStageElems;
  src.bars = reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(WARPS) * STAGES * Src::kStageElems * sizeof(T)) +
             warp * STAGES;
  src.lane = lane;
  src.cols = a.cols;
  src.init_barriers(&tmap0, &tmap1, &tmap2, &tmap3);
  // PDL: let the next kernel on the stream start its own prologue, then wait
  // for the previous one (our input) to complete before any global access.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  int wk = warp;  // which strip of the current super-strip this warp runs
#pragma unroll 1
  for (;;) {
#pragma unroll 1
  while (f < f_end) {
    int b = span ? 0 : static_cast<int>(f / item_cost);
    const int64_t fi = f - b * item_cost;
    // super-strip containing cost offset fi (piecewise-linear inverse of super_cost0)
    int sup;
    if (span) {
      sup = static_cast<int>(fi / (wi * rows_out));
    } else {
      const int64_t c_s0 = static_cast<int64_t>(s0) * we * rows_out;
      const int64_t c_s1 = super_cost0(s1) * rows_out;
      if (fi < c_s0)
        sup = static_cast<int>(fi / (we * rows_out));
      else if (fi < c_s1)
        sup = s0 + static_cast<int>((fi - c_s0) / (wi * rows_out));
      else
        sup = s1 + static_cast<int>((fi - c_s1) / (we * rows_out));
      if (sup >= n_super) sup = n_super - 1;
    }
    const bool edge_super = !span && (sup < s0 || sup >= s1);
    const int64_t wr = edge_super ? we : wi;
    const int64_t c0 = span ? wi * rows_out * sup : b * item_cost + super_cost0(sup) * rows_out;  // cost of row 0
    // rows whose start cost lies in [f, f_end)
    const int r0 = static_cast<int>((f - c0 + wr - 1) / wr);
    const int r1 = static_cast<int>(min(static_cast<int64_t>(rows_out), (f_end - c0 + wr - 1) / wr));
    f = c0 + wr * rows_out;  // next super-strip
    int strip = sup * WARPS + wk;
    if (span) {  // global strip -> (item, strip)
      const int64_t g = static_cast<int64_t>(sup) * WARPS + wk;
      if (g >= n_gstrips) continue;
      b = static_cast<int>(g / a.n_strips);
      strip = static_cast<int>(g - static_cast<int64_t>(b) * a.n_strips);
    }
    if (r0 >= r1 || strip >= a.n_strips) continue;
    const int r = r0;
    const int seg_len = r1 - r0;
    dbg_rows += seg_len;
    dbg_edge_rows += (strip < h0 || strip >= h1) ? seg_len : 0;

    Ctx cx;
    cx.rows = a.rows;
    cx.cols = a.cols;
    cx.fold1 = a.cols >= 2 * qspan;
    cx.m_strip = strip * a.strip_w - a.halo_l;
    cx.m_lane = cx.m_strip + Q * lane;
    const bool hedge = cx.m_strip < 0 || cx.m_strip + Q * kLaneCount > a.cols;
    cx.hedge = hedge;
    cx.n0 = a.row_begin + r;
    cx.n1 = cx.n0 + seg_len;
    cx.first = max(0, cx.n0 - G::up);
    const int last_load = min(a.rows - 1, cx.n1 - 1 + G::down);
    const int last_tick = cx.n1 - 1 + G::down;

    // Vertically interior segment: every row the stored rows depend on lies
    // inside the image and the input buffer, so no stage ever reflects a row.
    // Run it entirely in the unchecked loop over whole periods: the extra fill
    // ticks before n0 compute rows outside the stored rows' cone (never read
    // by them), and the sink masks rows outside [n0, n1).
    const int t_lo = (cx.first / kPS) * kPS;
    const int t_hi = ((last_tick + kPS) / kPS) * kPS;  // one past the last tick
    // (edge strips of narrow images need the generic column map: checked ticks only)
    const bool steady_ok = !hedge || cx.fold1;
    const bool unchecked = steady_ok && cx.n0 - G::up >= 0 && last_tick < a.rows && t_lo >= a.in_row0 &&
                           t_hi <= a.in_row_end;
    src.first = unchecked ? t_lo : cx.first;
    src.last_load = unchecked ? t_hi - 1 : last_load;
    src.m_lane = cx.m_lane;
    src.m_strip = cx.m_strip;
    src.b = b;
    src.boff = static_cast<int64_t>(b) * a.in_bstride;
    src.start(a, &tmap0, &tmap1, &tmap2, &tmap3);

    Sink sink;
    sink.init(a, static_cast<int64_t>(b) * a.out_bstride, cx.m_lane, max(strip * a.strip_w, 0),
              min(strip * a.strip_w + a.strip_w, a.cols));

    // Window rows above the segment's first loaded row only ever feed rows
    // that are not stored; start them at zero so nothing uninitialised is read.
    Pipe pipe{};

    // Steady range: every stage interior, every row loaded and stored.  The
    // checked ticks before and after it share one code copy (two rounds of
    // the outer loop); the steady ticks run in their own tight inner loop.
    const int steady_lo = G::down + max(cx.n0, G::kMaxUp);
    const int steady_hi = min(a.rows - 1, cx.n1 - 1 + G::down);
    int t = unchecked ? t_lo : cx.first;
    // first tick of the steady loop: >= steady_lo and a multiple of the period
    const int s0 = unchecked ? t_lo : ((max(steady_lo, t) + kPS - 1) / kPS) * kPS;
    const bool has_steady = unchecked || (steady_ok && s0 + kPS - 1 <= steady_hi);
    const int s1 = unchecked ? t_hi : has_steady ? s0 + ((steady_hi - s0 + 1) / kPS) * kPS : s0;  // one past the steady ticks
    const int t_end = unchecked ? t_hi : last_tick + 1;
#pragma unroll 1
    for (int round = 0; round < 2; ++round) {
      const int stop = (round == 0 && has_steady) ? s0 : t_end;
#pragma unroll 1
      for (; t < stop; ++t) {
        T row[4][Q];
        if (t <= last_load) {
          src.next(row, a, &tmap0, &tmap1, &tmap2, &tmap3);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < Q; ++q) row[c][q] = T(0);
        }
        checked_tick<kP>(pipe, row, t, cx, a, sink, Phases{});
      }
      if (round == 0 && has_steady) {
        if (hedge || sink.any_scalar) {
#pragma unroll 1
          for (; t < s1; t += kPS)
            steady_chunk<1, T, Q>(pipe, src, t, cx, a, sink, &tmap0, &tmap1, &tmap2, &tmap3, SteadyPhases{});
        } else {
          // interior strip: no halo folding, vector stores only
#pragma unroll 1
          for (; t < s1; t += kPS)
            steady_chunk<0, T, Q>(pipe, src, t, cx, a, sink, &tmap0, &tmap1, &tmap2, &tmap3, SteadyPhases{});
        }
      }
      if (!has_steady) break;
    }
    src.finish();
  }
    if (static_end >= total) break;
#if B2DWT_WARP_CLAIM
    {
      // every warp draws its own tail tickets: ticket t = strip t % WARPS of
      // fixed chunk t / WARPS (a CTA-wide claim parked the CTA's early warps at
      // a barrier until its slowest one finished: ~10% of the stall samples of
      // cdf97 convolution, profiles/r02_ncu_conv97_counters.txt)
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(a.tail_counter, 1ull);
      t = __shfl_sync(0xffffffffu, t, 0);
      wk = static_cast<int>(t % WARPS);
      f = static_end + static_cast<int64_t>(t / WARPS) * a.tail_chunk;
      if (f >= total) break;
      f_end = min(total, f + static_cast<int64_t>(a.tail_chunk));
      continue;
    }
#endif
    // the CTA's warps claim the next tail range together (same rows, adjacent strips)
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t sz = 0;
      s_claim[0] = claim_guided(a.tail_counter, total - static_end, a.tail_chunk, a.n_warps, a.guided, &sz);
      s_claim[1] = sz;
    }
    __syncthreads();
    f = static_end + s_claim[0];
    if (f >= total) break;
    f_end = min(total, f + static_cast<int64_t>(s_claim[1]));
  }
#if B2DWT_WARP_CLAIM
  if (a.tail_counter != nullptr) __syncthreads();  // every warp of the CTA has drawn its last ticket
#endif
  if (a.tail_counter != nullptr && threadIdx.x == 0) {
    // every CTA has drawn its last ticket before it gets here
    if (atomicAdd(a.tail_counter + 1, 1ull) == static_cast<unsigned long long>(a.n_warps) - 1) {
      a.tail_counter[0] = 0;
      a.tail_counter[1] = 0;
      a.tail_counter[2] = 0;
      __threadfence();
    }
  }
  if (a.dbg != nullptr && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int gw = cta * WARPS + warp;
    a.dbg[4 * gw + 0] = clock64() - clk0;
    a.dbg[4 * gw + 1] = dbg_rows;
    a.dbg[4 * gw + 2] = dbg_edge_rows;
    a.dbg[4 * gw + 3] = smid;
  }
}

}  // namespace b2dwt
