// fused2_kernel.cuh -- TWO pyramid levels in one kernel (sm_100a).
//
// The multi-level forward transform (level l+1 is
// `forward` of level l's LL, liftfuse/engine.py:481-487 iterated) normally
// writes level l's LL band to HBM and reads it back for level l+1.  Here the
// LL band never leaves the SM: each CTA runs level l's register pipeline
// (stream_kernel.cuh, Q = 2 quads per lane) over a super-strip of columns,
// passes the LL rows between its four warps through a small shared-memory
// ring, and the same warps run level l+1's pipeline (Q = 1) on them.  HBM
// traffic per pair of levels drops from 1 read + 1 write of each level's input
// to 1 read of level l's input + 1 write of level l's HL/LH/HH and of level
// l+1's four planes -- the paper's "keep intermediate results on chip across
// overlapping blocks" applied across levels.
//
// Geometry (all built-in lifting programs: per-sub-step horizontal reach <= 1,
// cone <= 2 quads per side):
//   CTA super-strip c owns level-l quad columns [224c, 224c + 224) and level
//   l+1 columns [112c, 112c + 112) (both whole 32-B sectors in f32) -- the
//   stream kernel's 256 loaded quads per 224 stored.
//   Level l:   warp w loads quads m0 + [0, 64), m0 = 224c - 8 + 60w (32-B
//              aligned); its valid lanes 1..30 (quads m0 + [2, 62)) publish
//              their LL and store HL/LH/HH of the CTA's columns among them.
//   Ring:      level-(l+1) quads: slot[j] = (c0, c1, c2, c3) of level-(l+1)
//              column 112c - 2 + j, j in [0, 116); level-l lane l of warp w
//              writes j = 30w + l - 2 (even LL row: c0/c1, odd row: c2/c3).
//   Level l+1: warp w, lane l runs column 112c - 2 + 28w + l (Q = 1) and stores
//              [112c + 28w, +28) (valid lanes are 2..29).
// Warp boundaries inside a super-strip are not sector-aligned; the warps of a
// CTA run in lockstep (below), so both halves of a shared sector reach L2
// together.
// Warp w reads ring columns of warps w-1 and w+1 and they read its columns, so
// each warp signals one mbarrier per ring slot (32 arrivals) and waits only for
// its neighbours' -- which also proves they are done reading the slot it is
// about to reuse (kF2Ring >= 2 steps later).  The ring depth is the slack
// between the warps of a CTA.
//
// Rows: a work unit is (super-strip, level-(l+1) rows [k0, k1)).  Level l then
// computes valid LL rows [2(k0 - up1), 2(k1 + down1)) (cone of level l+1) and
// stores HL/LH/HH rows [2 k0, 2 k1); vertically interior units run both
// pipelines entirely unchecked (the stream kernel's fill argument: extra ticks
// compute rows outside every stored row's cone).  Boundary semantics, term
// order and arithmetic are exactly the stream kernel's, so results are
// bit-identical to two separate launches (tests/test_gpu_fused2.py).
#pragma once

#include "stream_kernel.cuh"

namespace b2dwt {

constexpr int kF2SuperW = 224;  // level-l quads per CTA super-strip
constexpr int kF2StripW = 60;   // level-l quads between the warps' strips
constexpr int kF2Lead = 8;      // level-l quads loaded left of the CTA's columns
#ifndef B2DWT_F2_RING
#define B2DWT_F2_RING 5  // 6 slots push a CTA past a third of the SM's shared memory (2 CTAs/SM)
#endif
constexpr int kF2Ring = B2DWT_F2_RING;  // ring slots (level-(l+1) rows)
constexpr int kF2J = 116;               // ring columns (level-(l+1) quads)
constexpr int kF2W1 = 28;               // level-(l+1) columns stored per warp
constexpr int kF2Edge = 8;      // level-(l+1) rows at the image top / bottom run as checked units
// level-(l+1) steps of a steady chunk in pairs: one neighbour wait per two
// steps (F2Level1::step2)
#ifndef B2DWT_F2_PAIR
#define B2DWT_F2_PAIR 1  // C3 strict levels 0+1 415 -> 408 us, fast unchanged (tools/ab_lib.sh)
#endif

template <class T>
struct Fused2Args {
  // level-l image (interleaved), buffer row 0 == global quad row 0
  const T* in_img;
  const T* in_pl[4];  // unused (RowSource interface)
  int64_t in_ld[4];
  int64_t in_bstride;
  int in_row0;
  int in_row_end;
  // level-l HL/LH/HH ([0] unused: the LL band stays on chip)
  T* out_pl[4];
  int64_t out_ld[4];
  int out_row0;
  // level-(l+1) LL/HL/LH/HH
  T* out1_pl[4];
  int64_t out1_ld[4];
  int out1_ldb[4];  // out1_ld in bytes (the host checks that it fits)
  int rows, cols;      // level-l quad grid
  int k_begin, k_end;  // level-(l+1) quad rows produced by this launch
  int n_super;         // CTA super-strips
  int n_ctas;
  unsigned long long* tail_counter;  // [0] claimed tail rows, [1] CTAs done, [2] edge tickets
                                     // (self-resetting), or null
  int tail_chunk;                    // level-(l+1) rows per dynamic chunk (the smallest, when guided)
  int guided;                        // tail claims: guided, a 1/k share of the rest (k > 0), or fixed chunks (0)
  // work space (f2_work_space on the host), in cost units of one interior
  // level-(l+1) row.  The rows near the image top / bottom (`top` / `bot` per
  // super-strip) need the checked path and run as n_edge units of unit_rows
  // rows, each costing unit_cost; the interior rows [ki0, ki0 + rows_in) of
  // every super-strip are the rest.
  //  * small launch (no tail counter), space 0: [0, edge_cost) = the edge
  //    units, [edge_cost, total) = the interior super-strip by super-strip;
  //    [0, total) is split evenly over the CTAs (a unit goes to the CTA whose
  //    share holds its first cost unit);
  //  * large launch: static space 1 = the first s_rows interior rows of every
  //    super-strip, split evenly over the first static_ctas CTAs -- a whole
  //    multiple of n_super, so every share lies inside ONE super-strip (one
  //    cone fill per CTA); then the dynamic queue: the edge units first
  //    (dyn_edges tickets), then space 2 = the remaining d_rows rows of every
  //    super-strip ([0, n_dyn_rows)) in guided claims.
  int top, bot, ki0, rows_in, n_edge, unit_cost, edge_cost;
  int unit_rows, units_top, units_bot;  // an edge band is cut into units of unit_rows rows
  int total;                                      // small launch: size of space 0
  int s_rows, d_rows, static_ctas, n_dyn_rows;   // large launch: spaces 1 and 2
  int dyn_edges;
};

// Host: fill the work-space fields of `a` (its k range, n_super, n_ctas,
// tail_counter, tail_chunk and rows already set).  The rows near the image top
// / bottom need the checked (reflecting) path at both levels and run as short
// separate units, so no long segment is ever checked.  Large launches (with a
// tail counter) hand them out first in the dynamic queue; small ones weight
// them into the static split and size them to one CTA's share.
template <class T>
inline void f2_work_space(Fused2Args<T>& a, int static_frac, int edge_rows = kF2Edge) {
  const int rows1 = a.rows / 2;
  int edge = edge_rows < 1 ? 1 : edge_rows;
  if (a.tail_counter == nullptr && edge_rows == kF2Edge) {
    // small launch, all static: its time is max(edge unit, CTA share), an edge
    // unit costing ~4 interior rows per row -- size it to one share (>= 3 rows,
    // the fewest that leave the interior units unchecked).  C3 levels 2+3
    // (share 23 rows): 6-row units 45 us, 8-row 49 us.
    const int share = static_cast<int>(int64_t{a.n_super} * (a.k_end - a.k_begin) / (a.n_ctas > 0 ? a.n_ctas : 1));
    edge = (share + 2) / 4;
    edge = edge < 3 ? 3 : edge > kF2Edge ? kF2Edge : edge;
  }
  a.top = a.k_begin == 0 ? (a.k_end - a.k_begin < edge ? a.k_end - a.k_begin : edge) : 0;
  const int rest = a.k_end - a.k_begin - a.top;
  a.bot = a.k_end == rows1 ? (rest < edge ? rest : edge) : 0;
  a.ki0 = a.k_begin + a.top;
  a.rows_in = a.k_end - a.bot - a.ki0;
  // one unit per edge band (cutting it finer multiplies the checked cones:
  // 2-row units took C3 levels 2+3 from 47 to 57 us)
  a.unit_rows = edge;
  a.units_top = (a.top + a.unit_rows - 1) / a.unit_rows;
  a.units_bot = (a.bot + a.unit_rows - 1) / a.unit_rows;
  a.n_edge = a.n_super * (a.units_top + a.units_bot);
  a.unit_cost = 4 * a.unit_rows;  // checked ticks at both levels plus both cones (measured ~4x an interior row)
  a.edge_cost = a.n_edge * a.unit_cost;
  a.total = a.edge_cost + a.n_super * a.rows_in;
  a.s_rows = a.d_rows = a.static_ctas = a.n_dyn_rows = a.dyn_edges = 0;
  if (a.tail_counter != nullptr) {
    // large launch: whole super-strip slices for the static CTAs (C3 levels
    // 0+1: 444 CTAs = 12 per super-strip); the slow edge units go to whichever
    // CTAs finish their static share first (head of the dynamic list)
    const int per_super = a.n_ctas / a.n_super;
    a.static_ctas = per_super >= 1 ? per_super * a.n_super : a.n_ctas;
    a.s_rows = static_cast<int>(static_cast<int64_t>(a.rows_in) * static_frac * a.static_ctas / (1024 * int64_t{a.n_ctas}));
    a.d_rows = a.rows_in - a.s_rows;
    a.n_dyn_rows = a.n_super * a.d_rows;
    a.dyn_edges = a.n_edge;
  }
}

// Level-l sink: HL/LH/HH straight to HBM (8-B vectors), LL into the ring.
template <class T>
struct F2Sink0 {
  char* base[4];
  int ldb[4];
  bool full, vec, any_scalar;
  unsigned mask;
  unsigned ring;  // shared address of this lane's ring column in slot 0, or 0 (lane does not publish)
  int slot;       // current ring slot
  int last_n;

  __device__ __forceinline__ void init(const Fused2Args<T>& a, int m_lane, int vlo, int vhi) {
    bool v = true;
    mask = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (m_lane + q >= vlo && m_lane + q < vhi) mask |= 1u << q;
    full = mask == 3u;
#pragma unroll
    for (int c = 1; c < 4; ++c) {
      ldb[c] = static_cast<int>(a.out_ld[c] * static_cast<int64_t>(sizeof(T)));
      T* p = a.out_pl[c] - static_cast<int64_t>(a.out_row0) * a.out_ld[c] + m_lane;
      base[c] = reinterpret_cast<char*>(p);
      v = v && (a.out_ld[c] % 2 == 0) && (reinterpret_cast<uintptr_t>(p) % (sizeof(T) * 2) == 0);
    }
    vec = v;
    any_scalar = __any_sync(0xffffffffu, mask != 0 && !(full && vec));
    last_n = -0x40000000;
  }

  template <bool kScalar>
  __device__ __forceinline__ void store(const T (&v)[4][2], int n, bool in_range) {
    const bool vok = in_range && full && vec;
#pragma unroll
    for (int c = 1; c < 4; ++c) {
      char* p = row_addr(base[c], n, ldb[c]);
      st_pred<T, 2>(p, v[c], vok);
      if (kScalar && any_scalar) {
        if (in_range && !(full && vec)) {
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (mask & (1u << q)) reinterpret_cast<T*>(p)[q] = v[c][q];
        }
      }
    }
    // LL row n: level-(l+1) components (n even: c0, c1; odd: c2, c3)
    if (ring != 0) {
      const unsigned r = ring + static_cast<unsigned>(slot * (kF2J * 4) + 2 * (n & 1)) * sizeof(T);
      if constexpr (sizeof(T) == 4) {
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(r), "f"(v[0][0]), "f"(v[0][1]) : "memory");
      } else {
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(r), "d"(v[0][0]), "d"(v[0][1]) : "memory");
      }
    }
    last_n = n;
  }
};

// Level-(l+1) sink: one value per plane and lane.  Addresses are formed from
// the kernel parameters (constant bank) at each store instead of being held in
// registers: the level-l pipeline needs those registers.
template <class T>
struct F2Sink1 {
  const Fused2Args<T>* a;  // the __grid_constant__ parameter block
  int m_lane;
  bool lane_ok;
  bool any_scalar;  // (StoreSink interface; never set)

  template <bool kScalar>
  __device__ __forceinline__ void store(const T (&v)[4][1], int n, bool in_range) {
    if (in_range && lane_ok) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const T* p = reinterpret_cast<const T*>(row_addr(a->out1_pl[c], n, a->out1_ldb[c])) + m_lane;
        if constexpr (sizeof(T) == 4)
          asm volatile("st.global.f32 [%0], %1;\n" ::"l"(p), "f"(v[c][0]) : "memory");
        else
          asm volatile("st.global.f64 [%0], %1;\n" ::"l"(p), "d"(v[c][0]) : "memory");
      }
    }
  }
};

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_sa(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Per-warp state of the level-(l+1) half.
template <class P, class T, bool kStrict>
struct F2Level1 {
  using Pipe = Stage<P, T, 1, kStrict, 0>;
  Pipe pipe;
  F2Sink1<T> sink;
  Ctx cx;
  unsigned rd;    // shared address of this lane's ring column (slot 0)
  unsigned bars;  // shared address of the ring mbarriers [slot][warp]
  int warp;
  unsigned u;     // level-(l+1) steps taken by this CTA (ring slot / phase)
  int last_load;  // last level-(l+1) input row that exists

  // Publish this warp's LL pair for step u, wait for the neighbour warps',
  // read this lane's level-(l+1) input row.
  __device__ __forceinline__ void gather(T (&row)[4][1]) {
    const unsigned s = u % kF2Ring, par = (u / kF2Ring) & 1u;
    const unsigned b = bars + (s * 4) * 8;
    mbar_arrive(b + warp * 8);
#ifndef B2DWT_F2_NOSYNC  // (timing experiment only: results are wrong without it)
    if (warp > 0) mbar_wait_sa(b + (warp - 1) * 8, par);
    if (warp < 3) mbar_wait_sa(b + (warp + 1) * 8, par);
#endif
    __syncwarp();  // the warp's own lanes' ring writes
    const unsigned p = rd + s * (kF2J * 4) * static_cast<unsigned>(sizeof(T));
    if constexpr (sizeof(T) == 4) {
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                   : "=f"(row[0][0]), "=f"(row[1][0]), "=f"(row[2][0]), "=f"(row[3][0])
                   : "r"(p)
                   : "memory");
    } else {
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(row[0][0]), "=d"(row[1][0]) : "r"(p) : "memory");
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(row[2][0]), "=d"(row[3][0]) : "r"(p + 16) : "memory");
    }
    ++u;
  }

  // Paired steps (B2DWT_F2_PAIR): the first of two consecutive steps only
  // signals its slot; the second signals, waits for the neighbours ONCE (their
  // arrival for the later step orders their ring writes for both: arrive is a
  // release, the wait an acquire) and reads both rows.  Slot reuse stays safe
  // with 5 slots: a warp's waits now lag its reads by one step, and the
  // rewrite of a slot is still >= 2 waited steps behind its last read.
  __device__ __forceinline__ void arrive_only() {
    const unsigned s = u % kF2Ring;
    mbar_arrive(bars + (s * 4) * 8 + warp * 8);
    ++u;
  }
  template <int PHA, int PHB, int HEDGE, class Args>
  __device__ __forceinline__ void step2(int t1a, const Args& a) {
    const unsigned s = u % kF2Ring, par = (u / kF2Ring) & 1u;
    const unsigned sp = (u + kF2Ring - 1) % kF2Ring;
    const unsigned b = bars + (s * 4) * 8;
    mbar_arrive(b + warp * 8);
    if (warp > 0) mbar_wait_sa(b + (warp - 1) * 8, par);
    if (warp < 3) mbar_wait_sa(b + (warp + 1) * 8, par);
    __syncwarp();
    T ra[4][1], rb[4][1];
    const unsigned pa = rd + sp * (kF2J * 4) * static_cast<unsigned>(sizeof(T));
    const unsigned pb = rd + s * (kF2J * 4) * static_cast<unsigned>(sizeof(T));
    static_assert(sizeof(T) == 4, "paired steps: f32 only");
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(ra[0][0]), "=f"(ra[1][0]), "=f"(ra[2][0]), "=f"(ra[3][0]) : "r"(pa) : "memory");
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(rb[0][0]), "=f"(rb[1][0]), "=f"(rb[2][0]), "=f"(rb[3][0]) : "r"(pb) : "memory");
    ++u;
    pipe.template tick<PHA, false, HEDGE>(ra, t1a, cx, a, sink);
    pipe.template tick<PHB, false, HEDGE>(rb, t1a + 1, cx, a, sink);
  }

  // Unchecked level-(l+1) tick at compile-time phase PH1.
  template <int PH1, int HEDGE, class Args>
  __device__ __forceinline__ void step(int t1, const Args& a) {
    T row[4][1];
    gather(row);
    pipe.template tick<PH1, false, HEDGE>(row, t1, cx, a, sink);
  }

  // Checked level-(l+1) tick (runtime phase, row-range tests, edge remaps).
  template <class Args>
  __device__ __forceinline__ void step_checked(int t1, const Args& a) {
    T row[4][1];
    gather(row);
    checked_tick<Geo<P>::kPeriod>(pipe, row, t1, cx, a, sink, std::make_integer_sequence<int, Geo<P>::kPeriod>{});
  }

  // Level-(l+1) rows past the image bottom: no input (zeros, never read).
  template <class Args>
  __device__ __forceinline__ void flush_checked(int t1, const Args& a) {
    const T row[4][1] = {{T(0)}, {T(0)}, {T(0)}, {T(0)}};
    checked_tick<Geo<P>::kPeriod>(pipe, row, t1, cx, a, sink, std::make_integer_sequence<int, Geo<P>::kPeriod>{});
  }
};

// 2kP unchecked level-l ticks t .. t+2kP-1 (t % 2kP == 0); after every tick
// that completes an LL row pair, one level-(l+1) tick (L1C: checked).
template <int HEDGE, class P, class T, bool kStrict, class Pipe0, class Src, class Sink0, class Args, int... I>
__device__ __forceinline__ void f2_steady_chunk(Pipe0& pipe0, Src& src, F2Level1<P, T, kStrict>& l1, int t,
                                                const Ctx& cx0, const Args& a, Sink0& sink0,
                                                const CUtensorMap* m, std::integer_sequence<int, I...>) {
  constexpr int kD0 = Geo<P>::down;
  constexpr int kP = Geo<P>::kPeriod;
  constexpr bool kNest = Src::kStageRows % static_cast<int>(sizeof...(I)) == 0;
  auto one = [&](auto ic) {
    constexpr int i = decltype(ic)::value;
    T row[4][2];
    if constexpr (kNest)
      src.next_row(row);
    else
      src.next(row, a, m, m, m, m);
    pipe0.template tick<i, false, HEDGE>(row, t + i, cx0, a, sink0);
    if constexpr (((i - kD0) % 2 + 2) % 2 == 1) {  // LL row t + i - kD0 is odd: a quad row is complete
      sink0.slot = static_cast<int>((l1.u + 1) % kF2Ring);
      // j-th level-(l+1) step of the chunk (kD0 fixes which ticks complete a row)
      constexpr int j = (i - (((kD0 + 1) % 2 + 2) % 2)) / 2;
      constexpr int n_steps = static_cast<int>(sizeof...(I)) / 2;
      if constexpr (B2DWT_F2_PAIR && sizeof(T) == 4 && n_steps % 2 == 0 && j % 2 == 0) {
        l1.arrive_only();
      } else if constexpr (B2DWT_F2_PAIR && sizeof(T) == 4 && n_steps % 2 == 0) {
        l1.template step2<cmod((i - kD0 - 1) / 2 - 1, kP), cmod((i - kD0 - 1) / 2, kP), HEDGE>(
            (t + i - kD0 - 1) / 2 - 1, a);
      } else {
        l1.template step<cmod((i - kD0 - 1) / 2, kP), HEDGE>((t + i - kD0 - 1) / 2, a);
      }
    }
  };
  if constexpr (kNest) src.advance_if_due(a, m, m, m, m);  // t % period == 0: the only possible stage switch
  (one(std::integral_constant<int, I>{}), ...);
}

#ifndef B2DWT_F2_MIN_CTAS
#define B2DWT_F2_MIN_CTAS 3
#endif
template <class P, class T, bool kStrict, int STAGES, int RPS>
__global__ void __launch_bounds__(4 * kLaneCount, B2DWT_F2_MIN_CTAS)
    fused2_kernel(const __grid_constant__ Fused2Args<T> a, const __grid_constant__ CUtensorMap tmap) {
  constexpr int WARPS = 4, Q0 = 2;
  using G = Geo<P>;
  using Src = RowSource<T, Q0, kLayoutInterleaved, true, STAGES, RPS>;
  using Pipe0 = Stage<P, T, Q0, kStrict, 0>;
  constexpr int kP = G::kPeriod;
  constexpr int kPF = 2 * kP * B2DWT_UNROLL;  // one fused chunk: 2kP level-l ticks = kP level-(l+1) ticks (x unroll)
  static_assert(G::left <= 2 && G::right <= 2, "fused levels need a cone of <= 2 quads per side");
  extern __shared__ __align__(128) unsigned char smem_raw[];

  const int warp = threadIdx.x / kLaneCount;
  const int lane = threadIdx.x % kLaneCount;
  const int cta = blockIdx.x;
  if (cta >= a.n_ctas) return;
  __shared__ long long s_claim[2];  // dynamic item: kind/offset, size

  // shared memory: per-warp TMA rings | their mbarriers | LL ring | its mbarriers [slot][warp]
  const size_t ring0_bytes = static_cast<size_t>(WARPS) * STAGES * Src::kStageElems * sizeof(T);
  const unsigned ll_ring = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) +
                           static_cast<unsigned>(ring0_bytes + WARPS * STAGES * sizeof(uint64_t));
  const unsigned ll_bars = ll_ring + kF2Ring * kF2J * 4 * static_cast<unsigned>(sizeof(T));

  Src src;
  src.ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(warp) * STAGES * Src::kStageElems;
  src.bars = reinterpret_cast<uint64_t*>(smem_raw + ring0_bytes) + warp * STAGES;
  src.lane = lane;
  src.cols = a.cols;
  src.init_barriers(&tmap, &tmap, &tmap, &tmap);
  for (int i = threadIdx.x; i < kF2Ring * kF2J * 4; i += WARPS * kLaneCount) {
    const unsigned p = ll_ring + static_cast<unsigned>(i * sizeof(T));
    if constexpr (sizeof(T) == 4)
      asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(p), "f"(0.0f) : "memory");
    else
      asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(p), "d"(0.0) : "memory");
  }
  if (threadIdx.x < kF2Ring * WARPS) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ll_bars + threadIdx.x * 8), "r"(kLaneCount));
  }
  fence_mbar_init();
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int rows1 = a.rows / 2, cols1 = a.cols / 2;
  // work space: see Fused2Args / f2_work_space
  int space, f = 0, f_end = 0;  // the current range [f, f_end) of work space `space`
  if (a.tail_counter == nullptr) {
    space = 0;
    f = static_cast<int>(int64_t{a.total} * cta / a.n_ctas);
    f_end = static_cast<int>(int64_t{a.total} * (cta + 1) / a.n_ctas);
  } else {
    space = 1;
    if (cta < a.static_ctas) {
      const int64_t span = int64_t{a.n_super} * a.s_rows;
      f = static_cast<int>(span * cta / a.static_ctas);
      f_end = static_cast<int>(span * (cta + 1) / a.static_ctas);
    }
  }

  F2Level1<P, T, kStrict> l1;
  l1.bars = ll_bars;
  l1.warp = warp;
  l1.u = 0;
  l1.rd = ll_ring + static_cast<unsigned>((kF2W1 * warp + lane) * 4 * sizeof(T));
  const int jw = kF2StripW / 2 * warp + lane - 2;  // ring column of this lane's LL
  const unsigned ring_w =                         // published by the valid lanes 1..30, or 0
      lane >= 1 && lane <= 30 && jw >= 0 && jw < kF2J ? ll_ring + static_cast<unsigned>(jw * 4 * sizeof(T)) : 0u;

#pragma unroll 1
  for (;;) {
    // next unit: super-strip `sup`, level-(l+1) rows [k0, k1) (CTA-uniform)
    int sup, k0, k1;
    if (f < f_end) {
      if (space == 0 && f < a.edge_cost) {  // edge units: this CTA's if their first cost unit lies in [f, f_end)
        const int e = (f + a.unit_cost - 1) / a.unit_cost;  // first unit starting at or after f
        if (e >= a.n_edge || e * a.unit_cost >= f_end) {  // none: continue with the interior rows
          f = min(a.edge_cost, f_end);
          continue;
        }
        f = (e + 1) * a.unit_cost;
        const int n_top = a.n_super * a.units_top;
        if (e < n_top) {  // top band: super-strip e / units_top, its sub-unit e % units_top
          sup = e / a.units_top;
          k0 = a.k_begin + (e - sup * a.units_top) * a.unit_rows;
          k1 = min(a.k_begin + a.top, k0 + a.unit_rows);
        } else {
          const int eb = e - n_top;
          sup = eb / a.units_bot;
          k0 = a.k_end - a.bot + (eb - sup * a.units_bot) * a.unit_rows;
          k1 = min(a.k_end, k0 + a.unit_rows);
        }
      } else {  // interior rows: row space 0 (after the edges), 1 (static) or 2 (dynamic)
        const int ib = space == 0 ? a.edge_cost : 0;
        const int rps = space == 0 ? a.rows_in : space == 1 ? a.s_rows : a.d_rows;
        const int kb = space == 2 ? a.ki0 + a.s_rows : a.ki0;
        const int g = f - ib;
        sup = g / rps;
        const int c0 = sup * rps;
        k0 = kb + (g - c0);
        k1 = kb + min(rps, f_end - ib - c0);
        f = ib + c0 + rps;
        if (k0 >= k1) continue;
      }
    } else {  // next dynamic item: an edge unit, then guided interior ranges
      if (a.tail_counter == nullptr) break;
      __syncthreads();
      if (threadIdx.x == 0) {
        const long long e = a.dyn_edges > 0 ? static_cast<long long>(atomicAdd(a.tail_counter + 2, 1ull)) : 0;
        if (e < a.dyn_edges) {
          s_claim[0] = -1 - e;  // edge unit e
          s_claim[1] = 0;
        } else {
          int64_t sz = 0;
          s_claim[0] = claim_guided(a.tail_counter, a.n_dyn_rows, a.tail_chunk, a.n_ctas, a.guided, &sz);
          s_claim[1] = sz;
        }
      }
      __syncthreads();
      const long long c = s_claim[0];
      if (c < 0) {  // edge unit: its cost range in space 0, taken whole by this CTA
        space = 0;
        f = static_cast<int>(-1 - c) * a.unit_cost;
        f_end = f + 1;
      } else {
        space = 2;
        f = static_cast<int>(c);
        if (f >= a.n_dyn_rows) break;
        f_end = min(a.n_dyn_rows, f + static_cast<int>(s_claim[1]));
      }
      continue;
    }
    // level l: valid LL rows [n0p, n1p), HL/LH/HH rows [2 k0, 2 k1) stored
    const int n0p = max(0, 2 * (k0 - G::up));
    const int n1p = min(a.rows, 2 * (k1 + G::down));
    Ctx cx;
    cx.rows = a.rows;
    cx.cols = a.cols;
    cx.fold1 = true;  // host guarantees cols >= 128
    cx.m_strip = kF2SuperW * sup - kF2Lead + kF2StripW * warp;
    cx.m_lane = cx.m_strip + Q0 * lane;
    const bool hedge0 = cx.m_strip < 0 || cx.m_strip + Q0 * kLaneCount > a.cols;
    cx.hedge = hedge0;
    cx.n0 = 2 * k0;
    cx.n1 = 2 * k1;
    cx.first = max(0, n0p - G::up);
    const int last_load = min(a.rows - 1, n1p - 1 + G::down);
    const int last_tick = n1p - 1 + G::down;

    // level l+1
    l1.cx.rows = rows1;
    l1.cx.cols = cols1;
    l1.cx.fold1 = true;  // cols1 >= 64
    l1.cx.m_strip = kF2SuperW / 2 * sup - 2 + kF2W1 * warp;
    l1.cx.m_lane = l1.cx.m_strip + lane;
    const bool hedge1 = l1.cx.m_strip < 0 || l1.cx.m_strip + kLaneCount > cols1;
    l1.cx.hedge = hedge1;
    l1.cx.n0 = k0;
    l1.cx.n1 = k1;
    l1.cx.first = max(0, k0 - G::up);
    l1.last_load = min(rows1 - 1, k1 + G::down - 1);
    const int last_tick1 = k1 - 1 + G::down;

    const int t_lo = (cx.first / kPF) * kPF;
    const int t_hi = ((last_tick + kPF) / kPF) * kPF;
    const bool unchecked = 2 * (k0 - G::up) - G::up >= 0 && last_tick < a.rows && t_hi <= a.rows &&
                           k0 - G::up >= 0 && last_tick1 < rows1;
    src.first = unchecked ? t_lo : cx.first;
    src.last_load = unchecked ? t_hi - 1 : last_load;
    src.m_lane = cx.m_lane;
    src.m_strip = cx.m_strip;
    src.b = 0;
    src.boff = 0;
    src.start(a, &tmap, &tmap, &tmap, &tmap);

    F2Sink0<T> sink0;
    {
      const int own0 = kF2SuperW * sup, own1 = min(a.cols, own0 + kF2SuperW);
      const int w0 = cx.m_strip + 2, w1 = cx.m_strip + 62;  // this warp's valid columns (lanes 1..30)
      sink0.init(a, cx.m_lane, max(own0, w0), min(own1, w1));
      sink0.ring = ring_w;
      sink0.slot = static_cast<int>(l1.u % kF2Ring);
    }
    {
      const int own0 = kF2SuperW / 2 * sup + kF2W1 * warp;
      l1.sink.a = &a;
      l1.sink.m_lane = l1.cx.m_lane;
      l1.sink.lane_ok = l1.cx.m_lane >= own0 && l1.cx.m_lane < min(cols1, own0 + kF2W1);
      l1.sink.any_scalar = false;
    }
    Pipe0 pipe0{};
    l1.pipe = typename F2Level1<P, T, kStrict>::Pipe{};
    const bool hedge_any = hedge0 || hedge1 || sink0.any_scalar || l1.sink.any_scalar;

    if (unchecked) {
      // both levels interior: whole fused periods, no tests
      if (hedge_any) {
#pragma unroll 1
        for (int t = t_lo; t < t_hi; t += kPF)
          f2_steady_chunk<1>(pipe0, src, l1, t, cx, a, sink0, &tmap, std::make_integer_sequence<int, kPF>{});
      } else {
#pragma unroll 1
        for (int t = t_lo; t < t_hi; t += kPF)
          f2_steady_chunk<0>(pipe0, src, l1, t, cx, a, sink0, &tmap, std::make_integer_sequence<int, kPF>{});
      }
    } else {
      // image top / bottom (short units): every tick checked at both levels
#pragma unroll 1
      for (int t = cx.first; t <= last_tick; ++t) {
        T row[4][2];
        if (t <= last_load) {
          src.next(row, a, &tmap, &tmap, &tmap, &tmap);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < 2; ++q) row[c][q] = T(0);
        }
        checked_tick<kP>(pipe0, row, t, cx, a, sink0, std::make_integer_sequence<int, kP>{});
        if ((sink0.last_n & 1) && sink0.last_n >= 0) {  // an LL row pair is complete
          const int t1 = (sink0.last_n - 1) / 2;
          sink0.last_n = -0x40000000;
          sink0.slot = static_cast<int>((l1.u + 1) % kF2Ring);
          l1.step_checked(t1, a);
        }
      }
      // level-(l+1) rows whose cone runs past the image bottom: flush ticks
#pragma unroll 1
      for (int t1 = l1.last_load + 1; t1 <= last_tick1; ++t1) l1.flush_checked(t1, a);
    }
    src.finish();
  }
  if (a.tail_counter != nullptr && threadIdx.x == 0) {
    if (atomicAdd(a.tail_counter + 1, 1ull) == static_cast<unsigned long long>(a.n_ctas) - 1) {
      a.tail_counter[0] = 0;
      a.tail_counter[1] = 0;
      a.tail_counter[2] = 0;
      __threadfence();
    }
  }
}

}  // namespace b2dwt
