// b2dwt_host.cu -- C ABI (include/b2dwt.h): plans, validation, dispatch.
//
// A plan is a compiled StencilProgram (liftfuse/engine.py:227-256).  At plan
// creation the program's structure -- the ordered (src, dm, dn) list of every
// sub-step/target and which coefficients are exactly 1.0 -- is matched against
// the built-in structures of programs.inc.  A match runs the fused streaming
// kernel (stream_kernel.cuh) with the plan's own coefficients; anything else
// runs the per-sub-step interpreter (generic_kernel.cuh).  Both evaluate the
// terms in the compiled order, so strict mode is bit-identical to the
// reference either way.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu (no link dependency)

#include "../../include/b2dwt.h"
#include "generic_kernel.cuh"
#include "generic_tile.cuh"
#include "launch.h"

namespace b2dwt {

#define B2DWT_DECLARE(ID, NAME)                                     \
  cudaError_t b2dwt_fused_##NAME(const FusedLaunch&, bool* used_tma); \
  cudaError_t b2dwt_tile_##NAME(const FusedLaunch&);                  \
  cudaError_t b2dwt_fused2_##NAME(const Fused2Launch&);               \
  ConeInfo b2dwt_cone_##NAME();
B2DWT_FOR_EACH_PROGRAM(B2DWT_DECLARE)
#undef B2DWT_DECLARE

namespace {

thread_local std::string g_error;
long long* g_dbg = nullptr;  // debug: per-warp timing records of the next fused launches
int64_t g_dbg_n = 0;

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(B2DWT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Builtin {
  const char* key;
  int nsub;
  int nterms;
  int (*begin)(int);
  TermInfo (*term)(int);
  double (*coef)(int);
  FusedLauncher launch;
  TileLauncher tile;
  ConeGetter cone;
  bool inverse;
  Fused2Launcher fused2;
};

template <class P>
int begin_of(int i) {
  return P::begin(i);
}
template <class P>
TermInfo term_of(int i) {
  return P::term(i);
}
template <class P>
double coef_of(int i) {
  return P::coef(i);
}

const Builtin* builtins() {
  static const Builtin table[] = {
#define B2DWT_ROW(ID, NAME)                                                                                      \
  {progs::NAME::kKey,        progs::NAME::kNumSub, progs::NAME::kNumTerms, &begin_of<progs::NAME>,             \
   &term_of<progs::NAME>,    &coef_of<progs::NAME>,    &b2dwt_fused_##NAME,  &b2dwt_tile_##NAME, &b2dwt_cone_##NAME,     std::strstr(progs::NAME::kKey, "/inv") \
   != nullptr, &b2dwt_fused2_##NAME},
      B2DWT_FOR_EACH_PROGRAM(B2DWT_ROW)
#undef B2DWT_ROW
  };
  return table;
}

}  // namespace

// Error reporting for the other host units (host_pipeline.cu).
int set_last_error(int code, const char* msg) { return fail(code, msg); }

// NVTX ranges around pyramid levels and host-pipeline bands (nsys timelines),
// only when B2DWT_NVTX is set so the default path makes no NVTX calls.
bool nvtx_on() {
  static const bool on = std::getenv("B2DWT_NVTX") != nullptr;
  return on;
}
NvtxRange::NvtxRange(const char* name) : active(nvtx_on()) {
  if (active) nvtxRangePushA(name);
}
NvtxRange::~NvtxRange() {
  if (active) nvtxRangePop();
}

}  // namespace b2dwt

using namespace b2dwt;

struct b2dwt_plan_s {
  int nsub = 0;
  std::vector<int32_t> counts;   // nsub * 4
  std::vector<b2dwt_term> terms;
  int dtype = 0;
  int flags = 0;
  int builtin = -1;              // index into builtins(), -1 = generic
  std::vector<double> coeffs;    // flat, compiled order
  ConeInfo cone{0, 0, 0, 0};
  std::string key;
};

namespace {

bool strict_of(const b2dwt_plan_s* p) { return (p->flags & B2DWT_FAST) == 0; }

// Zero-initialised counter slots (kSlotWords words) for the dynamic work tail.
// The kernel's last CTA resets its pair, so launches ordered on ONE stream can
// share pairs safely; launches that may run concurrently must not.  Hence:
//   * eager launches draw round-robin from a pool owned by their stream;
//   * launches recorded into a CUDA graph draw from a capture arena whose pairs
//     are never handed out again (a graph may replay concurrently with anything).
// Pools are allocated and zeroed synchronously the first time a device is used
// outside a capture; inside a capture with no arena left the launch runs a fully
// static split (tail counter null), which is slower but exact.
namespace {
constexpr int kStreamSlots = 64;
constexpr int kArenaSlots = 4096;
constexpr int kSlotWords = 4;  // [0] claimed tail units, [1] CTAs done, [2] edge tickets, [3] spare
struct DeviceCounters {
  std::unordered_map<cudaStream_t, std::pair<unsigned long long*, unsigned>> streams;
  unsigned long long* arena = nullptr;
  int arena_used = 0;
};
unsigned long long* zeroed_pairs(int n) {
  void* p = nullptr;
  if (cudaMalloc(&p, static_cast<size_t>(n) * kSlotWords * sizeof(unsigned long long)) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  // synchronous zeroing, complete before any stream can use the pairs
  if (cudaMemset(p, 0, static_cast<size_t>(n) * kSlotWords * sizeof(unsigned long long)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    (void)cudaGetLastError();
    cudaFree(p);
    return nullptr;
  }
  return static_cast<unsigned long long*>(p);
}
}  // namespace

unsigned long long* tail_counter_slot(cudaStream_t stream) {
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static DeviceCounters dev_counters[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  DeviceCounters& d = dev_counters[dev];
  if (cap != cudaStreamCaptureStatusNone) {
    if (!d.arena || d.arena_used >= kArenaSlots) return nullptr;  // no allocation inside a capture
    return d.arena + kSlotWords * (d.arena_used++);
  }
  if (!d.arena || d.arena_used >= kArenaSlots) {  // (re)fill the capture arena while we may allocate
    d.arena = zeroed_pairs(kArenaSlots);
    d.arena_used = 0;
  }
  auto it = d.streams.find(stream);
  if (it == d.streams.end()) {
    unsigned long long* p = zeroed_pairs(kStreamSlots);
    if (!p) return nullptr;
    it = d.streams.emplace(stream, std::make_pair(p, 0u)).first;
  }
  return it->second.first + kSlotWords * (it->second.second++ % kStreamSlots);
}

// Guided self-scheduling of the dynamic tail (claim_guided, stream_kernel.cuh).
// Measured: the two-level fused kernel gains (C3 levels 0+1 427 -> 408 us with a
// 768/1024 static share), the stream kernel does not (C4 +1.6%, C5 -1%), so the
// defaults differ.  The value k > 0 sizes a claim as remaining / (k x CTAs); 0
// means fixed chunks.  B2DWT_GUIDED / B2DWT_F2_GUIDED override (defaults 0 / 1: for the
// fused kernel a full fair share, tools/guided_sweep.sh: levels 0+1 403 -> 392 us vs k = 2).
int guided_tail(bool fused2) {
  static const int v[2] = {[] {
                             const char* e = std::getenv("B2DWT_GUIDED");
                             return e ? std::atoi(e) : 0;
                           }(),
                           [] {
                             const char* e = std::getenv("B2DWT_F2_GUIDED");
                             return e ? std::atoi(e) : 1;
                           }()};
  return v[fused2 ? 1 : 0];
}

// Lower bound on rows per CTA (B2DWT_MIN_ROWS overrides).
int min_rows() {
  static int v = [] {
    const char* e = std::getenv("B2DWT_MIN_ROWS");
    return e ? std::atoi(e) : 16;  // measured on the C3 pyramid (level 3: 22.5 -> 18.4 us)
  }();
  return v;
}

// Work split: [0] share of the rows split statically (1/1024), [1] rows per
// dynamically claimed tail chunk.  B2DWT_STATIC_FRAC / B2DWT_TAIL_ROWS override.
int split_param(int which) {
  static const int v[5] = {[] {
                             const char* e = std::getenv("B2DWT_STATIC_FRAC");
                             return e ? std::atoi(e) : 768;
                           }(),
                           [] {
                             const char* e = std::getenv("B2DWT_TAIL_ROWS");
                             return e ? std::atoi(e) : 16;  // C3 level 0: 396 -> 392 us
                           }(),
                           [] {
                             const char* e = std::getenv("B2DWT_STRIP_ALIGN");
                             return e ? std::atoi(e) : 0;
                           }(),
                           [] {
                             const char* e = std::getenv("B2DWT_FULL_ROWS");
                             return e ? std::atoi(e) : 0;
                           }(),
                           [] {
                             const char* e = std::getenv("B2DWT_PDL");
                             return e ? std::atoi(e) : 1;
                           }()};
  return v[which];
}

// Largest level (batch x quads) served by the tile kernel; B2DWT_TILE_MAX_QUADS overrides.
int64_t tile_max_quads() {
  static int64_t v = [] {
    const char* e = std::getenv("B2DWT_TILE_MAX_QUADS");
    return e ? std::atoll(e) : int64_t{1} << 18;  // measured: levels <= 512^2 quads
  }();
  return v;
}

// Input bytes per stream-kernel launch before a request is split (0: never);
// B2DWT_MAX_LAUNCH_BYTES overrides.
int64_t max_launch_bytes() {
  const char* e = std::getenv("B2DWT_MAX_LAUNCH_BYTES");  // read per call: tests vary it
  return e ? std::atoll(e) : int64_t{512} << 20;
}

// Tile window rows (16 or 32); 0 = the launcher decides.  B2DWT_TILE_ROWS overrides.
int tile_rows_for() {
  static int forced = [] {
    const char* e = std::getenv("B2DWT_TILE_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  return forced;
}

// Relative cost of an image-edge strip row (eighths of an interior row) used to
// balance the work split; B2DWT_EDGE_COST8 overrides it for tuning.
int edge_cost8() {
  static int v = [] {
    const char* e = std::getenv("B2DWT_EDGE_COST8");
    const int x = e ? std::atoi(e) : 8;
    return x < 8 ? 8 : x;
  }();
  return v;
}

int match_builtin(const b2dwt_plan_s& p) {
  const Builtin* tab = builtins();
  for (int id = 0; id < B2DWT_NUM_PROGRAMS; ++id) {
    const Builtin& b = tab[id];
    if (b.nsub != p.nsub || b.nterms != static_cast<int>(p.terms.size())) continue;
    bool ok = true;
    for (int st = 0; st < p.nsub * 4 && ok; ++st)
      ok = (b.begin(st + 1) - b.begin(st)) == p.counts[st];
    for (int i = 0; i < b.nterms && ok; ++i) {
      const TermInfo ti = b.term(i);
      const b2dwt_term& t = p.terms[i];
      // same term, same coefficient bits (they are compiled into the kernel)
      ok = ti.src == t.src && ti.dm == t.dm && ti.dn == t.dn && b.coef(i) == t.coeff;
    }
    if (ok) return id;
  }
  return -1;
}

size_t esize(int dtype) { return dtype == B2DWT_F32 ? 4 : 8; }

// ---------------------------------------------------------------------------
// Generic path: one interpreter launch per sub-step, ping-pong scratch.

// Stream-ordered scratch comes from the device's default memory pool; by
// default the pool returns freed memory to the OS at every synchronisation, so
// each call would map its scratch afresh (milliseconds for a 4096^2 image).
// Keep it cached instead (once per device).
void keep_pool_memory() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~uint64_t{0};
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  (void)cudaGetLastError();
  done[dev] = true;
}
struct ViewSet {
  const void* p[4];
  int64_t rs[4], cs[4];
};

ViewSet planar_views(const b2dwt_planes* pl, size_t es) {
  ViewSet v;
  for (int c = 0; c < 4; ++c) {
    v.p[c] = pl->ptr[c];
    v.rs[c] = pl->ld[c];
    v.cs[c] = 1;
  }
  (void)es;
  return v;
}

ViewSet image_views(const void* img, int64_t ld, size_t es) {
  ViewSet v;
  for (int c = 0; c < 4; ++c) {
    v.p[c] = static_cast<const char*>(img) + ((c >> 1) * ld + (c & 1)) * static_cast<int64_t>(es);
    v.rs[c] = 2 * ld;
    v.cs[c] = 2;
  }
  return v;
}

template <class T>
cudaError_t launch_generic_substep(const b2dwt_plan_s& p, int s, const int32_t* term_base, const ViewSet& in,
                                   int64_t in_b, const ViewSet& out, int64_t out_b, int64_t rows, int64_t cols,
                                   int batch, cudaStream_t stream) {
  GenericSubstep sub{};
  int k = 0;
  for (int t = 0; t < 4; ++t) {
    sub.count[t] = p.counts[s * 4 + t];
    for (int j = 0; j < sub.count[t]; ++j, ++k) {
      const b2dwt_term& src = p.terms[term_base[0] + k];
      sub.terms[k].src = static_cast<int8_t>(src.src);
      sub.terms[k].dm = static_cast<int8_t>(src.dm);
      sub.terms[k].dn = static_cast<int8_t>(src.dn);
      sub.terms[k].tgt = static_cast<int8_t>(t);
      sub.terms[k].coeff = src.coeff;
    }
  }
  PlaneView<const T> iv[4];
  PlaneView<T> ov[4];
  for (int c = 0; c < 4; ++c) {
    iv[c] = PlaneView<const T>{static_cast<const T*>(in.p[c]), in.rs[c], in.cs[c]};
    ov[c] = PlaneView<T>{static_cast<T*>(const_cast<void*>(out.p[c])), out.rs[c], out.cs[c]};
  }
  const int64_t total = rows * cols;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  dim3 g(grid, batch);
  if (strict_of(&p))
    generic_substep_kernel<T, true><<<g, 256, 0, stream>>>(sub, iv[0], iv[1], iv[2], iv[3], ov[0], ov[1], ov[2],
                                                           ov[3], in_b, out_b, static_cast<int>(rows),
                                                           static_cast<int>(cols));
  else
    generic_substep_kernel<T, false><<<g, 256, 0, stream>>>(sub, iv[0], iv[1], iv[2], iv[3], ov[0], ov[1], ov[2],
                                                            ov[3], in_b, out_b, static_cast<int>(rows),
                                                            static_cast<int>(cols));
  return cudaGetLastError();
}

int run_generic(const b2dwt_plan_s& p, const ViewSet& in, int64_t in_b, const ViewSet& out, int64_t out_b,
                int64_t rows, int64_t cols, int batch, cudaStream_t stream) {
  const size_t es = esize(p.dtype);
  const int64_t plane = rows * cols;
  void* scratch = nullptr;
  if (p.nsub > 1) {
    keep_pool_memory();
    const size_t bytes = static_cast<size_t>(2 * 4 * plane * batch) * es;
    cudaError_t e = cudaMallocAsync(&scratch, bytes, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(generic scratch)");
  }
  auto scratch_views = [&](int which) {
    ViewSet v;
    for (int c = 0; c < 4; ++c) {
      v.p[c] = static_cast<char*>(scratch) + ((which * 4 + c) * plane * batch) * static_cast<int64_t>(es);
      v.rs[c] = cols;
      v.cs[c] = 1;
    }
    return v;
  };
  int32_t base = 0;
  cudaError_t err = cudaSuccess;
  for (int s = 0; s < p.nsub && err == cudaSuccess; ++s) {
    const ViewSet vin = s == 0 ? in : scratch_views((s - 1) & 1);
    const int64_t bin = s == 0 ? in_b : plane;
    const ViewSet vout = s == p.nsub - 1 ? out : scratch_views(s & 1);
    const int64_t bout = s == p.nsub - 1 ? out_b : plane;
    err = p.dtype == B2DWT_F32
              ? launch_generic_substep<float>(p, s, &base, vin, bin, vout, bout, rows, cols, batch, stream)
              : launch_generic_substep<double>(p, s, &base, vin, bin, vout, bout, rows, cols, batch, stream);
    base += p.counts[s * 4] + p.counts[s * 4 + 1] + p.counts[s * 4 + 2] + p.counts[s * 4 + 3];
  }
  if (scratch) cudaFreeAsync(scratch, stream);
  if (err != cudaSuccess) return cuda_fail(err, "generic stencil kernel");
  return B2DWT_OK;
}

void keep_pool_memory();

// ---------------------------------------------------------------------------
// Fused generic interpreter (generic_tile.cuh) for plans without a built-in
// kernel: B2DWT_EUNSUPPORTED when the program does not fit it (the caller
// then runs the per-sub-step interpreter).
template <class T>
cudaError_t launch_gtile(const b2dwt_plan_s& p, const GTileProgram& g, const FusedLaunch& r) {
  GTileArgs<T> a{};
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
  a.lin = r.lin;
  a.lout = r.lout;
  a.rows = r.rows;
  a.cols = r.cols;
  a.batch = r.batch;
  a.tr = kGTileWR - g.up - g.down;
  a.tc = kGTileWC - g.left - g.right;
  a.tiles_r = (r.rows + a.tr - 1) / a.tr;
  a.tiles_c = (r.cols + a.tc - 1) / a.tc;
  const int64_t n = static_cast<int64_t>(a.tiles_r) * a.tiles_c * r.batch;
  if (n > 0x7fffffff) return cudaErrorNotSupported;
  const size_t smem = gtile_smem_bytes(sizeof(T));
  // the term table travels in stream-ordered device memory (too large for the
  // parameter block); the pool keeps it cached between calls
  keep_pool_memory();
  void* dg = nullptr;
  cudaError_t e = cudaMallocAsync(&dg, sizeof(GTileProgram), r.stream);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(dg, &g, sizeof(GTileProgram), cudaMemcpyHostToDevice, r.stream);
  if (e == cudaSuccess) {
    // opt in to the large dynamic shared memory once per instantiation and device
    static PerDevice once;
    static cudaError_t attr[kMaxDevices][2] = {};
    const int dev = once.run([&](int d) {
      attr[d][0] = cudaFuncSetAttribute(generic_tile_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem));
      attr[d][1] = cudaFuncSetAttribute(generic_tile_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem));
    });
    const cudaError_t attr_strict = dev < 0 ? cudaErrorNotSupported : attr[dev][0];
    const cudaError_t attr_fast = dev < 0 ? cudaErrorNotSupported : attr[dev][1];
    if (strict_of(&p)) {
      e = attr_strict;
      if (e == cudaSuccess)
        generic_tile_kernel<T, true><<<static_cast<unsigned>(n), kGTileThreads, smem, r.stream>>>(
            a, static_cast<const GTileProgram*>(dg));
    } else {
      e = attr_fast;
      if (e == cudaSuccess)
        generic_tile_kernel<T, false><<<static_cast<unsigned>(n), kGTileThreads, smem, r.stream>>>(
            a, static_cast<const GTileProgram*>(dg));
    }
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  cudaFreeAsync(dg, r.stream);
  return e;
}

int try_gtile(const b2dwt_plan_s& p, const FusedLaunch& r) {
  if ((p.flags & B2DWT_NO_TILE) || p.builtin >= 0 && !(p.flags & B2DWT_FORCE_GENERIC)) return B2DWT_EUNSUPPORTED;
  if (p.nsub > kGTileMaxSub || static_cast<int>(p.terms.size()) > kGTileMaxTerms) return B2DWT_EUNSUPPORTED;
  GTileProgram g{};
  g.n_sub = p.nsub;
  int k = 0;
  for (int s = 0; s < p.nsub; ++s) {
    int ru = 0, rd = 0, rl = 0, rr = 0;
    for (int t = 0; t < 4; ++t) {
      const int n = p.counts[s * 4 + t];
      g.count[s][t] = static_cast<int16_t>(n);
      g.first[s][t] = static_cast<int16_t>(k);
      for (int j = 0; j < n; ++j, ++k) {
        const b2dwt_term& tm = p.terms[k];
        if (tm.dn < -kGTileMaxReach || tm.dn > kGTileMaxReach || tm.dm < -kGTileMaxReach ||
            tm.dm > kGTileMaxReach)
          return B2DWT_EUNSUPPORTED;
        g.src[k] = static_cast<int16_t>(tm.src);
        g.off[k] = static_cast<int16_t>(tm.dn * kGTileWC + tm.dm);
        g.unit[k] = tm.coeff == 1.0;  // x * 1.0 == x: skipping it is exact
        g.coef[k] = tm.coeff;
        ru = std::max(ru, -tm.dn);
        rd = std::max(rd, tm.dn);
        rl = std::max(rl, -tm.dm);
        rr = std::max(rr, tm.dm);
      }
      const b2dwt_term* t0 = n == 1 ? &p.terms[k - 1] : nullptr;
      g.identity[s][t] = t0 && t0->src == t && t0->dm == 0 && t0->dn == 0 && t0->coeff == 1.0;
    }
    g.up += ru;
    g.down += rd;
    g.left += rl;
    g.right += rr;
  }
  // the window must leave an output tile, and every ghost cell inside the
  // output's cone must mirror a cell inside the window (near-symmetric cone)
  if (kGTileWR - g.up - g.down < 2 || kGTileWC - g.left - g.right < 2) return B2DWT_EUNSUPPORTED;
  if (std::abs(g.up - g.down) > 1 || std::abs(g.left - g.right) > 1) return B2DWT_EUNSUPPORTED;
  const cudaError_t e = p.dtype == B2DWT_F32 ? launch_gtile<float>(p, g, r) : launch_gtile<double>(p, g, r);
  if (e == cudaErrorNotSupported) return B2DWT_EUNSUPPORTED;
  if (e != cudaSuccess) return cuda_fail(e, "generic tile kernel");
  return B2DWT_OK;
}

int run_fused(const b2dwt_plan_s& p, FusedLaunch& r) {
  const Builtin& b = builtins()[p.builtin];
  r.dtype = p.dtype;
  r.strict = strict_of(&p);
  r.allow_tma = (p.flags & B2DWT_NO_TMA) == 0;
  r.coeffs = p.coeffs.data();
  r.n_coeffs = static_cast<int>(p.coeffs.size());
  // Small levels are latency-bound (a tick is a long dependent chain), so
  // spread them over the whole machine; 16 rows keeps the cone re-read <= 25%
  // there and negligible on large levels, which fill the machine anyway.
  r.min_rows_per_warp = min_rows();
  r.edge_cost8 = edge_cost8();
  r.dbg = g_dbg;
  // dynamic tail: a counter slot from the per-device pool (self-resetting)
  r.tail_counter = split_param(0) < 1024 ? tail_counter_slot(r.stream) : nullptr;
  r.static_frac = split_param(0);
  r.tail_rows = split_param(1);
  r.guided = guided_tail(false);
  r.strip_align = split_param(2);
  r.full_rows = split_param(3);
  r.pdl = split_param(4) != 0;
  // Small whole-image levels run the 2-D tile kernel: the streaming kernel's
  // per-warp row pipelines are too short there to hide their latency.
  const int64_t quads = static_cast<int64_t>(r.batch) * r.rows * r.cols;
  const bool whole = r.row_begin == 0 && r.row_end == r.rows && r.in_row0 == 0 && r.out_row0 == 0 &&
                     r.in_rows == r.rows;
  const bool tile_ok = (p.flags & B2DWT_NO_TILE) == 0 &&
                       (quads <= tile_max_quads() || (p.flags & B2DWT_FORCE_TILE) != 0);
  if (whole && tile_ok) {
    r.use_tile = true;
    r.tile_rows = tile_rows_for();
    const cudaError_t e = b.tile(r);
    if (e == cudaSuccess) return B2DWT_OK;
    if (e != cudaErrorNotSupported) return cuda_fail(e, "fused tile kernel");
    (void)cudaGetLastError();
    r.use_tile = false;
  }
  // Footprint-bounded launches: one launch spreads its CTAs over the whole
  // request (each takes a contiguous share of the rows), and past ~1 GiB the
  // concurrently touched pages outgrow the GPU's translation reach (measured
  // on 65536^2: 0.70 of copy bandwidth as one launch, 0.82 as 16 row bands).
  // Large requests therefore run as a sequence of launches of at most
  // max_launch_bytes of input each: batch chunks, or row bands of one image.
  const size_t es = r.dtype == 1 ? 8 : 4;
  const int64_t in_bytes = quads * 4 * static_cast<int64_t>(es);
  const int64_t cap = max_launch_bytes();
  int64_t parts = cap > 0 ? (in_bytes + cap - 1) / cap : 1;
  if (r.batch > 1) parts = std::min<int64_t>(parts, r.batch);
  else parts = std::min<int64_t>(parts, std::max(1, (r.row_end - r.row_begin) / 256));
  bool used_tma = false;
  cudaError_t e = cudaSuccess;
  if (parts <= 1) {
    e = b.launch(r, &used_tma);
  } else if (r.batch > 1) {
    const int batch = r.batch;
    for (int64_t i = 0; i < parts && e == cudaSuccess; ++i) {
      const int i0 = static_cast<int>(batch * i / parts), i1 = static_cast<int>(batch * (i + 1) / parts);
      FusedLaunch q = r;
      const int64_t ib = static_cast<int64_t>(i0) * r.in_bstride * static_cast<int64_t>(es);
      const int64_t ob = static_cast<int64_t>(i0) * r.out_bstride * static_cast<int64_t>(es);
      if (q.in_img) q.in_img = static_cast<const char*>(q.in_img) + ib;
      if (q.out_img) q.out_img = static_cast<char*>(q.out_img) + ob;
      for (int c = 0; c < 4; ++c) {
        if (q.in_pl[c]) q.in_pl[c] = static_cast<const char*>(q.in_pl[c]) + ib;
        if (q.out_pl[c]) q.out_pl[c] = static_cast<char*>(q.out_pl[c]) + ob;
      }
      q.batch = i1 - i0;
      if (i > 0) q.tail_counter = r.tail_counter ? tail_counter_slot(r.stream) : nullptr;
      e = b.launch(q, &used_tma);
    }
  } else {
    const int rb = r.row_begin, re = r.row_end;
    for (int64_t i = 0; i < parts && e == cudaSuccess; ++i) {
      FusedLaunch q = r;
      q.row_begin = rb + static_cast<int>((re - rb) * i / parts);
      q.row_end = rb + static_cast<int>((re - rb) * (i + 1) / parts);
      if (i > 0) q.tail_counter = r.tail_counter ? tail_counter_slot(r.stream) : nullptr;
      e = b.launch(q, &used_tma);
    }
  }
  if (e == cudaErrorNotSupported) return fail(B2DWT_EUNSUPPORTED, "no compiled fused variant for this request");
  if (e != cudaSuccess) return cuda_fail(e, "fused stream kernel");
  return B2DWT_OK;
}

// Smallest level (quads) the two-level fused kernel takes; below it the levels
// run one launch each.  B2DWT_FUSE2_MIN_QUADS overrides (0 disables fusion).
int64_t fuse2_min_quads() {
  const char* e = std::getenv("B2DWT_FUSE2_MIN_QUADS");  // read per call: tests vary it
  return e ? std::atoll(e) : int64_t{1} << 20;
}

// Levels at which b2dwt_dwt may start a fused pair (greedy from level 0 by
// default); B2DWT_FUSE2_PAIRS="0,3" e.g. pairs (0,1) and (3,4) only.
// B2DWT_FUSE2_STRICT=0 keeps strict plans at one launch per level (measured
// C3 strict: 0.5105 ms fused vs 0.567 ms unfused; fast 0.476 vs 0.546 ms).
bool fuse2_starts_at(const b2dwt_plan_s& p, int level) {
  if (strict_of(&p)) {
    const char* s = std::getenv("B2DWT_FUSE2_STRICT");
    if (s && std::atoi(s) == 0) return false;
  }
  const char* e = std::getenv("B2DWT_FUSE2_PAIRS");
  if (!e) return true;
  for (const char* p = e; *p;) {
    char* end = nullptr;
    const long v = std::strtol(p, &end, 10);
    if (end == p) break;
    if (v == level) return true;
    p = *end ? end + 1 : end;
  }
  return false;
}

// Levels l and l+1 of a forward pyramid in one kernel (fused2_kernel.cuh):
// level l's LL never reaches HBM.  B2DWT_EUNSUPPORTED when the request does not
// fit it (the caller then runs the two levels separately).
int run_fused2_pair(const b2dwt_plan_s& p, const void* in, int64_t in_ld, int64_t h, int64_t w,
                    const b2dwt_planes& det0, const b2dwt_planes& det1, void* ll1, int64_t ll1_ld,
                    cudaStream_t stream, bool any_size = false) {
  if (p.builtin < 0 || (p.flags & (B2DWT_FORCE_GENERIC | B2DWT_NO_TMA | B2DWT_NO_FUSE)) || p.dtype != B2DWT_F32)
    return B2DWT_EUNSUPPORTED;
  const Builtin& b = builtins()[p.builtin];
  if (b.inverse) return B2DWT_EUNSUPPORTED;
  const int64_t rows = h / 2, cols = w / 2;
  const int64_t minq = fuse2_min_quads();
  if (!any_size && (minq <= 0 || rows * cols < minq)) return B2DWT_EUNSUPPORTED;
  if ((rows & 1) || (cols & 1)) return B2DWT_EUNSUPPORTED;
  Fused2Launch r{};
  r.dtype = 0;
  r.strict = strict_of(&p);
  r.in_img = in;
  r.in_ld = in_ld;
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  for (int c = 1; c < 4; ++c) {
    r.out0_pl[c] = det0.ptr[c];
    r.out0_ld[c] = det0.ld[c];
    r.out1_pl[c] = det1.ptr[c];
    r.out1_ld[c] = det1.ld[c];
  }
  r.out1_pl[0] = ll1;
  r.out1_ld[0] = ll1_ld;
  // work split of the fused kernel: a unit re-reads the cones of BOTH levels
  // (~14 level-l rows), so its dynamic tail chunks are longer than the stream
  // kernel's.  B2DWT_F2_STATIC_FRAC / B2DWT_F2_TAIL_ROWS override.
  // static share, measured on C3 with k = 1 claims (tools/guided_sweep.sh,
  // tools/sf_ab.sh): 832/1024 for fast plans (768: +0.4%), 768 for strict ones
  // (832: +1.1%, the slower pipeline wants the longer dynamic tail)
  static const int f2_static_env = [] {
    const char* e = std::getenv("B2DWT_F2_STATIC_FRAC");
    return e ? std::atoi(e) : -1;
  }();
  static const int f2_tail = [] {
    const char* e = std::getenv("B2DWT_F2_TAIL_ROWS");
    return e ? std::atoi(e) : 16;
  }();
  static const int f2_edge = [] {  // 8 (kF2Edge): sized per launch for small ones (f2_work_space)
    const char* e = std::getenv("B2DWT_F2_EDGE_ROWS");
    return e ? std::atoi(e) : 8;
  }();
  const int f2_static = f2_static_env >= 0 ? f2_static_env : (r.strict ? 768 : 832);
  r.static_frac = f2_static;
  r.tail_rows1 = f2_tail;
  r.guided = guided_tail(true);
  r.edge_rows1 = f2_edge;
  static const int f2_min_rows = [] {  // fewest level-(l+1) rows per CTA (0: from min_rows())
    const char* e = std::getenv("B2DWT_F2_MIN_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  r.min_rows1 = f2_min_rows > 0 ? f2_min_rows : std::max(8, min_rows() / 2);
  r.pdl = split_param(4) != 0;
  r.stream = stream;
  // footprint-bounded launches, as run_fused: row bands of <= 1 GiB of input
  // (B2DWT_F2_MAX_LAUNCH_BYTES): measured on C3 (1 GiB in), one launch runs
  // levels 0+1 in 437 us against 460 us as two 512 MiB bands -- each band
  // pays a ramp and a tail, and the translation-reach penalty that makes the
  // stream kernel split (65536^2) only sets in beyond that
  const int64_t rows1 = rows / 2;
  const int64_t in_bytes = rows * cols * 16;
  const char* cap_env = std::getenv("B2DWT_F2_MAX_LAUNCH_BYTES");
  const int64_t cap = cap_env ? std::atoll(cap_env) : int64_t{1} << 30;
  int64_t parts = cap > 0 ? (in_bytes + cap - 1) / cap : 1;
  parts = std::max<int64_t>(1, std::min<int64_t>(parts, rows1 / 128));
  cudaError_t e = cudaSuccess;
  for (int64_t i = 0; i < parts && e == cudaSuccess; ++i) {
    r.k_begin = static_cast<int>(rows1 * i / parts);
    r.k_end = static_cast<int>(rows1 * (i + 1) / parts);
    r.tail_counter = f2_static < 1024 ? tail_counter_slot(stream) : nullptr;
    e = b.fused2(r);
    if (e == cudaErrorNotSupported) {
      (void)cudaGetLastError();
      if (i == 0) return B2DWT_EUNSUPPORTED;
      return fail(B2DWT_ECUDA, "two-level fused kernel refused a later row band");
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "two-level fused kernel");
  return B2DWT_OK;
}

bool fused_layout_ok(const b2dwt_plan_s& p, int lin, int lout) {
  if (p.builtin < 0 || (p.flags & B2DWT_FORCE_GENERIC)) return false;
  const bool inv = builtins()[p.builtin].inverse;
  if (lin == 1 && lout == 1) return true;  // planar -> planar
  return inv ? (lin == 1 && lout == 0) : (lin == 0 && lout == 1);
}

int check_plan(b2dwt_plan p) {
  if (!p) return fail(B2DWT_EINVAL, "null plan");
  return B2DWT_OK;
}

int check_planes(const b2dwt_planes* pl, const char* what) {
  if (!pl) return fail(B2DWT_EINVAL, std::string(what) + ": null planes");
  for (int c = 0; c < 4; ++c)
    if (!pl->ptr[c]) return fail(B2DWT_EINVAL, std::string(what) + ": null plane pointer");
  return B2DWT_OK;
}

int check_dims(int64_t height, int64_t width) {
  if (height < 1 || width < 1) return fail(B2DWT_EINVAL, "image data must be a non-empty 2-D array");
  if (height % 2 || width % 2) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), "dimensions must be even, got %lldx%lld", static_cast<long long>(width),
                  static_cast<long long>(height));
    return fail(B2DWT_EINVAL, buf);
  }
  // the reflection map works in 32-bit pixel coordinates (period 4*cs - 2)
  if (height / 2 > (1LL << 29) || width / 2 > (1LL << 29))
    return fail(B2DWT_EUNSUPPORTED, "image too large for 32-bit quad indexing");
  return B2DWT_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int32_t b2dwt_abi_version(void) { return B2DWT_ABI_VERSION; }

const char* b2dwt_last_error(void) { return g_error.c_str(); }

int32_t b2dwt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

int b2dwt_plan_create(const b2dwt_program* program, int32_t dtype, int32_t flags, b2dwt_plan* out) {
  if (!out) return fail(B2DWT_EINVAL, "null output plan pointer");
  *out = nullptr;
  if (!program) return fail(B2DWT_EINVAL, "null program");
  if (program->abi_version != B2DWT_ABI_VERSION) return fail(B2DWT_EINVAL, "program ABI version mismatch");
  if (dtype != B2DWT_F32 && dtype != B2DWT_F64) return fail(B2DWT_EINVAL, "dtype must be B2DWT_F32 or B2DWT_F64");
  if (program->n_substeps < 1) return fail(B2DWT_EINVAL, "program has no sub-steps");
  if (!program->term_counts) return fail(B2DWT_EINVAL, "null term_counts");
  auto* p = new b2dwt_plan_s();
  p->nsub = program->n_substeps;
  p->dtype = dtype;
  p->flags = flags;
  p->counts.assign(program->term_counts, program->term_counts + 4 * p->nsub);
  size_t total = 0;
  for (int st = 0; st < 4 * p->nsub; ++st) {
    if (p->counts[st] < 0 || p->counts[st] > kGenericMaxTerms) {
      delete p;
      return fail(B2DWT_EUNSUPPORTED, "too many terms in one sub-step target");
    }
    total += static_cast<size_t>(p->counts[st]);
  }
  for (int s = 0; s < p->nsub; ++s) {
    int sub = 0;
    for (int t = 0; t < 4; ++t) sub += p->counts[s * 4 + t];
    if (sub > kGenericMaxTerms) {
      delete p;
      return fail(B2DWT_EUNSUPPORTED, "too many terms in one sub-step");
    }
  }
  if (total && !program->terms) {
    delete p;
    return fail(B2DWT_EINVAL, "null terms");
  }
  p->terms.assign(program->terms, program->terms + total);
  for (const b2dwt_term& t : p->terms) {
    if (t.src < 0 || t.src > 3 || t.dm < -64 || t.dm > 64 || t.dn < -64 || t.dn > 64) {
      delete p;
      return fail(B2DWT_EINVAL, "term out of range (src 0..3, |dm|,|dn| <= 64)");
    }
  }
  p->builtin = (flags & B2DWT_FORCE_GENERIC) ? -1 : match_builtin(*p);
  if (p->builtin >= 0) {
    const Builtin& b = builtins()[p->builtin];
    p->key = b.key;
    for (const b2dwt_term& t : p->terms) p->coeffs.push_back(t.coeff);
    p->cone = b.cone();
  } else {
    p->key = "generic";
  }
  *out = p;
  return B2DWT_OK;
}

// Debug hooks (not part of the public header): per-warp cycle counts of the
// fused kernel, used to tune the work split.
int b2dwt_debug_enable(int64_t max_warps) {
  if (g_dbg) cudaFree(g_dbg);
  g_dbg = nullptr;
  g_dbg_n = 0;
  if (max_warps <= 0) return B2DWT_OK;
  if (cudaMalloc(&g_dbg, static_cast<size_t>(max_warps) * 4 * sizeof(long long)) != cudaSuccess)
    return fail(B2DWT_ECUDA, "debug buffer");
  cudaMemset(g_dbg, 0, static_cast<size_t>(max_warps) * 4 * sizeof(long long));
  g_dbg_n = max_warps;
  return B2DWT_OK;
}

int b2dwt_debug_fetch(long long* host, int64_t max_warps) {
  if (!g_dbg) return fail(B2DWT_EINVAL, "debug timing not enabled");
  const int64_t n = max_warps < g_dbg_n ? max_warps : g_dbg_n;
  if (cudaMemcpy(host, g_dbg, static_cast<size_t>(n) * 4 * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(B2DWT_ECUDA, "debug fetch");
  return B2DWT_OK;
}

int b2dwt_plan_destroy(b2dwt_plan plan) {
  delete plan;
  return B2DWT_OK;
}

int b2dwt_plan_get_info(b2dwt_plan plan, b2dwt_plan_info* info) {
  if (int rc = check_plan(plan)) return rc;
  if (!info) return fail(B2DWT_EINVAL, "null info");
  std::memset(info, 0, sizeof(*info));
  info->kernel = plan->builtin >= 0 ? 1 : 0;
  info->program_id = plan->builtin;
  info->halo_left = plan->cone.left;
  info->halo_right = plan->cone.right;
  info->halo_up = plan->cone.up;
  info->halo_down = plan->cone.down;
  info->dtype = plan->dtype;
  info->flags = plan->flags;
  std::snprintf(info->key, sizeof(info->key), "%s", plan->key.c_str());
  return B2DWT_OK;
}

int b2dwt_run_components(b2dwt_plan plan, const b2dwt_planes* in, const b2dwt_planes* out, int64_t rows,
                         int64_t cols, int32_t batch, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_planes(in, "input")) return rc;
  if (int rc = check_planes(out, "output")) return rc;
  if (rows < 1 || cols < 1 || batch < 1) return fail(B2DWT_EINVAL, "empty component grid");
  if (int rc = check_dims(2 * rows, 2 * cols)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FusedLaunch r{};
  r.lin = 1;
  r.lout = 1;
  for (int c = 0; c < 4; ++c) {
    r.in_pl[c] = in->ptr[c];
    r.out_pl[c] = out->ptr[c];
  }
  for (int c = 0; c < 4; ++c) {
    r.in_ld[c] = in->ld[c];
    r.out_ld[c] = out->ld[c];
  }
  r.in_bstride = in->bstride;
  r.in_rows = static_cast<int>(rows);
  r.out_bstride = out->bstride;
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  r.row_begin = 0;
  r.row_end = static_cast<int>(rows);
  r.batch = batch;
  r.stream = s;
  if (fused_layout_ok(*plan, 1, 1)) {
    const int rc = run_fused(*plan, r);
    if (rc != B2DWT_EUNSUPPORTED) return rc;
  }
  if (int rc = try_gtile(*plan, r); rc != B2DWT_EUNSUPPORTED) return rc;
  const size_t es = esize(plan->dtype);
  return run_generic(*plan, planar_views(in, es), in->bstride, planar_views(out, es), out->bstride, rows, cols,
                     batch, s);
}

int b2dwt_forward(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t image_bstride, int64_t height,
                  int64_t width, const b2dwt_planes* out, int32_t batch, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_dims(height, width)) return rc;
  if (!image) return fail(B2DWT_EINVAL, "null image");
  if (int rc = check_planes(out, "output")) return rc;
  if (batch < 1) return fail(B2DWT_EINVAL, "batch must be >= 1");
  if (image_ld < width) return fail(B2DWT_EINVAL, "image_ld < width");
  const int64_t rows = height / 2, cols = width / 2;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FusedLaunch r{};
  r.lin = 0;
  r.lout = 1;
  r.in_img = image;
  r.in_ld[0] = image_ld;
  r.in_bstride = image_bstride;
  r.in_rows = static_cast<int>(rows);
  for (int c = 0; c < 4; ++c) {
    r.out_pl[c] = out->ptr[c];
    r.out_ld[c] = out->ld[c];
  }
  r.out_bstride = out->bstride;
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  r.row_begin = 0;
  r.row_end = static_cast<int>(rows);
  r.batch = batch;
  r.stream = s;
  if (fused_layout_ok(*plan, 0, 1)) {
    const int rc = run_fused(*plan, r);
    if (rc != B2DWT_EUNSUPPORTED) return rc;
  }
  if (int rc = try_gtile(*plan, r); rc != B2DWT_EUNSUPPORTED) return rc;
  const size_t es = esize(plan->dtype);
  return run_generic(*plan, image_views(image, image_ld, es), image_bstride, planar_views(out, es), out->bstride,
                     rows, cols, batch, s);
}

int b2dwt_inverse(b2dwt_plan plan, const b2dwt_planes* in, void* image, int64_t image_ld, int64_t image_bstride,
                  int64_t height, int64_t width, int32_t batch, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_dims(height, width)) return rc;
  if (!image) return fail(B2DWT_EINVAL, "null image");
  if (int rc = check_planes(in, "input")) return rc;
  if (batch < 1) return fail(B2DWT_EINVAL, "batch must be >= 1");
  if (image_ld < width) return fail(B2DWT_EINVAL, "image_ld < width");
  const int64_t rows = height / 2, cols = width / 2;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FusedLaunch r{};
  r.lin = 1;
  r.lout = 0;
  for (int c = 0; c < 4; ++c) {
    r.in_pl[c] = in->ptr[c];
    r.in_ld[c] = in->ld[c];
  }
  r.in_bstride = in->bstride;
  r.in_rows = static_cast<int>(rows);
  r.out_img = image;
  r.out_ld[0] = image_ld;
  r.out_bstride = image_bstride;
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  r.row_begin = 0;
  r.row_end = static_cast<int>(rows);
  r.batch = batch;
  r.stream = s;
  if (fused_layout_ok(*plan, 1, 0)) {
    const int rc = run_fused(*plan, r);
    if (rc != B2DWT_EUNSUPPORTED) return rc;
  }
  if (int rc = try_gtile(*plan, r); rc != B2DWT_EUNSUPPORTED) return rc;
  const size_t es = esize(plan->dtype);
  return run_generic(*plan, planar_views(in, es), in->bstride, image_views(image, image_ld, es), image_bstride,
                     rows, cols, batch, s);
}

int b2dwt_forward_rows(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t image_row0,
                       int64_t image_rows, int64_t global_height, int64_t width, int64_t out_row_begin,
                       int64_t out_row_end, const b2dwt_planes* out, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_dims(global_height, width)) return rc;
  if (!image) return fail(B2DWT_EINVAL, "null image");
  if (int rc = check_planes(out, "output")) return rc;
  if (image_row0 % 2 || image_rows % 2 || image_row0 < 0 || image_rows < 2 ||
      image_row0 + image_rows > global_height)
    return fail(B2DWT_EINVAL, "image band must be an even-aligned row range inside the image");
  const int64_t rows = global_height / 2, cols = width / 2;
  if (out_row_begin < 0 || out_row_end > rows || out_row_begin >= out_row_end)
    return fail(B2DWT_EINVAL, "bad output row range");
  if (!fused_layout_ok(*plan, 0, 1))
    return fail(B2DWT_EUNSUPPORTED, "row-band transform needs a fused built-in forward program");
  const int64_t in_r0 = image_row0 / 2, in_r1 = in_r0 + image_rows / 2;
  const int64_t need0 = std::max<int64_t>(0, out_row_begin - plan->cone.up);
  const int64_t need1 = std::min<int64_t>(rows, out_row_end + plan->cone.down);
  if (need0 < in_r0 || need1 > in_r1) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "band holds quad rows [%lld,%lld) but rows [%lld,%lld) are needed",
                  static_cast<long long>(in_r0), static_cast<long long>(in_r1), static_cast<long long>(need0),
                  static_cast<long long>(need1));
    return fail(B2DWT_EINVAL, buf);
  }
  FusedLaunch r{};
  r.lin = 0;
  r.lout = 1;
  r.in_img = image;
  r.in_ld[0] = image_ld;
  r.in_bstride = image_ld * image_rows;
  r.in_row0 = static_cast<int>(in_r0);
  r.in_rows = static_cast<int>(in_r1 - in_r0);
  for (int c = 0; c < 4; ++c) {
    r.out_pl[c] = out->ptr[c];
    r.out_ld[c] = out->ld[c];
  }
  r.out_bstride = out->bstride;
  r.out_row0 = static_cast<int>(out_row_begin);
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  r.row_begin = static_cast<int>(out_row_begin);
  r.row_end = static_cast<int>(out_row_end);
  r.batch = 1;
  r.stream = static_cast<cudaStream_t>(stream);
  return run_fused(*plan, r);
}

int b2dwt_inverse_rows(b2dwt_plan plan, const b2dwt_planes* in, int64_t in_row0, int64_t in_rows, void* image,
                       int64_t image_ld, int64_t global_height, int64_t width, int64_t out_row_begin,
                       int64_t out_row_end, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (int rc = check_dims(global_height, width)) return rc;
  if (!image) return fail(B2DWT_EINVAL, "null image");
  if (int rc = check_planes(in, "input")) return rc;
  const int64_t rows = global_height / 2, cols = width / 2;
  if (in_row0 < 0 || in_rows < 1 || in_row0 + in_rows > rows)
    return fail(B2DWT_EINVAL, "subband band must be a quad-row range inside the image");
  if (out_row_begin < 0 || out_row_end > rows || out_row_begin >= out_row_end)
    return fail(B2DWT_EINVAL, "bad output row range");
  if (image_ld < width) return fail(B2DWT_EINVAL, "image_ld < width");
  if (!fused_layout_ok(*plan, 1, 0))
    return fail(B2DWT_EUNSUPPORTED, "row-band inverse needs a fused built-in inverse program");
  const int64_t need0 = std::max<int64_t>(0, out_row_begin - plan->cone.up);
  const int64_t need1 = std::min<int64_t>(rows, out_row_end + plan->cone.down);
  if (need0 < in_row0 || need1 > in_row0 + in_rows) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "band holds quad rows [%lld,%lld) but rows [%lld,%lld) are needed",
                  static_cast<long long>(in_row0), static_cast<long long>(in_row0 + in_rows),
                  static_cast<long long>(need0), static_cast<long long>(need1));
    return fail(B2DWT_EINVAL, buf);
  }
  FusedLaunch r{};
  r.lin = 1;
  r.lout = 0;
  for (int c = 0; c < 4; ++c) {
    r.in_pl[c] = in->ptr[c];
    r.in_ld[c] = in->ld[c];
  }
  r.in_bstride = in->bstride;
  r.in_row0 = static_cast<int>(in_row0);
  r.in_rows = static_cast<int>(in_rows);
  r.out_img = image;
  r.out_ld[0] = image_ld;
  r.out_bstride = image_ld * 2 * (out_row_end - out_row_begin);
  r.out_row0 = static_cast<int>(out_row_begin);
  r.rows = static_cast<int>(rows);
  r.cols = static_cast<int>(cols);
  r.row_begin = static_cast<int>(out_row_begin);
  r.row_end = static_cast<int>(out_row_end);
  r.batch = 1;
  r.stream = static_cast<cudaStream_t>(stream);
  return run_fused(*plan, r);
}

int b2dwt_dwt(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width, int32_t levels,
              const b2dwt_planes* details, void* ll_out, int64_t ll_ld, void* scratch, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (levels < 1) return fail(B2DWT_EINVAL, "levels must be >= 1");
  if (!details || !ll_out || !image) return fail(B2DWT_EINVAL, "null pointer");
  if ((height % (2LL << (levels - 1))) || (width % (2LL << (levels - 1))))
    return fail(B2DWT_EINVAL, "height and width must be divisible by 2^levels");
  if (levels > 1 && !scratch) return fail(B2DWT_EINVAL, "scratch required for levels > 1");
  const size_t es = esize(plan->dtype);
  char* sc[2] = {static_cast<char*>(scratch), nullptr};
  if (scratch) sc[1] = sc[0] + static_cast<size_t>((height / 2) * (width / 2)) * es;
  const void* in = image;
  int64_t in_ld = image_ld;
  int in_sc = -1;  // scratch half holding the current input (-1: the image)
  // a level's LL (unless final) goes to the scratch half it does not read:
  // level 0's to sc[0] (the only one large enough), later ones alternate
  auto ll_half = [&](int level) { return in_sc == 0 ? 1 : in_sc == 1 ? 0 : (level == 0 ? 0 : 1); };
  for (int l = 0; l < levels; ++l) {
    const int64_t h = height >> l, w = width >> l;
    if (l + 1 < levels && fuse2_starts_at(*plan, l)) {
      // levels l and l+1 in one kernel when the plan and geometry allow it
      const int half = ll_half(l + 1);
      void* ll1 = l + 1 == levels - 1 ? ll_out : sc[half];
      const int64_t ll1_ld = l + 1 == levels - 1 ? ll_ld : w / 4;
      char name[40];
      std::snprintf(name, sizeof(name), "b2dwt dwt levels %d+%d", l, l + 1);
      NvtxRange range(name);
      const int rc = run_fused2_pair(*plan, in, in_ld, h, w, details[l], details[l + 1], ll1, ll1_ld,
                                     static_cast<cudaStream_t>(stream));
      if (rc == B2DWT_OK) {
        in = ll1;
        in_ld = ll1_ld;
        in_sc = half;
        ++l;
        continue;
      }
      if (rc != B2DWT_EUNSUPPORTED) return rc;
    }
    const b2dwt_planes& o = details[l];
    b2dwt_planes lv = o;
    lv.bstride = 0;
    if (l == levels - 1) {
      lv.ptr[0] = ll_out;
      lv.ld[0] = ll_ld;
    } else {
      in_sc = ll_half(l);
      lv.ptr[0] = sc[in_sc];
      lv.ld[0] = w / 2;
    }
    char name[32];
    std::snprintf(name, sizeof(name), "b2dwt dwt level %d", l);
    NvtxRange range(name);
    if (int rc = b2dwt_forward(plan, in, in_ld, 0, h, w, &lv, 1, stream)) return rc;
    in = lv.ptr[0];
    in_ld = lv.ld[0];
  }
  return B2DWT_OK;
}

int b2dwt_forward2(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width,
                   const b2dwt_planes* det0, const b2dwt_planes* out1, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (!image || !det0 || !out1) return fail(B2DWT_EINVAL, "null pointer");
  if (height % 4 || width % 4 || height < 4 || width < 4)
    return fail(B2DWT_EINVAL, "height and width must be divisible by 4");
  if (int rc = check_dims(height, width)) return rc;
  if (image_ld < width) return fail(B2DWT_EINVAL, "image_ld < width");
  for (int c = 1; c < 4; ++c)
    if (!det0->ptr[c] || det0->ld[c] < width / 2) return fail(B2DWT_EINVAL, "bad level-0 detail plane");
  for (int c = 0; c < 4; ++c)
    if (!out1->ptr[c] || out1->ld[c] < width / 4) return fail(B2DWT_EINVAL, "bad level-1 plane");
  const int rc = run_fused2_pair(*plan, image, image_ld, height, width, *det0, *out1, out1->ptr[0], out1->ld[0],
                                 static_cast<cudaStream_t>(stream), /*any_size=*/true);
  if (rc == B2DWT_EUNSUPPORTED) return fail(rc, "request does not fit the two-level fused kernel");
  return rc;
}

int b2dwt_idwt(b2dwt_plan plan, const void* ll, int64_t ll_ld, const b2dwt_planes* details, int32_t levels,
               void* image, int64_t image_ld, int64_t height, int64_t width, void* scratch, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (levels < 1) return fail(B2DWT_EINVAL, "levels must be >= 1");
  if (!details || !ll || !image) return fail(B2DWT_EINVAL, "null pointer");
  if ((height % (2LL << (levels - 1))) || (width % (2LL << (levels - 1))))
    return fail(B2DWT_EINVAL, "height and width must be divisible by 2^levels");
  if (levels > 1 && !scratch) return fail(B2DWT_EINVAL, "scratch required for levels > 1");
  const size_t es = esize(plan->dtype);
  char* sc[2] = {static_cast<char*>(scratch), nullptr};
  if (scratch) sc[1] = sc[0] + static_cast<size_t>((height / 2) * (width / 2)) * es;
  const void* cur = ll;
  int64_t cur_ld = ll_ld;
  for (int l = levels - 1; l >= 0; --l) {
    const int64_t h = height >> l, w = width >> l;
    void* dst;
    int64_t dst_ld;
    if (l == 0) {
      dst = image;
      dst_ld = image_ld;
    } else {
      // level l rebuilds an (H>>l) x (W>>l) LL: level 1 needs the big buffer
      dst = sc[(l + 1) & 1];
      dst_ld = w;
    }
    b2dwt_planes in = details[l];
    in.ptr[0] = const_cast<void*>(cur);
    in.ld[0] = cur_ld;
    in.bstride = 0;
    char name[32];
    std::snprintf(name, sizeof(name), "b2dwt idwt level %d", l);
    NvtxRange range(name);
    if (int rc = b2dwt_inverse(plan, &in, dst, dst_ld, 0, h, w, 1, stream)) return rc;
    cur = dst;
    cur_ld = dst_ld;
  }
  return B2DWT_OK;
}

}  // extern "C"
