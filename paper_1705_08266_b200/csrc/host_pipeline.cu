// host_pipeline.cu -- b2dwt_dwt_host: the multi-level forward pyramid of a
// HOST image into HOST subbands, with the PCIe copies overlapped against each
// other and against the kernels.
//
// The reference's public call (liftfuse forward(), engine.py:481-487) takes
// and returns host arrays.  Done naively on a GPU that is upload -> pyramid ->
// download, three serial phases, and for a 16384^2 f32 image the two copies
// (1 GiB each way) are ~98% of the time.  Host-to-device and device-to-host
// copies use different copy engines and PCIe directions, so they can run at
// the same time if the work is cut into row bands:
//
//   s_in  : H2D of image row chunk 0, 1, ..., K-1 (one event per chunk)
//   s_comp: level-l band k (b2dwt_forward_rows) as soon as its input rows plus
//           the program's cone exist -- H2D chunks for level 0, bands of
//           level l-1 for level l (a wavefront down the pyramid)
//   s_out : D2H of each finished band's HL/LH/HH rows (and the final LL)
//
// so the download of level 0 runs under the upload, and only the last band's
// work is exposed.  Every level keeps its own LL buffer in the workspace (all
// levels are in flight at once, so the ping-pong of b2dwt_dwt cannot be used).
// Results are bit-identical to b2dwt_dwt: row bands reproduce the whole-image
// transform exactly (b2dwt_forward_rows).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/b2dwt.h"
#include "launch.h"

namespace b2dwt {
int set_last_error(int code, const char* msg);  // b2dwt_host.cu: b2dwt_last_error() text
}

namespace {

constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  size_t image = 0;               // device copy of the input image
  std::vector<size_t> ll;         // LL output of level l (input of level l+1; last = final LL)
  std::vector<size_t> det;        // HL/LH/HH of level l, three planes back to back
  size_t total = 0;
};

Layout layout_of(int64_t h, int64_t w, int levels, size_t es) {
  Layout L;
  size_t off = 0;
  L.image = off;
  off = align_up(off + static_cast<size_t>(h * w) * es);
  for (int l = 0; l < levels; ++l) {
    const size_t q = static_cast<size_t>((h >> (l + 1)) * (w >> (l + 1))) * es;
    L.ll.push_back(off);
    off = align_up(off + q);
    L.det.push_back(off);
    off = align_up(off + 3 * align_up(q));
  }
  L.total = off;
  return L;
}

struct Resources {
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> events;
  bool timing = false;  // B2DWT_PIPE_TRACE: timed events, timeline printed after the call
  ~Resources() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);  // released once the GPU is past them
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
  }
  cudaError_t event(cudaEvent_t* e) {
    const cudaError_t r = cudaEventCreateWithFlags(e, timing ? cudaEventDefault : cudaEventDisableTiming);
    if (r == cudaSuccess) events.push_back(*e);
    return r;
  }
};

int pipe_fail(int code, const std::string& msg) { return b2dwt::set_last_error(code, msg.c_str()); }

}  // namespace

extern "C" {

int64_t b2dwt_dwt_host_workspace(b2dwt_plan plan, int64_t height, int64_t width, int32_t levels) {
  b2dwt_plan_info info;
  if (b2dwt_plan_get_info(plan, &info) != B2DWT_OK || levels < 1 || height < 2 || width < 2) return -1;
  return static_cast<int64_t>(layout_of(height, width, levels, info.dtype == B2DWT_F32 ? 4 : 8).total);
}

int b2dwt_dwt_host(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width,
                   int32_t levels, const b2dwt_planes* details, void* ll_out, int64_t ll_ld, void* workspace,
                   int64_t workspace_bytes, int32_t bands, void* stream) {
  b2dwt_plan_info info;
  if (int rc = b2dwt_plan_get_info(plan, &info)) return rc;
  if (levels < 1) return pipe_fail(B2DWT_EINVAL, "levels must be >= 1");
  if (!image || !details || !ll_out || !workspace) return pipe_fail(B2DWT_EINVAL, "null pointer");
  if (height < 2 || width < 2 || (height % (2LL << (levels - 1))) || (width % (2LL << (levels - 1))))
    return pipe_fail(B2DWT_EINVAL, "height and width must be divisible by 2^levels");
  if (image_ld < width || ll_ld < (width >> levels)) return pipe_fail(B2DWT_EINVAL, "row pitch smaller than width");
  if (info.kernel != 1 || std::strstr(info.key, "/fwd") == nullptr)
    return pipe_fail(B2DWT_EUNSUPPORTED, "host pipeline needs a fused built-in forward program");
  const size_t es = info.dtype == B2DWT_F32 ? 4 : 8;
  const Layout L = layout_of(height, width, levels, es);
  if (workspace_bytes < static_cast<int64_t>(L.total)) return pipe_fail(B2DWT_EINVAL, "workspace too small");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return pipe_fail(B2DWT_EINVAL, "workspace must be 256-B aligned");
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s_comp = static_cast<cudaStream_t>(stream);
  // K row chunks for the upload and level 0; level l uses K >> l bands (at
  // least one, never thinner than the cone) so the small levels are not cut
  // into copies too small to run at PCIe speed
  const int64_t cone = std::max<int64_t>(1, std::max(info.halo_up, info.halo_down));
  const int K0 = std::max(1, bands > 0 ? bands : 16);
  // Upload chunks: K0 equal chunks plus a ramp of `ramp` chunks at each end
  // whose sizes halve towards the image edges (1/2, 1/4, ... of a middle
  // chunk), so the pipeline fills (first upload, nothing to download yet) and
  // drains (last download, nothing left to upload) in a fraction of a chunk's
  // copy time.  B2DWT_PIPE_RAMP overrides (0 = equal chunks).
  static const int ramp_env = [] {
    const char* v = std::getenv("B2DWT_PIPE_RAMP");
    return v ? std::atoi(v) : 0;  // measured: no gain on C3 (the pipeline sits at the PCIe floor)
  }();
  const int64_t R0 = height / 2;
  int ramp = std::max(0, std::min(ramp_env, K0 / 4));
  std::vector<int64_t> qb;  // chunk boundaries in quad rows of level 0
  for (;; --ramp) {
    std::vector<double> wts;
    for (int r = ramp; r >= 1; --r) wts.push_back(std::ldexp(1.0, -r));
    for (int c = 0; c < K0; ++c) wts.push_back(1.0);
    for (int r = 1; r <= ramp; ++r) wts.push_back(std::ldexp(1.0, -r));
    double tot = 0;
    for (double x : wts) tot += x;
    qb.assign(1, 0);
    double acc = 0;
    for (double x : wts) {
      acc += x;
      qb.push_back(std::min<int64_t>(R0, static_cast<int64_t>(std::llround(R0 * acc / tot))));
    }
    qb.back() = R0;
    // every ramp chunk must still hold more rows than the cone (small images: no ramp)
    bool ok = true;
    for (size_t c = 1; c < qb.size() && ok; ++c) ok = qb[c] - qb[c - 1] > 2 * cone;
    if (ok || ramp == 0) break;
  }
  const int K = static_cast<int>(qb.size()) - 1;
  std::vector<int> KL(levels);
  for (int l = 0; l < levels; ++l) {
    const int64_t R = height >> (l + 1);
    KL[l] = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::max(1, K >> l), R / cone)));
  }

  Resources res;
  res.timing = std::getenv("B2DWT_PIPE_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> trace;  // (label, event) for the timeline
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&res.s_in, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&res.s_out, cudaStreamNonBlocking)) != cudaSuccess)
    return pipe_fail(B2DWT_ECUDA, std::string("stream create: ") + cudaGetErrorString(e));
  cudaEvent_t ev_start;
  if ((e = res.event(&ev_start)) != cudaSuccess || (e = cudaEventRecord(ev_start, s_comp)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(res.s_in, ev_start, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(res.s_out, ev_start, 0)) != cudaSuccess)
    return pipe_fail(B2DWT_ECUDA, std::string("event: ") + cudaGetErrorString(e));

  // 1. upload in K row chunks (even pixel rows), all enqueued up front so every
  //    event exists before a compute band waits on it
  char* dimg = ws + L.image;
  std::vector<cudaEvent_t> ev_in(K);
  std::vector<int64_t> chunk_end(K);  // pixel rows uploaded after chunk c
  for (int c = 0; c < K; ++c) {
    const int64_t p0 = 2 * qb[c], p1 = 2 * qb[c + 1];
    chunk_end[c] = p1;
    if (p1 > p0) {
      e = cudaMemcpy2DAsync(dimg + static_cast<size_t>(p0 * width) * es, width * es,
                            static_cast<const char*>(image) + static_cast<size_t>(p0 * image_ld) * es, image_ld * es,
                            width * es, p1 - p0, cudaMemcpyHostToDevice, res.s_in);
      if (e != cudaSuccess) return pipe_fail(B2DWT_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
    }
    if ((e = res.event(&ev_in[c])) != cudaSuccess || (e = cudaEventRecord(ev_in[c], res.s_in)) != cudaSuccess)
      return pipe_fail(B2DWT_ECUDA, std::string("event: ") + cudaGetErrorString(e));
    if (res.timing) trace.emplace_back("in" + std::to_string(c), ev_in[c]);
  }

  // 2. wavefront of bands; 3. downloads behind each band
  std::vector<std::vector<cudaEvent_t>> ev_band(levels);
  for (int l = 0; l < levels; ++l) ev_band[l].resize(KL[l]);
  // Band boundaries: each band ends `halo_down` quad rows short of what its
  // producer (H2D chunk / band of the level above) completes, so a band needs
  // exactly one producer and runs the moment that producer lands.  Level l's
  // input pixel rows are level l-1's output quad rows.
  std::vector<std::vector<int64_t>> ends(levels);  // exclusive quad-row ends
  std::vector<std::vector<int>> deps(levels);      // producer index of each band
  for (int l = 0; l < levels; ++l) {
    const int64_t R = height >> (l + 1);
    const int nprod = l == 0 ? K : KL[l - 1];
    int64_t prev = 0;
    for (int k = 0; k < KL[l]; ++k) {
      const int j = static_cast<int>((static_cast<int64_t>(k) + 1) * nprod / KL[l]) - 1;
      const int64_t pend = l == 0 ? chunk_end[j] : ends[l - 1][j];  // pixel rows of level-l input
      int64_t end = k == KL[l] - 1 ? R : std::min<int64_t>(R, pend / 2 - info.halo_down);
      end = std::max(end, prev);
      ends[l].push_back(end);
      deps[l].push_back(j);
      prev = end;
    }
  }
  // emission order = execution order on the compute stream: after each
  // level-0 band, every band of a coarser level whose producer is enqueued
  auto emit = [&](int l, int k) -> int {
    cudaStream_t s_o = res.s_out;
    char name[40];
    std::snprintf(name, sizeof(name), "b2dwt dwt_host level %d band %d", l, k);
    b2dwt::NvtxRange range(name);
    cudaEvent_t wait = l == 0 ? ev_in[deps[l][k]] : ev_band[l - 1][deps[l][k]];
    if ((e = cudaStreamWaitEvent(s_comp, wait, 0)) != cudaSuccess)
      return pipe_fail(B2DWT_ECUDA, std::string("wait: ") + cudaGetErrorString(e));
    const int64_t h = height >> l, w = width >> l, R = h / 2, C = w / 2;
    const int64_t b0 = k == 0 ? 0 : ends[l][k - 1], b1 = ends[l][k];
    if (b1 > b0) {
      const char* in = l == 0 ? dimg : ws + L.ll[l - 1];
      char* det = ws + L.det[l];
      const size_t plane = align_up(static_cast<size_t>(R * C) * es);
      b2dwt_planes out;
      out.ptr[0] = ws + L.ll[l] + static_cast<size_t>(b0 * C) * es;
      for (int c = 1; c < 4; ++c) out.ptr[c] = det + (c - 1) * plane + static_cast<size_t>(b0 * C) * es;
      for (int c = 0; c < 4; ++c) out.ld[c] = C;
      out.bstride = 0;
      if (int rc = b2dwt_forward_rows(plan, in, w, 0, h, h, w, b0, b1, &out, s_comp)) return rc;
    }
    if ((e = res.event(&ev_band[l][k])) != cudaSuccess || (e = cudaEventRecord(ev_band[l][k], s_comp)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s_o, ev_band[l][k], 0)) != cudaSuccess)
      return pipe_fail(B2DWT_ECUDA, std::string("event: ") + cudaGetErrorString(e));
    if (b1 > b0) {
      const size_t plane = align_up(static_cast<size_t>(R * C) * es);
      for (int c = 1; c < 4; ++c) {
        const char* src = ws + L.det[l] + (c - 1) * plane + static_cast<size_t>(b0 * C) * es;
        char* dst = static_cast<char*>(details[l].ptr[c]) + static_cast<size_t>(b0 * details[l].ld[c]) * es;
        e = cudaMemcpy2DAsync(dst, details[l].ld[c] * es, src, C * es, C * es, b1 - b0, cudaMemcpyDeviceToHost,
                              s_o);
        if (e != cudaSuccess) return pipe_fail(B2DWT_ECUDA, std::string("D2H: ") + cudaGetErrorString(e));
      }
      if (l == levels - 1) {
        const char* src = ws + L.ll[l] + static_cast<size_t>(b0 * C) * es;
        char* dst = static_cast<char*>(ll_out) + static_cast<size_t>(b0 * ll_ld) * es;
        e = cudaMemcpy2DAsync(dst, ll_ld * es, src, C * es, C * es, b1 - b0, cudaMemcpyDeviceToHost, s_o);
        if (e != cudaSuccess) return pipe_fail(B2DWT_ECUDA, std::string("D2H: ") + cudaGetErrorString(e));
      }
    }
    if (res.timing) {
      cudaEvent_t ev_o;
      if (res.event(&ev_o) == cudaSuccess && cudaEventRecord(ev_o, s_o) == cudaSuccess) {
        trace.emplace_back("c" + std::to_string(l) + "." + std::to_string(k), ev_band[l][k]);
        trace.emplace_back("o" + std::to_string(l) + "." + std::to_string(k), ev_o);
      }
    }
    return B2DWT_OK;
  };
  std::vector<int> next(levels, 0);
  for (int k0 = 0; k0 < KL[0]; ++k0) {
    if (int rc = emit(0, k0)) return rc;
    next[0] = k0 + 1;
    for (int l = 1; l < levels; ++l)
      while (next[l] < KL[l] && deps[l][next[l]] < next[l - 1]) {
        if (int rc = emit(l, next[l])) return rc;
        ++next[l];
      }
  }
  // the caller's stream sees everything complete after this point
  cudaEvent_t ev_done;
  if ((e = res.event(&ev_done)) != cudaSuccess || (e = cudaEventRecord(ev_done, res.s_out)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(s_comp, ev_done, 0)) != cudaSuccess)
    return pipe_fail(B2DWT_ECUDA, std::string("event: ") + cudaGetErrorString(e));
  if (res.timing && cudaEventSynchronize(ev_done) == cudaSuccess) {
    std::string line = "[b2dwt pipe] ms:";
    for (auto& t : trace) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev_start, t.second);
      char buf[48];
      std::snprintf(buf, sizeof(buf), " %s=%.2f", t.first.c_str(), ms);
      line += buf;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev_start, ev_done);
    std::fprintf(stderr, "%s done=%.2f\n", line.c_str(), ms);
  }
  return B2DWT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Inverse: host subbands -> host image.  The coarse levels (a quarter of the
// data) are uploaded first and inverted whole; level 0 -- three quarters of the
// input and all of the output -- runs in row bands: upload chunk k of its
// HL/LH/HH (and LL when there is one level), invert rows as soon as the chunk
// plus the cone is present, download the image rows while later chunks upload.

namespace {

struct InvLayout {
  std::vector<size_t> det;  // HL/LH/HH of level l (three planes back to back)
  std::vector<size_t> rec;  // image rebuilt by level l (l >= 1) = LL input of level l-1
  size_t ll = 0;            // coarsest LL
  size_t image = 0;
  size_t total = 0;
};

InvLayout inv_layout_of(int64_t h, int64_t w, int levels, size_t es) {
  InvLayout L;
  size_t off = 0;
  L.rec.assign(levels, 0);
  for (int l = 0; l < levels; ++l) {
    const size_t q = static_cast<size_t>((h >> (l + 1)) * (w >> (l + 1))) * es;
    L.det.push_back(off);
    off = align_up(off + 3 * align_up(q));
    if (l >= 1) {
      L.rec[l] = off;
      off = align_up(off + static_cast<size_t>((h >> l) * (w >> l)) * es);
    }
  }
  L.ll = off;
  off = align_up(off + static_cast<size_t>((h >> levels) * (w >> levels)) * es);
  L.image = off;
  off = align_up(off + static_cast<size_t>(h * w) * es);
  L.total = off;
  return L;
}

cudaError_t h2d_rows(void* dst, int64_t dld, const void* src, int64_t sld, int64_t cols, int64_t r0, int64_t r1,
                     size_t es, cudaStream_t s) {
  if (r1 <= r0) return cudaSuccess;
  return cudaMemcpy2DAsync(static_cast<char*>(dst) + static_cast<size_t>(r0 * dld) * es, dld * es,
                           static_cast<const char*>(src) + static_cast<size_t>(r0 * sld) * es, sld * es, cols * es,
                           r1 - r0, cudaMemcpyHostToDevice, s);
}

}  // namespace

extern "C" {

int64_t b2dwt_idwt_host_workspace(b2dwt_plan plan, int64_t height, int64_t width, int32_t levels) {
  b2dwt_plan_info info;
  if (b2dwt_plan_get_info(plan, &info) != B2DWT_OK || levels < 1 || height < 2 || width < 2) return -1;
  return static_cast<int64_t>(inv_layout_of(height, width, levels, info.dtype == B2DWT_F32 ? 4 : 8).total);
}

int b2dwt_idwt_host(b2dwt_plan plan, const void* ll, int64_t ll_ld, const b2dwt_planes* details, int32_t levels,
                    void* image, int64_t image_ld, int64_t height, int64_t width, void* workspace,
                    int64_t workspace_bytes, int32_t bands, void* stream) {
  b2dwt_plan_info info;
  if (int rc = b2dwt_plan_get_info(plan, &info)) return rc;
  if (levels < 1) return pipe_fail(B2DWT_EINVAL, "levels must be >= 1");
  if (!image || !details || !ll || !workspace) return pipe_fail(B2DWT_EINVAL, "null pointer");
  if (height < 2 || width < 2 || (height % (2LL << (levels - 1))) || (width % (2LL << (levels - 1))))
    return pipe_fail(B2DWT_EINVAL, "height and width must be divisible by 2^levels");
  if (image_ld < width || ll_ld < (width >> levels)) return pipe_fail(B2DWT_EINVAL, "row pitch smaller than width");
  if (info.kernel != 1 || std::strstr(info.key, "/inv") == nullptr)
    return pipe_fail(B2DWT_EUNSUPPORTED, "host pipeline needs a fused built-in inverse program");
  const size_t es = info.dtype == B2DWT_F32 ? 4 : 8;
  const InvLayout L = inv_layout_of(height, width, levels, es);
  if (workspace_bytes < static_cast<int64_t>(L.total)) return pipe_fail(B2DWT_EINVAL, "workspace too small");
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign) return pipe_fail(B2DWT_EINVAL, "workspace must be 256-B aligned");
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s_comp = static_cast<cudaStream_t>(stream);
  const int64_t R0 = height / 2, C0 = width / 2;
  const int K = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(bands > 0 ? bands : 16, R0 / std::max<int64_t>(1, std::max(info.halo_up, info.halo_down)))));

  Resources res;
  res.timing = false;
  cudaError_t e;
  auto fail_e = [&](const char* what) { return pipe_fail(B2DWT_ECUDA, std::string(what) + cudaGetErrorString(e)); };
  if ((e = cudaStreamCreateWithFlags(&res.s_in, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&res.s_out, cudaStreamNonBlocking)) != cudaSuccess)
    return fail_e("stream create: ");
  cudaEvent_t ev_start, ev_coarse;
  if ((e = res.event(&ev_start)) != cudaSuccess || (e = cudaEventRecord(ev_start, s_comp)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(res.s_in, ev_start, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(res.s_out, ev_start, 0)) != cudaSuccess)
    return fail_e("event: ");
  auto det_plane = [&](int l, int c) {  // device plane c (1..3) of level l
    const size_t q = static_cast<size_t>((height >> (l + 1)) * (width >> (l + 1))) * es;
    return ws + L.det[l] + (c - 1) * align_up(q);
  };
  // 1. coarse levels: LL and details of levels >= 1, uploaded whole
  const int64_t Rl = height >> levels, Cl = width >> levels;
  if (levels > 1 && (e = h2d_rows(ws + L.ll, Cl, ll, ll_ld, Cl, 0, Rl, es, res.s_in)) != cudaSuccess)
    return fail_e("H2D: ");
  for (int l = levels - 1; l >= 1; --l) {
    const int64_t R = height >> (l + 1), C = width >> (l + 1);
    for (int c = 1; c < 4; ++c)
      if ((e = h2d_rows(det_plane(l, c), C, details[l].ptr[c], details[l].ld[c], C, 0, R, es, res.s_in)) !=
          cudaSuccess)
        return fail_e("H2D: ");
  }
  if ((e = res.event(&ev_coarse)) != cudaSuccess || (e = cudaEventRecord(ev_coarse, res.s_in)) != cudaSuccess)
    return fail_e("event: ");
  // 2. level-0 inputs in K row chunks (LL too when there is a single level)
  char* ll0 = levels > 1 ? ws + L.rec[1] : ws + L.ll;
  std::vector<cudaEvent_t> ev_in(K);
  std::vector<int64_t> chunk_end(K);
  for (int k = 0; k < K; ++k) {
    const int64_t r0 = R0 * k / K, r1 = R0 * (k + 1) / K;
    chunk_end[k] = r1;
    if (levels == 1 && (e = h2d_rows(ll0, C0, ll, ll_ld, C0, r0, r1, es, res.s_in)) != cudaSuccess)
      return fail_e("H2D: ");
    for (int c = 1; c < 4; ++c)
      if ((e = h2d_rows(det_plane(0, c), C0, details[0].ptr[c], details[0].ld[c], C0, r0, r1, es, res.s_in)) !=
          cudaSuccess)
        return fail_e("H2D: ");
    if ((e = res.event(&ev_in[k])) != cudaSuccess || (e = cudaEventRecord(ev_in[k], res.s_in)) != cudaSuccess)
      return fail_e("event: ");
  }
  // 3. invert the coarse levels whole (LL of level l = image rebuilt by level l+1)
  if ((e = cudaStreamWaitEvent(s_comp, ev_coarse, 0)) != cudaSuccess) return fail_e("wait: ");
  for (int l = levels - 1; l >= 1; --l) {
    const int64_t h = height >> l, w = width >> l, C = w / 2;
    b2dwt_planes in;
    in.ptr[0] = l == levels - 1 ? ws + L.ll : ws + L.rec[l + 1];
    for (int c = 1; c < 4; ++c) in.ptr[c] = det_plane(l, c);
    for (int c = 0; c < 4; ++c) in.ld[c] = C;
    in.bstride = 0;
    if (int rc = b2dwt_inverse(plan, &in, ws + L.rec[l], w, 0, h, w, 1, s_comp)) return rc;
  }
  // 4. level 0 in bands that end a cone short of their chunk; 5. downloads
  char* dimg = ws + L.image;
  b2dwt_planes in0;
  in0.ptr[0] = ll0;
  for (int c = 1; c < 4; ++c) in0.ptr[c] = det_plane(0, c);
  for (int c = 0; c < 4; ++c) in0.ld[c] = C0;
  in0.bstride = 0;
  int64_t prev = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t end = k == K - 1 ? R0 : std::max(prev, std::min<int64_t>(R0, chunk_end[k] - info.halo_down));
    if ((e = cudaStreamWaitEvent(s_comp, ev_in[k], 0)) != cudaSuccess) return fail_e("wait: ");
    if (end > prev) {
      if (int rc = b2dwt_inverse_rows(plan, &in0, 0, R0, dimg + static_cast<size_t>(2 * prev * width) * es, width,
                                      height, width, prev, end, s_comp))
        return rc;
      cudaEvent_t ev_b;
      if ((e = res.event(&ev_b)) != cudaSuccess || (e = cudaEventRecord(ev_b, s_comp)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(res.s_out, ev_b, 0)) != cudaSuccess)
        return fail_e("event: ");
      e = cudaMemcpy2DAsync(static_cast<char*>(image) + static_cast<size_t>(2 * prev * image_ld) * es, image_ld * es,
                            dimg + static_cast<size_t>(2 * prev * width) * es, width * es, width * es,
                            2 * (end - prev), cudaMemcpyDeviceToHost, res.s_out);
      if (e != cudaSuccess) return fail_e("D2H: ");
    }
    prev = end;
  }
  cudaEvent_t ev_done;
  if ((e = res.event(&ev_done)) != cudaSuccess || (e = cudaEventRecord(ev_done, res.s_out)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(s_comp, ev_done, 0)) != cudaSuccess)
    return fail_e("event: ");
  return B2DWT_OK;
}

}  // extern "C"
