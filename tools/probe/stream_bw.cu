// Microbenchmark: ceiling of the fused kernel's data movement on B200.
//   each warp walks a 64-quad (128 px) column strip of a 16384^2 f32 image,
//   reads it with TMA 3-D boxes {128 px, 2*RPS rows} through an S-stage ring,
//   and (optionally) writes 4 planes of float2 per lane per quad row.
// Variants: read-only / write-only / both, stages, rows per stage, warps per SM,
// strip order (row-front vs column-major), and a plain LDG/STG copy for reference.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_1705_08266_b200/csrc/stream_kernel.cuh"
using namespace b2dwt;

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int N = 16384, QR = N / 2;  // quad rows/cols

template <int STAGES, int RPS, bool READ, bool WRITE>
__global__ void __launch_bounds__(128) strips(const __grid_constant__ CUtensorMap map, float* out0, float* out1,
                                              float* out2, float* out3, int n_warps, int strip_w, float* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gw = blockIdx.x * 4 + warp;
  if (gw >= n_warps) return;
  constexpr int kStage = RPS * 2 * 128;  // floats
  float* ring = reinterpret_cast<float*>(smem) + warp * STAGES * kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * STAGES * kStage * 4) + warp * STAGES;
  const int n_strips = (QR + strip_w - 1) / strip_w;
  const long long total = (long long)n_strips * QR;
  long long f = total * gw / n_warps, f_end = total * (gw + 1) / n_warps;
  if (lane == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1); fence_mbar_init(); }
  __syncwarp();
  float acc = 0.f;
  int g = 0;
  while (f < f_end) {
    const int strip = (int)(f / QR);
    const int r0 = (int)(f - (long long)strip * QR);
    const long long rem = f_end - f; const int r1 = (int)(rem < QR - r0 ? r0 + rem : QR);
    f += r1 - r0;
    const int m0 = strip * strip_w - 4;
    const int nst = (r1 - r0 + RPS - 1) / RPS;
    auto issue = [&](int k) {
      if (!READ) return;
      if (lane == 0) {
        uint64_t* bar = bars + ((g + k) % STAGES);
        mbar_expect_tx(bar, kStage * 4);
        tma_load_3d(ring + ((g + k) % STAGES) * kStage, &map, bar, 2 * m0, 2 * (r0 + k * RPS), 0);
      }
    };
    for (int k = 0; k < STAGES - 1 && k < nst; ++k) issue(k);
    for (int k = 0; k < nst; ++k) {
      if (READ) {
        mbar_wait(bars + ((g + k) % STAGES), ((g + k) / STAGES) & 1);
        __syncwarp();
        if (k + STAGES - 1 < nst) { if (lane == 0) fence_proxy_async(); issue(k + STAGES - 1); }
      }
      const float* st = ring + ((g + k) % STAGES) * kStage;
      for (int j = 0; j < RPS; ++j) {
        const int r = r0 + k * RPS + j;
        if (r >= r1) break;
        float4 a = *reinterpret_cast<const float4*>(st + (2 * j) * 128 + 4 * lane);
        float4 b = *reinterpret_cast<const float4*>(st + (2 * j + 1) * 128 + 4 * lane);
        if (WRITE) {
          const int m = m0 + 2 * lane;
          if (lane >= 2 && lane < 30 && m + 2 <= QR) {
            const long long o = (long long)r * QR + m;
            *reinterpret_cast<float2*>(out0 + o) = make_float2(a.x, a.z);
            *reinterpret_cast<float2*>(out1 + o) = make_float2(a.y, a.w);
            *reinterpret_cast<float2*>(out2 + o) = make_float2(b.x, b.z);
            *reinterpret_cast<float2*>(out3 + o) = make_float2(b.y, b.w);
          }
        } else {
          acc += a.x + b.w;
        }
      }
    }
    g += nst;
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int STAGES, int RPS>
__global__ void __launch_bounds__(128) strips_cta(const __grid_constant__ CUtensorMap map, float* out0, float* out1,
                                                  float* out2, float* out3, int n_ctas, int strip_w, float* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kStage = RPS * 2 * 128;
  float* ring = reinterpret_cast<float*>(smem) + warp * STAGES * kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * STAGES * kStage * 4) + warp * STAGES;
  const int n_strips = (QR + strip_w - 1) / strip_w;
  const int n_super = (n_strips + 3) / 4;
  const long long total = (long long)n_super * QR;
  long long f = total * blockIdx.x / n_ctas, f_end = total * (blockIdx.x + 1) / n_ctas;
  if (lane == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1); fence_mbar_init(); }
  __syncwarp();
  int g = 0;
  while (f < f_end) {
    const int sup = (int)(f / QR);
    const int r0 = (int)(f - (long long)sup * QR);
    const long long rem = f_end - f;
    const int r1 = (int)(rem < QR - r0 ? r0 + rem : QR);
    f += r1 - r0;
    const int strip = sup * 4 + warp;
    if (strip >= n_strips) continue;
    const int m0 = strip * strip_w - 4;
    const int nst = (r1 - r0 + RPS - 1) / RPS;
    auto issue = [&](int k) {
      if (lane == 0) {
        uint64_t* bar = bars + ((g + k) % STAGES);
        mbar_expect_tx(bar, kStage * 4);
        tma_load_3d(ring + ((g + k) % STAGES) * kStage, &map, bar, 2 * m0, 2 * (r0 + k * RPS), 0);
      }
    };
    for (int k = 0; k < STAGES - 1 && k < nst; ++k) issue(k);
    for (int k = 0; k < nst; ++k) {
      mbar_wait(bars + ((g + k) % STAGES), ((g + k) / STAGES) & 1);
      __syncwarp();
      if (k + STAGES - 1 < nst) { if (lane == 0) fence_proxy_async(); issue(k + STAGES - 1); }
      const float* st = ring + ((g + k) % STAGES) * kStage;
      for (int j = 0; j < RPS; ++j) {
        const int r = r0 + k * RPS + j;
        if (r >= r1) break;
        float4 a = *reinterpret_cast<const float4*>(st + (2 * j) * 128 + 4 * lane);
        float4 b = *reinterpret_cast<const float4*>(st + (2 * j + 1) * 128 + 4 * lane);
        const int m = m0 + 2 * lane;
        if (lane >= 2 && lane < 30 && m + 2 <= QR) {
          const long long o = (long long)r * QR + m;
          *reinterpret_cast<float2*>(out0 + o) = make_float2(a.x, a.z);
          *reinterpret_cast<float2*>(out1 + o) = make_float2(a.y, a.w);
          *reinterpret_cast<float2*>(out2 + o) = make_float2(b.x, b.z);
          *reinterpret_cast<float2*>(out3 + o) = make_float2(b.y, b.w);
        }
      }
    }
    g += nst;
  }
}

__device__ __forceinline__ void tma_store_3d_(const CUtensorMap* map, const void* smem, int x, int y, int z) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(s), "r"(x), "r"(y), "r"(z) : "memory");
}
// CTA-adjacent strips, TMA loads per warp, outputs staged in smem per CTA and written with
// TMA tensor stores of {224 quads, RPS rows} per plane (double-buffered).
template <int STAGES, int RPS>
__global__ void __launch_bounds__(128) strips_cta_tmastore(const __grid_constant__ CUtensorMap map,
    const __grid_constant__ CUtensorMap o0, const __grid_constant__ CUtensorMap o1,
    const __grid_constant__ CUtensorMap o2, const __grid_constant__ CUtensorMap o3, int n_ctas, int strip_w) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kStage = RPS * 2 * 128;
  float* ring = reinterpret_cast<float*>(smem) + warp * STAGES * kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * STAGES * kStage * 4) + warp * STAGES;
  constexpr int TW = 4 * 56;
  float* outbuf = reinterpret_cast<float*>(smem + 4 * STAGES * kStage * 4 + 128);  // 2 x 4 planes x RPS x TW
  const int n_strips = (QR + strip_w - 1) / strip_w;
  const int n_super = (n_strips + 3) / 4;
  const long long total = (long long)n_super * QR;
  long long f = total * blockIdx.x / n_ctas, f_end = total * (blockIdx.x + 1) / n_ctas;
  if (lane == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1); fence_mbar_init(); }
  __syncwarp();
  int g = 0, ob = 0;
  while (f < f_end) {
    const int sup = (int)(f / QR);
    const int r0 = (int)(f - (long long)sup * QR);
    const long long rem = f_end - f;
    const int r1 = (int)(rem < QR - r0 ? r0 + rem : QR);
    f += r1 - r0;
    const int strip = sup * 4 + warp;
    const int m0 = strip * strip_w - 4;
    const int nst = (r1 - r0 + RPS - 1) / RPS;
    auto issue = [&](int k) {
      if (lane == 0) {
        uint64_t* bar = bars + ((g + k) % STAGES);
        mbar_expect_tx(bar, kStage * 4);
        tma_load_3d(ring + ((g + k) % STAGES) * kStage, &map, bar, 2 * m0, 2 * (r0 + k * RPS), 0);
      }
    };
    for (int k = 0; k < STAGES - 1 && k < nst; ++k) issue(k);
    for (int k = 0; k < nst; ++k) {
      mbar_wait(bars + ((g + k) % STAGES), ((g + k) / STAGES) & 1);
      __syncwarp();
      if (k + STAGES - 1 < nst) { if (lane == 0) fence_proxy_async(); issue(k + STAGES - 1); }
      const float* st = ring + ((g + k) % STAGES) * kStage;
      float* o = outbuf + ob * (4 * RPS * TW);
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
      for (int j = 0; j < RPS; ++j) {
        float4 a = *reinterpret_cast<const float4*>(st + (2 * j) * 128 + 4 * lane);
        float4 b = *reinterpret_cast<const float4*>(st + (2 * j + 1) * 128 + 4 * lane);
        if (lane >= 2 && lane < 30) {
          const int x = warp * 56 + 2 * (lane - 2);
          *reinterpret_cast<float2*>(o + (0 * RPS + j) * TW + x) = make_float2(a.x, a.z);
          *reinterpret_cast<float2*>(o + (1 * RPS + j) * TW + x) = make_float2(a.y, a.w);
          *reinterpret_cast<float2*>(o + (2 * RPS + j) * TW + x) = make_float2(b.x, b.z);
          *reinterpret_cast<float2*>(o + (3 * RPS + j) * TW + x) = make_float2(b.y, b.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const int y = r0 + k * RPS, x = sup * TW;
        tma_store_3d_(&o0, o + 0 * RPS * TW, x, y, 0);
        tma_store_3d_(&o1, o + 1 * RPS * TW, x, y, 0);
        tma_store_3d_(&o2, o + 2 * RPS * TW, x, y, 0);
        tma_store_3d_(&o3, o + 3 * RPS * TW, x, y, 0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ob ^= 1;
    }
    g += nst;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void copy_kernel(const float4* in, float4* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

template <int S, int R, bool RD, bool WR>
float run(const CUtensorMap& map, float** outs, float* sink, int warps_per_sm, int strip_w) {
  auto k = strips<S, R, RD, WR>;
  size_t smem = 4 * S * R * 2 * 128 * 4 + 4 * S * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n_warps = 148 * warps_per_sm;
  int grid = (n_warps + 3) / 4;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) k<<<grid, 128, smem>>>(map, outs[0], outs[1], outs[2], outs[3], n_warps, strip_w, sink);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) k<<<grid, 128, smem>>>(map, outs[0], outs[1], outs[2], outs[3], n_warps, strip_w, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms / 10;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  float *img, *outs[4], *sink;
  size_t bytes = (size_t)N * N * 4;
  cudaMalloc(&img, bytes); cudaMemset(img, 0, bytes);
  for (int c = 0; c < 4; ++c) cudaMalloc(&outs[c], bytes / 4);
  cudaMalloc(&sink, 16);
  const double alg = 8.0 * N * N;  // read + write bytes of the transform
  for (int rps : {4, 8}) {
    if (getenv("ONLY_TMASTORE")) break;
    CUtensorMap map; memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {N, N, 1}; cuuint64_t str[2] = {N * 4ull, (cuuint64_t)N * N * 4};
    cuuint32_t box[3] = {128, (cuuint32_t)(2 * rps), 1}; cuuint32_t es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int wps : {8, 12, 16}) {
      float t;
      if (rps == 4) {
        t = run<4, 4, true, false>(map, outs, sink, wps, 56); printf("rps=%d wps=%2d read-only   %.3f ms  (%.0f GB/s of reads)\n", rps, wps, t, 4.0*N*N*64/56/t/1e6);
        t = run<4, 4, false, true>(map, outs, sink, wps, 56); printf("rps=%d wps=%2d write-only  %.3f ms  (%.0f GB/s of writes)\n", rps, wps, t, 4.0*N*N/t/1e6);
        t = run<4, 4, true, true>(map, outs, sink, wps, 56);  printf("rps=%d wps=%2d read+write  %.3f ms  (%.0f GB/s alg)\n", rps, wps, t, alg/t/1e6);
      } else {
        if (wps > 12) continue;
        t = run<2, 8, true, false>(map, outs, sink, wps, 56); printf("rps=%d wps=%2d read-only   %.3f ms\n", rps, wps, t);
        t = run<2, 8, true, true>(map, outs, sink, wps, 56);  printf("rps=%d wps=%2d read+write  %.3f ms  (%.0f GB/s alg)\n", rps, wps, t, alg/t/1e6);
      }
    }
  }
  {
    CUtensorMap map; memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {N, N, 1}; cuuint64_t str[2] = {N * 4ull, (cuuint64_t)N * N * 4};
    cuuint32_t box[3] = {128, 8, 1}; cuuint32_t es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int cps : {2, 3}) {
      auto k = strips_cta<4, 4>;
      size_t smem = 4 * 4 * 4 * 2 * 128 * 4 + 4 * 4 * 8;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int n = 148 * cps;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int it = 0; it < 3; ++it) k<<<n, 128, smem>>>(map, outs[0], outs[1], outs[2], outs[3], n, 56, sink);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) k<<<n, 128, smem>>>(map, outs[0], outs[1], outs[2], outs[3], n, 56, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      printf("CTA-adjacent read+write ctas/sm=%d  %.3f ms  (%.0f GB/s alg)\n", cps, ms, alg / ms / 1e6);
    }
  }
  {
    CUtensorMap map; memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {N, N, 1}; cuuint64_t str[2] = {N * 4ull, (cuuint64_t)N * N * 4};
    cuuint32_t box[3] = {128, 8, 1}; cuuint32_t es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap om[4];
    for (int c = 0; c < 4; ++c) {
      memset(&om[c], 0, sizeof(CUtensorMap));
      cuuint64_t d2[3] = {QR, QR, 1}; cuuint64_t s2[2] = {QR * 4ull, (cuuint64_t)QR * QR * 4};
      cuuint32_t b2[3] = {224, 4, 1};
      int rc = (int)enc(&om[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, outs[c], d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("encode out map %d rc=%d\n", c, rc);
    }
    for (int cps : {2, 3}) {
      auto k = strips_cta_tmastore<3, 4>;
      size_t smem = 4 * 3 * 4 * 2 * 128 * 4 + 4 * 3 * 8 + 128 + 2 * 4 * 4 * 224 * 4;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int n = 148 * cps;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int it = 0; it < 3; ++it) k<<<n, 128, smem>>>(map, om[0], om[1], om[2], om[3], n, 56);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) k<<<n, 128, smem>>>(map, om[0], om[1], om[2], om[3], n, 56);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      cudaError_t e = cudaGetLastError();
      printf("CTA-adjacent read + TMA-store ctas/sm=%d  %.3f ms  (%.0f GB/s alg) %s\n", cps, ms, alg / ms / 1e6, e ? cudaGetErrorString(e) : "");
    }
  }
  // plain copy
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float* dst; cudaMalloc(&dst, bytes);
  for (int it = 0; it < 3; ++it) copy_kernel<<<148 * 8, 256>>>((const float4*)img, (float4*)dst, bytes / 16);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) copy_kernel<<<148 * 8, 256>>>((const float4*)img, (float4*)dst, bytes / 16);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("plain float4 copy 1 GiB: %.3f ms (%.0f GB/s)\n", ms / 10, 2.0 * bytes / (ms / 10) / 1e6);
  return 0;
}
