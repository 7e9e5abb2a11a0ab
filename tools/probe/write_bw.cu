// Write-path microbenchmark: 4 output planes (8192^2 f32 each) written by warps
// walking 56/120-quad column strips, one quad row per step.
//   mode 0: STG.64 per lane (current kernel)      mode 1: STG.64 .cs (streaming)
//   mode 2: STG.128 per lane, 120-quad strips      mode 3: TMA tensor store of RPS-row tiles from smem
//   mode 4: linear float4 memset (ceiling)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include "../../paper_1705_08266_b200/csrc/stream_kernel.cuh"
using namespace b2dwt;
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int QR = 8192;

__device__ __forceinline__ void st_cs_v2(float* p, float a, float b) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem, int x, int y, int z) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(s), "r"(x), "r"(y), "r"(z) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// CTA = WARPS adjacent strips at the same rows (super-strip), flat split over CTAs.
//   mode 5: each warp STG.64 its own strip   mode 6: warps stage into smem, one TMA store {WARPS*56, RPS} per plane
template <int MODE, int RPS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) writer_cta(float* o0, float* o1, float* o2, float* o3, int n_ctas,
                                                         const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                         const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int SW = 56;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_super = (QR + WARPS * SW - 1) / (WARPS * SW);
  const long long total = (long long)n_super * QR;
  long long f = total * blockIdx.x / n_ctas, f_end = total * (blockIdx.x + 1) / n_ctas;
  float* tile = reinterpret_cast<float*>(smem);  // 2 bufs x 4 planes x RPS rows x (WARPS*SW)
  constexpr int TW = WARPS * SW;
  int buf = 0;
  while (f < f_end) {
    const int ss = (int)(f / QR);
    const int r0 = (int)(f - (long long)ss * QR);
    const long long rem = f_end - f;
    const int r1 = (int)(rem < QR - r0 ? r0 + rem : QR);
    f += r1 - r0;
    const int mstrip = (ss * WARPS + warp) * SW;
    if (MODE == 6) {
      for (int r = r0; r < r1; r += RPS) {
        float* t = tile + buf * (4 * RPS * TW);
        if (threadIdx.x == 0) bulk_wait_read<1>();
        __syncthreads();
        for (int j = 0; j < RPS; ++j)
          for (int c = 0; c < 4; ++c)
            if (lane >= 2 && lane < 30)
              *reinterpret_cast<float2*>(t + (c * RPS + j) * TW + warp * SW + 2 * (lane - 2)) = make_float2((float)r + j, (float)c);
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          const int x = ss * TW;
          tma_store_3d(&m0, t + 0 * RPS * TW, x, r, 0);
          tma_store_3d(&m1, t + 1 * RPS * TW, x, r, 0);
          tma_store_3d(&m2, t + 2 * RPS * TW, x, r, 0);
          tma_store_3d(&m3, t + 3 * RPS * TW, x, r, 0);
          bulk_commit();
        }
        buf ^= 1;
      }
      continue;
    }
    for (int r = r0; r < r1; ++r) {
      const int m = mstrip - 4 + 2 * lane;
      if (lane >= 2 && lane < 30 && m + 2 <= QR) {
        const long long o = (long long)r * QR + m;
        *reinterpret_cast<float2*>(o0 + o) = make_float2((float)r, (float)lane);
        *reinterpret_cast<float2*>(o1 + o) = make_float2((float)r, (float)lane);
        *reinterpret_cast<float2*>(o2 + o) = make_float2((float)r, (float)lane);
        *reinterpret_cast<float2*>(o3 + o) = make_float2((float)r, (float)lane);
      }
    }
  }
  if (MODE == 6 && threadIdx.x == 0) bulk_wait_read<0>();
}

template <int MODE, int RPS, int WARPS>
void run_cta(float** o, const CUtensorMap* maps, int ctas_per_sm, const char* name) {
  auto k = writer_cta<MODE, RPS, WARPS>;
  size_t smem = MODE == 6 ? 2 * 4 * RPS * WARPS * 56 * 4 : 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 148 * ctas_per_sm;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<n, WARPS * 32, smem>>>(o[0], o[1], o[2], o[3], n, maps[0], maps[1], maps[2], maps[3]);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) k<<<n, WARPS * 32, smem>>>(o[0], o[1], o[2], o[3], n, maps[0], maps[1], maps[2], maps[3]);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
  cudaError_t e = cudaGetLastError();
  printf("%-40s ctas/sm=%d %.3f ms  %.0f GB/s %s\n", name, ctas_per_sm, ms, 4.0 * QR * QR * 4 / ms / 1e6, e ? cudaGetErrorString(e) : "");
}

template <int MODE, int RPS>
__global__ void __launch_bounds__(128) writer(float* o0, float* o1, float* o2, float* o3, int n_warps, int strip_w,
                                              const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                              const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, gw = blockIdx.x * 4 + warp;
  if (gw >= n_warps) return;
  const int n_strips = (QR + strip_w - 1) / strip_w;
  const long long total = (long long)n_strips * QR;
  long long f = total * gw / n_warps, f_end = total * (gw + 1) / n_warps;
  float* tile = reinterpret_cast<float*>(smem) + warp * (2 * 4 * RPS * 128);  // 2 buffers x 4 planes x RPS x 128
  int buf = 0;
  while (f < f_end) {
    const int strip = (int)(f / QR);
    const int r0 = (int)(f - (long long)strip * QR);
    const long long rem = f_end - f;
    const int r1 = (int)(rem < QR - r0 ? r0 + rem : QR);
    f += r1 - r0;
    const int mbase = strip * strip_w;
    if (MODE == 3) {
      for (int r = r0; r < r1; r += RPS) {
        float* t = tile + buf * (4 * RPS * 128);
        bulk_wait_read<1>();  // the store issued from this buffer two rounds ago has read smem
        __syncwarp();
        for (int j = 0; j < RPS; ++j)
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<float2*>(t + (c * RPS + j) * 128 + 2 * lane) = make_float2((float)r + j, (float)c);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&m0, t + 0 * RPS * 128, mbase, r, 0);
          tma_store_3d(&m1, t + 1 * RPS * 128, mbase, r, 0);
          tma_store_3d(&m2, t + 2 * RPS * 128, mbase, r, 0);
          tma_store_3d(&m3, t + 3 * RPS * 128, mbase, r, 0);
          bulk_commit();
        }
        buf ^= 1;
      }
      continue;
    }
    for (int r = r0; r < r1; ++r) {
      const float va = (float)r, vb = (float)lane;
      if (MODE == 2) {
        const int m = mbase - 4 + 4 * lane;
        if (lane >= 1 && lane < 31 && m + 4 <= QR) {
          const long long o = (long long)r * QR + m;
          *reinterpret_cast<float4*>(o0 + o) = make_float4(va, vb, va, vb);
          *reinterpret_cast<float4*>(o1 + o) = make_float4(va, vb, va, vb);
          *reinterpret_cast<float4*>(o2 + o) = make_float4(va, vb, va, vb);
          *reinterpret_cast<float4*>(o3 + o) = make_float4(va, vb, va, vb);
        }
      } else {
        const int m = mbase - 4 + 2 * lane;
        if (lane >= 2 && lane < 30 && m + 2 <= QR) {
          const long long o = (long long)r * QR + m;
          if (MODE == 0) {
            *reinterpret_cast<float2*>(o0 + o) = make_float2(va, vb);
            *reinterpret_cast<float2*>(o1 + o) = make_float2(va, vb);
            *reinterpret_cast<float2*>(o2 + o) = make_float2(va, vb);
            *reinterpret_cast<float2*>(o3 + o) = make_float2(va, vb);
          } else {
            st_cs_v2(o0 + o, va, vb); st_cs_v2(o1 + o, va, vb); st_cs_v2(o2 + o, va, vb); st_cs_v2(o3 + o, va, vb);
          }
        }
      }
    }
  }
  if (MODE == 3) bulk_wait_read<0>();
}

__global__ void memset4(float4* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

template <int MODE, int RPS>
void run(float** o, const CUtensorMap* maps, int wps, int strip_w, const char* name) {
  auto k = writer<MODE, RPS>;
  size_t smem = MODE == 3 ? 4 * 2 * 4 * RPS * 128 * 4 : 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nw = 148 * wps, grid = (nw + 3) / 4;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, 128, smem>>>(o[0], o[1], o[2], o[3], nw, strip_w, maps[0], maps[1], maps[2], maps[3]);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) k<<<grid, 128, smem>>>(o[0], o[1], o[2], o[3], nw, strip_w, maps[0], maps[1], maps[2], maps[3]);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
  cudaError_t e = cudaGetLastError();
  printf("%-34s wps=%2d %.3f ms  %.0f GB/s %s\n", name, wps, ms, 4.0 * QR * QR * 4 / ms / 1e6, e ? cudaGetErrorString(e) : "");
}

int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  float* o[4];
  for (int c = 0; c < 4; ++c) cudaMalloc(&o[c], (size_t)QR * QR * 4);
  CUtensorMap maps[4];
  for (int c = 0; c < 4; ++c) {
    memset(&maps[c], 0, sizeof(CUtensorMap));
    cuuint64_t dims[3] = {QR, QR, 1}; cuuint64_t str[2] = {QR * 4ull, (cuuint64_t)QR * QR * 4};
    cuuint32_t box[3] = {56, 4, 1}; cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, o[c], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode %d\n", (int)r);
  }
  for (int wps : {8, 12}) {
    run<0, 4>(o, maps, wps, 56, "STG.64, 56-quad strips");
    run<1, 4>(o, maps, wps, 56, "STG.64.cs, 56-quad strips");
    run<2, 4>(o, maps, wps, 120, "STG.128, 120-quad strips");
    run<3, 4>(o, maps, wps, 56, "TMA store 4x{56,4} tiles, 2 buffers");
  }
  CUtensorMap wide[2][4];
  for (int wv = 0; wv < 2; ++wv)
  for (int c = 0; c < 4; ++c) {
    memset(&wide[wv][c], 0, sizeof(CUtensorMap));
    cuuint64_t dims[3] = {QR, QR, 1}; cuuint64_t str[2] = {QR * 4ull, (cuuint64_t)QR * QR * 4};
    cuuint32_t box[3] = {(cuuint32_t)(wv == 0 ? 224 : 112), 4, 1}; cuuint32_t es[3] = {1, 1, 1};
    enc(&wide[wv][c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, o[c], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  for (int cps : {2, 3}) {
    run_cta<5, 4, 4>(o, wide[0], cps, "CTA 4 adjacent strips, STG.64");
    run_cta<6, 4, 4>(o, wide[0], cps, "CTA 4 adjacent strips, TMA {224,4}");
    run_cta<5, 4, 2>(o, wide[1], cps * 2, "CTA 2 adjacent strips, STG.64");
    run_cta<6, 4, 2>(o, wide[1], cps * 2, "CTA 2 adjacent strips, TMA {112,4}");
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) memset4<<<148 * 8, 256>>>((float4*)o[0], (long long)QR * QR / 4);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) for (int c = 0; c < 4; ++c) memset4<<<148 * 8, 256>>>((float4*)o[c], (long long)QR * QR / 4);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
  printf("linear float4 writes (4 planes)    %.3f ms  %.0f GB/s\n", ms, 4.0 * QR * QR * 4 / ms / 1e6);
}
