// Standalone probe: planar 3-D TMA loads of 4 planes into one mbarrier stage.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../../paper_1705_08266_b200/csrc/stream_kernel.cuh"
using namespace b2dwt;
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
template <int NMAP>
__global__ void probe(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                      const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3, float* out, int x0) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* s = reinterpret_cast<float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4096);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, NMAP * 64 * 2 * 4);
    tma_load_3d(s, &m0, bar, x0, 0, 0);
    if (NMAP > 1) tma_load_3d(s + 128, &m1, bar, x0, 0, 0);
    if (NMAP > 2) tma_load_3d(s + 256, &m2, bar, x0, 0, 0);
    if (NMAP > 3) tma_load_3d(s + 384, &m3, bar, x0, 0, 0);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < NMAP * 128; i += blockDim.x) out[i] = s[i];
}
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  const int W = 256, H = 64;
  float* planes[4]; float* out;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  for (int c = 0; c < 4; ++c) { cudaMalloc(&planes[c], W * H * 4); cudaMemcpy(planes[c], h.data(), W * H * 4, cudaMemcpyHostToDevice); }
  cudaMalloc(&out, 4096 * 4);
  CUtensorMap maps[4]; memset(maps, 0, sizeof(maps));
  for (int c = 0; c < 4; ++c) {
    cuuint64_t dims[3] = {W, H, 1}; cuuint64_t str[2] = {W * 4, (cuuint64_t)W * H * 4};
    cuuint32_t box[3] = {64, 2, 1}; cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, planes[c], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d -> %d\n", c, (int)r);
  }
  for (int x0 : {0, -2}) {
    probe<1><<<1, 32, 8192>>>(maps[0], maps[1], maps[2], maps[3], out, x0);
    printf("nmap=1 x0=%d: %s\n", x0, cudaGetErrorString(cudaDeviceSynchronize()));
    probe<4><<<1, 32, 8192>>>(maps[0], maps[1], maps[2], maps[3], out, x0);
    printf("nmap=4 x0=%d: %s\n", x0, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  float ho[512]; cudaMemcpy(ho, out, 512 * 4, cudaMemcpyDeviceToHost);
  printf("out[0..3]=%g %g %g %g  out[128]=%g out[64]=%g\n", ho[0], ho[1], ho[2], ho[3], ho[128], ho[64]);
  return 0;
}
