// lift1d.cu -- batched 1-D lifting on the GPU.
//
// The reference's 1-D executor (liftfuse/schemes.py:806-856, apply_plan_1d /
// invert_plan_1d) lifts one signal at a time in Python: split into even/odd
// samples, then for every (P, U) pair  odd[i] += sum_k p_k even[ext(i-k)]  and
// even[i] += sum_k u_k odd[ext(i-k)]  (terms in ascending k, each product and
// sum rounded separately), then scale (lo, hi).  The inverse divides by the
// scale and runs the pairs backwards with negated polynomials.
//
// Here a signal batch [B, N] is lifted in place in the low/high output planes:
// one split (or merge) launch, one launch per lifting step, one scale launch.
// A step reads only the OTHER plane, so every thread updates its sample in
// place without a race, exactly like the reference's sequential loop.  The
// work is a handful of HBM passes over small data; it needs no tiling.
// Strict arithmetic (__dmul_rn / __dadd_rn, division for the inverse scale)
// makes the f64 path bit-identical to the reference's Python floats.
#include <cuda_runtime.h>

#include <string>

#include "../../include/b2dwt.h"

namespace b2dwt {
int set_last_error(int code, const char* msg);  // b2dwt_host.cu
}

namespace {

constexpr int kMaxTerms = 16;

template <class T>
struct Ar1;
template <>
struct Ar1<float> {
  static __device__ __forceinline__ float mac(float a, float c, float x) { return __fadd_rn(a, __fmul_rn(c, x)); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <>
struct Ar1<double> {
  static __device__ __forceinline__ double mac(double a, double c, double x) {
    return __dadd_rn(a, __dmul_rn(c, x));
  }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

// Whole-sample symmetric extension of pixel index i over n samples (engine.py:55-71).
__device__ __forceinline__ int64_t extend1(int64_t i, int64_t n) {
  if (n == 1) return 0;
  const int64_t period = 2 * n - 2;
  int64_t r = i % period;
  if (r < 0) r += period;
  return r >= n ? period - r : r;
}

struct Step {
  int count;
  int shift[kMaxTerms];
  double coef[kMaxTerms];
};

template <class T>
__global__ void split_kernel(const T* __restrict__ in, int64_t in_ld, T* lo, T* hi, int64_t out_ld, int64_t half,
                             int batch) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= half || b >= batch) return;
  lo[b * out_ld + i] = in[b * in_ld + 2 * i];
  hi[b * out_ld + i] = in[b * in_ld + 2 * i + 1];
}

template <class T>
__global__ void merge_kernel(const T* lo, const T* hi, int64_t in_ld, T* __restrict__ out, int64_t out_ld, int64_t half,
                             int batch) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= half || b >= batch) return;
  out[b * out_ld + 2 * i] = lo[b * in_ld + i];
  out[b * out_ld + 2 * i + 1] = hi[b * in_ld + i];
}

// target[i] += sum_k c_k * source[ext(i - k)]; source parity sp (0 even, 1 odd)
template <class T>
__global__ void step_kernel(T* target, const T* source, int64_t ld, int64_t half, int64_t size, int sp, int batch,
                            const Step st) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= half || b >= batch) return;
  const T* src = source + b * ld;
  T acc = target[b * ld + i];
  for (int t = 0; t < st.count; ++t) {
    const int64_t j = i - st.shift[t];
    // component index -> pixel 2j + sp -> extend -> component index
    const int64_t k = (extend1(2 * j + sp, size) - sp) / 2;
    acc = Ar1<T>::mac(acc, static_cast<T>(st.coef[t]), src[k]);
  }
  target[b * ld + i] = acc;
}

template <class T>
__global__ void scale_kernel(T* lo, T* hi, int64_t ld, int64_t half, int batch, double s_lo, double s_hi, int divide) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= half || b >= batch) return;
  T* l = lo + b * ld + i;
  T* h = hi + b * ld + i;
  if (divide) {
    *l = Ar1<T>::div(*l, static_cast<T>(s_lo));
    *h = Ar1<T>::div(*h, static_cast<T>(s_hi));
  } else {
    *l = Ar1<T>::mul(static_cast<T>(s_lo), *l);
    *h = Ar1<T>::mul(static_cast<T>(s_hi), *h);
  }
}

int fail(int code, const char* msg) { return b2dwt::set_last_error(code, msg); }

template <class T>
int run(int inverse, int32_t n_steps, const int32_t* target, const int32_t* count, const int32_t* shifts,
        const double* coefs, const double* scale, const void* in, int64_t in_ld, void* lo_, void* hi_,
        int64_t out_ld, void* out, int64_t length, int32_t batch, cudaStream_t s) {
  const int64_t half = length / 2;
  T* lo = static_cast<T*>(lo_);
  T* hi = static_cast<T*>(hi_);
  const dim3 block(256);
  const dim3 grid(static_cast<unsigned>((half + 255) / 256), static_cast<unsigned>(batch));
  if (!inverse) {
    split_kernel<T><<<grid, block, 0, s>>>(static_cast<const T*>(in), in_ld, lo, hi, out_ld, half, batch);
  } else if (scale) {
    scale_kernel<T><<<grid, block, 0, s>>>(lo, hi, out_ld, half, batch, scale[0], scale[1], 1);
  }
  int off = 0;
  for (int st = 0; st < n_steps; ++st) {
    Step p{};
    p.count = count[st];
    for (int t = 0; t < p.count; ++t) {
      p.shift[t] = shifts[off + t];
      p.coef[t] = coefs[off + t];
    }
    off += p.count;
    // target 1 = odd/high (reads even), 0 = even/low (reads odd)
    if (target[st] == 1)
      step_kernel<T><<<grid, block, 0, s>>>(hi, lo, out_ld, half, length, 0, batch, p);
    else
      step_kernel<T><<<grid, block, 0, s>>>(lo, hi, out_ld, half, length, 1, batch, p);
  }
  if (!inverse) {
    if (scale) scale_kernel<T><<<grid, block, 0, s>>>(lo, hi, out_ld, half, batch, scale[0], scale[1], 0);
  } else {
    merge_kernel<T><<<grid, block, 0, s>>>(lo, hi, out_ld, static_cast<T*>(out), in_ld, half, batch);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(B2DWT_ECUDA, (std::string("lift1d: ") + cudaGetErrorString(e)).c_str());
  return B2DWT_OK;
}

int check(int32_t dtype, int32_t n_steps, const int32_t* target, const int32_t* count, const int32_t* shifts,
          const double* coefs, int64_t length, int32_t batch) {
  if (dtype != B2DWT_F32 && dtype != B2DWT_F64) return fail(B2DWT_EINVAL, "dtype must be B2DWT_F32 or B2DWT_F64");
  if (length < 2 || length % 2) return fail(B2DWT_EINVAL, "signal length must be even");
  if (batch < 1 || batch > 65535) return fail(B2DWT_EINVAL, "batch must be in [1, 65535]");
  if (n_steps < 0 || (n_steps > 0 && (!target || !count || !shifts || !coefs)))
    return fail(B2DWT_EINVAL, "null lifting step arrays");
  for (int s = 0; s < n_steps; ++s) {
    if (count[s] < 0 || count[s] > kMaxTerms) return fail(B2DWT_EUNSUPPORTED, "too many terms in one lifting step");
    if (target[s] != 0 && target[s] != 1) return fail(B2DWT_EINVAL, "step target must be 0 (even) or 1 (odd)");
  }
  int32_t dev = 0;
  if (cudaGetDeviceCount(&dev) != cudaSuccess || dev == 0) {
    (void)cudaGetLastError();
    return fail(B2DWT_ECUDA, "no CUDA device");
  }
  return B2DWT_OK;
}

}  // namespace

extern "C" {

int b2dwt_lift1d(int32_t dtype, int32_t n_steps, const int32_t* step_target, const int32_t* step_count,
                 const int32_t* shifts, const double* coefs, const double* scale, const void* signal,
                 int64_t signal_ld, void* low, void* high, int64_t out_ld, int64_t length, int32_t batch,
                 void* stream) {
  if (int rc = check(dtype, n_steps, step_target, step_count, shifts, coefs, length, batch)) return rc;
  if (!signal || !low || !high) return fail(B2DWT_EINVAL, "null pointer");
  if (signal_ld < length || out_ld < length / 2) return fail(B2DWT_EINVAL, "row pitch smaller than the signal");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dtype == B2DWT_F32 ? run<float>(0, n_steps, step_target, step_count, shifts, coefs, scale, signal, signal_ld,
                                         low, high, out_ld, nullptr, length, batch, s)
                            : run<double>(0, n_steps, step_target, step_count, shifts, coefs, scale, signal,
                                          signal_ld, low, high, out_ld, nullptr, length, batch, s);
}

int b2dwt_unlift1d(int32_t dtype, int32_t n_steps, const int32_t* step_target, const int32_t* step_count,
                   const int32_t* shifts, const double* coefs, const double* scale, void* low, void* high,
                   int64_t band_ld, void* signal, int64_t signal_ld, int64_t length, int32_t batch, void* stream) {
  if (int rc = check(dtype, n_steps, step_target, step_count, shifts, coefs, length, batch)) return rc;
  if (!signal || !low || !high) return fail(B2DWT_EINVAL, "null pointer");
  if (signal_ld < length || band_ld < length / 2) return fail(B2DWT_EINVAL, "row pitch smaller than the signal");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dtype == B2DWT_F32 ? run<float>(1, n_steps, step_target, step_count, shifts, coefs, scale, nullptr,
                                         signal_ld, low, high, band_ld, signal, length, batch, s)
                            : run<double>(1, n_steps, step_target, step_count, shifts, coefs, scale, nullptr,
                                          signal_ld, low, high, band_ld, signal, length, batch, s);
}

}  // extern "C"
