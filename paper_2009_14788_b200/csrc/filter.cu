// Ramp-filter kernel (sm_100a): per detector row, zero-pad to P, FFT,
// multiply by the real frequency response, inverse FFT, crop and scale by
// pi / (2 n_angles) — sino_filter.cpp:98-124 (filtration always fp32,
// :106-123).
//
// One CTA filters the four rows (b = 4g..4g+3, angle a) that share one
// packed float4 sinogram cell, as two complex shared-memory FFTs: the
// response is real and even, so for z = x + i y, IFFT(FFT(z) H) = x*h + i (y*h)
// filters two real rows at once.  The forward transform is
// decimation-in-frequency (natural in, bit-reversed out), the response is
// applied in bit-reversed order, and the inverse is decimation-in-time with
// conjugate twiddles (bit-reversed in, natural out): no permutation pass.
#include <cuda_fp16.h>

#include "rk_internal.hpp"

namespace rk {

namespace {

template <class T>
__device__ __forceinline__ float ld_f32(const T* p);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld_f32<__half>(const __half* p) { return __half2float(*p); }
template <>
__device__ __forceinline__ float ld_f32<double>(const double* p) { return float(__ldg(p)); }

template <class T>
__device__ __forceinline__ T st_cast(float v);
template <>
__device__ __forceinline__ float st_cast<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half st_cast<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ double st_cast<double>(float v) { return double(v); }

constexpr int kFilterThreads = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Shared-memory slot of complex element i: an XOR swizzle inside each block of
// 16 (128 bytes) that makes every access pattern of the fused passes below
// bank-conflict free (64-bit loads, half warps).
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 3) & 15); }

__device__ __forceinline__ float2 cmul_conj(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// R consecutive radix-2 stages of an in-place FFT of 2^logn points fused in
// registers: the group of element i0 holds i0 + m 2^lh (m < 2^R), so stages
// lh+1 .. lh+R pair elements inside the group.  DIF (natural in, bit-reversed
// out, W = exp(-2 pi i/n)): u + v, (u - v) W; DIT (bit-reversed in, natural
// out): u + v W, u - v W, with conj(W) when CONJ (the unnormalised inverse).
// Each butterfly is the radix-2 one with the stage's table twiddle; a
// transform is ceil(logn / 3) shared-memory passes and barriers.  Two signals
// (z, z + stride).
template <int R, bool DIF, bool CONJ>
__device__ __forceinline__ void fft_pass(float2* z, int stride, int logn, int lh, const float2* __restrict__ tw) {
  const int gl = logn - R;  // log2(groups per signal)
  for (int t = threadIdx.x; t < (2 << gl); t += blockDim.x) {
    const int sig = t >> gl, g = t & ((1 << gl) - 1);
    const int lo = g & ((1 << lh) - 1), hi = g >> lh;
    const int i0 = lo + (hi << (lh + R));
    float2* a = z + sig * stride;
    float2 x[1 << R];
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) x[m] = a[swz(i0 + (m << lh))];
#pragma unroll
    for (int l = 0; l < R; ++l) {
      const int bit = DIF ? R - 1 - l : l;  // partner bit of m in this layer
#pragma unroll
      for (int m = 0; m < (1 << R); ++m) {
        if (m & (1 << bit)) continue;
        const int q = m | (1 << bit);
        const int k = lo + ((m & ((1 << bit) - 1)) << lh);
        const float2 w = __ldg(tw + (k << (logn - lh - 1 - bit)));
        const float2 u = x[m];
        if (DIF) {
          const float2 v = x[q];
          x[m] = make_float2(u.x + v.x, u.y + v.y);
          x[q] = cmul(make_float2(u.x - v.x, u.y - v.y), w);
        } else {
          const float2 v = CONJ ? cmul_conj(x[q], w) : cmul(x[q], w);
          x[m] = make_float2(u.x + v.x, u.y + v.y);
          x[q] = make_float2(u.x - v.x, u.y - v.y);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) a[swz(i0 + (m << lh))] = x[m];
  }
  __syncthreads();
}

// forward: natural -> bit-reversed (the short pass first, at the widest stride)
__device__ void fft_dif(float2* z, int stride, int logn, const float2* __restrict__ tw) {
  int lh = logn - logn % 3;
  if (logn % 3 == 2) fft_pass<2, true, false>(z, stride, logn, lh, tw);
  if (logn % 3 == 1) fft_pass<1, true, false>(z, stride, logn, lh, tw);
  while (lh >= 3) {
    lh -= 3;
    fft_pass<3, true, false>(z, stride, logn, lh, tw);
  }
}

// unnormalised inverse: bit-reversed -> natural
__device__ void ifft_dit(float2* z, int stride, int logn, const float2* __restrict__ tw) {
  int lh = 0;
  for (; lh + 3 <= logn; lh += 3) fft_pass<3, false, true>(z, stride, logn, lh, tw);
  if (logn - lh == 2) fft_pass<2, false, true>(z, stride, logn, lh, tw);
  if (logn - lh == 1) fft_pass<1, false, true>(z, stride, logn, lh, tw);
}

template <class TIn, class TOut, bool PACKED>
__global__ void __launch_bounds__(kFilterThreads) filter_kernel(const TIn* __restrict__ in, int64_t batch, int na,
                                                                int nd, int P, int logP,
                                                                const float* __restrict__ resp,
                                                                const float2* __restrict__ tw, float scale,
                                                                TOut* __restrict__ out, float4* __restrict__ packed) {
  extern __shared__ float2 fsm[];
  float2* za = fsm;      // rows q=0 (re) and q=1 (im), swizzled slots (swz)
  float2* zb = fsm + P;  // rows q=2 (re) and q=3 (im)
  const int a = blockIdx.x;
  const int64_t g = blockIdx.y;
  const int shift = 32 - logP;
  // ---- load (zero pad), natural order
  const TIn* rows[4];
  bool valid[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t b = g * kPack + q;
    valid[q] = b < batch;
    rows[q] = in + (valid[q] ? (b * na + a) * int64_t(nd) : 0);
  }
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (k < nd) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (valid[q]) v[q] = ld_f32(rows[q] + k);
    }
    za[swz(k)] = make_float2(v[0], v[1]);
    zb[swz(k)] = make_float2(v[2], v[3]);
  }
  __syncthreads();
  fft_dif(fsm, P, logP, tw);
  // ---- multiply by the real, even response; slot q holds frequency brev(q)
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int f = int(__brev(unsigned(q)) >> shift);
    const float h = __ldg(resp + (f <= P / 2 ? f : P - f));
    const int sq = swz(q);
    const float2 x = za[sq], y = zb[sq];
    za[sq] = make_float2(x.x * h, x.y * h);
    zb[sq] = make_float2(y.x * h, y.y * h);
  }
  __syncthreads();
  ifft_dit(fsm, P, logP, tw);
  // ---- crop, x 1/P (irfft normalisation, fft.cpp:117-118), x pi/(2 na)
  const float inv = 1.0f / float(P);
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const float2 x = za[swz(k)], y = zb[swz(k)];
    const float v[4] = {(x.x * inv) * scale, (x.y * inv) * scale, (y.x * inv) * scale, (y.y * inv) * scale};
    if (PACKED) {
      // fbp = backprojection(filter_sinogram(sino)) narrows the filtered rows
      // to the storage precision first (sino_filter.cpp:123, 126-128)
      packed[(g * na + a) * int64_t(nd) + k] =
          make_float4(float(st_cast<TOut>(v[0])), float(st_cast<TOut>(v[1])), float(st_cast<TOut>(v[2])),
                      float(st_cast<TOut>(v[3])));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (valid[q]) out[((g * kPack + q) * na + a) * int64_t(nd) + k] = st_cast<TOut>(v[q]);
    }
  }
}

template <class F>
void dispatch(int dtype, F&& f) {
  switch (dtype) {
    case RK_F16: f(__half{}); break;
    case RK_F32: f(float{}); break;
    case RK_F64: f(double{}); break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

}  // namespace

void launch_filter(const Filter& f, int dtype, const void* in, int64_t batch, int64_t n_angles, void* out,
                   float4* packed_out, cudaStream_t st) {
  const int P = int(f.padded);
  int logP = 0;
  while ((1 << logP) < P) ++logP;
  const size_t smem = size_t(2) * P * sizeof(float2);
  const float scale = float(M_PI / (2.0 * double(n_angles)));  // sino_filter.cpp:108
  dim3 grid(unsigned(n_angles), unsigned(groups_of(batch)));
  dispatch(dtype, [&](auto tag) {
    using T = decltype(tag);
    auto kern = packed_out ? filter_kernel<T, T, true> : filter_kernel<T, T, false>;
    if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    KernelTimer timer(RK_KERNEL_FILTER, st);
    kern<<<grid, kFilterThreads, smem, st>>>(static_cast<const T*>(in), batch, int(n_angles), int(f.det_count), P,
                                             logP, f.d_response.as<float>(), f.d_twiddle.as<float2>(), scale,
                                             static_cast<T*>(out), packed_out);
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
