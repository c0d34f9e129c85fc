// Ramp-filter kernel (sm_100a): per detector row, zero-pad to P, FFT,
// multiply by the real frequency response, inverse FFT, crop and scale by
// pi / (2 n_angles) — sino_filter.cpp:98-124 (filtration always fp32,
// :106-123).
//
// One CTA filters four rows of one packed group — images 2r, 2r + 1 of the
// group's four at an angle pair (a0, a0 + 1) — as two complex shared-memory
// FFTs: the response is real and even, so for z = x + i y,
// IFFT(FFT(z) H) = x*h + i (y*h) filters two real rows at once.
// The two rows of a sequence are one image's rows at the two angles, never two
// images': the complex butterflies mix the real and imaginary parts at the
// rounding level, so pairing images made a row's result depend on its batch
// neighbour (FBP of a batch differed from per-image calls in the last bit).  The forward transform is
// decimation-in-frequency (natural in, bit-reversed out), the response is
// applied in bit-reversed order, and the inverse is decimation-in-time with
// conjugate twiddles (bit-reversed in, natural out): no permutation pass.
// The row load, the response multiply and the crop/scale/store are fused into
// the first forward, last forward and last inverse passes (filter_kernel).
#include <cuda_fp16.h>

#include <cooperative_groups.h>

#include <type_traits>

#include "fft_smem.cuh"
#include "rk_internal.hpp"

namespace rk {

namespace cg = cooperative_groups;

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

// One fused radix-2^R pass over the two complex sequences (fft_smem.cuh's
// fft_pass with the same butterflies, twiddles and order, so the transform is
// bit-identical to it), with the element I/O supplied by the caller:
//   load(seq, i, m) -> float2    (m: the element's index within the group)
//   store(seq, i, m, float2)
// so the first forward pass can read the rows straight from global memory,
// the last forward pass can apply the response before its store, and the
// last inverse pass can crop, scale and write the output from registers.
// ZERO_TOP: inputs i >= n/2 are known zero (the zero-padded half of the row):
// the group's upper elements are not loaded and the first butterfly layer
// (partner bit R-1 of a DIF pass at the widest stride) reduces to u, u W.
// NSEQ: complex sequences per CTA (2; the split kernel below runs 1).
template <int R, bool DIF, bool CONJ, bool ZERO_TOP, class Load, class Store, int NSEQ = 2>
__device__ __forceinline__ void filter_pass(int logn, int lh, const float2* tw, Load load, Store store) {
  const int gl = logn - R;
#pragma unroll 4
  for (int t = threadIdx.x; t < (NSEQ << gl); t += kFilterThreads) {
    const int seq = t >> gl, g = t & ((1 << gl) - 1);
    const int lo = g & ((1 << lh) - 1), hi = g >> lh;
    const int i0 = lo + (hi << (lh + R));
    float2 x[1 << R];
#pragma unroll
    for (int m = 0; m < (1 << R); ++m)
      x[m] = (ZERO_TOP && m >= (1 << (R - 1))) ? make_float2(0.f, 0.f) : load(seq, i0 + (m << lh), m);
#pragma unroll
    for (int l = 0; l < R; ++l) {
      const int bit = DIF ? R - 1 - l : l;
#pragma unroll
      for (int m = 0; m < (1 << R); ++m) {
        if (m & (1 << bit)) continue;
        const int q = m | (1 << bit);
        const int k = lo + ((m & ((1 << bit) - 1)) << lh);
        const float2 w = __ldg(tw + ((1 << (lh + bit)) - 1) + k);  // stage lh + bit, entry k (= W^(k << ...))
        const float2 u = x[m];
        if (DIF) {
          if (ZERO_TOP && l == 0) {  // v = 0: u + v = u, (u - v) W = u W
            x[q] = fft_cmul(u, w);
          } else {
            const float2 v = x[q];
            x[m] = make_float2(u.x + v.x, u.y + v.y);
            x[q] = fft_cmul(make_float2(u.x - v.x, u.y - v.y), w);
          }
        } else {
          const float2 v = CONJ ? fft_cmul_conj(x[q], w) : fft_cmul(x[q], w);
          x[m] = make_float2(u.x + v.x, u.y + v.y);
          x[q] = make_float2(u.x - v.x, u.y - v.y);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) store(seq, i0 + (m << lh), m, x[m]);
  }
  __syncthreads();
}

// PACKED 0: user layout; 1: packed float4 cells (four images); 2: half of a
// packed half8 cell (fp16 storage, use_h8): this CTA's images 4g .. 4g+3 are
// the low or high four halves of group g / 2's cells.
//
// Round r = blockIdx.z (0, 1): sequence s is image q = 2r + s,
// z = row(q, a0) + i row(q, a0 + 1) (zero when a0 + 1 = n_angles).  Passes (P = 2^logP points, two sequences):
//   forward DIF: the first pass reads the rows from global memory (the upper
//   half is the zero padding: not read, first layer pruned), the middle
//   passes run in shared memory, the last pass multiplies by the response
//   (slot q holds frequency brev(q)) before storing;
//   inverse DIT: the middle passes in shared memory, the last pass crops to
//   det_count, scales and writes the result from registers.
// Twiddles come from a per-stage table (the stage's entries consecutive), so
// a warp's twiddle loads are coalesced; the strided gathers of the flat table
// made the kernel LSU-bound (ncu r2c: L1TEX 96 %, mio_throttle).
//
// LOGP > 0 fixes the transform size at compile time (the common sizes,
// launch_filter): every stride, shift and loop bound folds into the code,
// which the issue-bound passes need (ncu r2d: 79 % issue active); LOGP = 0
// takes the size at run time.
template <class TIn, class TOut, int PACKED, int LOGP>
// CTAs per SM: four up to 2^11 points (64 registers: without the bound the half8
// variant took 74 and three CTAs, +20 % at cfg4), three at 2^12 (64 KB of shared
// memory each)
__global__ void __launch_bounds__(kFilterThreads, (LOGP > 0 && LOGP <= 11) ? 4 : LOGP == 12 ? 3 : 1)
    filter_kernel(const TIn* __restrict__ in, int64_t batch, int na, int nd, int P_rt, int logP_rt,
                  const float* __restrict__ resp, const float2* __restrict__ tw, float scale, TOut* __restrict__ out,
                  float4* __restrict__ packed) {
  const int logP = LOGP ? LOGP : logP_rt;
  const int P = LOGP ? (1 << LOGP) : P_rt;
  extern __shared__ float2 fsm[];
  float2* za = fsm;  // sequences 0 and 1, swizzled slots (fft_swz)
  const float2* tws = tw;  // per-stage twiddle table (plan.cpp build_filter): consecutive per butterfly lane
  const int a0 = 2 * int(blockIdx.x);
  const bool has1 = a0 + 1 < na;  // the pair's second angle (odd n_angles: the last pair has one)
  const int64_t g = blockIdx.y;
  const int shift = 32 - logP;
  auto sm_load = [&](int seq, int i, int) { return za[seq * P + fft_swz(i)]; };
  auto sm_store = [&](int seq, int i, int, float2 v) { za[seq * P + fft_swz(i)] = v; };
  auto mul_store = [&](int seq, int i, int, float2 v) {
    const int f = int(__brev(unsigned(i)) >> shift);
    const float h = __ldg(resp + (f <= P / 2 ? f : P - f));
    za[seq * P + fft_swz(i)] = make_float2(v.x * h, v.y * h);
  };
  const float inv = 1.0f / float(P);
  const int r0 = logP % 3 == 0 ? 3 : logP % 3;  // the short forward pass first, at the widest stride
  // round = blockIdx.z: one CTA per round (a loop over both rounds kept values
  // live across them: 116 registers)
  const int round = int(blockIdx.z);
  // sequence seq: image q = 2 round + seq of the group, rows (q, a0) (re) and (q, a0 + 1) (im)
  const int64_t b0 = g * kPack + 2 * round, b1 = b0 + 1;
  const bool v0 = b0 < batch, v1 = b1 < batch;
  if (!v0) return;  // the group's remaining images are missing
  const TIn* row0 = in + (b0 * na + a0) * int64_t(nd);
  const TIn* row1 = in + (v1 ? (b1 * na + a0) * int64_t(nd) : 0);
  // (selects, not arrays indexed by seq: a dynamic index would put them in local memory)
  auto gl_load = [&](int seq, int i, int) {
    float re = 0.f, im = 0.f;
    if (i < nd && (seq ? v1 : v0)) {
      const TIn* r = seq ? row1 : row0;
      re = ld_f32(r + i);
      if (has1) im = ld_f32(r + nd + i);
    }
    return make_float2(re, im);
  };
  // ---- forward DIF (natural -> bit-reversed), fft_dif_seq's pass order
  int lh = logP - r0;
  const bool single = lh == 0;  // one pass (P <= 8): it both reads the rows and applies the response
  if (r0 == 1) {
    if (single) filter_pass<1, true, false, true>(logP, lh, tws, gl_load, mul_store);
    else filter_pass<1, true, false, true>(logP, lh, tws, gl_load, sm_store);
  } else if (r0 == 2) {
    if (single) filter_pass<2, true, false, true>(logP, lh, tws, gl_load, mul_store);
    else filter_pass<2, true, false, true>(logP, lh, tws, gl_load, sm_store);
  } else {
    if (single) filter_pass<3, true, false, true>(logP, lh, tws, gl_load, mul_store);
    else filter_pass<3, true, false, true>(logP, lh, tws, gl_load, sm_store);
  }
#pragma unroll
  while (lh >= 3) {
    lh -= 3;
    if (lh == 0)
      filter_pass<3, true, false, false>(logP, lh, tws, sm_load, mul_store);
    else
      filter_pass<3, true, false, false>(logP, lh, tws, sm_load, sm_store);
  }
  // ---- inverse DIT (bit-reversed -> natural), conjugate twiddles; the last
  // pass crops, x 1/P (irfft normalisation, fft.cpp:117-118), x pi/(2 na)
  // user layout: the last inverse pass writes the rows from registers
  auto out_store = [&](int seq, int i, int, float2 v) {
    if (i >= nd || !(seq ? v1 : v0)) return;
    TOut* o = out + ((g * kPack + 2 * round + seq) * na + a0) * int64_t(nd) + i;
    o[0] = st_cast<TOut>((v.x * inv) * scale);
    if (has1) o[nd] = st_cast<TOut>((v.y * inv) * scale);
  };
  auto inverse = [&](auto last) {
    int lq = 0;
#pragma unroll
    for (; lq + 3 <= logP; lq += 3) {
      if (lq + 3 == logP)
        filter_pass<3, false, true, false>(logP, lq, tws, sm_load, last);
      else
        filter_pass<3, false, true, false>(logP, lq, tws, sm_load, sm_store);
    }
    if (logP - lq == 2) filter_pass<2, false, true, false>(logP, lq, tws, sm_load, last);
    if (logP - lq == 1) filter_pass<1, false, true, false>(logP, lq, tws, sm_load, last);
  };
  if constexpr (PACKED == 0) {
    inverse(out_store);
  } else {
    // packed cells: the two sequences (images 2 round, 2 round + 1) share each cell, so the
    // last pass leaves them in shared memory and one thread writes both lanes per (angle, cell)
    // — 8-byte float2 / 4-byte half2 stores instead of two scalar ones
    inverse(sm_store);
    for (int i = threadIdx.x; i < nd; i += kFilterThreads) {
      const float2 z0 = za[fft_swz(i)], z1 = za[P + fft_swz(i)];  // (re, im) = (angle a0, a0 + 1)
      // fbp = backprojection(filter_sinogram(sino)) narrows the filtered rows to the
      // storage precision first (sino_filter.cpp:123, 126-128); a missing image's lane gets 0
      auto narrow = [&](float v) { return float(st_cast<TOut>((v * inv) * scale)); };
      const float r00 = narrow(z0.x), r01 = v1 ? narrow(z1.x) : 0.f;  // angle a0
      const float r10 = narrow(z0.y), r11 = v1 ? narrow(z1.y) : 0.f;  // angle a0 + 1
      if (PACKED == 2) {
        // this CTA's two of the cell's eight halves: the values the float4 path narrows through fp16
        __half2* c =
            reinterpret_cast<__half2*>(packed) + (((g >> 1) * na + a0) * int64_t(nd) + i) * 4 + (g & 1) * 2 + round;
        c[0] = __floats2half2_rn(r00, r01);
        if (has1) c[int64_t(nd) * 4] = __floats2half2_rn(r10, r11);
      } else {
        float2* c = reinterpret_cast<float2*>(packed) + ((g * na + a0) * int64_t(nd) + i) * 2 + round;
        c[0] = make_float2(r00, r01);
        if (has1) c[int64_t(nd) * 2] = make_float2(r10, r11);
      }
    }
  }
}

// Transforms of P = 2^14 and 2^15 points (det_count 4097 .. 16384) no longer
// fit one CTA's shared memory, so a two-CTA cluster splits each sequence into
// its even and odd frequencies.  The row is zero beyond det_count <= P/2, so
// the first DIF layer needs no exchange: y_0[i] = x[i] and y_1[i] = x[i] W_P^i
// (i < P/2) are the two half-size inputs, whose P/2-point DIF transforms are
// the even (rank 0) and odd (rank 1) frequency bins.  Each CTA applies the
// response to its bins (frequency 2 brev(q) + rank) and runs the P/2-point
// inverse DIT; the last inverse layer would combine the halves,
//   out[i] = a[i] + conj(W_P^i) b[i]   (only i < det_count <= P/2 is kept),
// so after a cluster barrier each CTA reads the other's half through
// distributed shared memory for its share of the outputs.  One complex
// sequence per cluster — image q = blockIdx.z of the group at the angle pair
// (a0, a0 + 1), as in filter_kernel; P/2 complex in each CTA (64 / 128 KB).
template <class TIn, class TOut, int PACKED, int LOGH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFilterThreads)
    filter_split_kernel(const TIn* __restrict__ in, int64_t batch, int na, int nd, const float* __restrict__ resp,
                        const float2* __restrict__ tw, float scale, TOut* __restrict__ out,
                        float4* __restrict__ packed) {
  constexpr int H = 1 << LOGH, P = 2 * H, logH = LOGH;
  extern __shared__ float2 fsm[];
  float2* za = fsm;  // this CTA's half, swizzled slots (fft_swz)
  const unsigned rank = blockIdx.x & 1u;  // cluster rank: 0 even, 1 odd frequencies
  const int a0 = 2 * int(blockIdx.x >> 1);
  const bool has1 = a0 + 1 < na;
  const int64_t g = blockIdx.y;
  const int q = int(blockIdx.z);  // image q of packed group g: rows (q, a0) (re) and (q, a0 + 1) (im)
  const int64_t b = g * kPack + q;
  if (b >= batch) return;  // both CTAs of the cluster leave together (same b)
  const TIn* pre = in + (b * na + a0) * int64_t(nd);
  const float2* wP = tw + (H - 1);  // stage logP - 1: W_P^k, k < P/2
  auto sm_load = [&](int, int i, int) { return za[fft_swz(i)]; };
  auto sm_store = [&](int, int i, int, float2 v) { za[fft_swz(i)] = v; };
  auto gl_load = [&](int, int i, int) {  // y_rank[i]
    float re = 0.f, im = 0.f;
    if (i < nd) {
      re = ld_f32(pre + i);
      if (has1) im = ld_f32(pre + nd + i);
    }
    float2 v = make_float2(re, im);
    if (rank) v = fft_cmul(v, __ldg(wP + i));
    return v;
  };
  constexpr int shift = 32 - logH;
  auto mul_store = [&](int, int i, int, float2 v) {
    const int f = 2 * int(__brev(unsigned(i)) >> shift) + int(rank);
    const float h = __ldg(resp + (f <= P / 2 ? f : P - f));
    za[fft_swz(i)] = make_float2(v.x * h, v.y * h);
  };
  // ---- forward DIF of the half (natural -> bit-reversed)
  constexpr int r0 = logH % 3 == 0 ? 3 : logH % 3;
  int lh = logH - r0;
  filter_pass<r0, true, false, false, decltype(gl_load), decltype(sm_store), 1>(logH, lh, tw, gl_load, sm_store);
#pragma unroll
  while (lh >= 3) {
    lh -= 3;
    if (lh == 0)
      filter_pass<3, true, false, false, decltype(sm_load), decltype(mul_store), 1>(logH, lh, tw, sm_load, mul_store);
    else
      filter_pass<3, true, false, false, decltype(sm_load), decltype(sm_store), 1>(logH, lh, tw, sm_load, sm_store);
  }
  // ---- inverse DIT of the half (bit-reversed -> natural), into shared memory
  int lq = 0;
#pragma unroll
  for (; lq + 3 <= logH; lq += 3)
    filter_pass<3, false, true, false, decltype(sm_load), decltype(sm_store), 1>(logH, lq, tw, sm_load, sm_store);
  if (logH - lq == 2) filter_pass<2, false, true, false, decltype(sm_load), decltype(sm_store), 1>(logH, lq, tw, sm_load, sm_store);
  if (logH - lq == 1) filter_pass<1, false, true, false, decltype(sm_load), decltype(sm_store), 1>(logH, lq, tw, sm_load, sm_store);
  // ---- combine across the cluster: out[i] = a[i] + conj(W_P^i) b[i], crop, x 1/P, x pi/(2 na)
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const float2* za0 = cluster.map_shared_rank(za, 0);
  const float2* za1 = cluster.map_shared_rank(za, 1);
  const float inv = 1.0f / float(P);
  const int half_nd = (nd + 1) / 2;
  for (int i = int(rank) * half_nd + threadIdx.x; i < min(nd, (int(rank) + 1) * half_nd); i += kFilterThreads) {
    const float2 av = za0[fft_swz(i)], bv = za1[fft_swz(i)];
    const float2 v = make_float2(av.x, av.y);
    const float2 wb = fft_cmul_conj(bv, __ldg(wP + i));
    const float v0 = ((v.x + wb.x) * inv) * scale, v1 = ((v.y + wb.y) * inv) * scale;
    if (PACKED == 2) {
      __half* c = reinterpret_cast<__half*>(packed) + (((g >> 1) * na + a0) * int64_t(nd) + i) * 8 + (g & 1) * 4 + q;
      c[0] = __float2half_rn(v0);
      if (has1) c[int64_t(nd) * 8] = __float2half_rn(v1);
    } else if (PACKED == 1) {
      float* c = reinterpret_cast<float*>(packed) + ((g * na + a0) * int64_t(nd) + i) * 4 + q;
      c[0] = float(st_cast<TOut>(v0));
      if (has1) c[int64_t(nd) * 4] = float(st_cast<TOut>(v1));
    } else {
      TOut* o = out + (b * na + a0) * int64_t(nd) + i;
      o[0] = st_cast<TOut>(v0);
      if (has1) o[nd] = st_cast<TOut>(v1);
    }
  }
  cluster.sync();  // the other CTA may still read this one's half
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
  const size_t smem = size_t(2) * P * sizeof(float2);  // two sequences
  const float scale = float(M_PI / (2.0 * double(n_angles)));  // sino_filter.cpp:108
  const unsigned pairs = unsigned((n_angles + 1) / 2);  // angle pairs (a0, a0 + 1)
  dim3 grid(pairs, unsigned(groups_of(batch)), 2u);  // z: the round (image pair of the group)
  if (logP >= 14) {  // 2^14, 2^15 (det_count 4097 .. 16384): the two-CTA cluster kernel
    const size_t hsmem = size_t(P / 2) * sizeof(float2);
    dim3 sgrid(2 * pairs, unsigned(groups_of(batch)), unsigned(kPack));
    dispatch(dtype, [&](auto tag) {
      using T = decltype(tag);
      auto pick = [&](auto packed_tag) {
        constexpr int PK = decltype(packed_tag)::value;
        return logP == 14 ? filter_split_kernel<T, T, PK, 13> : filter_split_kernel<T, T, PK, 14>;
      };
      auto kern = packed_out ? pick(std::integral_constant<int, 1>{}) : pick(std::integral_constant<int, 0>{});
      if constexpr (std::is_same<T, __half>::value)
        if (packed_out && use_h8(dtype, batch)) kern = pick(std::integral_constant<int, 2>{});
      allow_dynamic_smem(reinterpret_cast<const void*>(kern), hsmem);
      KernelTimer timer(RK_KERNEL_FILTER, st);
      kern<<<sgrid, kFilterThreads, hsmem, st>>>(static_cast<const T*>(in), batch, int(n_angles), int(f.det_count),
                                                 f.d_response.as<float>(), f.d_twiddle_stage.as<float2>(), scale,
                                                 static_cast<T*>(out), packed_out);
    });
    RK_CUDA(cudaGetLastError());
    return;
  }
  dispatch(dtype, [&](auto tag) {
    using T = decltype(tag);
    // compile-time sizes for P = 2^9 .. 2^13 (det_count 129 .. 4096), run-time size otherwise
    auto pick = [&](auto packed_tag) {
      constexpr int PK = decltype(packed_tag)::value;
      switch (logP) {
        case 9: return filter_kernel<T, T, PK, 9>;
        case 10: return filter_kernel<T, T, PK, 10>;
        case 11: return filter_kernel<T, T, PK, 11>;
        case 12: return filter_kernel<T, T, PK, 12>;
        case 13: return filter_kernel<T, T, PK, 13>;
        default: return filter_kernel<T, T, PK, 0>;
      }
    };
    auto kern = packed_out ? pick(std::integral_constant<int, 1>{}) : pick(std::integral_constant<int, 0>{});
    if constexpr (std::is_same<T, __half>::value)
      if (packed_out && use_h8(dtype, batch)) kern = pick(std::integral_constant<int, 2>{});
    allow_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    KernelTimer timer(RK_KERNEL_FILTER, st);
    kern<<<grid, kFilterThreads, smem, st>>>(static_cast<const T*>(in), batch, int(n_angles), int(f.det_count), P,
                                             logP, f.d_response.as<float>(), f.d_twiddle_stage.as<float2>(), scale,
                                             static_cast<T*>(out), packed_out);
  });
  RK_CUDA(cudaGetLastError());
}

}  // namespace rk
