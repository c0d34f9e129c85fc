// Alpha-shearlet analysis / synthesis on the device (§8f rank 3; reference
// shearlet.cpp:253-330): coefficient k of an image x is
// Re(ifft2(fft2(x) * M_k)); synthesis sums fft2(c_k) * M_k over k and takes
// Re(ifft2(.)).  Arithmetic follows the reference's precision split
// (shearlet.cpp:303-310): fp64 storage computes in fp64, fp32 / fp16 storage
// in fp32; power-of-two grids (other sizes: shearlet_generic.cu).
//
// Layout and passes (no transposes, no bit-reversal permutes):
//   * 2-D FFTs are a row pass and a column pass over natural [row][col]
//     planes, each a shared-memory FFT of a CTA tile (rows, or a tile of
//     adjacent columns read with coalesced row segments) with three radix-2
//     stages fused per register pass (fft_smem.cuh).
//   * Forward transforms are decimation-in-frequency (natural in, bit-reversed
//     out) and inverse ones decimation-in-time (bit-reversed in, natural out),
//     so spectra live in bit-reversed (row, col) order and the multipliers are
//     stored in that order on the host side of the plan.
//   * Two coefficients share one complex transform.  Analysis: M_k and
//     M_k+1 are real and even, so ifft2(X (M_k + i M_k+1)) = c_k + i c_k+1
//     (both real).  Synthesis: with Z = fft2(c_k + i c_k+1),
//     Z (M_k - i M_k+1) = [C_k M_k + C_k+1 M_k+1] + i[C_k+1 M_k - C_k M_k+1]
//     whose second term is anti-Hermitian, so Re(ifft2(sum)) is exactly the
//     synthesis.  This halves the FFT work and the intermediate traffic.
//   * Analysis walks (coefficient pair, image) items pair-major so one pair's
//     multipliers stay in L2 across the batch; synthesis accumulates a fixed
//     chunk of pairs per column tile in registers (a batch-independent order).
//
// ADMM hooks (admm.cu, admm.cpp:146-156): analysis can fuse the shrink and
// dual update into its store (z1 = shrink(c + u1, t_k), u1 += c - z1, with a
// non-finite flag), and synthesis can read (z1 - u1) instead of c.
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "fft_smem.cuh"
#include "rk_internal.hpp"

namespace rk {

namespace {

template <class R>
struct Cx;
template <>
struct Cx<float> {
  using T = float2;
};
template <>
struct Cx<double> {
  using T = double2;
};

template <class R, class T>
__device__ __forceinline__ R ld_r(const T* p) {
  return R(*p);
}
template <>
__device__ __forceinline__ float ld_r<float, __half>(const __half* p) {
  return __half2float(*p);
}
template <class T, class R>
__device__ __forceinline__ T st_r(R v) {
  return T(v);
}
template <>
__device__ __forceinline__ __half st_r<__half, float>(float v) {
  return __float2half_rn(v);
}

template <class C>
__device__ __forceinline__ C cmul(C a, C b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <class C>
__device__ __forceinline__ C cmul_conj(C a, C b) {  // a * conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}

constexpr int kTileMin = 4096;  // complex elements per CTA tile (>= one row, <= one plane)
constexpr int kPerThread = 16;  // tile elements per thread
constexpr int kAccPerThread = 8;  // synthesis accumulation: tile elements per thread (2x the threads, half the registers)
// analysis scratch per launch (the column pass's output planes): large enough
// that a launch covers many (pair, image) items — small chunks leave the GPU
// with short, tail-dominated launches (64 MB: 1.15 ms, 1 GB: 0.85 ms at 512^2,
// batch 8)
constexpr int kWkChunkMB = 1024;
constexpr int kPairChunk = 8;   // coefficient pairs per synthesis accumulation (fixed: batch-independent order)

// shared-memory slot of tile element e (row e >> logn of the tile, swizzled within the row)
__device__ __forceinline__ int srow(int e, int logn) {
  return ((e >> logn) << logn) | fft_swz(e & ((1 << logn) - 1));
}

// tile elements for an n x n plane: kTileMin, at least one row, at most the plane
__host__ __device__ inline int tile_of(int n) { return min(max(kTileMin, n), n * n); }

// ADMM analysis epilogue (admm.cpp:150-153), fp32 like the reference's float path
struct AdmmStore {
  float* z1 = nullptr;  // null: plain store
  float* u1 = nullptr;
  const float* thresh = nullptr;  // per coefficient, float((p0/p1) w_k)
  int* flag = nullptr;            // atomicMin(*iteration) when u1 turns non-finite
  const int* iteration = nullptr;  // device counter: the outer iteration (admm.cu; graph-replay safe)
};

// soft(a, b) = sign(a) max(|a| - b, 0) (admm.cpp:46-51)
__device__ __forceinline__ float soft(float a, float b) {
  float m = __fsub_rn(fabsf(a), b);
  if (m < 0.f) m = 0.f;
  return a < 0.f ? -m : (a > 0.f ? m : 0.f);
}

__device__ __forceinline__ void admm_update(const AdmmStore& a, int64_t gi, int k, float c) {
  const float u = a.u1[gi];
  const float z = soft(__fadd_rn(c, u), a.thresh[k]);
  const float un = __fadd_rn(u, __fsub_rn(c, z));
  a.z1[gi] = z;
  a.u1[gi] = un;
  if (!isfinite(un)) atomicMin(a.flag, *a.iteration);
}

// ---------------------------------------------------------------- row passes
// A CTA owns `nr` consecutive rows of one plane (nr * n = tile elements).

// forward row DIF of real input rows: out[p] = rowDIF(in0[p] (- sub0[p]) + i (in1[p] (- sub1[p])))
// plane p -> sources by `map`:
//   map 0 (images):        in0 = src + p * n^2, no imaginary part
//   map 1 (synthesis pair): p = b * J + jj, j = j0 + jj: in0 = c[b][2j], in1 = c[b][2j+1] (when < K)
struct RowSrc {
  int map;
  int64_t J, j0, K;
};
template <class T, class R>
__global__ void __launch_bounds__(512, 3) row_fwd_kernel(const T* __restrict__ src, const T* __restrict__ sub, RowSrc m,
                                                       int logn, const typename Cx<R>::T* __restrict__ tw,
                                                       typename Cx<R>::T* __restrict__ out) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int n = 1 << logn;
  const int64_t plane = int64_t(n) * n;
  const int tile = tile_of(n), nr = tile / n;
  const int64_t row0 = int64_t(blockIdx.x) * nr;  // global row over planes
  const int64_t p = row0 >> logn, lr0 = row0 - (p << logn);
  const T* in0;
  const T* in1 = nullptr;
  const T* s0 = nullptr;
  const T* s1 = nullptr;
  if (m.map == 0) {
    in0 = src + p * plane;
    if (sub) s0 = sub + p * plane;
  } else {
    const int64_t b = p / m.J, j = m.j0 + p % m.J, k0 = 2 * j;
    in0 = src + (b * m.K + k0) * plane;
    if (sub) s0 = sub + (b * m.K + k0) * plane;
    if (k0 + 1 < m.K) {
      in1 = in0 + plane;
      if (sub) s1 = s0 + plane;
    }
  }
  const int64_t base = lr0 * n;
  bool loaded = false;
  if constexpr (std::is_same<T, float>::value && std::is_same<R, float>::value) {
    // four reals per 16-byte load (memory-level parallelism: the pass is
    // latency-bound on its global reads); caller buffers may be misaligned
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(sub)) & 15) == 0;
    if (n >= 4 && aligned) {
#pragma unroll 4
      for (int e = 4 * threadIdx.x; e < tile; e += 4 * blockDim.x) {
        float4 re = *reinterpret_cast<const float4*>(in0 + base + e), im = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s0) {  // sub(z1, u1) (admm.cpp:147)
          const float4 d = *reinterpret_cast<const float4*>(s0 + base + e);
          re = make_float4(re.x - d.x, re.y - d.y, re.z - d.z, re.w - d.w);
        }
        if (in1) {
          im = *reinterpret_cast<const float4*>(in1 + base + e);
          if (s1) {
            const float4 d = *reinterpret_cast<const float4*>(s1 + base + e);
            im = make_float4(im.x - d.x, im.y - d.y, im.z - d.z, im.w - d.w);
          }
        }
        sm[srow(e, logn)] = {re.x, im.x};
        sm[srow(e + 1, logn)] = {re.y, im.y};
        sm[srow(e + 2, logn)] = {re.z, im.z};
        sm[srow(e + 3, logn)] = {re.w, im.w};
      }
      loaded = true;
    }
  }
  if (!loaded) {
#pragma unroll 8
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
      R re = ld_r<R>(in0 + base + e), im = R(0);
      if (s0) re = re - ld_r<R>(s0 + base + e);  // sub(z1, u1) (admm.cpp:147)
      if (in1) {
        im = ld_r<R>(in1 + base + e);
        if (s1) im = im - ld_r<R>(s1 + base + e);
      }
      sm[srow(e, logn)] = {re, im};
    }
  }
  __syncthreads();
  fft_dif_seq(sm, nr, n, logn, tw);
  C* o = out + p * plane + base;
  if constexpr (std::is_same<R, float>::value) {
    if (n >= 2) {  // two complex per 16-byte store
#pragma unroll 4
      for (int e = 2 * threadIdx.x; e < tile; e += 2 * blockDim.x) {
        const C u = sm[srow(e, logn)], v = sm[srow(e + 1, logn)];
        *reinterpret_cast<float4*>(o + e) = make_float4(u.x, u.y, v.x, v.y);
      }
      return;
    }
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < tile; e += blockDim.x) o[e] = sm[srow(e, logn)];
}

// inverse row DIT of complex rows, scaled: Re -> out0, Im -> out1 (when present)
// plane p -> destinations by `map`:
//   map 0 (images):        out0 = dst + p * n^2
//   map 1 (analysis pair): q = q0 + p, j = q / B, b = q % B: out0 = c[b][2j], out1 = c[b][2j+1] (when < K)
struct RowDst {
  int map;
  int64_t q0, B, K;
};
template <class T, class R>
__global__ void __launch_bounds__(512, 3) row_inv_kernel(const typename Cx<R>::T* __restrict__ in, RowDst m, int logn,
                                                       const typename Cx<R>::T* __restrict__ tw, R scale,
                                                       T* __restrict__ dst, AdmmStore admm) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int n = 1 << logn;
  const int64_t plane = int64_t(n) * n;
  const int tile = tile_of(n), nr = tile / n;
  const int64_t row0 = int64_t(blockIdx.x) * nr;
  const int64_t p = row0 >> logn, lr0 = row0 - (p << logn);
  const int64_t base = lr0 * n;
  const C* src = in + p * plane + base;
  bool vec = false;
  if constexpr (std::is_same<R, float>::value) {
    if (n >= 2) {  // two complex per 16-byte load
      vec = true;
#pragma unroll 4
      for (int e = 2 * threadIdx.x; e < tile; e += 2 * blockDim.x) {
        const float4 u = *reinterpret_cast<const float4*>(src + e);
        sm[srow(e, logn)] = {u.x, u.y};
        sm[srow(e + 1, logn)] = {u.z, u.w};
      }
    }
  }
  if (!vec) {
#pragma unroll 8
    for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[srow(e, logn)] = src[e];
  }
  __syncthreads();
  ifft_dit_seq(sm, nr, n, logn, tw);
  int64_t o0, o1 = -1;  // element offsets of the two output planes
  int k0 = 0;
  if (m.map == 0) {
    o0 = p * plane;
  } else {
    const int64_t q = m.q0 + p, j = q / m.B, b = q % m.B;
    k0 = int(2 * j);
    o0 = (b * m.K + k0) * plane;
    if (k0 + 1 < m.K) o1 = o0 + plane;
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < tile; e += blockDim.x) {
    const C v = sm[srow(e, logn)];
    const R re = v.x * scale, im = v.y * scale;
    if (admm.z1 == nullptr) {
      dst[o0 + base + e] = st_r<T>(re);
      if (o1 >= 0) dst[o1 + base + e] = st_r<T>(im);
    } else {
      admm_update(admm, o0 + base + e, k0, float(re));
      if (o1 >= 0) admm_update(admm, o1 + base + e, k0 + 1, float(im));
    }
  }
}

// ---------------------------------------------------------------- column passes
// A CTA owns `tc` adjacent columns of one plane (tc * n = tile elements),
// staged column-major in shared memory with a padded stride.
__host__ __device__ inline int col_ld(int n) { return n + 4; }

// (fp32: two adjacent columns per 16-byte access — scratch planes are aligned)
template <class C>
__device__ __forceinline__ void load_cols(C* sm, const C* __restrict__ src, int n, int tc, int c0, int ld) {
  if constexpr (std::is_same<C, float2>::value) {
    if ((tc & 1) == 0) {
      const int hp = tc >> 1;
#pragma unroll 8
      for (int e = threadIdx.x; e < hp * n; e += blockDim.x) {
        const int r = e / hp, c = 2 * (e - r * hp);
        const float4 u = *reinterpret_cast<const float4*>(src + int64_t(r) * n + c0 + c);
        sm[c * ld + fft_swz(r)] = make_float2(u.x, u.y);
        sm[(c + 1) * ld + fft_swz(r)] = make_float2(u.z, u.w);
      }
      return;
    }
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < tc * n; e += blockDim.x) {
    const int r = e / tc, c = e - r * tc;
    sm[c * ld + fft_swz(r)] = src[int64_t(r) * n + c0 + c];
  }
}
template <class C>
__device__ __forceinline__ void store_cols(C* __restrict__ dst, const C* sm, int n, int tc, int c0, int ld) {
  if constexpr (std::is_same<C, float2>::value) {
    if ((tc & 1) == 0) {
      const int hp = tc >> 1;
#pragma unroll 8
      for (int e = threadIdx.x; e < hp * n; e += blockDim.x) {
        const int r = e / hp, c = 2 * (e - r * hp);
        const C u = sm[c * ld + fft_swz(r)], v = sm[(c + 1) * ld + fft_swz(r)];
        *reinterpret_cast<float4*>(dst + int64_t(r) * n + c0 + c) = make_float4(u.x, u.y, v.x, v.y);
      }
      return;
    }
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < tc * n; e += blockDim.x) {
    const int r = e / tc, c = e - r * tc;
    dst[int64_t(r) * n + c0 + c] = sm[c * ld + fft_swz(r)];
  }
}

// mode 0: out = colDIF(in)                          (plane p -> p)
// mode 1: out = colDIT^-1(in[b] * (M_2j + i M_2j+1)) (analysis item q = q0 + p: j = q / B, b = q % B)
// mode 2: out = colDIT^-1(in)                       (plane p -> p)
// mode 3: out = colDIT^-1(sum_c in[p][c])             (B = chunk partials per plane, summed in order)
template <class R>
__global__ void __launch_bounds__(512, 3) col_kernel(const typename Cx<R>::T* __restrict__ in, int mode, int logn,
                                                   const typename Cx<R>::T* __restrict__ tw,
                                                   const typename Cx<R>::T* __restrict__ mult2, int64_t q0, int64_t B,
                                                   typename Cx<R>::T* __restrict__ out) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int n = 1 << logn, ld = col_ld(n);
  const int64_t plane = int64_t(n) * n;
  const int tile = tile_of(n), tc = tile / n;
  const int tiles = n / tc;
  const int64_t p = blockIdx.x / tiles;
  const int c0 = int(blockIdx.x - p * tiles) * tc;
  if (mode == 1) {
    const int64_t q = q0 + p, j = q / B, b = q % B;
    const C* src = in + b * plane;
    const C* mk = mult2 + j * plane;
    bool done = false;
    if constexpr (std::is_same<C, float2>::value) {
      if ((tc & 1) == 0) {  // two adjacent columns per 16-byte load
        const int hp = tc >> 1;
#pragma unroll 8
        for (int e = threadIdx.x; e < hp * n; e += blockDim.x) {
          const int r = e / hp, c = 2 * (e - r * hp);
          const int64_t gi = int64_t(r) * n + c0 + c;
          const float4 x = *reinterpret_cast<const float4*>(src + gi), w = *reinterpret_cast<const float4*>(mk + gi);
          sm[c * ld + fft_swz(r)] = cmul(make_float2(x.x, x.y), make_float2(w.x, w.y));
          sm[(c + 1) * ld + fft_swz(r)] = cmul(make_float2(x.z, x.w), make_float2(w.z, w.w));
        }
        done = true;
      }
    }
    if (!done) {
#pragma unroll 8
      for (int e = threadIdx.x; e < tc * n; e += blockDim.x) {
        const int r = e / tc, c = e - r * tc;
        const int64_t gi = int64_t(r) * n + c0 + c;
        sm[c * ld + fft_swz(r)] = cmul(src[gi], mk[gi]);
      }
    }
  } else if (mode == 3) {
  #pragma unroll 8
    for (int e = threadIdx.x; e < tc * n; e += blockDim.x) {
      const int r = e / tc, c = e - r * tc;
      const int64_t gi = int64_t(r) * n + c0 + c;
      C a = {R(0), R(0)};
      for (int64_t k = 0; k < B; ++k) {
        const C v = in[(p * B + k) * plane + gi];
        a = {a.x + v.x, a.y + v.y};
      }
      sm[c * ld + fft_swz(r)] = a;
    }
  } else {
    load_cols(sm, in + p * plane, n, tc, c0, ld);
  }
  __syncthreads();
  if (mode == 0)
    fft_dif_seq(sm, tc, ld, logn, tw);
  else
    ifft_dit_seq(sm, tc, ld, logn, tw);
  store_cols(out + p * plane, sm, n, tc, c0, ld);
}

// synthesis accumulation: for image b, a column tile and a chunk c of
// kPairChunk coefficient pairs, over the chunk's pairs in ascending order:
// acc += colDIF(W[b][pair]) * (M_2j - i M_2j+1); the chunk's sum goes to its
// own partial plane Sp[b][c] (the final column pass adds the partials in
// chunk order).  Each thread owns the same kPerThread tile elements
// throughout, so the sum order per bin is fixed and batch-independent.
// W holds the wave's pairs p0 .. p0 + np - 1 of every image (b * np + pair - p0).
template <class R>
__global__ void __launch_bounds__(512, 2) col_acc_kernel(const typename Cx<R>::T* __restrict__ W, int64_t np, int64_t p0,
                                                       int64_t P, int64_t c0, int64_t ncw, int64_t nch, int logn,
                                                       const typename Cx<R>::T* __restrict__ tw,
                                                       const typename Cx<R>::T* __restrict__ mult2,
                                                       typename Cx<R>::T* __restrict__ Sp) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int n = 1 << logn, ld = col_ld(n);
  const int64_t plane = int64_t(n) * n;
  const int tile = tile_of(n), tc = tile / n;
  const int tiles = n / tc;
  // image fastest: the CTAs of one (chunk, tile) run together and share the
  // chunk's multiplier tiles in L2
  const int64_t batch = gridDim.x / (int64_t(tiles) * ncw);
  const int64_t b = blockIdx.x % batch, ct = blockIdx.x / batch;
  const int64_t cw = ct / tiles;
  const int c0t = int(ct - cw * tiles) * tc;
  const int64_t chunk = c0 + cw;
  const int64_t ja = chunk * kPairChunk, jb = min(ja + kPairChunk, P);
  C acc[kAccPerThread];
#pragma unroll
  for (int m = 0; m < kAccPerThread; ++m) acc[m] = {R(0), R(0)};
  for (int64_t j = ja; j < jb; ++j) {
    load_cols(sm, W + (b * np + (j - p0)) * plane, n, tc, c0t, ld);
    __syncthreads();
    fft_dif_seq(sm, tc, ld, logn, tw);
    const C* mk = mult2 + j * plane;
#pragma unroll
    for (int m = 0; m < kAccPerThread; ++m) {
      const int e = threadIdx.x + m * blockDim.x;
      if (e >= tile) break;
      const int r = e / tc, c = e - r * tc;
      const C v = cmul_conj(sm[c * ld + fft_swz(r)], mk[int64_t(r) * n + c0t + c]);
      acc[m] = {acc[m].x + v.x, acc[m].y + v.y};
    }
    __syncthreads();
  }
  C* s = Sp + (b * nch + chunk) * plane;
#pragma unroll
  for (int m = 0; m < kAccPerThread; ++m) {
    const int e = threadIdx.x + m * blockDim.x;
    if (e >= tile) break;
    const int r = e / tc, c = e - r * tc;
    s[int64_t(r) * n + c0t + c] = acc[m];
  }
}

// ---------------------------------------------------------------- host side
int log2_of(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

struct Launch {
  unsigned threads;
  size_t row_smem, col_smem;
  int tile, per_plane_rows, per_plane_cols;  // CTAs per plane in the row / column passes
};
template <class R>
Launch launch_cfg(int n) {
  using C = typename Cx<R>::T;
  Launch l;
  l.tile = tile_of(n);
  l.threads = unsigned(std::max(32, l.tile / kPerThread));
  l.row_smem = size_t(l.tile) * sizeof(C);
  const int tc = l.tile / n;
  l.col_smem = size_t(tc) * size_t(col_ld(n)) * sizeof(C);
  l.per_plane_rows = n / (l.tile / n);
  l.per_plane_cols = n / tc;
  return l;
}

template <class K>
void smem_opt_in(K kernel, size_t smem) {
  allow_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
}

template <class R>
struct Tables {
  const typename Cx<R>::T* tw;
  const typename Cx<R>::T* mult2;
};

// {M_2j, M_2j+1}[r][c] = M[brev r][brev c], zero for a missing odd partner
template <class R>
void build_tables(const Shearlet& sp, std::vector<typename Cx<R>::T>& mult2, std::vector<typename Cx<R>::T>& tw) {
  const int64_t n = sp.height, bins = n * n, K = sp.n_coeff, P = (K + 1) / 2;
  const int logn = log2_of(n);
  std::vector<int64_t> rev(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = 0;
    for (int bit = 0; bit < logn; ++bit)
      if (i & (int64_t(1) << bit)) r |= int64_t(1) << (logn - 1 - bit);
    rev[size_t(i)] = r;
  }
  mult2.assign(size_t(P * bins), {R(0), R(0)});
  for (int64_t k = 0; k < K; ++k) {
    const double* m = sp.multipliers.data() + k * bins;
    auto* d = mult2.data() + (k / 2) * bins;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        const R v = R(m[rev[size_t(r)] * n + rev[size_t(c)]]);
        if (k % 2 == 0)
          d[r * n + c].x = v;
        else
          d[r * n + c].y = v;
      }
  }
  tw.assign(size_t(std::max<int64_t>(n / 2, 1)), {R(0), R(0)});
  for (int64_t k = 0; k < n / 2; ++k) {
    const double ang = 2.0 * M_PI * double(k) / double(n);
    tw[size_t(k)] = {R(std::cos(ang)), R(-std::sin(ang))};
  }
}

template <class R>
Tables<R> tables(Shearlet& sp);
template <>
Tables<float> tables<float>(Shearlet& sp) {
  return {sp.d_twiddle.as<float2>(), sp.d_mult2.as<float2>()};
}
template <>
Tables<double> tables<double>(Shearlet& sp) {
  if (!sp.d_mult2_64.ptr) {
    std::vector<double2> m2, tw;
    build_tables<double>(sp, m2, tw);
    sp.d_twiddle64.reserve(tw.size() * sizeof(double2));
    RK_CUDA(cudaMemcpy(sp.d_twiddle64.ptr, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    sp.d_mult2_64.reserve(m2.size() * sizeof(double2));
    RK_CUDA(cudaMemcpy(sp.d_mult2_64.ptr, m2.data(), m2.size() * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return {sp.d_twiddle64.as<double2>(), sp.d_mult2_64.as<double2>()};
}

template <class T, class R>
void row_fwd(const T* src, const T* sub, RowSrc m, int64_t planes, int logn, const Launch& l,
             const typename Cx<R>::T* tw, typename Cx<R>::T* out, cudaStream_t st) {
  smem_opt_in(row_fwd_kernel<T, R>, l.row_smem);
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  row_fwd_kernel<T, R><<<unsigned(planes * l.per_plane_rows), l.threads, l.row_smem, st>>>(src, sub, m, logn, tw, out);
  RK_CUDA(cudaGetLastError());
}

template <class T, class R>
void row_inv(const typename Cx<R>::T* in, RowDst m, int64_t planes, int logn, const Launch& l,
             const typename Cx<R>::T* tw, R scale, T* dst, const AdmmStore& admm, cudaStream_t st) {
  smem_opt_in(row_inv_kernel<T, R>, l.row_smem);
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  row_inv_kernel<T, R><<<unsigned(planes * l.per_plane_rows), l.threads, l.row_smem, st>>>(in, m, logn, tw, scale, dst,
                                                                                          admm);
  RK_CUDA(cudaGetLastError());
}

template <class R>
void col(const typename Cx<R>::T* in, int mode, int64_t planes, int logn, const Launch& l, const Tables<R>& tb,
         int64_t q0, int64_t B, typename Cx<R>::T* out, cudaStream_t st) {
  smem_opt_in(col_kernel<R>, l.col_smem);
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  col_kernel<R><<<unsigned(planes * l.per_plane_cols), l.threads, l.col_smem, st>>>(in, mode, logn, tb.tw, tb.mult2,
                                                                                     q0, B, out);
  RK_CUDA(cudaGetLastError());
}

// shearlet.cpp:253-270: image [B][n][n] -> coefficients [B][K][n][n]
template <class T, class R>
void forward_impl(Shearlet& sp, const T* image, int64_t batch, T* coeff, const AdmmStore& admm, cudaStream_t st) {
  using C = typename Cx<R>::T;
  const int n = int(sp.height), logn = log2_of(n);
  const int64_t plane = int64_t(n) * n, K = sp.n_coeff, P = (K + 1) / 2;
  const Tables<R> tb = tables<R>(sp);
  const Launch l = launch_cfg<R>(n);
  // (pair, image) items per chunk: the column pass's scratch planes, <= kWkChunkMB
  const int64_t items = P * batch;
  const int64_t chunk =
      std::max<int64_t>(1, std::min<int64_t>(items, (int64_t(kWkChunkMB) << 20) / (plane * int64_t(sizeof(C)))));
  sp.work_a.reserve(size_t(batch) * plane * sizeof(C));  // X = fft2(x), bit-reversed order
  sp.work_b.reserve(size_t(chunk) * plane * sizeof(C));
  C* X = sp.work_a.as<C>();
  C* Wk = sp.work_b.as<C>();
  row_fwd<T, R>(image, nullptr, RowSrc{0, 1, 0, K}, batch, logn, l, tb.tw, X, st);
  col<R>(X, 0, batch, logn, l, tb, 0, 1, X, st);
  const R scale = R(1) / R(plane);
  for (int64_t q0 = 0; q0 < items; q0 += chunk) {
    const int64_t nq = std::min(chunk, items - q0);
    col<R>(X, 1, nq, logn, l, tb, q0, batch, Wk, st);
    row_inv<T, R>(Wk, RowDst{1, q0, batch, K}, nq, logn, l, tb.tw, scale, coeff, admm, st);
  }
}

// shearlet.cpp:272-294: coefficients [B][K][n][n] (minus `sub` when given) -> image [B][n][n]
template <class T, class R>
void backward_impl(Shearlet& sp, const T* coeff, const T* sub, int64_t batch, T* image, cudaStream_t st) {
  using C = typename Cx<R>::T;
  const int n = int(sp.height), logn = log2_of(n);
  const int64_t plane = int64_t(n) * n, K = sp.n_coeff, P = (K + 1) / 2;
  const Tables<R> tb = tables<R>(sp);
  const Launch l = launch_cfg<R>(n);
  // pairs in chunks of kPairChunk (a fixed, batch-independent reduction
  // order); a wave of chunks is transformed and accumulated concurrently,
  // each chunk into its own partial spectrum
  const int64_t nch = (P + kPairChunk - 1) / kPairChunk;
  const int64_t chunk_bytes = batch * int64_t(kPairChunk) * plane * int64_t(sizeof(C));
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(nch, (int64_t(1) << 30) / chunk_bytes));
  sp.work_a.reserve(size_t(batch * nch) * plane * sizeof(C));
  sp.work_b.reserve(size_t(std::max<int64_t>(batch * std::min(cap * kPairChunk, P), batch)) * plane * sizeof(C));
  C* Sp = sp.work_a.as<C>();  // per-chunk partial spectra, bit-reversed order
  C* Wk = sp.work_b.as<C>();
  smem_opt_in(col_acc_kernel<R>, l.col_smem);
  for (int64_t c0 = 0; c0 < nch; c0 += cap) {
    const int64_t ncw = std::min(cap, nch - c0), p0 = c0 * kPairChunk, np = std::min(ncw * kPairChunk, P - p0);
    row_fwd<T, R>(coeff, sub, RowSrc{1, np, p0, K}, batch * np, logn, l, tb.tw, Wk, st);
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    col_acc_kernel<R><<<unsigned(batch * l.per_plane_cols * ncw), unsigned(std::max(32, l.tile / kAccPerThread)),
                        l.col_smem, st>>>(
        Wk, np, p0, P, c0, ncw, nch, logn, tb.tw, tb.mult2, Sp);
    RK_CUDA(cudaGetLastError());
  }
  // image = Re(ifft2(sum of the partials)) / (n n)
  col<R>(Sp, 3, batch, logn, l, tb, 0, nch, Wk, st);
  row_inv<T, R>(Wk, RowDst{0, 0, 1, 1}, batch, logn, l, tb.tw, R(1) / R(plane), image, AdmmStore{}, st);
}

}  // namespace

void upload_shearlet(Shearlet& sp) {
  if (sp.device < 0) return;
  if (!shearlet_pow2(sp.height)) return upload_shearlet_generic(sp);
  std::vector<float2> m2, tw;
  build_tables<float>(sp, m2, tw);
  rk::set_device(sp.device);
  sp.d_mult2.reserve(m2.size() * sizeof(float2));
  sp.d_twiddle.reserve(tw.size() * sizeof(float2));
  RK_CUDA(cudaMemcpy(sp.d_mult2.ptr, m2.data(), m2.size() * sizeof(float2), cudaMemcpyHostToDevice));
  RK_CUDA(cudaMemcpy(sp.d_twiddle.ptr, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
}

void shearlet_forward(Shearlet& sp, int dtype, const void* image, int64_t batch, void* coeff, cudaStream_t st) {
  if (!shearlet_pow2(sp.height)) return shearlet_forward_generic(sp, dtype, image, batch, coeff, GenericAdmm{}, st);
  switch (dtype) {
    case RK_F16:
      forward_impl<__half, float>(sp, static_cast<const __half*>(image), batch, static_cast<__half*>(coeff), {}, st);
      break;
    case RK_F32:
      forward_impl<float, float>(sp, static_cast<const float*>(image), batch, static_cast<float*>(coeff), {}, st);
      break;
    case RK_F64:
      forward_impl<double, double>(sp, static_cast<const double*>(image), batch, static_cast<double*>(coeff), {}, st);
      break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

void shearlet_backward(Shearlet& sp, int dtype, const void* coeff, int64_t batch, void* image, cudaStream_t st) {
  if (!shearlet_pow2(sp.height)) return shearlet_backward_generic(sp, dtype, coeff, nullptr, batch, image, st);
  switch (dtype) {
    case RK_F16:
      backward_impl<__half, float>(sp, static_cast<const __half*>(coeff), nullptr, batch, static_cast<__half*>(image), st);
      break;
    case RK_F32:
      backward_impl<float, float>(sp, static_cast<const float*>(coeff), nullptr, batch, static_cast<float*>(image), st);
      break;
    case RK_F64:
      backward_impl<double, double>(sp, static_cast<const double*>(coeff), nullptr, batch, static_cast<double*>(image),
                                    st);
      break;
    default: throw ValidationError("unknown dtype " + std::to_string(dtype));
  }
}

void shearlet_admm_shrink(Shearlet& sp, const float* f, int64_t batch, float* z1, float* u1, const float* thresh,
                          int* flag, const int* iteration, cudaStream_t st) {
  if (!shearlet_pow2(sp.height)) {
    GenericAdmm g;
    g.z1 = z1;
    g.u1 = u1;
    g.thresh = thresh;
    g.flag = flag;
    g.iteration = iteration;
    return shearlet_forward_generic(sp, RK_F32, f, batch, nullptr, g, st);
  }
  AdmmStore a;
  a.z1 = z1;
  a.u1 = u1;
  a.thresh = thresh;
  a.flag = flag;
  a.iteration = iteration;
  forward_impl<float, float>(sp, f, batch, nullptr, a, st);
}

void shearlet_admm_synth(Shearlet& sp, const float* z1, const float* u1, int64_t batch, float* image,
                         cudaStream_t st) {
  if (!shearlet_pow2(sp.height)) return shearlet_backward_generic(sp, RK_F32, z1, u1, batch, image, st);
  backward_impl<float, float>(sp, z1, u1, batch, image, st);
}

}  // namespace rk
