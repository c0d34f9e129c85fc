// Shared-memory FFTs for the ramp filter (filter.cu) and the alpha-shearlet
// transform (shearlet.cu): in-place radix-2 DIF / DIT transforms of 2^logn
// points whose stages are fused three at a time in registers.
//
// A pass covers stages lh+1 .. lh+R: the group of element i0 holds
// i0 + m 2^lh (m < 2^R, i0 with bits lh .. lh+R-1 clear), each thread loads a
// group, runs the R butterfly layers and stores it back, so a transform is
// ceil(logn / 3) shared-memory passes and barriers instead of logn.  Every
// butterfly is the plain radix-2 one with the stage's table twiddle
// (tw[k] = exp(-2 pi i k / n), k < n/2):
//   DIF (natural in, bit-reversed out):  u + v, (u - v) W
//   DIT (bit-reversed in, natural out):  u + v W, u - v W   (conj(W) if CONJ)
// so the results are those of the stage-by-stage radix-2 transform, bit for bit.
//
// Elements live at swizzled slots inside their sequence (fft_swz): an XOR
// swizzle within each block of 16 that makes every access pattern of the
// passes (element strides 1, 8, 64, 512, 4096; half warps of 64-bit
// accesses) bank-conflict free — checked exhaustively for 2^8 .. 2^13 points.
// Callers index shared memory with seq * ld + fft_swz(i).
#pragma once

#include <cuda_runtime.h>

namespace rk {

__device__ __forceinline__ int fft_swz(int i) { return i ^ ((i >> 3) & 15); }

template <class C>
__device__ __forceinline__ C fft_cmul(C a, C b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <class C>
__device__ __forceinline__ C fft_cmul_conj(C a, C b) {  // a * conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}

// One fused pass over `cnt` sequences at stride `ld`, stages lh+1 .. lh+R.
template <int R, bool DIF, bool CONJ, class C>
__device__ __forceinline__ void fft_pass(C* z, int cnt, int ld, int logn, int lh, const C* __restrict__ tw) {
  const int gl = logn - R;  // log2(groups per sequence)
  for (int t = threadIdx.x; t < (cnt << gl); t += blockDim.x) {
    const int seq = t >> gl, g = t & ((1 << gl) - 1);
    const int lo = g & ((1 << lh) - 1), hi = g >> lh;
    const int i0 = lo + (hi << (lh + R));
    C* a = z + seq * ld;
    C x[1 << R];
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) x[m] = a[fft_swz(i0 + (m << lh))];
#pragma unroll
    for (int l = 0; l < R; ++l) {
      const int bit = DIF ? R - 1 - l : l;  // partner bit of m (stage lh + bit + 1)
#pragma unroll
      for (int m = 0; m < (1 << R); ++m) {
        if (m & (1 << bit)) continue;
        const int q = m | (1 << bit);
        const int k = lo + ((m & ((1 << bit) - 1)) << lh);
        const C w = tw[k << (logn - lh - 1 - bit)];
        const C u = x[m];
        if (DIF) {
          const C v = x[q];
          x[m] = {u.x + v.x, u.y + v.y};
          x[q] = fft_cmul(C{u.x - v.x, u.y - v.y}, w);
        } else {
          const C v = CONJ ? fft_cmul_conj(x[q], w) : fft_cmul(x[q], w);
          x[m] = {u.x + v.x, u.y + v.y};
          x[q] = {u.x - v.x, u.y - v.y};
        }
      }
    }
#pragma unroll
    for (int m = 0; m < (1 << R); ++m) a[fft_swz(i0 + (m << lh))] = x[m];
  }
  __syncthreads();
}

// Forward DIF, natural -> bit-reversed (the short pass first, at the widest stride).
template <class C>
__device__ void fft_dif_seq(C* z, int cnt, int ld, int logn, const C* __restrict__ tw) {
  int lh = logn - logn % 3;
  if (logn % 3 == 2) fft_pass<2, true, false>(z, cnt, ld, logn, lh, tw);
  if (logn % 3 == 1) fft_pass<1, true, false>(z, cnt, ld, logn, lh, tw);
  while (lh >= 3) {
    lh -= 3;
    fft_pass<3, true, false>(z, cnt, ld, logn, lh, tw);
  }
}

// Unnormalised inverse DIT, bit-reversed -> natural.
template <class C>
__device__ void ifft_dit_seq(C* z, int cnt, int ld, int logn, const C* __restrict__ tw) {
  int lh = 0;
  for (; lh + 3 <= logn; lh += 3) fft_pass<3, false, true>(z, cnt, ld, logn, lh, tw);
  if (logn - lh == 2) fft_pass<2, false, true>(z, cnt, ld, logn, lh, tw);
  if (logn - lh == 1) fft_pass<1, false, true>(z, cnt, ld, logn, lh, tw);
}

}  // namespace rk
