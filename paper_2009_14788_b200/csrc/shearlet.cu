// Alpha-shearlet analysis / synthesis on the device (§8f rank 3; reference
// shearlet.cpp:253-330): coefficient k of an image x is
// Re(ifft2(fft2(x) * M_k)); synthesis sums fft2(c_k) * M_k over k in
// ascending order and takes Re(ifft2(.)).  Arithmetic follows the reference's
// precision split (shearlet.cpp:303-310): fp64 storage computes in fp64
// (spec_d), fp32 / fp16 storage in fp32 (spec_f); power-of-two grids.
//
// 2-D FFT = row FFTs, a tiled transpose, row FFTs: the spectra are kept in
// the transposed layout Xt[b][col][row] so every pass is a row pass of a
// shared-memory radix-2 FFT, and the multipliers are pre-transposed on the
// host.  The multiply, the inverse transform's conjugations, the 1/(h w)
// normalisation, the real-part extraction and the synthesis accumulation are
// fused into the load / store of the row passes.  Analysis walks the
// (image, coefficient) planes in chunks small enough that a chunk's two
// complex scratch planes stay resident in L2 between passes.
//
// ADMM hooks (admm.cu, admm.cpp:146-156): analysis can fuse the shrink and
// dual update into its store (z1 = shrink(c + u1, t_k), u1 += c - z1, with a
// non-finite flag), and synthesis can read (z1 - u1) instead of c.
#include <cuda_fp16.h>

#include "rk_internal.hpp"

namespace rk {

namespace {

constexpr int kFftThreads = 256;

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

// R rows of n complex values in shared memory (bit-reversed order on entry) ->
// forward DFT of each row (natural order).
template <class C>
__device__ void fft_rows_smem(C* a, int rows, int n, const C* __restrict__ tw) {
  const int halfn = n >> 1;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1, stride = n / len;
    for (int b = tid; b < rows * halfn; b += nt) {
      const int r = b / halfn, bb = b - r * halfn;
      const int grp = bb / half, k = bb - grp * half;
      C* row = a + r * n;
      const int i = grp * len + k;
      const C u = row[i], v = cmul(row[i + half], tw[k * stride]);
      row[i] = {u.x + v.x, u.y + v.y};
      row[i + half] = {u.x - v.x, u.y - v.y};
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int brev(int k, int logn) { return int(__brev(unsigned(k)) >> (32 - logn)); }

// forward FFT of real rows: out[r] = fft(in[r] (- sub[r])); rows are contiguous
// in planes of rpp rows, plane p of the source at p * pstride
template <class T, class R>
__global__ void __launch_bounds__(kFftThreads)
    rowfft_real_kernel(const T* __restrict__ in, const T* __restrict__ sub, int64_t pstride, int64_t rows, int n,
                       int logn, const typename Cx<R>::T* __restrict__ tw, typename Cx<R>::T* __restrict__ out) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int nr = int(min(int64_t(blockDim.y), rows - int64_t(blockIdx.x) * blockDim.y));
  const int64_t r0 = int64_t(blockIdx.x) * blockDim.y;
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y) {
    const int r = e / n, c = e - r * n;
    const int64_t rr = r0 + r, p = rr / n, lr = rr - p * n;
    const int64_t off = p * pstride + lr * n + c;
    R v = ld_r<R>(in + off);
    if (sub) v = v - ld_r<R>(sub + off);  // sub(z1, u1) (admm.cpp:147)
    sm[r * n + brev(c, logn)] = {v, R(0)};
  }
  __syncthreads();
  fft_rows_smem(sm, nr, n, tw);
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y)
    out[(r0 + e / n) * n + (e % n)] = sm[e];
}

// Complex row pass over planes of n rows.
// mode 0: forward, out = fft(in)                        in plane = p
// mode 1: inverse with multiplier, out = conj(fft(conj(in * m)))  (= n ifft(in m));
//         plane p of the chunk is (image, coeff) q = q0 + p: in plane q / K, m plane q % K
// mode 2: forward + accumulate, out += fft(in) * m      in plane = p, m plane = q0
// mode 3: inverse, out = conj(fft(conj(in)))            in plane = p
template <class R>
__global__ void __launch_bounds__(kFftThreads)
    rowfft_c2c_kernel(const typename Cx<R>::T* __restrict__ in, int64_t rows, int n, int logn,
                      const typename Cx<R>::T* __restrict__ tw, int mode, const R* __restrict__ mult, int64_t q0,
                      int64_t K, typename Cx<R>::T* __restrict__ out) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int nr = int(min(int64_t(blockDim.y), rows - int64_t(blockIdx.x) * blockDim.y));
  const int64_t r0 = int64_t(blockIdx.x) * blockDim.y;
  const int64_t plane = int64_t(n) * n;
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y) {
    const int r = e / n, c = e - r * n;
    const int64_t rr = r0 + r, p = rr / n, lr = rr - p * n;
    C v;
    if (mode == 1) {
      const int64_t q = q0 + p;
      v = in[(q / K) * plane + lr * n + c];
      const R m = mult[(q % K) * plane + lr * n + c];
      v = {v.x * m, -(v.y * m)};
    } else {
      v = in[rr * n + c];
      if (mode == 3) v.y = -v.y;
    }
    sm[r * n + brev(c, logn)] = v;
  }
  __syncthreads();
  fft_rows_smem(sm, nr, n, tw);
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y) {
    const int r = e / n, c = e - r * n;
    const int64_t rr = r0 + r;
    const C v = sm[e];
    if (mode == 1 || mode == 3) {
      out[rr * n + c] = {v.x, -v.y};
    } else if (mode == 2) {
      const int64_t lr = rr % n;
      const R m = mult[q0 * plane + lr * n + c];
      const C a = out[rr * n + c];
      out[rr * n + c] = {a.x + v.x * m, a.y + v.y * m};
    } else {
      out[rr * n + c] = v;
    }
  }
}

// ADMM analysis epilogue (admm.cpp:150-153), fp32 like the reference's float path
struct AdmmStore {
  float* z1 = nullptr;  // null: plain store
  float* u1 = nullptr;
  const float* thresh = nullptr;  // per coefficient, float((p0/p1) w_k)
  int* flag = nullptr;            // atomicMin(iteration) when u1 turns non-finite
  int iteration = 0;
};

// soft(a, b) = sign(a) max(|a| - b, 0) (admm.cpp:46-51)
__device__ __forceinline__ float soft(float a, float b) {
  float m = __fsub_rn(fabsf(a), b);
  if (m < 0.f) m = 0.f;
  return a < 0.f ? -m : (a > 0.f ? m : 0.f);
}

// inverse row pass with real output: Re(conj(fft(conj(in)))) * scale stored
// contiguously at out + (row r0 + r) * n (+ the ADMM update when requested)
template <class T, class R>
__global__ void __launch_bounds__(kFftThreads)
    rowifft_real_kernel(const typename Cx<R>::T* __restrict__ in, int64_t rows, int n, int logn,
                        const typename Cx<R>::T* __restrict__ tw, R scale, int64_t q0, int64_t K,
                        T* __restrict__ out, AdmmStore admm) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  const int nr = int(min(int64_t(blockDim.y), rows - int64_t(blockIdx.x) * blockDim.y));
  const int64_t r0 = int64_t(blockIdx.x) * blockDim.y;
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y) {
    const int r = e / n, c = e - r * n;
    const C v = in[(r0 + r) * n + c];
    sm[r * n + brev(c, logn)] = {v.x, -v.y};
  }
  __syncthreads();
  fft_rows_smem(sm, nr, n, tw);
  const int64_t plane = int64_t(n) * n;
  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < nr * n; e += blockDim.x * blockDim.y) {
    const int64_t idx = (r0 + e / n) * n + (e % n);
    const R c = sm[e].x * scale;
    if (admm.z1 == nullptr) {
      out[idx] = st_r<T>(c);
    } else {
      const float cf = float(c);
      const int64_t gi = q0 * plane + idx;  // global (image, coeff, row, col) index
      const float u = admm.u1[gi];
      const float z = soft(__fadd_rn(cf, u), admm.thresh[(q0 + idx / plane) % K]);
      const float un = __fadd_rn(u, __fsub_rn(cf, z));
      admm.z1[gi] = z;
      admm.u1[gi] = un;
      if (!isfinite(un)) atomicMin(admm.flag, admm.iteration);
    }
  }
}

// out[p][c][r] = in[p][r][c] (complex, tiled)
template <class C>
__global__ void transpose_c_kernel(const C* __restrict__ in, int nr, int nc, C* __restrict__ out) {
  __shared__ C tile[32][33];
  const int64_t plane = int64_t(nr) * nc;
  const C* s = in + blockIdx.z * plane;
  C* d = out + blockIdx.z * plane;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = by + r, j = bx + threadIdx.x;
    if (i < nr && j < nc) tile[r][threadIdx.x] = s[int64_t(i) * nc + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + r, j = by + threadIdx.x;
    if (i < nc && j < nr) d[int64_t(i) * nr + j] = tile[threadIdx.x][r];
  }
}

struct Rows {
  dim3 block;
  unsigned grid;
  size_t smem;
};
template <class R>
Rows rows_cfg(int64_t rows, int n) {
  const size_t row_bytes = size_t(n) * sizeof(typename Cx<R>::T);
  const int nr = int(std::max<size_t>(1, std::min<size_t>(8, 32768 / row_bytes)));  // rows per CTA
  Rows c;
  c.block = dim3(unsigned(kFftThreads / nr), unsigned(nr));
  c.grid = unsigned((rows + nr - 1) / nr);
  c.smem = size_t(nr) * row_bytes;
  return c;
}

template <class K>
void smem_opt_in(K kernel, size_t smem) {
  if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
}

template <class C>
void transpose_c(const C* in, int64_t planes, int n, C* out, cudaStream_t st) {
  dim3 grid(unsigned((n + 31) / 32), unsigned((n + 31) / 32), unsigned(planes));
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  transpose_c_kernel<C><<<grid, dim3(32, 8), 0, st>>>(in, n, n, out);
  RK_CUDA(cudaGetLastError());
}

template <class R>
void c2c(const typename Cx<R>::T* in, int64_t rows, int n, int logn, const typename Cx<R>::T* tw, int mode,
         const R* mult, int64_t q0, int64_t K, typename Cx<R>::T* out, cudaStream_t st) {
  Rows c = rows_cfg<R>(rows, n);
  smem_opt_in(rowfft_c2c_kernel<R>, c.smem);
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  rowfft_c2c_kernel<R><<<c.grid, c.block, c.smem, st>>>(in, rows, n, logn, tw, mode, mult, q0, K, out);
  RK_CUDA(cudaGetLastError());
}

int log2_of(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

// device tables in the working precision: fp32 ones are built with the plan,
// fp64 ones on first use (multipliers transposed per coefficient)
template <class R>
struct Tables {
  const typename Cx<R>::T* tw;
  const R* mult;
};
template <class R>
Tables<R> tables(Shearlet& sp);
template <>
Tables<float> tables<float>(Shearlet& sp) {
  return {sp.d_twiddle.as<float2>(), sp.d_mult_t.as<float>()};
}
template <>
Tables<double> tables<double>(Shearlet& sp) {
  if (!sp.d_mult_t64.ptr) {
    const int64_t h = sp.height, w = sp.width, bins = h * w;
    std::vector<double> mt(size_t(sp.n_coeff * bins));
    for (int64_t k = 0; k < sp.n_coeff; ++k)
      for (int64_t i = 0; i < h; ++i)
        for (int64_t j = 0; j < w; ++j) mt[size_t(k * bins + j * h + i)] = sp.multipliers[size_t(k * bins + i * w + j)];
    std::vector<double2> tw(size_t(std::max<int64_t>(h / 2, 1)));
    for (int64_t k = 0; k < h / 2; ++k) {
      const double ang = 2.0 * M_PI * double(k) / double(h);
      tw[size_t(k)] = make_double2(std::cos(ang), -std::sin(ang));
    }
    sp.d_twiddle64.reserve(tw.size() * sizeof(double2));
    RK_CUDA(cudaMemcpy(sp.d_twiddle64.ptr, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    sp.d_mult_t64.reserve(mt.size() * sizeof(double));
    RK_CUDA(cudaMemcpy(sp.d_mult_t64.ptr, mt.data(), mt.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  return {sp.d_twiddle64.as<double2>(), sp.d_mult_t64.as<double>()};
}

// shearlet.cpp:253-270: image [B][n][n] -> coefficients [B][K][n][n]
template <class T, class R>
void forward_impl(Shearlet& sp, const T* image, int64_t batch, T* coeff, AdmmStore admm, cudaStream_t st) {
  using C = typename Cx<R>::T;
  const int n = int(sp.height), logn = log2_of(n);
  const int64_t plane = int64_t(n) * n, K = sp.n_coeff;
  const Tables<R> tb = tables<R>(sp);
  // (image, coeff) planes per chunk: two complex scratch planes each, ~32 MB
  // in flight so the transpose and the last row pass hit L2
  const int64_t total = batch * K;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(total, (int64_t(32) << 20) / (2 * plane * int64_t(sizeof(C)))));
  sp.work_a.reserve(size_t(batch) * plane * sizeof(C));  // spectrum of every image, transposed
  sp.work_b.reserve(size_t(std::max(chunk, batch)) * plane * sizeof(C) * 2);
  C* X = sp.work_a.as<C>();
  C* A = sp.work_b.as<C>();
  C* Bt = A + size_t(std::max(chunk, batch)) * plane;
  // X^T = columns-FFT(transpose(rows-FFT(x)))
  {
    Rows c = rows_cfg<R>(batch * n, n);
    smem_opt_in(rowfft_real_kernel<T, R>, c.smem);
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    rowfft_real_kernel<T, R><<<c.grid, c.block, c.smem, st>>>(image, nullptr, plane, batch * n, n, logn, tb.tw, A);
    RK_CUDA(cudaGetLastError());
  }
  transpose_c(A, batch, n, Bt, st);
  c2c<R>(Bt, batch * n, n, logn, tb.tw, 0, nullptr, 0, 1, X, st);
  const R scale = R(1) / R(plane);
  for (int64_t q0 = 0; q0 < total; q0 += chunk) {
    const int64_t planes = std::min(chunk, total - q0);
    // inverse along columns of X^T * M_k^T (rows of the transposed layout)
    c2c<R>(X, planes * n, n, logn, tb.tw, 1, tb.mult, q0, K, A, st);
    transpose_c(A, planes, n, Bt, st);
    Rows c = rows_cfg<R>(planes * n, n);
    smem_opt_in(rowifft_real_kernel<T, R>, c.smem);
    KernelTimer t(RK_KERNEL_SHEARLET, st);
    rowifft_real_kernel<T, R><<<c.grid, c.block, c.smem, st>>>(Bt, planes * n, n, logn, tb.tw, scale, q0, K,
                                                               coeff ? coeff + q0 * plane : nullptr, admm);
    RK_CUDA(cudaGetLastError());
  }
}

// shearlet.cpp:272-294: coefficients [B][K][n][n] (minus `sub` when given) -> image [B][n][n]
template <class T, class R>
void backward_impl(Shearlet& sp, const T* coeff, const T* sub, int64_t batch, T* image, cudaStream_t st) {
  using C = typename Cx<R>::T;
  const int n = int(sp.height), logn = log2_of(n);
  const int64_t plane = int64_t(n) * n, K = sp.n_coeff;
  const Tables<R> tb = tables<R>(sp);
  sp.work_a.reserve(size_t(batch) * plane * sizeof(C));
  sp.work_b.reserve(size_t(batch) * plane * sizeof(C) * 2);
  C* S = sp.work_a.as<C>();  // accumulated spectrum, transposed
  C* A = sp.work_b.as<C>();
  C* Bt = A + size_t(batch) * plane;
  RK_CUDA(cudaMemsetAsync(S, 0, size_t(batch) * plane * sizeof(C), st));
  Rows c = rows_cfg<R>(batch * n, n);
  smem_opt_in(rowfft_real_kernel<T, R>, c.smem);
  for (int64_t k = 0; k < K; ++k) {  // ascending k: a fixed reduction order (shearlet.cpp:286-291)
    {
      KernelTimer t(RK_KERNEL_SHEARLET, st);
      rowfft_real_kernel<T, R><<<c.grid, c.block, c.smem, st>>>(coeff + k * plane, sub ? sub + k * plane : nullptr,
                                                                K * plane, batch * n, n, logn, tb.tw, A);
      RK_CUDA(cudaGetLastError());
    }
    transpose_c(A, batch, n, Bt, st);
    // forward along columns, S += result * M_k^T
    c2c<R>(Bt, batch * n, n, logn, tb.tw, 2, tb.mult, k, K, S, st);
  }
  // image = Re(ifft2(S)) / (n n)
  c2c<R>(S, batch * n, n, logn, tb.tw, 3, nullptr, 0, 1, A, st);
  transpose_c(A, batch, n, Bt, st);
  smem_opt_in(rowifft_real_kernel<T, R>, c.smem);
  KernelTimer t(RK_KERNEL_SHEARLET, st);
  rowifft_real_kernel<T, R><<<c.grid, c.block, c.smem, st>>>(Bt, batch * n, n, logn, tb.tw, R(1) / R(plane), 0, 1,
                                                             image, AdmmStore{});
  RK_CUDA(cudaGetLastError());
}

}  // namespace

void shearlet_forward(Shearlet& sp, int dtype, const void* image, int64_t batch, void* coeff, cudaStream_t st) {
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
                          int* flag, int iteration, cudaStream_t st) {
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
  backward_impl<float, float>(sp, z1, u1, batch, image, st);
}

}  // namespace rk
