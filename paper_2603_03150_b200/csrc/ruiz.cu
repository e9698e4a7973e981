// ruiz.cu -- device Ruiz equilibration.
//
// Restates hybridlp.transform.ruiz_equilibrate (transform.py:35-77) on the
// device with the reference's exact arithmetic, so scales and scaled values
// are bit-identical to scipy's:
//   row_norm = max_j |a_ij|, col_norm = max_i |a_ij|         (exact maxima)
//   stop when every norm lies in [1/(1+tol), 1+tol]           (transform.py:63-67)
//   r = 1/sqrt(row_norm), c = 1/sqrt(col_norm)               (IEEE sqrt and division)
//   a_ij <- (r_i * a_ij) * c_j                               (diags(r) @ A @ diags(c))
//   row_scale *= r, col_scale *= c                           (transform.py:72-73)
// Column maxima use an integer atomicMax on the bit patterns of |a_ij|
// (non-negative doubles order like their bits), so the result is exact and
// independent of the atomic order.
#include "../../include/pdhg_b200.h"

#include <cuda_runtime.h>

#include <climits>
#include <string>

namespace pdhg_internal {
int set_error(int code, const std::string& msg);
}

namespace {

using pdhg_internal::set_error;

#define RZ_TRY(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

__global__ void k_fill1(double* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = 1.0;
}

// warp per row: row max |a| and column max via bit-pattern atomicMax
__global__ void k_norms(int m, const int* __restrict__ ptr, const int* __restrict__ col,
                        const double* __restrict__ val, double* __restrict__ row_norm,
                        unsigned long long* __restrict__ colbits) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int s = ptr[w], e = ptr[w + 1];
  double mx = 0.0;
  for (int k = s + lane; k < e; k += 32) {
    const double a = fabs(val[k]);
    mx = a > mx ? a : mx;
    atomicMax(&colbits[col[k]], (unsigned long long)__double_as_longlong(a));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if (lane == 0) row_norm[w] = mx;
}

// flag |= any norm outside [lo, hi]; NaN counts as outside (numpy comparisons are False)
__global__ void k_range(const double* __restrict__ v, int n, double lo, double hi, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(v[i] >= lo && v[i] <= hi)) atomicOr(flag, 1);
}

__global__ void k_colnorm(const unsigned long long* __restrict__ bits, double* __restrict__ out, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = __longlong_as_double((long long)bits[j]);
}

// v <- 1/sqrt(v); scale *= v
__global__ void k_recip_sqrt(double* __restrict__ v, double* __restrict__ scale, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = __ddiv_rn(1.0, __dsqrt_rn(v[i]));
  v[i] = r;
  scale[i] = __dmul_rn(scale[i], r);
}

__global__ void k_apply(int m, const int* __restrict__ ptr, const int* __restrict__ col,
                        double* __restrict__ val, const double* __restrict__ r,
                        const double* __restrict__ c) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const double ri = r[w];
  const int s = ptr[w], e = ptr[w + 1];
  for (int k = s + lane; k < e; k += 32) val[k] = __dmul_rn(__dmul_rn(ri, val[k]), c[col[k]]);
}

unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

extern "C" {

size_t pdhg_ruiz_tmp_bytes(int32_t m, int32_t n) {
  return a256((size_t)m * 8) + a256((size_t)n * 8) + a256((size_t)n * 8) + a256(64);
}

int pdhg_ruiz(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col, double* val,
              double* row_scale, double* col_scale, int32_t max_iters, double lo, double hi,
              void* tmp, size_t tmp_bytes, void* stream, int32_t* applied_out) {
  if (m <= 0 || n <= 0 || nnz < 0 || !ptr || !col || !val || !row_scale || !col_scale || !tmp)
    return set_error(PDHG_ERR_ARG, "ruiz: bad argument");
  if (tmp_bytes < pdhg_ruiz_tmp_bytes(m, n)) return set_error(PDHG_ERR_ARG, "ruiz: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)tmp;
  double* rnorm = (double*)p; p += a256((size_t)m * 8);
  double* cnorm = (double*)p; p += a256((size_t)n * 8);
  unsigned long long* cbits = (unsigned long long*)p; p += a256((size_t)n * 8);
  int* flag = (int*)p;
  k_fill1<<<nb(m, 256), 256, 0, s>>>(row_scale, m);
  k_fill1<<<nb(n, 256), 256, 0, s>>>(col_scale, n);
  int applied = 0;
  for (int it = 0; it < max_iters; ++it) {
    RZ_TRY(cudaMemsetAsync(cbits, 0, (size_t)n * 8, s));
    RZ_TRY(cudaMemsetAsync(flag, 0, 4, s));
    k_norms<<<nb((long long)m * 32, 256), 256, 0, s>>>(m, ptr, col, val, rnorm, cbits);
    k_colnorm<<<nb(n, 256), 256, 0, s>>>(cbits, cnorm, n);
    k_range<<<nb(m, 256), 256, 0, s>>>(rnorm, m, lo, hi, flag);
    k_range<<<nb(n, 256), 256, 0, s>>>(cnorm, n, lo, hi, flag);
    int hflag = 0;
    RZ_TRY(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, s));
    RZ_TRY(cudaStreamSynchronize(s));
    if (!hflag) break;
    k_recip_sqrt<<<nb(m, 256), 256, 0, s>>>(rnorm, row_scale, m);
    k_recip_sqrt<<<nb(n, 256), 256, 0, s>>>(cnorm, col_scale, n);
    k_apply<<<nb((long long)m * 32, 256), 256, 0, s>>>(m, ptr, col, val, rnorm, cnorm);
    ++applied;
  }
  RZ_TRY(cudaGetLastError());
  RZ_TRY(cudaStreamSynchronize(s));
  if (applied_out) *applied_out = applied;
  return 0;
}

}  // extern "C"
